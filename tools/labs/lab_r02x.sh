mkdir -p gpurun_out
OUT=gpurun_out/lab_r02x.txt
: > $OUT
for args in "--config c3 --lanes 2 --subring-size 2" "--config c3 --lanes 2 --subring-size 2 --merged-lanes" "--config c2 --dtype mixed"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 100)) \
    bench.py --gpus 4 --steps 5 --warmup 3 $args 2>/dev/null | grep -E '^\{' | tail -1 > /tmp/l.json
  python -c "import json; d=json.load(open('/tmp/l.json')); print('$args', '%.3e'%d['value'], d['config'].get('lane_pipelines'), d['config']['parallelism'], 'traffic', d['roofline']['traffic'], 'e2e %.3e'%d['e2e']['value'])" >> $OUT 2>&1
done
