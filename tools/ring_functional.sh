# functional: ring bench for config 3 (8 ranks = 2 sub-rings of 4, 2 lanes) and config 2 at 2 ranks,
# all sharing the one GPU of the box (timings are not meaningful); reference arm under torchrun
cd $GRAFT_REPO_ROOT
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $R --nproc-per-node 8 --master-port 29521 bench.py --gpus 8 --config c3 --steps 3 --warmup 3 2>&1 | grep -E '^\{|Error|error' | tail -3 > gpurun_out/ring_c3_n8.json
timeout 300 $R --nproc-per-node 2 --master-port 29522 bench.py --gpus 2 --steps 5 --warmup 3 2>&1 | grep -E '^\{|Error|error' | tail -3 > gpurun_out/ring_c2_n2.json
timeout 300 $R --nproc-per-node 2 --master-port 29523 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 2>&1 | grep -E '^\{|Error|error' | tail -3 > gpurun_out/ref_n2.json
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep -E '^\{' | tail -1 > gpurun_out/n1_e2efix.json
for f in ring_c3_n8 ring_c2_n2 ref_n2 n1_e2efix; do echo "== $f"; python -c "
import json,sys
for line in open('gpurun_out/$f.json'):
    try: d=json.loads(line)
    except Exception: print(line[:300]); continue
    print({k: d.get(k) for k in ('value','n_gpus','ms_per_step','impl')}, d.get('config',{}).get('parallelism'), 'e2e', d.get('e2e',{}).get('value'), 'model', d.get('model',{}).get('round_ms'), 'host', d.get('host',{}).get('enqueue_ms_per_step'))
"; done
