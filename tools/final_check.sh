# the driver's round-end sequence, approximately: smoke, default bench (N=1), reference arm, ring bench (2 ranks, 1 GPU)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
( time python bench.py ) > gpurun_out/final_bench.log 2>&1
grep -E '^\{' gpurun_out/final_bench.log | tail -1 > gpurun_out/final_bench.json
grep real gpurun_out/final_bench.log
python bench.py --impl reference --steps 3 --warmup 1 2>/dev/null | grep -E '^\{' | tail -1 > gpurun_out/final_ref.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --steps 5 --warmup 3 2>&1 | grep -E '^\{' | tail -1 > gpurun_out/final_ring2.json
for f in final_bench final_ref final_ring2; do python -c "
import json; d=json.load(open('gpurun_out/$f.json'))
print('$f', '%.3e'%d['value'], d.get('n_gpus'), 'ms/step %.3f'%d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'], 'roofline', {k: d.get('roofline',{}).get(k) for k in ('frac','traffic')}, 'onchip', d.get('onchip',{}).get('smem_frac'), 'cpu', d.get('cpu_baseline',{}).get('value'), 'h2d', d['e2e'].get('h2d_gbs_achieved'), d['e2e'].get('h2d_peak_gbs'), 'nvlink', d.get('nvlink'))"; done
