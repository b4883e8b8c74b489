# ring engine: native round program vs host loop (tests), and the 2/4-rank bench on one GPU
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_engine.py -x -q 2>&1 | tail -3
for N in 2 4; do
  for nat in 1 0; do
    G4RING_NATIVE=$nat timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 10 --warmup 3 2>&1 | grep -E '^\{' | tail -1 > gpurun_out/ring_n${N}_native$nat.json
    python -c "
import json; d=json.load(open('gpurun_out/ring_n${N}_native$nat.json'))
print('N=$N native=$nat', '%.3e'%d['value'], 'ms/step %.3f'%d['ms_per_step'], 'host', d['host'], 'k1 roofline %.3f'%d['roofline']['frac'], 'model', {k: d['model'][k] for k in ('round_ms','k1_ms','step_transfer_ms','ring_hidden')})"
  done
done
