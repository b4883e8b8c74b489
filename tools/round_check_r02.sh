# round-2 validation bundle on the GPU box: GPU tests, smoke, sanitizers on the warp-specialised
# kernels, config-5 sweeps (message size, K1 batch x N), the N=2 ring bench line on one GPU
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_r02c.log 2>&1
tail -5 gpurun_out/gpu_tests_r02c.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/gpu_tests_r02c.log 2>&1
timeout 600 python tools/copy_bench.py --sweep > gpurun_out/r02_copy_sweep.txt 2>&1
VARIANTS="G4RING_V2GEOM=-1" BATCHES="1 2 4 8 16" SHAPES="512:64 1024:64 1024:16 4608:72" ARITHS="fused exact" \
  timeout 1500 bash tools/k1_sweep.sh > gpurun_out/r02_k1_sweep.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r02_bench_ring2.log 2>&1
grep -E '^\{' gpurun_out/r02_bench_ring2.log | tail -1 > gpurun_out/r02_bench_ring2_one_gpu.json
timeout 2400 bash tools/sanitize_v3.sh > gpurun_out/r02_sanitizer_v3.txt 2>&1
