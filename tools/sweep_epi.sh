# deferred-update epilogue A/B: word-contiguous reds (parked block) vs per-lane re/im reds
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "fused or bench_workload or deferred" 2>&1 | tail -2
L="timeout 120 python tools/k1_lab.py --arith fused"
for rep in 1 2; do
for b in 4 8 16; do $L --batch $b --tag "fused default"; done
$L --batch 8 --dtype c64 --tag "fused c64"
$L --batch 8 --dtype mixed --tag "fused mixed"
done
$L --batch 8 --n 4608 --planes 72 --iters 3 --tag "fused c4"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 3 -c 1 -o gpurun_out/epi_g12 python tools/k1_lab.py --arith fused --batch 8 --iters 2 > /dev/null 2>&1
