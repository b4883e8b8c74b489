# chained deferred passes extended to the v2 kernels (P = 8 geometry 19, complex64 geometry 12,
# 4-7 walkers geometry 25), then the round bundle r02j on the final code
mkdir -p gpurun_out
OUT=gpurun_out/lab_r02af.txt
: > $OUT
timeout 900 python -m pytest tests/test_gpu_chain.py -x -q 2>&1 | tail -3 | tee -a $OUT | grep -q " passed" || exit 1
for c in 0 1 0 1; do
  G4RING_V3_CHAIN=$c timeout 120 python tools/k1_lab.py --n 512 --planes 8 --batch 8 --iters 40 --arith fused --tag "chain$c P8" >> $OUT 2>&1
  G4RING_V3_CHAIN=$c timeout 120 python tools/k1_lab.py --n 512 --planes 64 --batch 8 --dtype c64 --iters 20 --arith fused --tag "chain$c c64" >> $OUT 2>&1
  G4RING_V3_CHAIN=$c timeout 120 python tools/k1_lab.py --n 512 --planes 64 --batch 5 --iters 20 --arith fused --tag "chain$c B5" >> $OUT 2>&1
  G4RING_V3_CHAIN=$c timeout 120 python tools/k1_lab.py --n 512 --planes 16 --batch 8 --iters 40 --arith fused --tag "chain$c P16" >> $OUT 2>&1
done
timeout 1500 bash tools/profile_round.sh r02j 8 >> $OUT 2>&1
timeout 900 bash tools/final_check.sh >> $OUT 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02j_gpu_tests.log 2>&1
tail -3 gpurun_out/r02j_gpu_tests.log >> $OUT
