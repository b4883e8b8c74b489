mkdir -p gpurun_out
OUT=gpurun_out/lab_r02ae.txt
: > $OUT
# chained fused passes (no wait for the previous pass before loads/reductions)
timeout 600 python -m pytest tests/test_gpu_chain.py tests/test_gpu_headline.py -x -q 2>&1 | tail -3 >> $OUT
bash tools/lab_v3_ab.sh "G4RING_V3_CHAIN=0" "G4RING_V3_CHAIN=1" "G4RING_V3_CHAIN=0" "G4RING_V3_CHAIN=1" >> $OUT 2>&1
for c in 0 1; do
  G4RING_V3_CHAIN=$c timeout 120 python tools/k1_lab.py --n 1024 --planes 64 --batch 8 --iters 10 --arith fused --tag "chain$c n1024" >> $OUT 2>&1
  G4RING_V3_CHAIN=$c timeout 120 python tools/k1_lab.py --n 4608 --planes 72 --batch 8 --iters 3 --arith fused --tag "chain$c c4" >> $OUT 2>&1
  G4RING_V3_CHAIN=$c timeout 120 python tools/k1_lab.py --n 512 --planes 32 --batch 8 --iters 20 --arith fused --tag "chain$c P32" >> $OUT 2>&1
done
