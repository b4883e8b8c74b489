mkdir -p gpurun_out
OUT=gpurun_out/lab_r02n.txt
: > $OUT
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_kernels.py -x -q 2>&1 | tail -3 >> $OUT
bash tools/lab_v3_ab.sh "G4RING_V3_EARLY_ST=0" "G4RING_V3_EARLY_ST=1" "G4RING_V3_EARLY_ST=0 G4RING_PDL=0" "G4RING_V3_EARLY_ST=1 G4RING_V3_HINTS=2" >> $OUT 2>&1
for e in "G4RING_V3_EARLY_ST=0" "G4RING_V3_EARLY_ST=1"; do
  env $e timeout 120 python tools/k1_lab.py --planes 256 --batch 8 --arith fused --tag "$e P256" >> $OUT 2>&1
  env $e timeout 120 python tools/k1_lab.py --n 4608 --planes 72 --batch 8 --iters 3 --arith fused --tag "$e c4" >> $OUT 2>&1
  env $e timeout 120 python tools/k1_lab.py --n 1024 --planes 64 --batch 8 --iters 10 --arith fused --tag "$e n1024" >> $OUT 2>&1
done
timeout 300 python tools/v3_trace.py --batch 8 --planes 64 >> $OUT 2>&1
