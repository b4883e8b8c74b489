mkdir -p gpurun_out
OUT=gpurun_out/lab_r02r.txt
: > $OUT
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_kernels.py -x -q 2>&1 | tail -3 >> $OUT
G4RING_V3_EXACT=1 timeout 900 python -m pytest tests/test_gpu_headline.py -x -q 2>&1 | tail -2 >> $OUT
bash tools/lab_v3_ab.sh "G4RING_PDL=1" >> $OUT 2>&1
timeout 300 python tools/v3_trace.py --batch 8 --planes 64 2>&1 | grep -E "drain|tready|span" >> $OUT
for e in "G4RING_V3_EXACT=0" "G4RING_V3_EXACT=1"; do
  env $e timeout 120 python tools/k1_lab.py --planes 64 --batch 8 --arith exact --tag "$e exact B=8" >> $OUT 2>&1
done
timeout 120 python tools/k1_lab.py --n 4608 --planes 72 --batch 8 --iters 3 --arith fused --tag "c4 fused" >> $OUT 2>&1
timeout 120 python tools/k1_lab.py --n 1024 --planes 64 --batch 8 --iters 10 --arith fused --tag "n1024 fused" >> $OUT 2>&1
timeout 120 python tools/k1_lab.py --n 1024 --planes 16 --batch 16 --iters 10 --arith fused --tag "c3 share fused" >> $OUT 2>&1
