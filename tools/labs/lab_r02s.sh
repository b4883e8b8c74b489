mkdir -p gpurun_out
OUT=gpurun_out/lab_r02s.txt
: > $OUT
G4RING_V3_HINTS=4 timeout 900 python -m pytest tests/test_gpu_headline.py -x -q 2>&1 | tail -2 >> $OUT
bash tools/lab_v3_ab.sh "G4RING_V3_HINTS=0" "G4RING_V3_HINTS=4" "G4RING_V3_HINTS=6" >> $OUT 2>&1
G4RING_V3_HINTS=4 timeout 300 python tools/v3_trace.py --batch 8 --planes 64 2>&1 | grep -E "drain|tready|span|tile \(" >> $OUT
for h in 0 4; do
  G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --planes 256 --batch 8 --arith fused --tag "hints=$h P256" >> $OUT 2>&1
  G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --n 4608 --planes 72 --batch 8 --iters 3 --arith fused --tag "hints=$h c4" >> $OUT 2>&1
  G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --n 1024 --planes 64 --batch 8 --iters 10 --arith fused --tag "hints=$h n1024" >> $OUT 2>&1
done
