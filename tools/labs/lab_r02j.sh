mkdir -p gpurun_out
OUT=gpurun_out/lab_r02j.txt
: > $OUT
G4RING_V3_HINTS=131072 timeout 900 python -m pytest tests/test_gpu_headline.py -x -q 2>&1 | tail -3 >> $OUT
for h in 0 131072 131074; do
  G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --planes 64 --batch 8 --arith fused --tag "hints=$h" >> $OUT 2>&1
  G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --planes 256 --batch 8 --arith fused --tag "hints=$h P256" >> $OUT 2>&1
  G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --planes 64 --batch 16 --arith fused --tag "hints=$h B16" >> $OUT 2>&1
  G4RING_V2GEOM=43 G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --planes 64 --batch 8 --arith fused --tag "g43 hints=$h" >> $OUT 2>&1
  G4RING_V2GEOM=43 G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --n 4608 --planes 72 --batch 8 --iters 3 --arith fused --tag "g43 c4 hints=$h" >> $OUT 2>&1
done
G4RING_V3_HINTS=131072 timeout 300 python tools/v3_trace.py --batch 8 --planes 64 >> $OUT 2>&1
