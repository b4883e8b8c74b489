mkdir -p gpurun_out
OUT=gpurun_out/lab_r02e.txt
: > $OUT
for h in 0 2 4096 8192 4098 8194 32 288; do
  G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --planes 64 --batch 8 --arith fused --tag "hints=$h" >> $OUT 2>&1
  G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --planes 256 --batch 8 --arith fused --tag "hints=$h P256" >> $OUT 2>&1
done
for h in 0 2 4096 8192; do
  G4RING_V2GEOM=43 G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --n 4608 --planes 72 --batch 8 --iters 3 --arith fused --tag "g43 c4 hints=$h" >> $OUT 2>&1
done
