mkdir -p gpurun_out
OUT=gpurun_out/lab_r02k.txt
: > $OUT
bash tools/lab_v3_ab.sh "G4RING_V3_HINTS=0" "G4RING_V3_HINTS=262144" "G4RING_V3_HINTS=262146" "G4RING_V3_HINTS=262145" >> $OUT 2>&1
for h in 0 262144; do
  G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --planes 256 --batch 8 --arith fused --tag "hints=$h P256" >> $OUT 2>&1
  G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --planes 32 --batch 8 --arith fused --tag "hints=$h P32" >> $OUT 2>&1
  G4RING_V2GEOM=43 G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --n 4608 --planes 72 --batch 8 --iters 3 --arith fused --tag "g43 c4 hints=$h" >> $OUT 2>&1
done
