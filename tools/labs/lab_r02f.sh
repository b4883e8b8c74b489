mkdir -p gpurun_out
OUT=gpurun_out/lab_r02f.txt
: > $OUT
for h in 0 64 66 96 352; do
  G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --planes 64 --batch 8 --arith fused --tag "hints=$h" >> $OUT 2>&1
  G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --planes 256 --batch 8 --arith fused --tag "hints=$h P256" >> $OUT 2>&1
done
