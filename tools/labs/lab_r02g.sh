mkdir -p gpurun_out
OUT=gpurun_out/lab_r02g.txt
: > $OUT
for h in 32 48 2080 0 16; do
  echo "== hints=$h" >> $OUT
  G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --planes 256 --batch 8 --arith fused --tag "hints=$h P256" >> $OUT 2>&1
  G4RING_V3_HINTS=$h timeout 300 python tools/v3_trace.py --batch 8 --planes 256 >> $OUT 2>&1
done
