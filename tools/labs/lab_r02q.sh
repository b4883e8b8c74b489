mkdir -p gpurun_out
OUT=gpurun_out/lab_r02q.txt
: > $OUT
for g in 148 111 74 37; do
  echo "== grid $g" >> $OUT
  G4RING_V3_GRID=$g timeout 300 python tools/v3_trace.py --batch 8 --planes 64 2>&1 | grep -E "span|tile \(|drain q0|tready|kernel span" >> $OUT
done
