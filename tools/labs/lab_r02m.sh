mkdir -p gpurun_out
OUT=gpurun_out/lab_r02m.txt
: > $OUT
for e in "G4RING_V3_SCHED=0 G4RING_PDL=0 G4RING_V2GEOM=40" "G4RING_V3_SCHED=0 G4RING_PDL=0 G4RING_V2GEOM=43" "G4RING_V3_SCHED=0 G4RING_PDL=1 G4RING_V2GEOM=43" "G4RING_V3_SCHED=1 G4RING_PDL=0 G4RING_V2GEOM=43"; do
  echo "== $e" >> $OUT
  env $e timeout 600 python -m pytest tests/test_gpu_headline.py -x -q -k "config4_share" 2>&1 | grep -E "passed|failed|Error|error|assert" | head -5 >> $OUT
done
