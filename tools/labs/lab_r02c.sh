# round-2 lab: v3 inner-loop ceiling, per-tile timeline, geometry / knob A/B (GPU box)
mkdir -p gpurun_out
OUT=gpurun_out/lab_r02c.txt
echo "== k1_core_bench" > $OUT
timeout 120 ./tools/k1_core_bench.bin >> $OUT 2>&1
echo "== v3_trace B=8" >> $OUT
timeout 300 python tools/v3_trace.py --batch 8 >> $OUT 2>&1
echo "== knob A/B (bench shape)" >> $OUT
timeout 1500 bash tools/lab_v3_ab.sh "G4RING_V3_HINTS=0" "G4RING_V3_HINTS=16" "G4RING_V3_HINTS=1" "G4RING_V3_HINTS=2" \
   "G4RING_V2GEOM=42" "G4RING_V2GEOM=43" "G4RING_V2GEOM=44" "G4RING_V2GEOM=25" "G4RING_V3_HINTS=256" >> $OUT 2>&1
echo "== c4 share" >> $OUT
for g in 40 43 25 12; do
  G4RING_V2GEOM=$g timeout 300 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --skip-extras 2>/dev/null | grep -E '^\{' | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 geom $g', '%.3e'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'ms %.2f'%d['ms_per_step'])" >> $OUT 2>&1
done
