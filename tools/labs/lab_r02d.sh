mkdir -p gpurun_out
OUT=gpurun_out/lab_r02d.txt
echo "== v3_trace B=8" > $OUT
timeout 300 python tools/v3_trace.py --batch 8 >> $OUT 2>&1
echo "== v3_trace B=8 G4RING_V3_HINTS=256" >> $OUT
G4RING_V3_HINTS=256 timeout 300 python tools/v3_trace.py --batch 8 >> $OUT 2>&1
echo "== plane sweep (fixed cost per launch)" >> $OUT
for p in 16 32 64 128 256; do timeout 300 python tools/k1_lab.py --planes $p --batch 8 --arith fused --tag "p=$p" >> $OUT 2>&1; done
