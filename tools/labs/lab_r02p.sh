mkdir -p gpurun_out
OUT=gpurun_out/lab_r02p.txt
: > $OUT
timeout 300 python tools/v3_trace.py --batch 8 --planes 256 >> $OUT 2>&1
timeout 300 python tools/v3_trace.py --batch 8 --planes 64 >> $OUT 2>&1
