mkdir -p gpurun_out
OUT=gpurun_out/lab_r02t.txt
: > $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "fused" 2>&1 | tail -2 >> $OUT
bash tools/lab_v3_ab.sh "G4RING_PDL=1" "G4RING_PDL=0" >> $OUT 2>&1
timeout 300 python tools/v3_trace.py --batch 8 --planes 64 2>&1 | grep -E "payload|span" >> $OUT
