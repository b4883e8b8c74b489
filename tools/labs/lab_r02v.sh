mkdir -p gpurun_out
OUT=gpurun_out/lab_r02v.txt
: > $OUT
timeout 1200 python -m pytest tests/test_gpu_headline.py tests/test_gpu_kernels.py -x -q 2>&1 | tail -2 >> $OUT
G4RING_V3_EXACT=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "fused or variant or random" 2>&1 | tail -1 >> $OUT
timeout 1800 bash tools/sanitize_v3.sh >> $OUT 2>&1
