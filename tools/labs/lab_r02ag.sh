# v3: consumer warps whose planes lie past the slice end (config 4's 72 planes = 4.5 chunks of 16)
# skip loads, math and TMEM stores; A/B via G4RING_V3_HINTS=128 (skip off)
mkdir -p gpurun_out
OUT=gpurun_out/lab_r02ag.txt
: > $OUT
timeout 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_headline.py -x -q 2>&1 | tail -2 | tee -a $OUT | grep -q " passed" || exit 1
timeout 600 python tools/geom_check.py 2>&1 | tail -12 >> $OUT
for h in 128 0 128 0; do
  G4RING_V3_HINTS=$h timeout 200 python tools/k1_lab.py --n 4608 --planes 72 --batch 8 --iters 4 --arith fused --tag "hints$h c4" >> $OUT 2>&1
  G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --n 1024 --planes 24 --batch 8 --iters 20 --arith fused --tag "hints$h n1024 P24" >> $OUT 2>&1
done
bash tools/lab_v3_ab.sh "G4RING_V3_HINTS=128" "G4RING_V3_HINTS=0" "G4RING_V3_HINTS=128" "G4RING_V3_HINTS=0" >> $OUT 2>&1
timeout 300 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -E '^\{' | tail -1 > gpurun_out/bench_r02ag_c4.json
