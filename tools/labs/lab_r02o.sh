mkdir -p gpurun_out
OUT=gpurun_out/lab_r02o.txt
: > $OUT
G4RING_V3_EXACT=1 timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_kernels.py -x -q 2>&1 | tail -3 >> $OUT
for e in "G4RING_V3_EXACT=0" "G4RING_V3_EXACT=1"; do
  for b in 8 16; do
    env $e timeout 120 python tools/k1_lab.py --planes 64 --batch $b --arith exact --tag "$e B=$b" >> $OUT 2>&1
  done
  env $e timeout 120 python tools/k1_lab.py --n 1024 --planes 64 --batch 8 --iters 10 --arith exact --tag "$e n1024" >> $OUT 2>&1
  env $e timeout 120 python tools/k1_lab.py --n 4608 --planes 72 --batch 8 --iters 3 --arith exact --tag "$e c4" >> $OUT 2>&1
done
G4RING_V3_EXACT=1 timeout 300 python bench.py --arith exact --steps 20 --warmup 5 --no-cpu-baseline --skip-extras 2>/dev/null | grep -E '^\{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench exact v3', '%.3e'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'parity', d['parity_check'])" >> $OUT 2>&1
