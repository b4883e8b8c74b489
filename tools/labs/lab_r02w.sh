mkdir -p gpurun_out
OUT=gpurun_out/lab_r02w.txt
: > $OUT
G4RING_V3_C64=1 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_headline.py -x -q -k "c64 or complex64 or fused or many or deferred" 2>&1 | tail -2 >> $OUT
for e in "G4RING_V3_C64=0" "G4RING_V3_C64=1"; do
  for b in 8 16; do
    env $e timeout 120 python tools/k1_lab.py --planes 64 --batch $b --dtype c64 --arith fused --tag "$e c64 B=$b" >> $OUT 2>&1
  done
  env $e timeout 120 python tools/k1_lab.py --n 4608 --planes 72 --batch 8 --iters 3 --dtype c64 --arith fused --tag "$e c64 c4" >> $OUT 2>&1
  env $e timeout 120 python tools/k1_lab.py --n 1024 --planes 64 --batch 8 --iters 10 --dtype c64 --arith fused --tag "$e c64 n1024" >> $OUT 2>&1
done
G4RING_V3_C64=1 timeout 300 python bench.py --dtype c64 --steps 20 --warmup 5 --no-cpu-baseline --skip-extras 2>/dev/null | grep -E '^\{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench c64 v3', '%.3e'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'parity', d['parity_check'])" >> $OUT 2>&1
