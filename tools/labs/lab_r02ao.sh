# L2 evict_last on the payload boxes (G4RING_V3_HINTS=2) with chaining: 5 alternations at B = 8, N = 1024
mkdir -p gpurun_out
OUT=gpurun_out/lab_r02ao.txt
: > $OUT
for rep in 1 2 3 4 5; do
  for h in 0 2; do
    G4RING_V3_HINTS=$h timeout 300 python bench.py --steps 40 --warmup 5 --batch 8 --no-cpu-baseline --skip-extras 2>/dev/null \
      | grep -E '^\{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('hints=$h B=8', '%.3e'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'us %.1f'%(d['ms_per_step']*1e3), 'clk', d['clocks']['sm_mhz'], 'parity', d['parity_check']['ok'])" >> $OUT 2>&1
  done
done
for h in 0 2 0 2; do
  G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --n 1024 --planes 64 --batch 8 --iters 10 --arith fused --tag "hints$h n1024" >> $OUT 2>&1
  G4RING_V3_HINTS=$h timeout 120 python tools/k1_lab.py --n 512 --planes 32 --batch 8 --iters 40 --arith fused --tag "hints$h P32" >> $OUT 2>&1
done
