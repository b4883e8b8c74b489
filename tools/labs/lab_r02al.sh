# 1-3 walkers a pass in fused mode: the exact kernel (default below 4 walkers) against the deferred,
# now chained, v2 kernel (G4RING_DEFER_MIN_WALKERS=1)
mkdir -p gpurun_out
OUT=gpurun_out/lab_r02al.txt
: > $OUT
for rep in 1 2; do
for cfg in "G4RING_DEFER_MIN_WALKERS=4" "G4RING_DEFER_MIN_WALKERS=1"; do
  for b in 1 2 3; do
    env $cfg timeout 300 python bench.py --steps 30 --warmup 5 --batch $b --no-cpu-baseline --skip-extras 2>/dev/null \
      | grep -E '^\{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg B=$b', '%.3e'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'us %.1f'%(d['ms_per_step']*1e3), 'clk', d['clocks']['sm_mhz'], 'geom', d.get('launched_k1_geometry'), 'parity', d['parity_check']['ok'])" >> $OUT 2>&1
  done
done
done
for cfg in "G4RING_DEFER_MIN_WALKERS=4" "G4RING_DEFER_MIN_WALKERS=1"; do
  env $cfg timeout 200 python tools/k1_lab.py --n 4608 --planes 72 --batch 1 --iters 3 --arith fused --tag "$cfg c4 B1" >> $OUT 2>&1
  env $cfg timeout 120 python tools/k1_lab.py --n 512 --planes 8 --batch 1 --iters 40 --arith fused --tag "$cfg P8 B1" >> $OUT 2>&1
done
