# K1 v3 A/B of environment knobs at the bench shape (GPU box):
#   bash tools/lab_v3_ab.sh "G4RING_V3_HINTS=0" "G4RING_V3_HINTS=1" ...
for cfg in "$@"; do
  for b in 8 16; do
    env $cfg timeout 300 python bench.py --steps 30 --warmup 5 --batch $b --no-cpu-baseline --skip-extras 2>/dev/null \
      | grep -E '^\{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg B=$b', '%.3e'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'us %.1f'%(d['ms_per_step']*1e3), 'clk', d['clocks']['sm_mhz'], 'parity', d['parity_check']['ok'])"
  done
done
