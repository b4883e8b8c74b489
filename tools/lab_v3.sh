# K1 v3 (persistent TMEM-handoff kernel) lab: parity then timing per geometry.
# usage (GPU box): bash tools/lab_v3.sh <tag> [geoms...]
TAG=${1:-v3}; shift
GEOMS=${@:-40 42}
mkdir -p gpurun_out
for g in $GEOMS; do
  echo "== parity geom $g"
  G4RING_V2GEOM=$g timeout 300 python tools/geom_check.py 2>&1 | grep -E "fused|Error|error" | head -14
done
for g in 25 $GEOMS; do
  for b in 8 16; do
    G4RING_V2GEOM=$g timeout 300 python bench.py --steps 20 --warmup 5 --batch $b --no-cpu-baseline 2>/dev/null \
      | grep -E '^\{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('geom $g B=$b', '%.3e'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'us %.1f'%(d['ms_per_step']*1e3), 'parity', d['parity_check']['ok'], d['parity_check']['max_rel_err'])"
  done
done
