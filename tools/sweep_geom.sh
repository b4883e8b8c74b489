# v2 geometry sweep: parity subset + throughput for each G4RING_V2GEOM and arith mode
for g in ${GEOMS:-0 1 2}; do
  G4RING_V2GEOM=$g timeout 300 python -m pytest tests -x -q -m gpu -k "variant or fused or full_size" 2>&1 | tail -1 | sed "s/^/geom $g tests: /"
  for a in exact fused; do for b in 8 16; do
    G4RING_V2GEOM=$g timeout 120 python bench.py --steps 10 --warmup 3 --batch $b --no-cpu-baseline --arith $a 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('geom $g', '$a', d['config']['walkers_per_pass'], '%.3e'%d['value'], 'frac %.3f'%d['roofline']['frac'])"
  done; done
done
