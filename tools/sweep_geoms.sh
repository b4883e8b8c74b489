# geometry sweep: parity subset + K1 timing per G4RING_V2GEOM
cd $GRAFT_REPO_ROOT
L="timeout 120 python tools/k1_lab.py"
for g in ${GEOMS:-3 13 19 12}; do
  G4RING_V2GEOM=$g timeout 300 python -m pytest tests -x -q -m gpu -k "variant or fused or full_size" 2>&1 | tail -1 | sed "s/^/geom $g tests: /"
  for a in exact fused; do for b in 8 16; do G4RING_V2GEOM=$g $L --batch $b --arith $a --tag "geom $g"; done; done
  G4RING_V2GEOM=$g $L --batch 8 --n 4608 --planes 72 --iters 3 --tag "geom $g c4"
done
