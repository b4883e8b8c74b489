# v3 (persistent) geometry sweep: parity subset + K1 timing per G4RING_V3GEOM
cd $GRAFT_REPO_ROOT
L="timeout 120 python tools/k1_lab.py"
timeout 600 python -m pytest tests -x -q -m gpu -k "variant or fused or mixed or complex64" 2>&1 | tail -2
for g in ${GEOMS:-0 1 2 3 4 5}; do
  G4RING_KERNEL=3 G4RING_V3GEOM=$g timeout 300 python -m pytest tests -x -q -m gpu -k "variant or fused or full_size" 2>&1 | tail -1 | sed "s/^/v3 geom $g tests: /"
  for a in exact fused; do for b in 8 16; do G4RING_KERNEL=3 G4RING_V3GEOM=$g $L --batch $b --arith $a --tag "v3 geom $g"; done; done
  G4RING_KERNEL=3 G4RING_V3GEOM=$g $L --batch 8 --n 4608 --planes 72 --iters 3 --tag "v3 geom $g c4"
done
