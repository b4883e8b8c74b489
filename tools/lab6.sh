# v4 (persistent, TMA-staged G4 blocks): parity subset + K1 timing per G4RING_V4GEOM
cd $GRAFT_REPO_ROOT
L="timeout 120 python tools/k1_lab.py"
timeout 600 python -m pytest tests -x -q -m gpu -k "variant or fused or mixed or complex64" 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -12
for g in ${GEOMS:-0 1 2 3}; do
  G4RING_KERNEL=3 G4RING_V4GEOM=$g timeout 300 python -m pytest tests -x -q -m gpu -k "variant or fused or full_size or mixed" 2>&1 | tail -1 | sed "s/^/v4 geom $g tests: /"
  for a in exact fused; do for b in 8 16; do G4RING_KERNEL=3 G4RING_V4GEOM=$g $L --batch $b --arith $a --tag "v4 geom $g"; done; done
  G4RING_KERNEL=3 G4RING_V4GEOM=$g $L --batch 1 --tag "v4 geom $g"
  G4RING_KERNEL=3 G4RING_V4GEOM=$g $L --batch 8 --dtype mixed --tag "v4 geom $g"
  G4RING_KERNEL=3 G4RING_V4GEOM=$g $L --batch 8 --n 4608 --planes 72 --iters 3 --tag "v4 geom $g c4"
done
