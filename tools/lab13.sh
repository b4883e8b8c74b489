# 8x3 thread tiles (24 entries): geometries 21-23 against 13
cd $GRAFT_REPO_ROOT
L="timeout 120 python tools/k1_lab.py"
for g in 21 22 23; do G4RING_V2GEOM=$g timeout 300 python -m pytest tests -x -q -m gpu -k "variant or fused or full_size" 2>&1 | tail -1 | sed "s/^/geom $g tests: /"; done
for g in 13 21 22 23; do for a in exact fused; do for b in 8 16; do G4RING_V2GEOM=$g $L --batch $b --arith $a --tag "geom $g"; done; done; done
for g in 13 21 23; do G4RING_V2GEOM=$g $L --batch 8 --n 4608 --planes 72 --iters 3 --tag "geom $g c4"; done
