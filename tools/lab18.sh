# 8x2 thread blocks in 8-warp CTAs (16x8 tile, fills 7.75 B/update): geometries 24/25 vs 13
cd $GRAFT_REPO_ROOT
L="timeout 120 python tools/k1_lab.py"
for g in 24 25; do G4RING_V2GEOM=$g timeout 300 python -m pytest tests -x -q -m gpu -k "variant or fused or full_size" 2>&1 | tail -1 | sed "s/^/geom $g tests: /"; done
for g in 13 24 25; do for b in 8 16; do G4RING_V2GEOM=$g $L --batch $b --tag "geom $g"; done; G4RING_V2GEOM=$g $L --batch 8 --arith fused --tag "geom $g"; done
for g in 13 24 25; do G4RING_V2GEOM=$g $L --batch 8 --n 4608 --planes 72 --iters 3 --tag "geom $g c4"; done
