# persistent v2 (geometry 30 = 13 persistent, 31 = 19 persistent) with next-tile L2 prefetch
cd $GRAFT_REPO_ROOT
L="timeout 120 python tools/k1_lab.py"
for g in 30 31; do G4RING_V2GEOM=$g timeout 300 python -m pytest tests -x -q -m gpu -k "variant or fused or full_size or mixed or complex64" 2>&1 | tail -1 | sed "s/^/geom $g tests: /"; done
for g in 13 30; do for b in 1 8 16; do G4RING_V2GEOM=$g $L --batch $b --tag "geom $g"; done; G4RING_V2GEOM=$g $L --batch 8 --arith fused --tag "geom $g"; done
for g in 19 31; do G4RING_V2GEOM=$g $L --batch 8 --planes 8 --tag "geom $g p8"; done
for g in 13 30; do G4RING_V2GEOM=$g $L --batch 8 --n 4608 --planes 72 --iters 3 --tag "geom $g c4"; done
