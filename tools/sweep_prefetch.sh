# shifted-operand prefetch distance (V2Geom PF): geometry 13 (PF 1) vs 26 (PF 2), 27 (PF 3); 3 (4x4, PF 1) vs 28 (PF 2)
cd $GRAFT_REPO_ROOT
L="timeout 120 python tools/k1_lab.py"
for g in 26 27 28; do G4RING_V2GEOM=$g timeout 300 python -m pytest tests -x -q -m gpu -k "variant or fused or full_size or mixed or complex64" 2>&1 | tail -1 | sed "s/^/geom $g tests: /"; done
for g in 13 26 27 3 28; do for b in 8 16; do G4RING_V2GEOM=$g $L --batch $b --tag "geom $g"; done; G4RING_V2GEOM=$g $L --batch 8 --arith fused --tag "geom $g"; G4RING_V2GEOM=$g $L --batch 8 --dtype mixed --tag "geom $g"; done
for g in 13 26 27; do G4RING_V2GEOM=$g $L --batch 8 --n 4608 --planes 72 --iters 3 --tag "geom $g c4"; done
