# plane-count dependence of the K1 choice (v1 vs v2 geometries), B = 8
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for g in 19 20 13; do G4RING_V2GEOM=$g timeout 300 python -m pytest tests -x -q -m gpu -k "variant or fused or full_size or mixed or complex64" 2>&1 | tail -1 | sed "s/^/geom $g tests: /"; done
L="timeout 120 python tools/k1_lab.py --batch 8"
for P in 4 8 16 64; do
  G4RING_KERNEL=1 $L --planes $P --tag "v1"
  for g in 19 20 13 3; do G4RING_V2GEOM=$g $L --planes $P --tag "geom $g"; done
done
for g in 19 13 3; do for d in c64 mixed; do G4RING_V2GEOM=$g $L --dtype $d --tag "geom $g"; done; done
G4RING_KERNEL=1 $L --n 4608 --planes 8 --iters 3 --tag "v1 c4-8"
G4RING_V2GEOM=19 $L --n 4608 --planes 8 --iters 3 --tag "geom 19 c4-8"
