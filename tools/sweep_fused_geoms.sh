# fused mode (deferred L2-reduction update) across geometries: big-tile layouts lose their G4 prologue
cd $GRAFT_REPO_ROOT
L="timeout 120 python tools/k1_lab.py --arith fused"
for g in 13 3 7 8 11 12 16 17; do for b in 8 16; do G4RING_V2GEOM=$g $L --batch $b --tag "fused geom $g"; done; done
for g in 13 8 12; do G4RING_V2GEOM=$g $L --batch 8 --n 4608 --planes 72 --iters 3 --tag "fused geom $g c4"; done
