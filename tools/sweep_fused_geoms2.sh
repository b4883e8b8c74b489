# fused mode across geometries after the TMA write-back (lab32)
cd $GRAFT_REPO_ROOT
L="timeout 120 python tools/k1_lab.py --arith fused"
for g in 12 13 3 7 11 16 17 20 8; do for b in 8 16; do G4RING_V2GEOM=$g $L --batch $b --tag "fused geom $g"; done; done
for g in 12 13 17; do G4RING_V2GEOM=$g $L --batch 8 --n 4608 --planes 72 --iters 3 --tag "fused geom $g c4"; done
for g in 19 20 13; do G4RING_V2GEOM=$g $L --batch 8 --planes 8 --tag "fused geom $g P8"; done
