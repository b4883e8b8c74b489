# Cluster-multicast K1 geometries (21/22 = fused default 12 with band multicast over
# 4/2 CTAs, 23/24 = exact default 13 likewise): parity first, then timing vs 12/13.
cd $GRAFT_REPO_ROOT
for g in 21 22 23 24; do echo "== parity geom $g"; G4RING_V2GEOM=$g timeout 300 python tools/cluster_check.py || echo "PARITY FAIL geom $g"; done
L="timeout 120 python tools/k1_lab.py"
for rep in 1 2; do
for g in 12 21 22; do for b in 8 16; do G4RING_V2GEOM=$g $L --arith fused --batch $b --tag "fused geom $g"; done; done
for g in 13 23 24; do for b in 1 8; do G4RING_V2GEOM=$g $L --arith exact --batch $b --tag "exact geom $g"; done; done
done
for g in 12 21; do G4RING_V2GEOM=$g $L --arith fused --batch 8 --n 4608 --planes 64 --iters 3 --tag "fused geom $g c4-64"; done
for g in 12 21; do G4RING_V2GEOM=$g $L --arith fused --batch 8 --dtype c64 --tag "fused geom $g c64"; done
