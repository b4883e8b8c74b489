# geometry 27 = geometry 19 (P < 16 default) + a producer warp group, 3 CTAs/SM (lab36)
cd $GRAFT_REPO_ROOT
G4RING_V2GEOM=27 timeout 300 python tools/cluster_check.py | grep -c " ok$"
L="timeout 120 python tools/k1_lab.py --arith fused --planes 8"
for rep in 1 2; do for g in 19 27; do
G4RING_V2GEOM=$g $L --batch 8 --tag "geom $g P8 B8"; G4RING_V2GEOM=$g $L --batch 16 --tag "geom $g P8 B16"; G4RING_V2GEOM=$g $L --batch 8 --n 1024 --tag "geom $g P8 N1024"
done; done
