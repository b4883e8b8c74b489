# warp-specialised K1: geometry 25 = geometry 12 + a producer warp group (setmaxnreg 24/232) (lab35; now the fused default)
cd $GRAFT_REPO_ROOT
G4RING_V2GEOM=25 timeout 300 python tools/cluster_check.py | grep -c " ok$"
L="timeout 120 python tools/k1_lab.py"
for rep in 1 2; do for g in 12 25; do
export G4RING_V2GEOM=$g
$L --batch 8 --arith fused --tag "geom $g fused B8"
$L --batch 16 --arith fused --tag "geom $g fused B16"
$L --batch 4 --arith fused --tag "geom $g fused B4"
$L --batch 8 --dtype mixed --arith fused --tag "geom $g mixed B8"
done; done
for g in 12 25; do G4RING_V2GEOM=$g $L --batch 8 --n 4608 --planes 72 --iters 3 --arith fused --tag "geom $g c4"; done
