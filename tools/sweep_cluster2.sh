cd $GRAFT_REPO_ROOT
G4RING_V2GEOM=21 timeout 300 python tools/cluster_check.py | grep -c " ok$"
L="timeout 120 python tools/k1_lab.py"
for g in 12 21 22; do for b in 8 16; do G4RING_V2GEOM=$g $L --arith fused --batch $b --tag "fused geom $g"; done; done
for g in 13 23 24; do for b in 1 8; do G4RING_V2GEOM=$g $L --arith exact --batch $b --tag "exact geom $g"; done; done
G4RING_V2GEOM=22 timeout 300 ncu --set full --clock-control none -k regex:k_accumulate -s 3 -c 1 -o gpurun_out/cl2_g22 python tools/k1_lab.py --arith fused --batch 8 --iters 2 > /dev/null 2>&1
