# persistent geometry 13 (30) vs 13: grid sizes, then one ncu capture each at B = 1
cd $GRAFT_REPO_ROOT
L="timeout 120 python tools/k1_lab.py --batch 1 --iters 20"
G4RING_V2GEOM=13 $L --tag "g13"
for grid in 592 1184 2368 4096 8192; do G4RING_PERS_GRID=$grid G4RING_V2GEOM=30 $L --tag "pers grid $grid"; done
G4RING_V2GEOM=30 ncu --set full --clock-control none -k regex:k_accumulate -s 3 -c 1 -o gpurun_out/pers_b1 python tools/k1_lab.py --batch 1 --iters 2 > /dev/null 2>&1
G4RING_V2GEOM=13 ncu --set full --clock-control none -k regex:k_accumulate -s 3 -c 1 -o gpurun_out/g13_b1 python tools/k1_lab.py --batch 1 --iters 2 > /dev/null 2>&1
ls gpurun_out | grep _b1
