cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L="timeout 120 python tools/k1_lab.py"
for b in 1 8 16; do $L --batch $b --tag "exp0"; done
for e in 3 4 7 8; do for b in 8 16; do G4RING_EXP=$e $L --batch $b --tag "exp$e"; done; done
for e in 0 3 8; do G4RING_EXP=$e $L --batch 8 --arith fused --tag "fused exp$e"; done
$L --batch 8 --dtype mixed --tag mixed
$L --batch 8 --dtype c64 --tag c64
$L --batch 8 --n 4608 --planes 72 --iters 3 --tag "c4 exp0"
G4RING_EXP=8 $L --batch 8 --n 4608 --planes 72 --iters 3 --tag "c4 exp8"
G4RING_EXP=3 $L --batch 8 --n 4608 --planes 72 --iters 3 --tag "c4 exp3"
