# deferred G4 update with red.global.add (G4RING_EXP=16) vs load/store (0), geometry 13
cd $GRAFT_REPO_ROOT
L="timeout 120 python tools/k1_lab.py"
for e in 0 16; do for b in 1 8 16; do for a in exact fused; do G4RING_EXP=$e $L --batch $b --arith $a --tag "exp$e"; done; done; done
for e in 0 16; do G4RING_EXP=$e $L --batch 8 --n 4608 --planes 72 --iters 3 --arith fused --tag "c4 exp$e"; done
