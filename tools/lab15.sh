# G4 load/store cache policies (geometry 13)
cd $GRAFT_REPO_ROOT
L="timeout 120 python tools/k1_lab.py"
for e in 0 32 64 256; do for b in 1 8 16; do G4RING_EXP=$e $L --batch $b --tag "g13 exp$e"; done; done
for e in 0 32 64 256; do G4RING_EXP=$e $L --batch 8 --n 4608 --planes 72 --iters 3 --tag "g13 c4 exp$e"; done
