# where the G4 phase costs go (geometry 13, B = 8 and 16): G4RING_EXP stripped variants
cd $GRAFT_REPO_ROOT
L="timeout 120 python tools/k1_lab.py"
for b in 8 16; do for e in 0 1 2 3 4 7; do G4RING_EXP=$e $L --batch $b --tag "g13 exp$e"; done; done
for e in 0 1 2 3; do G4RING_EXP=$e $L --batch 8 --arith fused --tag "g13 fused exp$e"; done
