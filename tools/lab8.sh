# payload-fill-only (G4RING_EXP=7x) timing: TMA stage depth vs CTA tile, B=8
cd $GRAFT_REPO_ROOT
for e in 7 70 71 72 73 74; do G4RING_EXP=$e timeout 120 python tools/k1_lab.py --batch 8 --tag "fills-only exp$e"; done
for e in 7 70 71 72 73 74; do G4RING_EXP=$e timeout 120 python tools/k1_lab.py --batch 32 --iters 5 --tag "fills-only exp$e"; done
