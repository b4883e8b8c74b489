# G4 stores interleaved into the last walker (default) vs at CTA end (G4RING_EXP=8)
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -x -q -m gpu -k "variant or fused or full_size or mixed or complex64 or guard or identity" 2>&1 | tail -1
L="timeout 120 python tools/k1_lab.py"
for e in 0 8; do for b in 1 8 16; do G4RING_EXP=$e $L --batch $b --tag "g13 exp$e"; done; G4RING_EXP=$e $L --batch 8 --arith fused --tag "g13 fused exp$e"; done
for e in 0 8; do G4RING_EXP=$e $L --batch 8 --n 4608 --planes 72 --iters 3 --tag "g13 c4 exp$e"; G4RING_EXP=$e $L --batch 8 --planes 8 --tag "p8 exp$e"; done
