# where does the deferred (bulk-reduce) update pay?  walkers 1/2/4 at P = 64, and P = 8 (ring share at 8 GPUs)
cd $GRAFT_REPO_ROOT
L="timeout 120 python tools/k1_lab.py --arith fused"
for rep in 1 2; do
for b in 1 2 4; do $L --batch $b --tag "fused"; G4RING_DEFER_MIN_WALKERS=1 $L --batch $b --tag "fused defer>=1"; done
for b in 1 8; do $L --batch $b --planes 8 --tag "fused P8"; G4RING_DEFER_MIN_WALKERS=1 G4RING_DEFER_MIN_PLANES=1 $L --batch $b --planes 8 --tag "fused P8 defer"; done
for b in 1 8; do $L --batch $b --planes 16 --n 1024 --tag "fused c3"; G4RING_DEFER_MIN_WALKERS=1 $L --batch $b --planes 16 --n 1024 --tag "fused c3 defer>=1"; done
done
