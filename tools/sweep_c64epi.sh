# complex64 slices through the park + TMA bulk epilogue (aligned segments, LSU edges)
cd $GRAFT_REPO_ROOT
timeout 300 python tools/cluster_check.py | grep -c " ok$"
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu 2>&1 | tail -1
L="timeout 120 python tools/k1_lab.py --dtype c64"
for rep in 1 2; do
for b in 1 8; do $L --batch $b --arith exact --tag "c64 exact"; G4RING_BULK_STORE=0 $L --batch $b --arith exact --tag "c64 exact st.cs"; done
for b in 8 16; do $L --batch $b --arith fused --tag "c64 fused"; done
$L --batch 8 --planes 8 --arith fused --tag "c64 fused P8"
$L --batch 8 --n 4608 --planes 72 --iters 3 --arith fused --tag "c64 fused c4"
done
