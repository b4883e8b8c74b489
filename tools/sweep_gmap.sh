# K1 write-back of interior blocks as ONE sheared tensor-map box per warp (G4RING_GMAP=1, default)
# vs 32 per-segment bulk ops (G4RING_GMAP=0)
cd $GRAFT_REPO_ROOT
timeout 300 python tools/cluster_check.py | grep -c " ok$"
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu 2>&1 | tail -1
L="timeout 120 python tools/k1_lab.py"
for rep in 1 2; do
for m in 1 0; do
export G4RING_GMAP=$m
$L --batch 8 --arith fused --tag "gmap=$m fused B8"
$L --batch 16 --arith fused --tag "gmap=$m fused B16"
$L --batch 1 --arith exact --tag "gmap=$m exact B1"
$L --batch 8 --arith exact --tag "gmap=$m exact B8"
$L --batch 8 --planes 8 --arith fused --tag "gmap=$m fused P8"
done
done
for m in 1 0; do G4RING_GMAP=$m $L --batch 8 --n 4608 --planes 72 --iters 3 --arith fused --tag "gmap=$m c4"; done
