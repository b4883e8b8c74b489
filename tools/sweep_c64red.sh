# complex64 deferred update: one red.global.add.v2.f32 per entry vs two scalar reds (G4RING_SCALAR_RED=1) (lab34)
cd $GRAFT_REPO_ROOT
timeout 300 python tools/cluster_check.py | grep -c " ok$"
L="timeout 120 python tools/k1_lab.py --dtype c64 --arith fused"
for rep in 1 2; do for sc in 0 1; do
export G4RING_SCALAR_RED=$sc
$L --batch 8 --tag "scalar=$sc c64 B8"; $L --batch 16 --tag "scalar=$sc c64 B16"; $L --batch 4 --tag "scalar=$sc c64 B4"; $L --batch 8 --planes 8 --tag "scalar=$sc c64 P8"
done; done
for sc in 0 1; do G4RING_SCALAR_RED=$sc $L --batch 8 --n 4608 --planes 72 --iters 3 --tag "scalar=$sc c64 c4"; done
