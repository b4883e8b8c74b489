# producer refill duty rotating over the warps (G4RING_ROTATE=1) vs lane 0 of warp 0.
# Record of lab33 only: the knob was removed after this measurement (no gain).
cd $GRAFT_REPO_ROOT
G4RING_ROTATE=1 timeout 300 python tools/cluster_check.py | grep -c " ok$"
L="timeout 120 python tools/k1_lab.py"
for rep in 1 2; do for r in 0 1; do
export G4RING_ROTATE=$r
$L --batch 8 --arith fused --tag "rot=$r fused B8"
$L --batch 16 --arith fused --tag "rot=$r fused B16"
$L --batch 8 --arith exact --tag "rot=$r exact B8"
$L --batch 8 --planes 8 --arith fused --tag "rot=$r fused P8"
done; done
