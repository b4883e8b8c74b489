# exact-mode write-back by TMA bulk store (G4RING_BULK_STORE=1) vs st.global.cs
cd $GRAFT_REPO_ROOT
G4RING_BULK_STORE=1 timeout 300 python tools/cluster_check.py | grep -c " ok$"
L="timeout 120 python tools/k1_lab.py --arith exact"
for rep in 1 2; do
for b in 1 8; do $L --batch $b --tag "exact"; G4RING_BULK_STORE=1 $L --batch $b --tag "exact bulkst"; done
for b in 1 8; do $L --batch $b --planes 8 --tag "exact P8"; G4RING_BULK_STORE=1 $L --batch $b --planes 8 --tag "exact P8 bulkst"; done
$L --batch 1 --arith fused --tag "fused B1"; G4RING_BULK_STORE=1 $L --batch 1 --arith fused --tag "fused B1 bulkst"
done
$L --batch 8 --n 4608 --planes 72 --iters 3 --tag "exact c4"; G4RING_BULK_STORE=1 $L --batch 8 --n 4608 --planes 72 --iters 3 --tag "exact c4 bulkst"
