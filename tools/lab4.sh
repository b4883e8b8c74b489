cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -x -q -m gpu -k "variant or fused or mixed or complex64" 2>&1 | grep -E "Error|error|assert|FAIL|passed|failed" | head -20
B="python tools/k1_lab.py --batch 8 --iters 2"
ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 3 -c 1 -o gpurun_out/g3_exact $B > /dev/null 2>&1
G4RING_V2GEOM=12 ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 3 -c 1 -o gpurun_out/g12_exact $B > /dev/null 2>&1
G4RING_V2GEOM=12 ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 3 -c 1 -o gpurun_out/g12_fused $B --arith fused > /dev/null 2>&1
G4RING_KERNEL=3 ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 3 -c 1 -o gpurun_out/v3g0_exact $B > /dev/null 2>&1
G4RING_EXP=3 ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 3 -c 1 -o gpurun_out/g3_exp3 $B --arith fused > /dev/null 2>&1
ls -la gpurun_out
