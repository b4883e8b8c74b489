# complex64 slices: v3 geometry 45 (opt-in) chained like the others, against geometry 12 (chained)
mkdir -p gpurun_out
OUT=gpurun_out/lab_r02ak.txt
: > $OUT
G4RING_V3_C64=1 timeout 600 python -m pytest tests/test_gpu_chain.py -x -q -k c64 2>&1 | tail -2 | tee -a $OUT | grep -q " passed" || exit 1
G4RING_V3_C64=1 G4RING_V2GEOM=45 timeout 600 python tools/geom_check.py 2>&1 | grep c64 >> $OUT
for v in 0 1 0 1; do
  G4RING_V3_C64=$v timeout 120 python tools/k1_lab.py --n 512 --planes 64 --batch 8 --dtype c64 --iters 20 --arith fused --tag "v3c64=$v B8" >> $OUT 2>&1
  G4RING_V3_C64=$v timeout 120 python tools/k1_lab.py --n 512 --planes 64 --batch 16 --dtype c64 --iters 20 --arith fused --tag "v3c64=$v B16" >> $OUT 2>&1
  G4RING_V3_C64=$v timeout 200 python tools/k1_lab.py --n 4608 --planes 72 --batch 8 --dtype c64 --iters 3 --arith fused --tag "v3c64=$v c4" >> $OUT 2>&1
done
