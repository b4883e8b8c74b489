mkdir -p gpurun_out
OUT=gpurun_out/lab_r02ab.txt
: > $OUT
for e in 0 1; do
  for a in "--n 1024 --planes 16 --batch 16 --iters 10" "--n 1024 --planes 64 --batch 16 --iters 10" "--n 1024 --planes 64 --batch 8 --iters 10" "--n 4608 --planes 72 --batch 16 --iters 3" "--n 4608 --planes 72 --batch 8 --iters 3"; do
    G4RING_V3_EARLY_ST=$e timeout 120 python tools/k1_lab.py $a --arith fused --tag "early=$e $a" >> $OUT 2>&1
  done
done
