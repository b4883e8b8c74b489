mkdir -p gpurun_out
OUT=gpurun_out/lab_r02u.txt
: > $OUT
for g in 13 25 12 17; do
  for b in 8 16; do
    G4RING_V2GEOM=$g timeout 120 python tools/k1_lab.py --planes 64 --batch $b --arith exact --tag "geom $g exact B=$b" >> $OUT 2>&1
  done
  G4RING_V2GEOM=$g timeout 120 python tools/k1_lab.py --n 1024 --planes 64 --batch 8 --iters 10 --arith exact --tag "geom $g exact n1024" >> $OUT 2>&1
  G4RING_V2GEOM=$g timeout 120 python tools/k1_lab.py --n 4608 --planes 72 --batch 8 --iters 3 --arith exact --tag "geom $g exact c4" >> $OUT 2>&1
done
