mkdir -p gpurun_out
OUT=gpurun_out/lab_r02z.txt
: > $OUT
for g in 46 47; do
  G4RING_V2GEOM=$g timeout 900 python tools/geom_check.py 2>&1 | tail -3 >> $OUT
done
bash tools/lab_v3_ab.sh "G4RING_V2GEOM=40" "G4RING_V2GEOM=46" "G4RING_V2GEOM=47" >> $OUT 2>&1
for g in 40 46; do
  G4RING_V2GEOM=$g timeout 120 python tools/k1_lab.py --n 1024 --planes 64 --batch 8 --iters 10 --arith fused --tag "g$g n1024" >> $OUT 2>&1
done
G4RING_V2GEOM=46 timeout 300 python tools/v3_trace.py --batch 8 --planes 64 2>&1 | grep -E "fill|span|tile \(" >> $OUT
