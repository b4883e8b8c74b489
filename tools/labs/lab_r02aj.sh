# v3 geometries 40/42/43/44 at the bench shape with chaining on; P = 16/32 shares 40 vs 43
mkdir -p gpurun_out
OUT=gpurun_out/lab_r02aj.txt
: > $OUT
bash tools/lab_v3_ab.sh "G4RING_V2GEOM=40" "G4RING_V2GEOM=42" "G4RING_V2GEOM=43" "G4RING_V2GEOM=44" "G4RING_V2GEOM=40" "G4RING_V2GEOM=42" >> $OUT 2>&1
for g in 40 43 40 43; do
  G4RING_V2GEOM=$g timeout 120 python tools/k1_lab.py --n 512 --planes 32 --batch 8 --iters 40 --arith fused --tag "g$g P32" >> $OUT 2>&1
  G4RING_V2GEOM=$g timeout 120 python tools/k1_lab.py --n 512 --planes 16 --batch 8 --iters 40 --arith fused --tag "g$g P16" >> $OUT 2>&1
done
