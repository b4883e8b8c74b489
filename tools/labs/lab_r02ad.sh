mkdir -p gpurun_out
OUT=gpurun_out/lab_r02ad.txt
: > $OUT
# geometry 48: geometry 40 in CTA pairs sharing the direct box by TMA multicast
G4RING_V2GEOM=48 timeout 600 python tools/geom_check.py 2>&1 | tail -8 >> $OUT
bash tools/lab_v3_ab.sh "G4RING_V2GEOM=40" "G4RING_V2GEOM=48" "G4RING_V2GEOM=40" "G4RING_V2GEOM=48" >> $OUT 2>&1
for g in 40 48; do
  G4RING_V2GEOM=$g timeout 120 python tools/k1_lab.py --n 1024 --planes 64 --batch 8 --iters 10 --arith fused --tag "g$g n1024" >> $OUT 2>&1
  G4RING_V2GEOM=$g timeout 120 python tools/k1_lab.py --n 4608 --planes 72 --batch 8 --iters 3 --arith fused --tag "g$g c4" >> $OUT 2>&1
done
