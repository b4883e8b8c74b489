mkdir -p gpurun_out
OUT=gpurun_out/lab_r02l.txt
: > $OUT
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_kernels.py -x -q 2>&1 | tail -3 >> $OUT
bash tools/lab_v3_ab.sh "G4RING_V3_SCHED=0 G4RING_PDL=0" "G4RING_V3_SCHED=1 G4RING_PDL=0" "G4RING_V3_SCHED=0 G4RING_PDL=1" "G4RING_V3_SCHED=1 G4RING_PDL=1" "G4RING_V3_SCHED=1 G4RING_PDL=1 G4RING_V3_HINTS=2" >> $OUT 2>&1
for e in "G4RING_V3_SCHED=0 G4RING_PDL=0" "G4RING_V3_SCHED=1 G4RING_PDL=1"; do
  env $e timeout 120 python tools/k1_lab.py --planes 256 --batch 8 --arith fused --tag "$e P256" >> $OUT 2>&1
  env $e G4RING_V2GEOM=43 timeout 120 python tools/k1_lab.py --n 4608 --planes 72 --batch 8 --iters 3 --arith fused --tag "$e g43 c4" >> $OUT 2>&1
done
timeout 300 python tools/v3_trace.py --batch 8 --planes 64 >> $OUT 2>&1
for b in 4 5 6 7; do
  for g in 25 40 13; do
    G4RING_V2GEOM=$g timeout 120 python tools/k1_lab.py --planes 64 --batch $b --arith fused --tag "geom $g B=$b" >> $OUT 2>&1
  done
done
