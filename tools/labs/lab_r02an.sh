# with chaining: in-walker TMEM stores at N = 512 and L2 evict_last payload hints, A/B at the bench shape
mkdir -p gpurun_out
OUT=gpurun_out/lab_r02an.txt
: > $OUT
bash tools/lab_v3_ab.sh "G4RING_V3_EARLY_ST=0" "G4RING_V3_EARLY_ST=1" "G4RING_V3_HINTS=2" "G4RING_V3_EARLY_ST=0" "G4RING_V3_EARLY_ST=1" "G4RING_V3_HINTS=2" >> $OUT 2>&1
