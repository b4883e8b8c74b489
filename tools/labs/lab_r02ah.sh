# chained passes: compute-sanitizer over chained v3 / v2 deferred passes (k1_lab runs 3 + iters
# passes back to back); geometry 40 vs 43 at config 4's share and N = 1024 with chaining on
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
OUT=gpurun_out/lab_r02ah.txt
: > $OUT
CS="compute-sanitizer --print-limit 20 --error-exitcode 9"
run() {  # env, k1_lab args, label
  timeout 900 env $1 $CS --tool $tool python tools/k1_lab.py $2 --iters 2 > /tmp/san.log 2>&1
  echo "$tool $3 [$2]: rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' /tmp/san.log | tail -1)" >> $OUT
}
for tool in memcheck racecheck synccheck; do
  run "G4RING_V3_CHAIN=1" "--n 160 --planes 40 --batch 8 --arith fused" "chained v3 geom 40"
  run "G4RING_V3_CHAIN=1" "--n 160 --planes 8 --batch 8 --arith fused" "chained v2 geom 19"
  run "G4RING_V3_CHAIN=1" "--n 128 --planes 32 --batch 8 --dtype c64 --arith fused" "chained v2 geom 12 c64"
done
for g in 43 40 43 40; do
  G4RING_V2GEOM=$g timeout 200 python tools/k1_lab.py --n 4608 --planes 72 --batch 8 --iters 4 --arith fused --tag "g$g c4" >> $OUT 2>&1
  G4RING_V2GEOM=$g timeout 120 python tools/k1_lab.py --n 1024 --planes 64 --batch 8 --iters 10 --arith fused --tag "g$g n1024" >> $OUT 2>&1
done
