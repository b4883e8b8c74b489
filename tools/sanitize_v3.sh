# compute-sanitizer over the warp-specialised K1 kernels (geometries 25 and 27 in both
# modes; K1 v3, the persistent TMEM hand-off kernel, geometries 40 and 43, both epilogues)
cd ${GRAFT_REPO_ROOT:-.}
CS="compute-sanitizer --print-limit 20 --error-exitcode 9"
run() {  # env, k1_lab args, label
  timeout 900 env $1 $CS --tool $tool python tools/k1_lab.py $2 --iters 1 > /tmp/san.log 2>&1
  echo "$tool $3 [$2]: rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' /tmp/san.log | tail -1)"
}
for tool in memcheck racecheck synccheck; do
  for a in exact fused; do
    run "G4RING_V2GEOM=25" "--n 128 --planes 32 --batch 6 --arith $a" "geom 25"
    run "G4RING_V2GEOM=27" "--n 128 --planes 16 --batch 6 --arith $a" "geom 27"
  done
  for g in 40 43; do for h in 0; do
    run "G4RING_V2GEOM=$g G4RING_V3_HINTS=$h" "--n 160 --planes 40 --batch 6 --arith fused" "v3 geom $g hints $h"
    run "G4RING_V2GEOM=$g G4RING_V3_HINTS=$h" "--n 128 --planes 32 --batch 9 --dtype mixed --arith fused" "v3 geom $g hints $h"
    run "G4RING_V2GEOM=$g" "--n 200 --planes 40 --batch 8 --arith exact" "v3 exact geom $g"
  done; done
done
