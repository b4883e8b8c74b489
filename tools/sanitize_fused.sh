# compute-sanitizer over the fused-mode kernels (deferred L2-reduction update, geometry 12)
cd $GRAFT_REPO_ROOT
CS="compute-sanitizer --print-limit 20 --error-exitcode 9"
for tool in memcheck racecheck synccheck; do
  for case in "--n 128 --planes 32 --batch 6" "--n 96 --planes 20 --batch 4 --dtype c64" "--n 160 --planes 17 --batch 5 --dtype mixed"; do
    timeout 600 $CS --tool $tool python tools/k1_lab.py $case --arith fused --iters 1 > /tmp/san.log 2>&1
    echo "$tool fused [$case]: rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' /tmp/san.log | tail -1)"
  done
done
