# compute-sanitizer over the fused-mode kernels (deferred update: TMA bulk-reduce epilogue for
# complex128 slices, red.global for complex64; geometries 12 and 19, and cluster geometry 22)
cd $GRAFT_REPO_ROOT
CS="compute-sanitizer --print-limit 20 --error-exitcode 9"
for tool in memcheck racecheck synccheck; do
  for case in "--n 128 --planes 32 --batch 6" "--n 96 --planes 20 --batch 4 --dtype c64" "--n 160 --planes 17 --batch 5 --dtype mixed" "--n 200 --planes 8 --batch 4"; do
    timeout 600 $CS --tool $tool python tools/k1_lab.py $case --arith fused --iters 1 > /tmp/san.log 2>&1
    echo "$tool fused [$case]: rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' /tmp/san.log | tail -1)"
  done
done
for tool in memcheck racecheck synccheck; do
  G4RING_V2GEOM=22 timeout 600 $CS --tool $tool python tools/k1_lab.py --n 128 --planes 32 --batch 5 --arith fused --iters 1 > /tmp/san.log 2>&1
  echo "$tool fused geom 22: rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' /tmp/san.log | tail -1)"
done
