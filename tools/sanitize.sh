# compute-sanitizer over small K1/K2/K3 cases and the ring (race detection)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CS="compute-sanitizer --print-limit 20 --error-exitcode 9"
for tool in memcheck racecheck synccheck initcheck; do
  for case in "--n 128 --planes 16 --batch 4" "--n 128 --planes 8 --batch 3" "--n 96 --planes 20 --batch 2 --dtype c64" "--n 160 --planes 17 --batch 3 --dtype mixed" "--n 48 --planes 3 --batch 2"; do
    timeout 600 $CS --tool $tool python tools/k1_lab.py $case --iters 1 > /tmp/san.log 2>&1
    echo "$tool [$case]: rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Error' /tmp/san.log | tail -1)"
  done
done
# the ring (2 ranks on one GPU) and K2/K3 through the engine test path, memcheck only
timeout 900 $CS --tool memcheck --target-processes all python -m pytest tests/test_gpu_engine.py -q -x -k "native and kw0" > /tmp/san_ring.log 2>&1
echo "memcheck ring: rc=$? $(grep -E 'ERROR SUMMARY' /tmp/san_ring.log | sort | uniq -c | tr '\n' ' ') $(tail -1 /tmp/san_ring.log)"
