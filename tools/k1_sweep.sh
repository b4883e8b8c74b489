# K1 sweeps on the GPU box (replaces round 1's per-experiment lab*.sh / sweep_*.sh scripts).
#   VARIANTS  library env settings to compare, one process each (e.g. "G4RING_V2GEOM=25 G4RING_V2GEOM=40")
#   BATCHES   walkers per pass                       (default "8 16")
#   SHAPES    n:planes pairs                         (default "512:64 4608:72")
#   ARITHS    exact / fused                          (default "fused")
#   DTYPES    c128 / c64 / mixed                     (default "c128")
#   PARITY=1  run the v2/v3 parity subset of the GPU tests under each variant first
#   usage: VARIANTS="G4RING_V2GEOM=25 G4RING_V2GEOM=40" BATCHES="1 2 4 8 16" bash tools/k1_sweep.sh
cd ${GRAFT_REPO_ROOT:-.}
for v in ${VARIANTS:-"G4RING_V2GEOM=-1"}; do
  if [ "${PARITY:-0}" = 1 ]; then
    env $v timeout 600 python -m pytest tests -x -q -m gpu -k "variant or fused or full_size or headline" 2>&1 | tail -1 | sed "s/^/$v tests: /"
  fi
  for sh in ${SHAPES:-512:64 4608:72}; do
    n=${sh%%:*}; p=${sh##*:}
    it=20; [ $n -gt 1024 ] && it=3
    for a in ${ARITHS:-fused}; do for d in ${DTYPES:-c128}; do for b in ${BATCHES:-8 16}; do
      env $v timeout 300 python tools/k1_lab.py --n $n --planes $p --batch $b --arith $a --dtype $d --iters $it \
        --tag "$v n=$n p=$p B=$b $a $d"
    done; done; done
  done
done
