# Round profile bundle (run on the GPU box via gpurun): bench lines, ncu launch list, ncu full capture.
# usage: bash tools/profile_round.sh <tag> [batch]
TAG=${1:-r01}; B=${2:-8}
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 --batch $B > gpurun_out/bench_$TAG.log 2>&1
grep -E '^\{' gpurun_out/bench_$TAG.log | tail -1 > gpurun_out/bench_$TAG.json
NC="--steps 20 --warmup 5 --no-cpu-baseline"
for dt in c64 mixed; do
  python bench.py $NC --batch $B --dtype $dt 2>/dev/null | grep -E '^\{' | tail -1 > gpurun_out/bench_${TAG}_$dt.json
done
python bench.py $NC --batch $B --arith exact 2>/dev/null | grep -E "^\{" | tail -1 > gpurun_out/bench_${TAG}_exact.json
for b in 1 16; do python bench.py $NC --batch $b 2>/dev/null | grep -E '^\{' | tail -1 > gpurun_out/bench_${TAG}_b$b.json; done
python bench.py $NC --batch $B --planes 8 2>/dev/null | grep -E '^\{' | tail -1 > gpurun_out/bench_${TAG}_p8.json
python bench.py --config c4 --steps 5 --warmup 3 --batch $B --no-cpu-baseline 2>/dev/null | grep -E '^\{' | tail -1 > gpurun_out/bench_${TAG}_c4.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 5 --warmup 3 --batch $B --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 4 -c 1 \
    -o gpurun_out/full_$TAG python bench.py --steps 2 --warmup 3 --batch $B --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out | grep $TAG
