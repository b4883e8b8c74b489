# DRAM traffic per K1 launch (ncu, read + write) for the launch configurations the
# bench lines use, N = 1 and the per-rank shares of N > 1 runs -> gpurun_out/traffic_*.csv
mkdir -p gpurun_out
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_accumulate -s 6 -c 1 --csv"
cap() {  # tag, bench args
  timeout 600 ncu $M --log-file gpurun_out/traffic_$1.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --skip-extras "${@:2}" > /dev/null 2>&1
  echo "$1: $(grep -c dram gpurun_out/traffic_$1.csv) rows"
}
cap p8 --planes 8
cap p16 --planes 16
cap p32 --planes 32
cap c64 --dtype c64
cap mixed --dtype mixed
cap b16 --batch 16
cap b1 --batch 1
cap c4 --config c4
