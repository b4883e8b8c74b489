# ncu capture of the headline K1 on the final code (payload evict_last default), launch list
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --skip-extras > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02m.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --skip-extras > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 4 -c 1 \
    -o gpurun_out/full_r02m python bench.py --steps 2 --warmup 3 --no-cpu-baseline --skip-extras > /dev/null 2>&1
ls -la gpurun_out | grep r02m
