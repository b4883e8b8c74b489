# final check on the final code: GPU suite, smoke, default bench, reference arm, 2-rank line, B = 3 line
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02k_gpu_tests.log 2>&1
timeout 900 bash tools/final_check.sh > gpurun_out/r02k_final_check.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --batch 3 --no-cpu-baseline --skip-extras 2>/dev/null | grep -E '^\{' | tail -1 > gpurun_out/r02k_bench_b3.json
