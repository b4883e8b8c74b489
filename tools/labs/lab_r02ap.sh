# final code: smoke, headline/chain parity, default bench
mkdir -p gpurun_out
OUT=gpurun_out/r02l_check.txt
: > $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 >> $OUT
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_chain.py -q 2>&1 | tail -2 >> $OUT
timeout 600 python tools/geom_check.py --repeat 2 2>&1 | tail -3 >> $OUT
timeout 600 python bench.py > gpurun_out/r02l_bench.log 2>&1
grep -E '^\{' gpurun_out/r02l_bench.log | tail -1 > gpurun_out/r02l_bench.json
