mkdir -p gpurun_out
OUT=gpurun_out/lab_r02aa.txt
: > $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -1 >> $OUT
for e in "G4RING_PDL=0" "G4RING_PDL=1"; do
  for a in "--planes 8" "--dtype c64" "--arith exact" "--batch 5" "--batch 1"; do
    env $e timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --skip-extras $a 2>/dev/null | grep -E '^\{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e $a', '%.3e'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'us %.1f'%(d['ms_per_step']*1e3), 'geom', d['launched_k1_geometry'], 'parity', d['parity_check']['ok'])" >> $OUT 2>&1
  done
done
