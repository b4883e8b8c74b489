# compute-sanitizer on chained passes, full logs (lab r02ah returned rc=86 without a summary)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for c in 1 0; do
  timeout 600 env G4RING_V3_CHAIN=$c compute-sanitizer --print-limit 20 --tool memcheck python tools/k1_lab.py --n 160 --planes 40 --batch 8 --arith fused --iters 2 > gpurun_out/san_chain$c.log 2>&1
  echo "rc=$?" >> gpurun_out/san_chain$c.log
done
timeout 600 compute-sanitizer --print-limit 20 --tool memcheck python tools/k1_lab.py --n 160 --planes 40 --batch 8 --arith exact --iters 2 > gpurun_out/san_exact.log 2>&1; echo "rc=$?" >> gpurun_out/san_exact.log
