# BASELINE config 5's ring sweep on one multi-GPU node (needs N visible B200s):
# every sub-ring size S | N, both wire payload formats, 1 and 2 lanes, and
# configs 2 / 3 / 4, one bench line each (torchrun, one rank per GPU).
#   bash tools/scale_sweep.sh [N=8] [out=gpurun_out/scale_sweep.jsonl]
N=${1:-8}; OUT=${2:-gpurun_out/scale_sweep.jsonl}
mkdir -p $(dirname $OUT); : > $OUT
run() {  # label, bench args
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 200)) bench.py --gpus $N --steps 10 --warmup 3 "${@:2}" 2>/dev/null \
    | grep -E '^\{' | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['sweep']='$1'; print(json.dumps(d))" >> $OUT
}
for S in 1 2 4 8; do
  [ $((N % S)) -eq 0 ] && [ $S -le $N ] || continue
  for wire in cores staged; do
    G4RING_WIRE=$wire run "c2 S=$S wire=$wire" --config c2 --subring-size $S
  done
  run "c2 S=$S c64 payloads" --config c2 --subring-size $S --dtype mixed
  run "c3 S=$S lanes=2" --config c3 --subring-size $S --lanes 2
  run "c3 S=$S lanes=2 merged" --config c3 --subring-size $S --lanes 2 --merged-lanes
done
run "c4 S=$N" --config c4 --subring-size $N
for B in 1 4 16; do run "c2 S=$N B=$B" --config c2 --batch $B; done
python - "$OUT" <<'PY'
import json, sys
for line in open(sys.argv[1]):
    d = json.loads(line)
    print(f"{d['sweep']:28s} {d['value']:.3e} upd/s  {d['ms_per_step']:.3f} ms/step  "
          f"K1 HBM {d['roofline']['frac']:.2f}  NVLink {d['nvlink']['achieved_gbs']:.0f} GB/s")
PY
