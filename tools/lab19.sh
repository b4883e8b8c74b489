cd $GRAFT_REPO_ROOT
R="timeout 60 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
p=29540
for combo in "1 1 1" "0 1 1" "1 0 1" "0 0 1" "0 0 0" "1 0 0"; do
  set -- $combo; p=$((p+1))
  r=$(G4RING_FLUSH=$1 G4RING_CORE_COPY=$2 G4RING_HALO=$3 $R --master-port $p tools/debug_deadlock.py 2>&1 | grep -E "raised|finished|Timeout" | head -2 | tr '\n' ' ')
  echo "flush=$1 core_copy=$2 halo=$3: $r"
done
