# Multi-GPU bench recipe for an 8 x B200 node (one process per GPU, NCCL over
# NVLink/NVSwitch).  Emits one JSON line per N (merge_ms is in each line).
# usage (repo root): bash tools/scale_recipe.sh [config] [merge] > scale.jsonl
#   config: caida | 10G | bigwin (default 10G); merge: sharded | delta | stamps |
#   sparse | p2p | nvls (default sharded)
set -u
CFG=${1:-10G}
MERGE=${2:-sharded}
EXTRA=""
[ "$CFG" = bigwin ] && EXTRA="--shard-state"
for N in 1 2 4 8; do
  if [ $N = 1 ]; then
    timeout 900 python bench.py --config $CFG --steps 20 --warmup 5 --no-cpu-baseline
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $((29600 + N)) bench.py --gpus $N \
      --config $CFG --steps 20 --warmup 5 --merge $MERGE $EXTRA
  fi
done
