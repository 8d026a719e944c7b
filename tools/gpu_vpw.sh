#!/bin/bash
# vocab-parallel across N GPUs at the P = 8 shard width: parked rows (RS) 0 / 1, cache vs ring
set -u
N=${2:-4}
for args in "3=2 5=1" "3=2 5=2" "3=1"; do for W in 18992 37984; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29552 \
    tools/vp_width_multi.py --width $W $args 2>&1 | grep VP_WIDTH; done
done
