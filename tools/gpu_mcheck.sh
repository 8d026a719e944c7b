#!/bin/bash
# multi-GPU correctness after a vocab-parallel change: mgpu_check, race_check (narrow / wide), the multi-GPU test
set -u
N=${2:-4}
O=gpurun_out/${1:-mcheck}; mkdir -p $O
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  tests/mgpu_check.py > $O/mgpu.log 2>&1; echo "mgpu rc=$?"; grep -a "MGPU\|FAIL" $O/mgpu.log | head -5
for V in $((N * 18992)) 151936; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port 29551 tools/race_check.py --vocab $V 3=2 2>&1 | grep RACE_CHECK | sed "s/^/V=$V /"; done
