#!/bin/bash
set -u
N=${2:-4}
O=gpurun_out/${1:-vpt}; mkdir -p $O
export RL_LIB_PATH=paper_2605_15565_b200/librlpolicy_trace.so
for cfg in "--pub 0" "--pub 1" "--pub 2" "--pub 1 --rs 0" "--pub 2 --rs 0"; do
  echo "== $cfg" >> $O/multi.log
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29543 \
    tools/vptrace.py $cfg 2>&1 | grep -o "\[rank 0\][^[]*" >> $O/multi.log
done
