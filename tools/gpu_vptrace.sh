#!/bin/bash
set -u
N=${2:-4}
O=gpurun_out/${1:-vpt}; mkdir -p $O
export RL_LIB_PATH=paper_2605_15565_b200/librlpolicy_trace.so
timeout 300 python tools/vptrace.py --width-of $N > $O/single.log 2>&1; echo "rc=$?" >> $O/single.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29543 \
  tools/vptrace.py > $O/multi.log 2>&1; echo "rc=$?" >> $O/multi.log
