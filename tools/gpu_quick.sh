#!/bin/bash
# quick 1-GPU check after a kernel change: fused-loss objectives, SV, vocab-parallel shards, GPU tests
set -u
O=gpurun_out/${1:-quick}; mkdir -p $O
timeout 300 python tools/objbench.py clip entropy full 2>&1 | tail -3
timeout 300 python tools/kbench.py 2>&1 | tail -2
for P in 4 8; do timeout 120 python tools/vpbench.py --P $P --peer 2>&1 | tail -1; done
timeout 120 python tools/vpbench.py --P 4 --peer --ring 2>&1 | tail -1
timeout 120 python tools/vpbench.py --P 2 --peer --ring 2>&1 | tail -1
timeout 120 python tools/vpbench.py --P 4 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
