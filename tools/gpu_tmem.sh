#!/bin/bash
# vp_cache_kernel with the parked rows in tensor memory: parity (one GPU), timings one GPU and N GPUs
set -u
N=${2:-4}
O=gpurun_out/${1:-tmem}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -x -k "tmem" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for P in 4 8; do echo "P=$P tmem $(timeout 120 python tools/vpbench.py --P $P --peer --tmem 2>&1 | tail -1 | cut -d: -f2)"; done
for W in 37984 18992; do for args in "3=2 10=2" "3=2" "3=1"; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29552 \
    tools/vp_width_multi.py --width $W $args > $O/w.log 2>&1; grep VP_WIDTH $O/w.log || tail -3 $O/w.log
done; done
