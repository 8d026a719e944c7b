#!/bin/bash
# vp_cache_kernel: rows parked in smem (RS) — single GPU timings, then across N GPUs; parity
set -u
N=${2:-4}
O=gpurun_out/${1:-vprs}; mkdir -p $O
for P in 8 4; do for rs in 0 1 2; do
  echo "P=$P rs=$rs" >> $O/single.log
  timeout 120 python tools/vpbench.py --P $P --rows 65536 --reps 10 --peer --rs $rs 2>&1 | grep shard >> $O/single.log
done; done
for rs in 0 1 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 \
    bench.py --gpus $N --config vocabpar --vc-rows $rs --steps 20 --warmup 3 > $O/vp_rs$rs.json 2> $O/vp_rs$rs.err; echo "rs=$rs rc=$?" >> $O/status.txt
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29542 \
  tests/mgpu_check.py > $O/mgpu.log 2>&1; echo "mgpu rc=$?" >> $O/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -p no:cacheprovider -k "vocab_parallel" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
