#!/bin/bash
# multi-GPU pass (gpurun --gpus N): mgpu parity, the vocab-parallel bench (peer and NCCL paths),
# token-parallel bench lines
set -u
N=${2:-2}
O=gpurun_out/${1:-multi}; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  tests/mgpu_check.py > $O/mgpu.log 2>&1; echo "mgpu rc=$?" >> $O/mgpu.log
for path in peer nccl; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --gpus $N --config vocabpar --vp-path $path --steps 20 --warmup 3 > $O/bench_vocabpar_$path.json 2> $O/bench_vocabpar_$path.err; echo "rc=$?" >> $O/bench_vocabpar_$path.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29535 \
  bench.py --gpus $N --steps 20 --warmup 3 > $O/bench_single.json 2> $O/bench_single.err; echo "rc=$?" >> $O/bench_single.err
for cfg in long multi; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29536 \
  bench.py --gpus $N --config $cfg --steps 20 --warmup 3 --no-e2e --no-cpu > $O/bench_$cfg.json 2> $O/bench_$cfg.err; echo "rc=$?" >> $O/bench_$cfg.err
done
