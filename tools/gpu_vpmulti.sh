#!/bin/bash
# vocab-parallel across N GPUs: kernel A/B (cache vs ring) and the NCCL path
set -u
N=${2:-4}
O=gpurun_out/${1:-vpm}; mkdir -p $O
for args in "--vp-kernel cache" "--vp-kernel ring" "--vp-path nccl"; do
  tag=$(echo $args | tr -d ' -')
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29540 \
    bench.py --gpus $N --config vocabpar $args --steps 20 --warmup 3 > $O/vp_$tag.json 2> $O/vp_$tag.err; echo "$tag rc=$?" >> $O/status.txt
done
