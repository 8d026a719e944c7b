#!/bin/bash
# configs[3] across N GPUs: the register-cache kernel forced vs the ring (and the library default)
set -u
N=${2:-4}
O=gpurun_out/${1:-vpx}; mkdir -p $O
for k in cache ring auto; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29540 \
    bench.py --gpus $N --config vocabpar --vp-kernel $k --steps 20 --warmup 3 --no-e2e --no-cpu > $O/vp_$k.json 2> $O/vp_$k.err
  echo "$k rc=$? $(python -c "import json;d=json.load(open('$O/vp_$k.json'));print(round(d['value']/1e6,2),'M',round(d['ms_per_step'],3),'ms',round(d['roofline']['frac'],3),d['roofline']['kernel'][:45])" 2>&1 | tail -1)"
done
