#!/bin/bash
# final multi-GPU pass: correctness (mgpu_check, race_check on both kernels) and the bench lines
set -u
N=${2:-4}
O=gpurun_out/${1:-fm}; mkdir -p $O
bash tools/gpu_mcheck.sh $1 $N
for V in $((N * 18992)) 151936; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port 29551 tools/race_check.py --vocab $V 3=1 2>&1 | grep RACE_CHECK | sed "s/^/ring V=$V /"; done
bash tools/gpu_multi.sh $1 $N > /dev/null 2>&1
for f in $O/bench_*.json; do python -c "import json;d=json.load(open('$f'));print('$f'.split('/')[-1],round(d['value']/1e6,2),'M',round(d['ms_per_step'],3),'ms',round(d['roofline']['frac'],3),d['roofline']['kernel'][26:45])" 2>&1 | tail -1; done
