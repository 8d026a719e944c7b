#!/bin/bash
# final multi-GPU pass at N GPUs: GPU test suite (cuda:0), multi-GPU parity, race check, bench lines
set -u
N=${2:-4}
O=gpurun_out/${1:-final}; mkdir -p $O
if [ "${3:-}" = "tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
fi
for i in 1 2; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29551 \
    tools/race_check.py 3=2 2>&1 | grep RACE_CHECK >> $O/race.log; done
cat $O/race.log
bash tools/gpu_multi.sh $1 $N
grep -a "MGPU\|rc=" $O/mgpu.log | tail -2
for f in $O/bench_*.json; do python -c "import json;d=json.load(open('$f'));print('$f',round(d['value']/1e6,2),'M',round(d['ms_per_step'],3),'ms',round(d['roofline']['frac'],3),d['roofline']['kernel'][:60])" 2>&1 | tail -1; done
