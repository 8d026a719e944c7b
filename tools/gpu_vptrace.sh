#!/bin/bash
# per-CTA vp_cache_kernel counters on every rank (trace build), P = N GPUs
set -u
N=${2:-4}
O=gpurun_out/${1:-vpt2}; mkdir -p $O
export RL_LIB_PATH=paper_2605_15565_b200/librlpolicy_trace.so
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29543 \
    tools/vptrace.py --dump $O/tr 2>&1 | grep -o "\[rank [0-9]\][^[]*" > $O/multi.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29544 \
    tools/vptrace.py --width-of $N --dump $O/single 2>&1 | grep -o "\[rank [0-9]\][^[]*" >> $O/multi.log
cat $O/multi.log
for k in cache ring; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29540 \
    bench.py --gpus $N --config vocabpar --vp-kernel $k --steps 20 --warmup 3 --no-e2e --no-cpu > $O/vp_$k.json 2> $O/vp_$k.err
  echo "$k rc=$? $(python -c "import json;d=json.load(open('$O/vp_$k.json'));print(round(d['value']/1e6,2),'M',round(d['ms_per_step'],3),'ms',round(d['roofline']['frac'],3))" 2>&1 | tail -1)"
done
