#!/bin/bash
# vp_cache_kernel deferral through L2: single-GPU parity of the VP tests, multi-GPU parity, then the
# configs[3] bench at N GPUs: library default, register cache (deferral default / off), ring
set -u
N=${2:-4}
O=gpurun_out/${1:-defer}; mkdir -p $O
timeout 300 python tools/kbench.py > $O/kbench.log 2>&1; tail -2 $O/kbench.log
timeout 300 python tools/vpbench.py --peer --P 4 > $O/vpbench4.log 2>&1; tail -1 $O/vpbench4.log
timeout 300 python tools/vpbench.py --peer --P 8 > $O/vpbench8.log 2>&1; tail -1 $O/vpbench8.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "vocab_parallel" > $O/pytest_vp.log 2>&1; echo "pytest rc=$?" >> $O/pytest_vp.log
tail -3 $O/pytest_vp.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  tests/mgpu_check.py > $O/mgpu.log 2>&1; echo "mgpu rc=$?" >> $O/mgpu.log
tail -2 $O/mgpu.log
for args in "--vp-kernel cache" "--vp-kernel cache --vc-defer 0" "--vp-kernel ring" "--vp-kernel cache --vc-defer 4" ; do
  tag=$(echo $args | tr -d ' -')
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29540 \
    bench.py --gpus $N --config vocabpar $args --steps 20 --warmup 3 --no-e2e --no-cpu > $O/vp_$tag.json 2> $O/vp_$tag.err
  echo "$tag rc=$? $(python -c "import json;d=json.load(open('$O/vp_$tag.json'));print(round(d['value']/1e6,2),'M',round(d['ms_per_step'],3),'ms',round(d['roofline']['frac'],3))" 2>&1 | tail -1)"
done
