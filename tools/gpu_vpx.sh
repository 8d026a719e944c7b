#!/bin/bash
# configs[3] across N GPUs: kernel choice and vp_cache_kernel knobs (collector groups, record send)
set -u
N=${2:-4}
O=gpurun_out/${1:-vpx}; mkdir -p $O
i=0
for args in "--vp-kernel ring" "--vp-kernel cache" "--vp-kernel cache --dev-opt 4=4" "--vp-kernel cache --dev-opt 4=2" \
            "--vp-kernel cache --dev-opt 6=3" "--vp-kernel cache --dev-opt 6=1" "--vp-kernel cache --vc-rows 0"; do
  i=$((i+1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29540 \
    bench.py --gpus $N --config vocabpar $args --steps 20 --warmup 3 --no-e2e --no-cpu > $O/vp_$i.json 2> $O/vp_$i.err
  echo "[$args] rc=$? $(python -c "import json;d=json.load(open('$O/vp_$i.json'));print(round(d['value']/1e6,2),'M',round(d['ms_per_step'],3),'ms',round(d['roofline']['frac'],3),d['roofline']['kernel'][26:45])" 2>&1 | tail -1)"
done
