#!/bin/bash
# GPU-box profiling pass for one round (run via gpurun from the repo root).
#   1. bench.py (the JSON line)            -> gpurun_out/bench.json
#   2. ncu launch list of a short bench    -> gpurun_out/launches_bench.csv
#   3. ncu --set full of the loss kernel   -> gpurun_out/prof_loss.ncu-rep (16,384-row launch)
#   4. ncu --set full of the logprob kernel-> gpurun_out/prof_logprob.ncu-rep
#   5. ncu --set full of the vocab-parallel finish pass (P = 4 shard on one GPU) -> prof_vpfin
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
ARGS="--steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 600 python bench.py $ARGS > gpurun_out/bench_short.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_bench.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 300 python tools/kbench.py --rows 16384 --reps 2 > gpurun_out/kb_small.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:loss_sv_kernel -s 1 -c 1 \
    -o gpurun_out/prof_loss python tools/kbench.py --rows 16384 --reps 2 > gpurun_out/ncu_loss.log 2>&1
echo "ncu loss rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:logprob_warp -s 1 -c 1 \
    -o gpurun_out/prof_logprob python tools/kbench.py --rows 16384 --reps 2 > gpurun_out/ncu_logprob.log 2>&1
echo "ncu logprob rc=$?"
timeout 300 python tools/vpbench.py --P 4 --rows 16384 --reps 2 > gpurun_out/vpb_small.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:vp_finish_tma -s 1 -c 1 \
    -o gpurun_out/prof_vpfin python tools/vpbench.py --P 4 --rows 16384 --reps 2 > gpurun_out/ncu_vpfin.log 2>&1
echo "ncu vp finish rc=$?"
