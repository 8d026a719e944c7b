#!/bin/bash
# Round measurement pass on ONE GPU (gpurun): every bench line, then the ncu evidence.
#   gpurun_out/$1/bench_*.json      one JSON line per config / objective
#   gpurun_out/$1/launches.csv      ncu launch list of a short default bench
#   gpurun_out/$1/prof_*.ncu-rep    ncu --set full of each hot kernel
set -u
O=gpurun_out/${1:-round}; mkdir -p $O
run() { local name=$1; shift; timeout 1200 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo "$name rc=$?" >> $O/status.txt; }
run single
run tiny --config tiny --steps 50
run objective_full --objective full --no-e2e --no-cpu
run objective_m2po --objective m2po --no-e2e --no-cpu
run long --config long --no-e2e --no-cpu --steps 10
run long_skip --config long --no-e2e --no-cpu --steps 10 --skip-masked
run multi --config multi --no-e2e --no-cpu --steps 10
run vp_w8 --config vocabpar --vp-width-of 8
run vp_w4 --config vocabpar --vp-width-of 4
run vp_w2 --config vocabpar --vp-width-of 2
run lmhead --config lmhead --steps 10
run resident --resident --no-e2e --no-cpu --steps 10
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > $O/bench_short.log 2>&1 && \
  timeout 900 ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > $O/ncu_launch.log 2>&1
echo "launch list rc=$?" >> $O/status.txt
prof() { local name=$1 kern=$2 skip=$3; shift 3; timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kern -s $skip -c 1 \
  -o $O/prof_$name "$@" > $O/ncu_$name.log 2>&1; echo "prof $name rc=$?" >> $O/status.txt; }
prof loss_sv loss_sv_kernel 1 python tools/kbench.py --rows 16384 --reps 2
prof vpcache8 vp_cache 1 python tools/vpbench.py --P 8 --rows 65536 --reps 2 --peer
prof vpcache4 vp_cache 1 python tools/vpbench.py --P 4 --rows 65536 --reps 2 --peer
prof ring4 vp_ring 1 python tools/vpbench.py --P 4 --rows 65536 --reps 2 --peer --ring
prof ring2 vp_ring 1 python tools/vpbench.py --P 2 --rows 65536 --reps 2 --peer --ring
# lmbench --bwd --reps 1 launches lmhead_kernel as: forward (warm), forward (timed), then the backward's
# gradient kernel once per 8,192-token chunk: skip 2 -> the first gradient launch; skip 1 -> a forward
prof lmgrad lmhead_kernel 2 python tools/lmbench.py --rows 16384 --reps 1 --bwd
prof lmfwd lmhead_kernel 1 python tools/lmbench.py --rows 16384 --reps 1
