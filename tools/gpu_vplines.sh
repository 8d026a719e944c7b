#!/bin/bash
# the one-rank vocab-parallel bench lines and their ncu captures (one GPU)
set -u
O=gpurun_out/${1:-vpl}; mkdir -p $O
for w in 8 4 2; do timeout 600 python bench.py --config vocabpar --vp-width-of $w > $O/bench_vp_w$w.json 2> $O/bench_vp_w$w.err; echo "w$w rc=$?"; done
prof() { local name=$1 kern=$2 skip=$3; shift 3; timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kern -s $skip -c 1 \
  -o $O/prof_$name "$@" > $O/ncu_$name.log 2>&1; echo "prof $name rc=$?"; }
prof vpcache8 vp_cache 1 python tools/vpbench.py --P 8 --rows 65536 --reps 2 --peer
prof vpcache4 vp_cache 1 python tools/vpbench.py --P 4 --rows 65536 --reps 2 --peer
