#!/bin/bash
# One GPU-box pass (run via gpurun from the repo root): quick kernel timings, the -m gpu suite,
# compute-sanitizer over tools/sanitize_tiny.py, the default bench line.  Output: gpurun_out/$1/
set -u
O=gpurun_out/${1:-check}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
echo "== vpbench" > $O/vpbench.log
for P in 4 8; do
  timeout 120 python tools/vpbench.py --P $P --rows 65536 --reps 10 --peer >> $O/vpbench.log 2>&1; echo "peer P=$P rc=$?" >> $O/vpbench.log
  timeout 120 python tools/vpbench.py --P $P --rows 65536 --reps 10 >> $O/vpbench.log 2>&1; echo "nccl P=$P rc=$?" >> $O/vpbench.log
done
timeout 300 python tools/kbench.py --rows 131072 --reps 5 > $O/kbench.log 2>&1; echo "kbench rc=$?" >> $O/kbench.log
timeout 2400 python -m pytest tests -q -m gpu -x -p no:cacheprovider -s > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_tiny.py > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $O/sanitize_$tool.log
done
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
