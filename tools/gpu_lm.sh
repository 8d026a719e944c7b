#!/bin/bash
set -u
O=gpurun_out/${1:-lm}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "lmhead" -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for mode in "" "--cublas"; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches$mode.csv \
  python tools/lmbench.py --rows 16384 --reps 2 --bwd --chunk 16384 $mode > $O/ncu$mode.log 2>&1; echo "rc=$?" >> $O/ncu$mode.log
timeout 300 python tools/lmbench.py --rows 16384 --reps 5 --bwd --chunk 16384 $mode >> $O/lmbench.log 2>&1
timeout 300 python tools/lmbench.py --rows 65536 --reps 3 --bwd --chunk 16384 $mode >> $O/lmbench.log 2>&1
done
