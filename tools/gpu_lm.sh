#!/bin/bash
set -u
O=gpurun_out/${1:-lm}; mkdir -p $O
timeout 120 python tools/lmbench.py --rows 16384 --reps 3 >> $O/lmbench.log 2>&1; echo "pair rc=$?" >> $O/lmbench.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "lmhead" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for N in 16384 65536 131072; do
  timeout 300 python tools/lmbench.py --rows $N --reps 3 --bwd --chunk 16384 >> $O/lmbench.log 2>&1; echo "pair N=$N rc=$?" >> $O/lmbench.log
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:lmhead_kernel -s 1 -c 1 -o $O/prof_lmfwd_pair \
  python tools/lmbench.py --rows 16384 --reps 1 > $O/ncu_fwd.log 2>&1; echo "ncu rc=$?" >> $O/ncu_fwd.log
