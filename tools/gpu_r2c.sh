#!/bin/bash
set -u
O=gpurun_out/r2c; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -p no:cacheprovider -s -k "lmhead or full_chain" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python tools/lmbench.py --rows 16384 --reps 3 --bwd > $O/lmbench.log 2>&1; echo "rc=$?" >> $O/lmbench.log
timeout 600 python tools/lmbench.py --rows 65536 --reps 3 --bwd --chunk 16384 >> $O/lmbench.log 2>&1; echo "rc=$?" >> $O/lmbench.log
