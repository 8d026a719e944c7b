#!/bin/bash
# vocab-parallel quick loop: kernel timings at the P = 4 / 8 widths (cache, ring) and the VP tests
set -u
O=gpurun_out/${1:-vpq}; mkdir -p $O
for rep in 1 2; do for P in 4 8; do timeout 120 python tools/vpbench.py --P $P --peer 2>&1 | tail -1; done; done
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "vocab_parallel or repeated" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
