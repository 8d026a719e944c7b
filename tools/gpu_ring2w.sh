#!/bin/bash
# vp_ring_kernel with two service warps: D sweep at the P = 2 / 4 / 8 widths (one GPU) + the VP tests
set -u
O=gpurun_out/${1:-r2w}; mkdir -p $O
for P in 2 4 8; do for dl in 0 1 2 3; do
  echo "P=$P D=$dl $(timeout 120 python tools/vpbench.py --P $P --peer --ring --delay $dl 2>&1 | tail -1 | cut -d: -f2)"
done; done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "vocab_parallel or repeated" > $O/pytest.log 2>&1; tail -1 $O/pytest.log
