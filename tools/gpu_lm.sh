#!/bin/bash
set -u
O=gpurun_out/${1:-lm}; mkdir -p $O
# one 8,192-token chunk: dh GEMM (lm_gemm_kernel<false,true>) then dW GEMM (<true,true>)
timeout 300 ncu --set full --clock-control none --import-source on -k regex:lm_gemm -c 2 -o $O/prof_gemm \
  python tools/lmbench.py --rows 8192 --reps 1 --bwd --chunk 8192 > $O/ncu_gemm.log 2>&1; echo "ncu rc=$?" >> $O/ncu_gemm.log
