#!/bin/bash
# vocab-parallel quick loop: timings of both peer kernels at the P = 8 / 4 widths, the VP parity tests
set -u
O=gpurun_out/${1:-vp}; mkdir -p $O
echo "== vpbench" > $O/vpbench.log
for P in 8 4; do
  for mode in "--peer" "--peer --ring" ""; do
    timeout 120 python tools/vpbench.py --P $P --rows 65536 --reps 10 $mode >> $O/vpbench.log 2>&1; echo "P=$P $mode rc=$?" >> $O/vpbench.log
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -p no:cacheprovider -k "vocab_parallel" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
if [ "${2:-}" = "ncu" ]; then
  for P in 8 4; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:vp_cache -s 1 -c 1 -o $O/prof_vpcache$P \
    python tools/vpbench.py --P $P --rows 65536 --reps 2 --peer > $O/ncu$P.log 2>&1; echo "ncu rc=$?" >> $O/ncu$P.log
  done
fi
