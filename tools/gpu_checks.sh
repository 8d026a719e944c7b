#!/bin/bash
# the GPU suite against the debug-checks build (device-side bounds assertions; the stand-in for
# compute-sanitizer, which this pool refuses)
set -u
O=gpurun_out/${1:-checks}; mkdir -p $O
RL_LIB_PATH=paper_2605_15565_b200/librlpolicy_checks.so timeout 3000 python -m pytest tests -q -m gpu \
  -p no:cacheprovider -k "not alternate" > $O/pytest_checks.log 2>&1; echo "pytest rc=$?" >> $O/pytest_checks.log
RL_LIB_PATH=paper_2605_15565_b200/librlpolicy_checks.so timeout 600 python tools/sanitize_tiny.py > $O/tiny_checks.log 2>&1; echo "tiny rc=$?" >> $O/tiny_checks.log
