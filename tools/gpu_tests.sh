#!/bin/bash
# the driver's round-end GPU tiers on one GPU: pytest -m gpu and smoke()
set -u
O=gpurun_out/${1:-tests}; mkdir -p $O
timeout 3000 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
