set -u
O=gpurun_out/t1; mkdir -p $O
for i in 1 2; do
timeout 300 python tools/vpbench.py --peer --P 4 2>&1 | tail -1
timeout 300 python tools/vpbench.py --peer --P 8 2>&1 | tail -1
done
timeout 300 python tools/kbench.py 2>&1 | tail -2
