timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "vocab" 2>&1 | tail -2
for cfg in "RL_VP2_PF=0" "RL_VP2_PF=1" "RL_VP2_PF=2" "RL_VP2_PF=1 RL_VP2_BUDGET_KB=300" "RL_VP2_PF=2 RL_VP2_BUDGET_KB=100" "RL_VP2_PF=1 RL_VP2_BUDGET_KB=80" "RL_VP2_PF=3 RL_VP2_BUDGET_KB=80"; do
  echo "$cfg"; env $cfg timeout 120 python tools/vpbench.py --P 4 --peer 2>&1 | grep shard
done
RL_VP2_PF=1 timeout 120 python tools/vpbench.py --P 4 --peer --adv0 2>&1 | grep shard
