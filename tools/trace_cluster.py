"""Phase timeline of the cluster loss kernels (RL_TRACE=1; development tool).
    RL_TRACE=1 [RL_LOSS_KERNEL=cluster] python tools/trace_cluster.py [--rows 131072]"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2605_15565_b200 as rl
    import synth
    lib = rl.load()
    N = int(sys.argv[sys.argv.index("--rows") + 1]) if "--rows" in sys.argv else 131072
    V = 151936
    x = torch.empty((N, V), dtype=torch.bfloat16, device="cuda")
    y = torch.empty(N, dtype=torch.int32, device="cuda")
    synth.device_logits(x, V, 0, 2, targets_out=y)
    dl = torch.empty_like(x)
    old = torch.zeros(N, dtype=torch.float32, device="cuda")
    tseq = torch.zeros(N, dtype=torch.int32, device="cuda")
    adv = torch.ones(1, dtype=torch.float32, device="cuda")
    stats = torch.zeros(12, dtype=torch.float64, device="cuda")
    ws = torch.empty(rl.policy_loss_workspace_size(N, V), dtype=torch.uint8, device="cuda")
    p = rl.LossParams(agg=rl.AGG_SUM)
    for _ in range(3):
        rl.policy_loss_fwd_bwd(x, y, old, tseq, adv, p, dl, stats, ws)
    torch.cuda.synchronize()
    buf = np.zeros((256, 64, 8), dtype=np.uint64)
    sv = os.environ.get("RL_LOSS_KERNEL", "sv") == "sv"
    fn = lib.rl_debug_trace_sv if sv else lib.rl_debug_trace
    fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    assert fn(buf.ctypes.data, buf.nbytes) == 0
    b = buf[:148].astype(np.float64)
    rows = slice(8, 60)
    d = lambda i, j: (b[:, rows, j] - b[:, rows, i])
    per_row = (b[:, 9:61, 0] - b[:, 8:60, 0])
    print(f"row period (consumer T0->T0 next)  : {np.median(per_row):8.0f} ns  (p10 {np.percentile(per_row,10):.0f}, p90 {np.percentile(per_row,90):.0f})")
    if sv:
        phases = [("ref wait T0->T1", 0, 1), ("chunk loop T1->T2", 1, 2), ("exchange T2->T3", 2, 3),
                  ("scale + next start T3->T0'", None, None), ("service: res seen -> stats E4->E5", 4, 5)]
    else:
        phases = [("passA(next) T0->T1", 0, 1), ("scale wait T1->T2", 1, 2), ("fused C+B T2->T3", 2, 3),
                  ("epi: wait sumbar E4->E5", 4, 5), ("epi: peer wait E5->E6", 5, 6), ("epi: compute E6->E7", 6, 7)]
    for name, i, j in phases:
        if i is None:
            v = b[:, 9:61, 0] - b[:, 8:60, 3]
        else:
            v = d(i, j)
        print(f"{name:36s}: {np.median(v):8.0f} ns  (p10 {np.percentile(v,10):.0f}, p90 {np.percentile(v,90):.0f})")
    if sv:
        v = b[:, rows, 1] - b[:, rows, 7]
        print(f"{'first copy issued -> ref received':36s}: {np.median(v):8.0f} ns  (p10 {np.percentile(v,10):.0f}, p90 {np.percentile(v,90):.0f})")
        v = b[:, 9:61, 7] - b[:, 8:60, 7]
        print(f"{'producer row period':36s}: {np.median(v):8.0f} ns")
        return
    # sumbar completes at E5: relative to the consumer's T3 of the previous row (send_sum)
    v = b[:, 9:61, 5] - b[:, 8:60, 3]
    print(f"{'send(i) -> epi sees sums':36s}: {np.median(v):8.0f} ns")
    v = b[:, 9:61, 2] - b[:, 9:61, 7]
    print(f"{'publish(i) -> consumer past scale':36s}: {np.median(v):8.0f} ns")

if __name__ == "__main__":
    main()
