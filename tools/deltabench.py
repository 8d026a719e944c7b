"""bf16 delta-scan throughput (development tool, NEXT 3): two synthetic snapshots of N 16-bit
words at sparsity s ("0.989-0.993"), timed encode and apply.
    python tools/deltabench.py [--words 2147483647] [--sparsity 0.99]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2605_15565_b200 as rl
    rl.load()
    n = int(sys.argv[sys.argv.index("--words") + 1]) if "--words" in sys.argv else (1 << 31) - 1
    s = float(sys.argv[sys.argv.index("--sparsity") + 1]) if "--sparsity" in sys.argv else 0.99
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    a = torch.randint(-32768, 32767, (n,), dtype=torch.int16, device="cuda", generator=g)
    b = a.clone()
    ch = torch.rand(n, device="cuda", generator=g) < (1 - s)
    b[ch] ^= 1
    del ch
    cap = int((1 - s) * n * 1.05) + 1024
    idx = torch.empty(cap, dtype=torch.int32, device="cuda")
    words = torch.empty(cap, dtype=torch.int16, device="cuda")
    count = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.empty(rl.delta_workspace_size(n), dtype=torch.uint8, device="cuda")
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")

    def timed(fn, reps=10):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return min(ts), sum(ts) / len(ts)

    t, avg = timed(lambda: rl.delta_encode(a, b, idx, words, count, ws))
    k = int(count.item())
    print(f"encode: {n} words, {k} changes (sparsity {1 - k / n:.4f}): {t:.3f} ms (avg {avg:.3f})  "
          f"{2 * n * 2 / t / 1e6:.1f} GB/s read, algorithmic {(4 * n + 6 * k) / t / 1e6:.1f} GB/s")
    base = a.clone()
    t, avg = timed(lambda: rl.delta_apply(base, idx, words, count, bad))
    print(f"apply : {k} changes: {t:.3f} ms (avg {avg:.3f})  {6 * k / t / 1e6:.1f} GB/s of changes")
    t2, _ = timed(lambda: b.copy_(a), reps=5)
    print(f"torch copy of one snapshot: {t2:.3f} ms  {2 * n * 2 / t2 / 1e6:.1f} GB/s (R+W)")


if __name__ == "__main__":
    main()
