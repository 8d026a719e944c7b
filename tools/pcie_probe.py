import torch, time
n = 1 << 30  # 1 GiB
h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=5):
    f(); torch.cuda.synchronize(); t0 = time.time()
    for _ in range(reps): f()
    torch.cuda.synchronize(); return (time.time() - t0) / reps
h2d = t(lambda: d1.copy_(h1, non_blocking=True)); print(f"H2D {n/h2d/1e9:.1f} GB/s")
d2h = t(lambda: h2.copy_(d2, non_blocking=True)); print(f"D2H {n/d2h/1e9:.1f} GB/s")
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
bi = t(both); print(f"bidirectional {2*n/bi/1e9:.1f} GB/s aggregate ({n/bi/1e9:.1f} per direction)")
