import torch, time
n = 268435456 // 4
h1 = torch.empty(n).pin_memory(); h2 = torch.empty(n).pin_memory()
d1 = torch.empty(n, device="cuda"); d2 = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, it=5):
    torch.cuda.synchronize(); a = time.perf_counter()
    for _ in range(it): f()
    torch.cuda.synchronize(); return (time.perf_counter() - a) / it
h2d = t(lambda: d1.copy_(h1, non_blocking=True))
d2h = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
bo = t(both)
print(f"H2D {n*4/h2d/1e9:.1f} GB/s  D2H {n*4/d2h/1e9:.1f} GB/s  concurrent: {2*n*4/bo/1e9:.1f} GB/s total ({bo*1e3:.2f} ms for both)")
