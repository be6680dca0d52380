import torch, time
n = 268435456
h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(n, dtype=torch.uint8).pin_memory(); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / reps
def h2d():
    d1.copy_(h1, non_blocking=True)
def d2h():
    h2.copy_(d2, non_blocking=True)
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
x = t(h2d); y = t(d2h); z = t(both)
print(f"H2D {n/x/1e9:.1f} GB/s  D2H {n/y/1e9:.1f} GB/s  both {2*n/z/1e9:.1f} GB/s total ({z*1e3:.2f} ms for 2x{n>>20} MiB)")
