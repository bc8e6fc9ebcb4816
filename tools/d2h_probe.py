import time, torch
n = 2097152
xd = torch.randn(n, dtype=torch.float64, device="cuda")
def a():
    return xd.cpu()
def b():
    xo = torch.empty(n, dtype=torch.float64, pin_memory=True)
    xo.copy_(xd, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return xo
bh = torch.randn(n, dtype=torch.float64).pin_memory()
def h2d():
    return bh.to("cuda", non_blocking=True)
for f in (a, b, a, b, h2d):
    for _ in range(3): r = f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20): r = f()
    torch.cuda.synchronize()
    print(f.__name__, (time.perf_counter() - t0) / 20 * 1e3, "ms")
