"""Host<->device staging costs for a 16 MB vector (pageable vs pinned)."""
import time

import numpy as np
import torch

n = 2097152
xd = torch.randn(n, dtype=torch.float64, device="cuda")
bn = np.random.default_rng(0).standard_normal(n)


def d2h_pageable():
    return xd.cpu()


def d2h_pinned():
    xo = torch.empty(n, dtype=torch.float64, pin_memory=True)
    xo.copy_(xd, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return xo


def h2d_pageable():
    return torch.from_numpy(bn).cuda()


def h2d_staged():
    p = torch.empty(n, dtype=torch.float64, pin_memory=True)
    p.numpy()[:] = bn
    return p.to("cuda", non_blocking=True)


for f in (d2h_pageable, d2h_pinned, h2d_pageable, h2d_staged):
    rs = [f() for _ in range(3)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        rs.append(f())
        rs.pop(0)
    torch.cuda.synchronize()
    print(f.__name__, round((time.perf_counter() - t0) / 20 * 1e3, 3), "ms")
