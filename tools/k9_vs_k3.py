"""Sinkhorn on several grid sizes: K9 (one cluster launch) vs the per-conv K3 path (CUDA graph)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2402_15322_b200 import Kernel, se2_sinkhorn
for (nx, ny, nt, R, eps) in [(16, 16, 8, 3, 0.05), (24, 24, 8, 3, 0.05), (28, 28, 16, 5, 0.02), (32, 32, 16, 3, 0.05), (40, 40, 8, 4, 0.03)]:
    rng = np.random.default_rng(0)
    mu = rng.random((nt, ny, nx)).astype(np.float32) ** 3 + 1e-6; mu /= mu.sum()
    nu = rng.random((nt, ny, nx)).astype(np.float32) ** 3 + 1e-6; nu /= nu.sum()
    k = Kernel(nx, ny, nt, eps, (1.0, 3.0, 1.0), R)
    m, n = torch.from_numpy(mu).cuda(), torch.from_numpy(nu).cuda()
    a, b = torch.empty_like(m), torch.empty_like(m)
    res = {}
    for pers in (True, False):
        se2_sinkhorn(k, m, n, a, b, 100, True, trace=True, persistent=pers)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            se2_sinkhorn(k, m, n, a, b, 100, True, trace=True, persistent=pers)
        e1.record(); torch.cuda.synchronize()
        res["K9" if pers else "K3"] = e0.elapsed_time(e1) / 3
    print(f"{nx}x{ny}x{nt} R{R}: N*box = {nx*ny*nt*(2*R+1)**2*nt:.3e}  K9 {res['K9']:.3f} ms  K3+graph {res['K3']:.3f} ms per 100 it")
