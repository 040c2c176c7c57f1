import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle as O
from paper_2402_15322_b200 import Kernel, se2_conv, _lib as L
nx, ny, nt, eps, w, R = 48, 64, 4, 0.01, (1.0, 4.0, 2.0), 7
k = Kernel(nx, ny, nt, eps, w, R, max_batch=1)
Lt = O.log_kernel_table(O.Grid(nx, ny, nt), R, eps, w)
X, Y = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
for gx, gy, curv in [(0, 0, 0.05), (8, 0, 0), (0, 8, 0), (8, 8, 0), (30, 0, 0), (0, 30, 0), (-20, 15, 0.02)]:
    lv = np.stack([gx * X + gy * Y + curv * (X - 20.0) ** 2 * 40 + 0.0 * t for t in range(nt)]).astype(np.float32)
    ref = O.lse_conv(Lt, lv.astype(np.float64))
    k.lse_path_stats(reset=True)
    y = se2_conv(k, torch.from_numpy(lv).cuda(), log_domain=True).cpu().numpy().astype(np.float64)
    ps = k.lse_path_stats(reset=True)
    d = np.abs(y - ref)
    i = np.unravel_index(np.nanargmax(np.where(np.isfinite(d), d, 1e30)), d.shape)
    print(f"g=({gx},{gy}) curv={curv}: {ps} maxerr {d.max():.3e} at {i} y={y[i]:.3f} ref={ref[i]:.3f}")
