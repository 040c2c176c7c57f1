import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle as O
from paper_2402_15322_b200 import Kernel, se2_conv, _lib as L
nx, ny, nt, eps, w, R = 64, 64, 32, 0.01, (1.0, 4.0, 2.0), 7
k = Kernel(nx, ny, nt, eps, w, R, max_batch=2)
rng = np.random.default_rng(7)
X, Y = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
lv = np.empty((2, nt, ny, nx))
for b in range(2):
    for t in range(nt):
        gx, gy = rng.uniform(-40, 40, 2)
        lv[b, t] = gx * X + gy * Y + 0.02 * (X - nx / 2) ** 2 + rng.uniform(-3, 3, (ny, nx)) + 50 * t
lv = lv.astype(np.float32)
ref = O.lse_conv(O.log_kernel_table(O.Grid(nx, ny, nt), R, eps, w), lv.astype(np.float64))
x = torch.from_numpy(lv).cuda()
for name, fl in [("default", 0), ("notilt", L.SE2_LSE_NOTILT), ("k3exact", L.SE2_LSE_K3EXACT)]:
    k.lse_path_stats(reset=True)
    y = se2_conv(k, x, log_domain=True, extra_flags=fl).cpu().numpy().astype(np.float64)
    ps = k.lse_path_stats(reset=True)
    bad = ~np.isfinite(y)
    d = np.abs(y - ref)
    d[bad] = np.inf
    print(name, ps, "nonfinite", bad.sum(), "maxerr finite", np.nanmax(np.where(bad, np.nan, d)), "ref range", ref.min(), ref.max())
    if bad.sum():
        idx = np.argwhere(bad)[:5]; print("  bad at", idx.tolist(), [y[tuple(i)] for i in idx])
