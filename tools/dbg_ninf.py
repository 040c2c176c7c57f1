"""Debug: log-domain conv of fields with many -inf entries (lifted +- parts) vs the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle as O
from oracle import se2_lift as LF
from test_gpu_lifting import _smooth_image
from paper_2402_15322_b200 import Kernel, se2_conv, se2_barycenter
ny = nx = 20; N, L, R, eps, w = 8, 9, 3, 0.05, (1.0, 3.0, 1.0)
f0, f1 = _smooth_image(ny, nx, 21), _smooth_image(ny, nx, 22)
B = LF.cake_bank(N, L).real
U = LF.lift_image(np.stack([f0, f1]), B)
Up, Un, mp, mn = LF.split_signed(U)
g = O.Grid(nx, ny, N)
Lt = O.log_kernel_table(g, R, eps, w)
k = Kernel(nx, ny, N, eps, w, R, max_batch=6)
with np.errstate(divide="ignore"):
    lx = np.log(Up).astype(np.float32)
x = torch.from_numpy(lx).cuda()
for exact in (False, True):
    y = se2_conv(k, x, log_domain=True, lse_exact=exact).cpu().numpy().astype(np.float64)
    ref = O.lse_conv(Lt, lx.astype(np.float64))
    bad = ~np.isclose(y, ref, rtol=1e-5, atol=1e-5) & ~((y == -np.inf) & (ref == -np.inf))
    print("exact" if exact else "K3", "nan", np.isnan(y).sum(), "+inf", np.isposinf(y).sum(), "-inf", np.isneginf(y).sum(),
          "ref -inf", np.isneginf(ref).sum(), "mismatch", bad.sum())
mus = torch.from_numpy(np.stack([Up[0], Up[1]]).astype(np.float32)).cuda()
for no_graph in (False, True):
    try:
        b, _ = se2_barycenter(k, mus, np.array([[0.5, 0.5]]), 30, True, no_graph=no_graph)
        print("bary ok", torch.isnan(b).sum().item())
    except Exception as e:
        print("bary error", e)
v = torch.empty((1, 2, N, ny, nx), device="cuda"); ww = torch.empty_like(v)
for it in (1, 2, 3, 5):
    try:
        b, _ = se2_barycenter(k, mus, np.array([[0.5, 0.5]]), it, True, v_state=v, w_state=ww)
        print(it, "ok")
    except Exception as e:
        vv, wv = v.cpu().numpy(), ww.cpu().numpy()
        print(it, "fail", np.isnan(vv).sum(), np.isnan(wv).sum(), np.isposinf(vv).sum(), np.isposinf(wv).sum(), np.isneginf(vv).sum(), np.isneginf(wv).sum())
