"""Where does a linear Sinkhorn on K10 drift from the oracle? (diagnostic)"""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np, torch
import oracle as O, se2_synth as S
from paper_2402_15322_b200 import Kernel, _lib as L, se2_conv
from paper_2402_15322_b200.api import _ptr, _stream
nx, ny, nt, R, eps, w = 48, 40, 16, 5, 0.02, (1.0, 3.0, 1.0)
k = Kernel(nx, ny, nt, eps, w, R, max_batch=2)
g = O.Grid(nx, ny, nt)
T, Lt = O.kernel_table(g, R, eps, w), O.log_kernel_table(g, R, eps, w)
mu = S.stroke_measure(nx, ny, nt, 3, seed=71).astype(np.float32).astype(np.float64)
nu = S.stroke_measure(nx, ny, nt, 3, seed=72).astype(np.float32).astype(np.float64)
for iters in (1, 5, 20, 60):
    ref = O.sinkhorn(T, Lt, mu, nu, iters, log_domain=False, trace=False)
    for eng, fl in (("tc", L.SE2_LIN_TC), ("ffma", L.SE2_LIN_FFMA)):
        a, b = torch.empty((1, nt, ny, nx), device="cuda"), torch.empty((1, nt, ny, nx), device="cuda")
        opts = L.se2_opts(iters, fl)
        mu_d = torch.from_numpy(mu[None].astype(np.float32)).cuda(); nu_d = torch.from_numpy(nu[None].astype(np.float32)).cuda()
        L.check(L.load().se2_sinkhorn(k.handle, _ptr(mu_d), _ptr(nu_d), _ptr(a), _ptr(b), 1, None, ctypes.byref(opts), None, _stream(mu_d.device)))
        torch.cuda.synchronize()
        la, lb = np.log(a.cpu().numpy()[0].astype(np.float64)), np.log(b.cpu().numpy()[0].astype(np.float64))
        ra, rb = np.log(ref["a"]), np.log(ref["b"])
        da, db = np.abs(la - ra), np.abs(lb - rb)
        i = np.unravel_index(np.argmax(da), da.shape)
        print(f"iters {iters:3d} {eng:5s}: max|dlog a| {da.max():.3e} at {i} (ref log a {ra[i]:.2f}, log mu {np.log(mu[i]):.2f}); "
              f"max|dlog b| {db.max():.3e}; median |dlog a| {np.median(da):.2e}; range log a [{ra.min():.1f},{ra.max():.1f}] log b [{rb.min():.1f},{rb.max():.1f}]")
# one conv on a wide-range input: relative error vs oracle, by magnitude
x = np.exp(np.random.default_rng(1).uniform(-80, 0, (1, nt, ny, nx)))
ref = O.conv(T, x)
for eng, fl in (("tc", L.SE2_LIN_TC), ("ffma", L.SE2_LIN_FFMA)):
    y = se2_conv(k, torch.from_numpy(x.astype(np.float32)).cuda(), extra_flags=fl).cpu().numpy().astype(np.float64)
    rel = np.abs(y - ref) / ref
    print(eng, "conv on e^U(-80,0): max rel", rel.max(), "median", np.median(rel))
