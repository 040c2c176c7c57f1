"""Small invocations of every hot kernel for compute-sanitizer (one workload per argument):

    compute-sanitizer --tool racecheck python tools/sanitize.py k10
    compute-sanitizer --tool synccheck python tools/sanitize.py k9 k3
    compute-sanitizer --tool memcheck  python tools/sanitize.py all

k10   : tensor-core linear conv, balanced mode (3 fields) and rows mode, incl. a thin grid (npad 16)
k2    : FFMA linear conv (TMA staging) + fused JKO prox epilogue
k3/k4 : log-domain convs (FFMA path, exact path with hints, theta_i split + combine)
k9    : one-launch cluster Sinkhorn (DSMEM exchange)
slab  : slab convs with peer-halo epilogue stores (3 slabs of one grid on one GPU)
bary  : barycenter solve (log domain) + fused reduce/update kernel
lift  : lifting / projection kernels
"""
import os
import sys

import ctypes

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2402_15322_b200 import _lib as L  # noqa: E402
from paper_2402_15322_b200 import (Kernel, make_prox, se2_barycenter, se2_conv, se2_jko_step,  # noqa: E402
                                   se2_sinkhorn)


def _f(shape, seed, lo=-3.0, hi=0.0):
    rng = np.random.default_rng(seed)
    return torch.from_numpy(np.exp(rng.uniform(lo, hi, shape)).astype(np.float32)).cuda()


def k10():
    for (nx, ny, nt, R, batch, pieces, eps) in [(37, 53, 32, 7, 3, "1", 0.01), (37, 53, 32, 7, 1, "0", 0.01),
                                                (16, 5, 32, 2, 2, "1", 0.01), (72, 44, 16, 15, 1, "1", 0.01),
                                                (40, 36, 64, 15, 2, "1", 0.003), (40, 36, 64, 15, 1, "0", 0.003)]:
        os.environ["SE2_TC_PIECES"] = pieces
        k = Kernel(nx, ny, nt, eps, (1.0, 3.0, 1.0), R, max_batch=batch)
        x = _f((batch, nt, ny, nx), nx + ny)
        se2_conv(k, x, extra_flags=L.SE2_LIN_TC)
        # narrow geometry (nt >= 32): tiles on the 16-orientation window and, with an e^80 input range,
        # on the 32-orientation fallback window
        se2_conv(k, _f((batch, nt, ny, nx), nx + ny + 1, lo=-80.0, hi=0.0), extra_flags=L.SE2_LIN_TC)
        mu = _f((nt, ny, nx), 3)
        mu /= mu.sum()
        a, b, nxt = torch.empty_like(mu), torch.empty_like(mu), torch.empty_like(mu)
        se2_jko_step(k, mu, nxt, a, b, 3, make_prox(k, 1e-3), False, trace=True, engine_flags=L.SE2_LIN_TC)
    os.environ.pop("SE2_TC_PIECES", None)


def k2():
    k = Kernel(40, 36, 16, 0.01, (1.0, 3.0, 1.0), 5, max_batch=2)
    se2_conv(k, _f((2, 16, 36, 40), 1), extra_flags=L.SE2_LIN_FFMA)
    mu = _f((16, 36, 40), 2)
    mu /= mu.sum()
    a, b, nxt = torch.empty_like(mu), torch.empty_like(mu), torch.empty_like(mu)
    se2_jko_step(k, mu, nxt, a, b, 3, make_prox(k, 1e-3), False, trace=True, engine_flags=L.SE2_LIN_FFMA)


def k3():
    rng = np.random.default_rng(5)
    k = Kernel(44, 40, 32, 0.005, (1.0, 3.0, 1.0), 10, max_batch=2)
    for span in (20.0, 2000.0):
        x = torch.from_numpy(rng.uniform(-span / 2, span / 2, (2, 32, 40, 44)).astype(np.float32)).cuda()
        se2_conv(k, x, log_domain=True)
        se2_conv(k, x, log_domain=True, lse_exact=True)


def k9():
    k = Kernel(16, 16, 8, 0.05, (1.0, 3.0, 1.0), 3, max_batch=1)
    mu, nu = _f((8, 16, 16), 1), _f((8, 16, 16), 2)
    mu /= mu.sum()
    nu /= nu.sum()
    a, b = torch.empty_like(mu), torch.empty_like(mu)
    se2_sinkhorn(k, mu, nu, a, b, 5, True, trace=True)


def bary():
    k = Kernel(28, 28, 16, 0.02, (1.0, 3.0, 1.0), 5, max_batch=4)
    mus = torch.stack([_f((16, 28, 28), s) for s in (1, 2)])
    mus /= mus.sum(dim=(1, 2, 3), keepdim=True)
    se2_barycenter(k, mus, np.array([[0.3, 0.7], [1.0, 0.0]]), 4, True, trace=True, no_graph=True)
    from paper_2402_15322_b200.api import se2_bary_reduce_update
    N = 1000
    parts = [torch.randn(N, device="cuda") for _ in range(3)]
    table = torch.tensor([p.data_ptr() for p in parts], dtype=torch.int64, device="cuda")
    lv, ld, lbar = torch.randn(2, N, device="cuda"), torch.randn(2, N, device="cuda"), torch.empty(N, device="cuda")
    se2_bary_reduce_update(table, 2, N, lv, ld, lbar)


def precise():
    """fp64-potential barycenter (K4P exact log-domain conv + fp64 epilogues)."""
    from paper_2402_15322_b200 import se2_barycenter_precise
    k = Kernel(28, 28, 16, 0.02, (1.0, 3.0, 1.0), 5, max_batch=4)
    mus = torch.stack([_f((16, 28, 28), s) for s in (1, 2)])
    mus /= mus.sum(dim=(1, 2, 3), keepdim=True)
    se2_barycenter_precise(k, mus, np.array([[0.3, 0.7], [1.0, 0.0]]), 3, trace=True)


def slab():
    """3 slabs of a 48 x 40 x 16 grid on one GPU; each conv's epilogue writes its boundary rows into the
    neighbours' halo rows (peer pointers = plain device pointers here), slab after slab on one stream."""
    from paper_2402_15322_b200.api import _ptr, se2_conv_update
    nx, ny, nt, R = 48, 40, 16, 4
    bounds = [(0, 14), (14, 27), (27, 40)]
    ks, xs, outs = [], [], []
    for (r0, r1) in bounds:
        rows = r1 - r0
        ks.append(Kernel(nx, rows + 2 * R, nt, 0.003, (1, 3, 1), R, hx=1.0 / nx, hy=1.0 / ny))
        xs.append(_f((nt, rows + 2 * R, nx), r0))
        outs.append(torch.zeros(nt, rows + 2 * R, nx, device="cuda"))
    for eng in (L.SE2_LIN_FFMA, L.SE2_LIN_TC):
        for i, (r0, r1) in enumerate(bounds):
            rows = r1 - r0
            up = outs[i - 1] if i > 0 else None
            dn = outs[i + 1] if i + 1 < len(bounds) else None
            # own rows [R, R + rows); up's halo rows below its own: row (R + rows_up) + (row - R)
            rows_up = bounds[i - 1][1] - bounds[i - 1][0] if i > 0 else 0
            sl = L.se2_slab(R, R + rows, R, _ptr(up) if up is not None else None, rows_up,
                            (rows_up + 2 * R) if up is not None else 0,
                            _ptr(dn) if dn is not None else None, rows,
                            (bounds[i + 1][1] - bounds[i + 1][0] + 2 * R) if dn is not None else 0)
            tgt = torch.ones_like(xs[i])
            L.check(L.load().se2_conv_update_slab(ks[i].handle, _ptr(xs[i]), _ptr(tgt), _ptr(outs[i]), 1,
                                                  L.SE2_EPI_DIVIDE, None, eng, ctypes.byref(sl), None))


def lift():
    from paper_2402_15322_b200.lifting import Cake, se2_lift_image, se2_project, se2_split_signed
    c = Cake(16, 11)
    img = torch.rand(2, 40, 36, device="cuda")
    U = se2_lift_image(c, img)
    se2_split_signed(c, U, floor_rel=1e-6)
    se2_project(c, U)


ALL = dict(k10=k10, k2=k2, k3=k3, k9=k9, bary=bary, precise=precise, slab=slab, lift=lift)

if __name__ == "__main__":
    names = sys.argv[1:] or ["all"]
    if names == ["all"]:
        names = list(ALL)
    for n in names:
        ALL[n]()
        torch.cuda.synchronize()
        print(f"sanitize workload {n}: ok", flush=True)
