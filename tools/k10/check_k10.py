"""K10 vs K2 on the config grids and odd grids: max relative difference and per-launch time.
    python tools/k10/check_k10.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import se2_synth as S  # noqa: E402
from paper_2402_15322_b200 import Kernel, se2_conv  # noqa: E402
from paper_2402_15322_b200 import _lib as L  # noqa: E402

cases = [("c1", None), ("c2", None), ("c3", None), ("c4", None),
         ("odd1", (72, 60, 16, 4)), ("odd2", (200, 130, 64, 15)), ("odd3", (37, 53, 32, 7)), ("odd4", (256, 9, 48, 2))]
for name, geo in cases:
    if geo is None:
        cfg = S.get_config(name)
        nx, ny, nt, R, eps, w = cfg.nx, cfg.ny, cfg.ntheta, cfg.R, cfg.eps, cfg.w
    else:
        nx, ny, nt, R = geo
        cfg = S.get_config("c4")
        eps, w = cfg.eps, cfg.w
    batch = 2
    k = Kernel(nx, ny, nt, eps, w, R, max_batch=batch)
    x = torch.from_numpy(S.random_positive_field((batch, nt, ny, nx), seed=3, log_range=10.0)).cuda()
    y10, y2 = torch.empty_like(x), torch.empty_like(x)
    se2_conv(k, x, y10)
    se2_conv(k, x, y2, extra_flags=L.SE2_LIN_FFMA)
    torch.cuda.synchronize()
    rel = ((y10 - y2).abs() / y2.abs().clamp_min(1e-30)).max().item()
    rel_floor = ((y10 - y2).abs() / y2.abs().clamp_min(1e-6 * y2.abs().max())).max().item()
    bias = ((y10 - y2) / y2.abs().clamp_min(1e-30)).mean().item()
    t = {}
    for tag, fl in (("k10", 0), ("k2", L.SE2_LIN_FFMA)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(2):
            se2_conv(k, x, y10, extra_flags=fl)
        e0.record()
        for _ in range(10):
            se2_conv(k, x, y10, extra_flags=fl)
        e1.record()
        torch.cuda.synchronize()
        t[tag] = e0.elapsed_time(e1) / 10 / batch
    print(f"{name:5s} {nx}x{ny}x{nt} R{R}: max rel {rel:.2e} (floored {rel_floor:.2e}, mean signed {bias:+.1e})  per field: K10 {t['k10']:.3f} ms  K2 {t['k2']:.3f} ms"
          f"  ({t['k2'] / t['k10']:.2f}x)", flush=True)
