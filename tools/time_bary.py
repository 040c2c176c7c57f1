"""Iterations/s of the fp32-potential (K3) and fp64-potential (K4P) barycenter engines on c1-c3 (CUDA events,
one warm-up solve).  python tools/time_bary.py [c1 c2 c3] [--iters N]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import se2_synth as S  # noqa: E402
from paper_2402_15322_b200 import Kernel, se2_barycenter, se2_barycenter_precise  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
iters_over = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else None
for name in (args or ["c1", "c2", "c3"]):
    if name.isdigit():
        continue
    cfg = S.get_config(name)
    d = S.config_inputs(cfg)
    lams = np.atleast_2d(np.stack(d["lambdas"]))
    n = len(d["mus"])
    k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=n * lams.shape[0])
    mus = torch.from_numpy(np.stack(d["mus"])).cuda()
    it = iters_over or cfg.iters
    for fn in (se2_barycenter, se2_barycenter_precise):
        call = (lambda: fn(k, mus, lams, it, True)) if fn is se2_barycenter else (lambda: fn(k, mus, lams, it))
        call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        torch.cuda.synchronize()
        extra = ""
        if fn is se2_barycenter_precise:
            ps = k.precise_path_stats(reset=True)
            extra = f", K4P channels on the FFMA path {ps['ffma']}/{ps['channels']}, hinted CTAs redone {ps['hint_redos']}"
        print(f"{name} {fn.__name__}: {it / (e0.elapsed_time(e1) / 1000.0):.1f} it/s ({it} iterations){extra}", flush=True)
    k.close()
