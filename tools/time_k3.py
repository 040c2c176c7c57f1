"""Iterations/s of the fp32-potential barycenter (K3) on c1-c3 with its path statistics (CUDA events, one
warm-up solve).  python tools/time_k3.py [c1 c2 c3] [--iters N]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import se2_synth as S  # noqa: E402
from paper_2402_15322_b200 import Kernel, se2_barycenter  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--") and not a.isdigit()]
iters_over = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else None
for name in (args or ["c1", "c2", "c3"]):
    cfg = S.get_config(name)
    d = S.config_inputs(cfg)
    lams = np.atleast_2d(np.stack(d["lambdas"]))
    n = len(d["mus"])
    k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=n * lams.shape[0])
    mus = torch.from_numpy(np.stack(d["mus"])).cuda()
    it = iters_over or cfg.iters
    se2_barycenter(k, mus, lams, it, True)
    torch.cuda.synchronize()
    k.lse_path_stats(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    se2_barycenter(k, mus, lams, it, True)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} se2_barycenter: {it / (e0.elapsed_time(e1) / 1000.0):.1f} it/s ({it} iterations) "
          f"stats {k.lse_path_stats(reset=True)}", flush=True)
    k.close()
