"""One fp64-potential barycenter solve of a config (for ncu captures).  python tools/run_bary_precise.py c2 [iters]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import se2_synth as S  # noqa: E402
from paper_2402_15322_b200 import Kernel, se2_barycenter_precise  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = S.get_config(name)
d = S.config_inputs(cfg)
lams = np.atleast_2d(np.stack(d["lambdas"]))
n = len(d["mus"])
k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=n * lams.shape[0])
mus = torch.from_numpy(np.stack(d["mus"])).cuda()
it = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.iters
se2_barycenter_precise(k, mus, lams, it, no_graph=True)
torch.cuda.synchronize()
print("done", name, it)
