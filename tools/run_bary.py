"""Run a config's barycenter solve (for ncu captures of the in-solver kernels, e.g. hinted K3)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import se2_synth as S
from paper_2402_15322_b200 import Kernel, se2_barycenter
ap = argparse.ArgumentParser(); ap.add_argument("--cfg", default="c3"); ap.add_argument("--iters", type=int, default=250)
ap.add_argument("--no-graph", action="store_true")
a = ap.parse_args()
cfg = S.get_config(a.cfg); d = S.config_inputs(cfg)
lams = np.atleast_2d(np.stack(d["lambdas"])); n = len(d["mus"])
k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=n * lams.shape[0])
mus = torch.from_numpy(np.stack(d["mus"])).cuda()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
se2_barycenter(k, mus, lams, a.iters, True, no_graph=a.no_graph)
e1.record(); torch.cuda.synchronize()
print(f"{a.cfg} barycenter {a.iters} iters: {e0.elapsed_time(e1):.1f} ms")
