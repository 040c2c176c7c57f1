"""Dump a config's barycenter v-state after --iters iterations (log domain) to gpurun_out/ (analysis)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import se2_synth as S
from paper_2402_15322_b200 import Kernel, se2_barycenter
ap = argparse.ArgumentParser(); ap.add_argument("--cfg", default="c3"); ap.add_argument("--iters", type=int, default=300)
a = ap.parse_args()
cfg = S.get_config(a.cfg); d = S.config_inputs(cfg)
lams = np.atleast_2d(np.stack(d["lambdas"])); n = len(d["mus"])
k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=n * lams.shape[0])
mus = torch.from_numpy(np.stack(d["mus"])).cuda()
v = torch.empty((lams.shape[0], n) + cfg.shape, device="cuda"); w = torch.empty_like(v)
bary, _ = se2_barycenter(k, mus, lams, a.iters, True, v_state=v, w_state=w)
np.savez_compressed(f"gpurun_out/state_{a.cfg}_{a.iters}.npz", v=v.cpu().numpy(), w=w.cpu().numpy(), bary=bary.cpu().numpy())
