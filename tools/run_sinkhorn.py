"""Run a config's Sinkhorn solve (c0) a few times (for ncu captures of K9 / the K3 path)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import se2_synth as S
from paper_2402_15322_b200 import Kernel, se2_sinkhorn
ap = argparse.ArgumentParser(); ap.add_argument("--cfg", default="c0"); ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--no-persistent", action="store_true")
a = ap.parse_args()
cfg = S.get_config(a.cfg); d = S.config_inputs(cfg)
k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=1)
mu, nu = (torch.from_numpy(m.astype(np.float32)).cuda() for m in d["mus"][:2])
al, be = torch.empty_like(mu), torch.empty_like(mu)
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    se2_sinkhorn(k, mu, nu, al, be, cfg.iters, True, trace=True, persistent=not a.no_persistent)
    e1.record(); torch.cuda.synchronize()
    print(f"{a.cfg} sinkhorn {cfg.iters} iters: {e0.elapsed_time(e1):.3f} ms")
