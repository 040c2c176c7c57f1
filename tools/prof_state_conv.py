"""Log-domain conv (K3) on a realistic state: run a config's barycenter for --iters iterations, then
apply se2_conv (log) to the resulting v-state a few times (for ncu / timing of K3 mid-solve).

    python tools/prof_state_conv.py --cfg c3 --iters 100 --reps 3 [--exact]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import se2_synth as S  # noqa: E402
from paper_2402_15322_b200 import Kernel, se2_barycenter, se2_conv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="c3")
ap.add_argument("--iters", type=int, default=100)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--exact", action="store_true")
a = ap.parse_args()
cfg = S.get_config(a.cfg)
d = S.config_inputs(cfg)
lams = np.atleast_2d(np.stack(d["lambdas"]))
n = len(d["mus"])
F = n * lams.shape[0]
k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=F)
mus = torch.from_numpy(np.stack(d["mus"])).cuda()
v = torch.empty((lams.shape[0], n) + cfg.shape, device="cuda")
w = torch.empty_like(v)
se2_barycenter(k, mus, lams, a.iters, True, v_state=v, w_state=w)
y = torch.empty_like(v)
se2_conv(k, v, y, log_domain=True, lse_exact=a.exact)
torch.cuda.synchronize()
k.lse_path_stats(reset=True)
k.lse_row_stats(reset=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    se2_conv(k, v, y, log_domain=True, lse_exact=a.exact)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
ps = k.lse_path_stats(reset=True)
rs = k.lse_row_stats(reset=True)
vv = v.cpu().numpy()
print(f"{a.cfg} state after {a.iters} iters: lv range [{vv.min():.1f}, {vv.max():.1f}]; "
      f"{'K4' if a.exact else 'K3'} conv over {F} fields: {ms:.3f} ms; pairs {ps}, "
      f"active {ps['active'] / max(ps['visited'], 1):.3f}, ffma/active {ps['ffma'] / max(ps['active'], 1):.3f}, "
      f"exact rows live {rs['live'] / max(rs['visited'], 1):.3f}")
