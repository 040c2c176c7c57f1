"""Run the group convolution of one config a few times (for ncu captures / quick timing).

    python tools/prof_conv.py --cfg c4 [--log] [--reps 5] [--batch B]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import se2_synth as S  # noqa: E402
from paper_2402_15322_b200 import Kernel, se2_conv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="c4")
ap.add_argument("--log", action="store_true")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--batch", type=int, default=1)
a = ap.parse_args()
cfg = S.get_config(a.cfg)
k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=a.batch)
st = k.stats()
x = torch.from_numpy(S.random_positive_field((a.batch,) + cfg.shape, seed=1, log_range=20.0)).cuda()
if a.log:
    x = torch.log(x)
y = torch.empty_like(x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
se2_conv(k, x, y, log_domain=a.log)
torch.cuda.synchronize()
e0.record()
for _ in range(a.reps):
    se2_conv(k, x, y, log_domain=a.log)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
work = 2.0 * cfg.N * a.batch * (st["box_taps"] if a.log else st["nnz_taps"])
ts = k.tc_tile_stats() if (not a.log and k.has_tensor_cores) else {}
print(f"{a.cfg} {'log' if a.log else 'linear'} batch {a.batch}: {ms:.3f} ms/conv, tc tiles {ts}, "
      f"{work / ms / 1e9:.2f} T(flop|tap-op)/s, nnz {st['nnz_taps']} box {st['box_taps']} band {st['theta_band']}")
