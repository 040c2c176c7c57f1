"""c4 JKO steps through se2_jko_step (no per-conv timing events), CUDA events around 5 steps after 3 warm-up steps.
python tools/time_jko.py   (SE2_GRAPH_MAX_LOG2=23: the step replayed as a CUDA graph)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import se2_synth as S  # noqa: E402
from paper_2402_15322_b200 import Kernel, make_prox, se2_jko_step  # noqa: E402

cfg = S.get_config("c4")
d = S.config_inputs(cfg)
k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=1)
prox = make_prox(k, cfg.tau)
mu = torch.from_numpy(d["mus"][0]).cuda()
nxt, a, b = torch.empty_like(mu), torch.empty_like(mu), torch.empty_like(mu)
for _ in range(4):
    se2_jko_step(k, mu, nxt, a, b, cfg.iters, prox, False)
    mu, nxt = nxt, mu
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(6):
    se2_jko_step(k, mu, nxt, a, b, cfg.iters, prox, False)
    mu, nxt = nxt, mu
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 6
print(f"c4 JKO step: {ms:.2f} ms, {cfg.iters / ms * 1e3:.0f} inner iterations/s (graph max log2 {os.environ.get('SE2_GRAPH_MAX_LOG2', '21')})")
