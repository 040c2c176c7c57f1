"""Per-conv absolute error of the log-domain engines on real solver states (the c2m golden's final lv/lw,
fp64 oracle): which part of the arithmetic limits end-to-end potential parity.  Diagnostic only."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import se2_synth as S  # noqa: E402
from paper_2402_15322_b200 import Kernel, _lib as L, se2_conv  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "c2m"
pc = S.get_parity_case(case)
cfg, d = S.parity_inputs(pc)
gold = dict(np.load(os.path.join(ROOT, "tests", "golden", f"{case}.npz")))
g = O.Grid(cfg.nx, cfg.ny, cfg.ntheta)
Lt = O.log_kernel_table(g, cfg.R, cfg.eps, cfg.w)
k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=1)
for name in ("lv", "lw"):
    X = gold[name].reshape((-1,) + g.shape)[:2]
    for i in range(X.shape[0]):
        x64 = X[i]
        x32 = x64.astype(np.float32)
        ref64 = O.lse_conv(Lt, x64)
        ref32in = O.lse_conv(Lt, x32.astype(np.float64))
        storage = np.abs(ref32in - ref64)
        for eng, fl in (("K3", 0), ("K3exact", L.SE2_LSE_K3EXACT), ("K4", L.SE2_LSE_EXACT)):
            y = se2_conv(k, torch.from_numpy(x32).cuda(), log_domain=True, extra_flags=fl).cpu().numpy().astype(np.float64)
            e = np.abs(y - ref32in)
            fin = np.isfinite(ref32in)
            sg = (y - ref32in)[fin]
            print(f"{case} {name}[{i}] range [{x64.min():.0f},{x64.max():.0f}] {eng:8s}: arith err max {e[fin].max():.2e} "
                  f"mean {e[fin].mean():.2e} signed mean {sg.mean():+.2e} | storage-rounding effect max "
                  f"{storage[fin].max():.2e} mean {storage[fin].mean():.2e}", flush=True)
