"""One rank's share of the c4 slab split on ONE GPU: the conv of slab `index` of `nslabs` (owned rows + R-row halos,
output window = the owned rows), CUDA events, default engine and K2.  The compute side of the strong-scaling
projection (the halo exchange is not timed here).   python tools/time_slab_conv.py [nslabs ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import se2_synth as S  # noqa: E402
from paper_2402_15322_b200 import _lib as L, se2_conv  # noqa: E402
from paper_2402_15322_b200.dist import slab_kernel  # noqa: E402

cfg = S.get_config("c4")
for nslabs in [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]:
    k, row0, rows, top, bot = slab_kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, nslabs, nslabs // 2)
    x = torch.rand((1, cfg.ntheta, top + rows + bot, cfg.nx), device="cuda") + 0.1
    y = torch.empty_like(x)
    out = []
    for name, fl in (("default", 0), ("K10", L.SE2_LIN_TC), ("K2", L.SE2_LIN_FFMA)):
        for _ in range(3):
            se2_conv(k, x, y, log_domain=False, extra_flags=fl)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            se2_conv(k, x, y, log_domain=False, extra_flags=fl)
        e1.record()
        torch.cuda.synchronize()
        out.append(f"{name} {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
    print(f"c4 slab {nslabs // 2} of {nslabs}: rows {rows} (+{top}+{bot} halo), uses_tensor_cores {k.uses_tensor_cores}: "
          + ", ".join(out), flush=True)
    if os.environ.get("SE2_TC_DIAG_PROF"):
        k.tc_tile_stats()   # prints the issuer's cycle counters (stderr)
    k.close()
