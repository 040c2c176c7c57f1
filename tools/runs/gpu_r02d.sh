#!/bin/bash
mkdir -p gpurun_out/r02d
timeout 1200 python -m pytest tests/test_gpu_ops.py tests/test_gpu_parity.py -q -rf --timeout 900 -k "precise and not c3m and not c3q" > gpurun_out/r02d/pytest_precise.log 2>&1; echo "precise rc $?"
python - > gpurun_out/r02d/timing.log 2>&1 <<'PY'
import numpy as np, torch, time, sys
sys.path.insert(0, '.')
import se2_synth as S
from paper_2402_15322_b200 import Kernel, se2_barycenter, se2_barycenter_precise
for name in ["c1", "c2", "c3"]:
    cfg = S.get_config(name); d = S.config_inputs(cfg)
    lams = np.atleast_2d(np.stack(d["lambdas"])); n = len(d["mus"])
    k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=n * lams.shape[0])
    mus = torch.from_numpy(np.stack(d["mus"])).cuda()
    it = 20 if name == "c3" else cfg.iters
    for fn in (se2_barycenter, se2_barycenter_precise):
        args = (k, mus, lams, it, True) if fn is se2_barycenter else (k, mus, lams, it)
        fn(*args); torch.cuda.synchronize()
        t = time.time(); fn(*args); torch.cuda.synchronize(); dt = time.time() - t
        print(name, fn.__name__, f"{it / dt:.1f} it/s", flush=True)
PY
echo "timing rc $?"
