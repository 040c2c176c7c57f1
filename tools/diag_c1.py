import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import se2_synth as S
from paper_2402_15322_b200 import Kernel, se2_barycenter
from gpu_util import potential_err
case = sys.argv[1] if len(sys.argv) > 1 else "c1"
pc = S.get_parity_case(case); cfg, d = S.parity_inputs(pc)
gold = dict(np.load(f"tests/golden/{case}.npz"))
lams = gold["lambdas"]; n, ns = len(d["mus"]), lams.shape[0]
k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=n * ns)
mus = torch.from_numpy(np.stack(d["mus"])).cuda()
v = torch.empty((ns, n) + cfg.shape, device="cuda"); w = torch.empty_like(v)
bary, tr = se2_barycenter(k, mus, lams, cfg.iters, True, v_state=v, w_state=w, trace=True)
V = v.cpu().numpy().astype(np.float64).reshape(ns, n, -1); W = w.cpu().numpy().astype(np.float64).reshape(ns, n, -1)
B = bary.cpu().numpy().astype(np.float64).reshape(ns, -1)
for s in range(ns):
    print("solve", s, lams[s], "lbary err", potential_err(B[s], gold["lbary"].reshape(ns, -1)[s]))
    for i in range(n):
        gv = gold["lv"].reshape(ns, n, -1)[s, i]; gw = gold["lw"].reshape(ns, n, -1)[s, i]
        dv = V[s, i] - gv; dw = W[s, i] - gw
        print(f"   input {i}: lv range [{gv.min():.1f},{gv.max():.1f}] err {potential_err(V[s,i], gv):.2e} mean diff {dv.mean():+.3e} std {dv.std():.2e} | lw err {potential_err(W[s,i], gw):.2e} mean {dw.mean():+.3e}")
import sys as _s
sys.path.insert(0, "tests")
from gpu_util import measure_err
G = gold["bary_lin"].reshape(ns, -1)
for s in range(ns):
    g = np.exp(B[s]); r = G[s]
    for fl in (1e-6, 1e-5, 1e-4):
        print(f"solve {s} measure err floor {fl:g}: {measure_err(g, r, fl):.3e}")
    rel = np.abs(g - r) / np.maximum(r, 1e-6 * r.max())
    i = np.argmax(rel); print("   worst at", i, "ref", r[i], "max ref", r.max(), "got", g[i])
