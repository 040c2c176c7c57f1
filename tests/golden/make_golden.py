"""Expected values of the GPU parity tests, computed with oracle/ ONLY (never the CUDA path).

    OMP_NUM_THREADS=$(nproc) python tests/golden/make_golden.py [case ...]

Writes tests/golden/<case>.npz for the cases of se2_synth.PARITY_CASES.  Whole fields are stored
for the small cases; for the full-size prefixes a seeded sample of entries (se2_synth.sample_indices).
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402
import se2_synth as S  # noqa: E402

N_SAMPLES = 20000


def _store(out, name, arr, pc, idx):
    arr = np.asarray(arr)
    if pc.full_fields:
        out[name] = arr
    else:
        out[name] = arr.reshape(arr.shape[:-3] + (-1,))[..., idx]


def make(pc):
    cfg, d = S.parity_inputs(pc)
    g = O.Grid(cfg.nx, cfg.ny, cfg.ntheta, cfg.cell, cfg.cell)
    T = O.kernel_table(g, cfg.R, cfg.eps, cfg.w)
    L = O.log_kernel_table(g, cfg.R, cfg.eps, cfg.w)
    N = cfg.N
    idx = S.sample_indices(N, N_SAMPLES, seed=7)
    out = dict(sample_idx=idx, log_domain=np.array(cfg.log_domain))
    mus = [m.astype(np.float64) for m in d["mus"]]
    if cfg.problem == "sinkhorn":
        r = O.sinkhorn(T, L, mus[0], mus[1], cfg.iters, cfg.log_domain)
        for k in ("alpha", "beta", "a", "b", "row", "col"):
            if k in r:
                _store(out, k, r[k], pc, idx)
        out["err"] = r["err"]
    elif cfg.problem == "barycenter":
        lams = d["lambdas"]
        res = [O.barycenter(T, L, mus, lam, cfg.iters, cfg.log_domain) for lam in lams]
        out["lambdas"] = np.stack([np.asarray(l) for l in lams])
        key_b = "lbary" if cfg.log_domain else "bary"
        _store(out, key_b, np.stack([r[key_b] for r in res]), pc, idx)
        _store(out, "bary_lin", np.stack([r["bary"] for r in res]), pc, idx)
        kv = "lv" if cfg.log_domain else "v"
        kw = "lw" if cfg.log_domain else "w"
        _store(out, kv, np.stack([r[kv] for r in res]), pc, idx)
        _store(out, kw, np.stack([r[kw] for r in res]), pc, idx)
        out["err"] = np.stack([r["err"] for r in res], axis=1)          # [iters][nsolve]
        out["errs"] = np.stack([r["errs"] for r in res], axis=1)        # [iters][nsolve][n]
    elif cfg.problem == "jko":
        r = O.jko(T, L, mus[0], g, cfg.eps, cfg.tau, cfg.jko_steps, cfg.iters, cfg.log_domain,
                  energy=pc.energy, m=pc.m)
        _store(out, "mus", r["mus"], pc, idx)
        out["masses"] = r["masses"]
        out["err"] = r["err"]
        for k in ("a", "b", "alpha", "beta"):
            if k in r:
                _store(out, k, r[k], pc, idx)
    np.savez_compressed(os.path.join(HERE, f"{pc.name}.npz"), **out)


if __name__ == "__main__":
    names = sys.argv[1:] or [pc.name for pc in S.PARITY_CASES]
    for n in names:
        t0 = time.time()
        make(S.get_parity_case(n))
        print(f"{n}: {time.time() - t0:.1f} s (threads {O.oracle_threads()})", flush=True)
