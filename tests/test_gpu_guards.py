"""Counted division guard (reading R9), the safeguarded porous-medium prox and
the barycenter warm start (resume) -- through the C ABI (-m gpu)."""
import warnings

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def _host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy().astype(np.float64)


def test_division_guard_counted(cuda_device):
    """One linear Sinkhorn iteration with mu supported on a small square: a = mu / K1 vanishes off it, so
    z = K^T a is EXACTLY 0 at every site farther than R (box) from the square, and b = nu / max(z, 1e-30)
    clamps exactly there: count = ntheta x those sites; the solve returns the SE2_WGUARD_HIT warning."""
    from paper_2402_15322_b200 import Kernel, se2_sinkhorn
    nx, ny, nt, R, eps = 24, 20, 8, 2, 0.5
    k = Kernel(nx, ny, nt, eps, (1.0, 2.0, 1.0), R, max_batch=1)
    mu = np.zeros((nt, ny, nx))
    mu[:, 8:11, 5:9] = 1.0
    mu /= mu.sum()
    nu = np.full((nt, ny, nx), 1.0 / (nt * ny * nx))
    a, b = torch.empty(nt, ny, nx, device="cuda"), torch.empty(nt, ny, nx, device="cuda")
    with pytest.warns(UserWarning, match="SE2_WGUARD_HIT"):
        se2_sinkhorn(k, _dev(mu), _dev(nu), a, b, 1, False)
    yy, xx = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    near = (yy >= 8 - R) & (yy <= 10 + R) & (xx >= 5 - R) & (xx <= 8 + R)
    want = nt * int((~near).sum())
    assert k.guard_stats()["div_clamps"] == want
    # the oracle's iteration clamps the same denominators (R9): b matches where z > 0 and is nu / 1e-30
    # elsewhere
    g = O.Grid(nx, ny, nt)
    ref = O.sinkhorn(O.kernel_table(g, R, eps, (1.0, 2.0, 1.0)), None, mu, nu, 1, False, trace=False)
    np.testing.assert_allclose(_host(b), ref["b"], rtol=2e-5)
    # a solve with no clamp reports none (counters reset per solve)
    mu2 = np.full((nt, ny, nx), 1.0 / (nt * ny * nx))
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        se2_sinkhorn(k, _dev(mu2), _dev(nu), a, b, 3, False)
    assert k.guard_stats()["div_clamps"] == 0


@pytest.mark.parametrize("log_domain", [False, True])
def test_porous_prox_extreme_inputs(log_domain, cuda_device):
    """The porous-medium prox on conv outputs spanning 1e-30 .. 1e12 (z = K x, x = 10^U(-40, 12)): the
    safeguarded Newton must converge everywhere (no NaN, no count) and satisfy the stationarity
    condition C (s/cell)^{m-1} + log(s/z) = 0 in fp64 to fp32 accuracy."""
    from paper_2402_15322_b200 import Kernel, _lib as L, make_porous_prox, se2_conv, se2_conv_update
    nx, ny, nt, R, eps, tau, m = 24, 20, 16, 2, 0.003, 1e-3, 5.0
    k = Kernel(nx, ny, nt, eps, (1.0, 10 ** 0.5, 2 ** 0.5), R, max_batch=1)
    rng = np.random.default_rng(9)
    x = 10.0 ** rng.uniform(-40, 12, (nt, ny, nx))
    xin = np.log(x) if log_domain else x
    xd = _dev(xin)
    z = _host(se2_conv(k, xd, log_domain=log_domain))
    lz = z if log_domain else np.log(np.maximum(z, 1e-30))
    out = torch.empty_like(xd)
    se2_conv_update(k, xd, None, out, L.SE2_EPI_PROX, log_domain, prox=make_porous_prox(tau, m))
    got = _host(out)
    assert np.all(np.isfinite(got))
    assert k.guard_stats()["prox_noconv"] == 0
    u = (got if log_domain else np.log(got)) + lz          # log s = log b + log z
    cell = O.haar_cell(O.Grid(nx, ny, nt))
    C = tau * m / (eps * (m - 1.0)) * cell ** (1.0 - m)
    ex = C * np.exp((m - 1.0) * u)
    res = ex + u - lz
    # the root's error: residual / g'(u), relative to 1 + |u| (fp32: a few ulps of u)
    assert np.max(np.abs(res) / ((m - 1.0) * ex + 1.0) / (1.0 + np.abs(u))) < 1e-6
    # same values as the oracle's prox (Newton + bisection) where it applies
    s_ref = O.porous_prox(np.exp(lz), eps, tau, m, cell)
    fin = s_ref > 0
    np.testing.assert_allclose(np.exp(u[fin]), s_ref[fin], rtol=5e-4)


@pytest.mark.parametrize("log_domain", [False, True])
def test_barycenter_warm_start_resume(log_domain, cuda_device):
    """App. A split into 12 + 13 iterations with SE2_WARM_START (resume from v_state) equals one
    25-iteration call: bit-identical in the linear domain, to fp32 rounding in logs (the compensated
    running sum restarts)."""
    import se2_synth as S
    from paper_2402_15322_b200 import Kernel, se2_barycenter
    nx, ny, nt, R, eps = 28, 28, 16, 5, 0.02
    k = Kernel(nx, ny, nt, eps, (1.0, 3.0, 1.0), R, max_batch=4)
    mus = np.stack([S.stroke_measure(nx, ny, nt, 3, 1000 + i) for i in range(2)])
    lams = np.array([[0.3, 0.7], [0.5, 0.5]])
    v1 = torch.empty((2, 2, nt, ny, nx), device="cuda")
    w1 = torch.empty_like(v1)
    bary1, _ = se2_barycenter(k, _dev(mus), lams, 25, log_domain, v_state=v1, w_state=w1, no_graph=True)
    v2 = torch.empty_like(v1)
    w2 = torch.empty_like(v1)
    se2_barycenter(k, _dev(mus), lams, 12, log_domain, v_state=v2, w_state=w2, no_graph=True)
    bary2, _ = se2_barycenter(k, _dev(mus), lams, 13, log_domain, v_state=v2, w_state=w2, warm_start=True,
                              no_graph=True)
    if log_domain:
        assert np.max(np.abs(_host(bary1) - _host(bary2))) < 1e-4
        assert np.max(np.abs(_host(v1) - _host(v2))) < 1e-4
    else:
        assert torch.equal(bary1, bary2) and torch.equal(v1, v2) and torch.equal(w1, w2)


def test_nvtx_ranges_do_not_change_results(cuda_device):
    """SE2_NVTX=1 (NVTX ranges per solve / iteration / conv, read once per process) in a fresh process: the same
    small Sinkhorn solve gives bit-identical scalings with and without the ranges."""
    import hashlib
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import hashlib, torch, numpy as np, se2_synth as S\n"
        "from paper_2402_15322_b200 import Kernel, se2_sinkhorn\n"
        "cfg = S.get_config('c0'); d = S.config_inputs(cfg)\n"
        "k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=1)\n"
        "mu, nu = (torch.from_numpy(m).cuda() for m in d['mus'][:2])\n"
        "a, b = torch.empty_like(mu), torch.empty_like(mu)\n"
        "se2_sinkhorn(k, mu, nu, a, b, 12, log_domain=True, trace=True, persistent=False, no_graph=True)\n"
        "torch.cuda.synchronize()\n"
        "print(hashlib.sha256(a.cpu().numpy().tobytes() + b.cpu().numpy().tobytes()).hexdigest())\n")
    outs = []
    for nvtx in ("0", "1"):
        env = dict(os.environ, SE2_NVTX=nvtx, PYTHONPATH=root)
        p = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        outs.append(p.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1] and len(outs[0]) == 64
