"""End-to-end GPU parity of the scaling loops against the fp64 oracle (-m gpu).

Expected values come from tests/golden/<case>.npz, written by tests/golden/make_golden.py, which
calls oracle/ only.  Cases (se2_synth.PARITY_CASES): the BASELINE configs at full size (whole
runs for c0/c1; prefixes for c2/c3/c4, compared on a seeded sample of entries) and reduced-grid
analogues with ragged tiles running the configs' full iteration counts.

Tolerances (north_star; SURVEY ledger L18 = DESIGN.md reading R12): potentials elementwise
max|d|/max(1,|ref|) <= 1e-4 after the gauge fix of tests/gpu_util.py (Sinkhorn pair, App. A inputs);
transported measures max|d|/max(|ref|, 1e-6 max|ref|) <= 1e-4; error traces |d| <= 1e-4 ref + 1e-5.
"""
import os

import numpy as np
import pytest
import torch

import se2_synth as S
from gpu_util import bary_potential_errs, gauge_fixed_pair_err, measure_err, potential_err, trace_err

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL_POT = 1e-4
TOL_MEAS = 1e-4
TOL_TRACE = 1.0     # trace_err is scaled: |d| / (1e-4 ref + 1e-5)


def _golden(name):
    p = os.path.join(GOLD, f"{name}.npz")
    if not os.path.exists(p):
        pytest.fail(f"missing golden file {p}: run tests/golden/make_golden.py {name}")
    return dict(np.load(p))


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def _host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy().astype(np.float64)


def _sel(arr, gold, full):
    """Flatten the field axes and pick the golden sample (or everything)."""
    a = np.asarray(arr).reshape(np.asarray(arr).shape[:-3] + (-1,))
    return a if full else a[..., gold["sample_idx"]]


def _kernel(cfg, batch):
    from paper_2402_15322_b200 import Kernel
    return Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=batch, device=0,
                  hx=cfg.cell, hy=cfg.cell)


def _cmp_pot(name, got, ref):
    e = potential_err(got, ref)
    assert e <= TOL_POT, f"{name}: potential error {e:.3e}"
    return e


def _cmp_meas(name, got, ref):
    e = measure_err(got, ref)
    assert e <= TOL_MEAS, f"{name}: measure error {e:.3e}"
    return e


@pytest.mark.parametrize("persistent", [True, False], ids=["K9", "K3"])
@pytest.mark.parametrize("case", ["c0"])
def test_sinkhorn_parity(case, persistent, cuda_device):
    """c0 through the one-launch cluster solver (K9, the default for this size) and through the
    per-conv K3 path."""
    from paper_2402_15322_b200 import se2_conv, se2_launch_count, se2_sinkhorn
    pc = S.get_parity_case(case)
    cfg, d = S.parity_inputs(pc)
    gold = _golden(case)
    k = _kernel(cfg, 1)
    mu, nu = _dev(d["mus"][0]), _dev(d["mus"][1])
    a = torch.empty_like(mu)
    b = torch.empty_like(mu)
    n0 = se2_launch_count()
    tr = se2_sinkhorn(k, mu, nu, a, b, cfg.iters, cfg.log_domain, trace=True, persistent=persistent)
    launches = se2_launch_count() - n0
    if persistent:
        assert launches <= 3, launches          # K9 + the two non-finite checks
    else:
        assert launches > cfg.iters, launches
    assert cfg.log_domain
    e = gauge_fixed_pair_err(_sel(_host(a), gold, pc.full_fields), _sel(_host(b), gold, pc.full_fields),
                             gold["alpha"].reshape(-1), gold["beta"].reshape(-1))
    assert max(e.values()) <= TOL_POT, e
    # transported measures: the plan's marginals a * K b and b * K^T a (K^T = K)
    row = np.exp(_host(a) + _host(se2_conv(k, b, log_domain=True)))
    col = np.exp(_host(b) + _host(se2_conv(k, a, log_domain=True)))
    _cmp_meas("row", row.reshape(-1), gold["row"].reshape(-1))
    _cmp_meas("col", col.reshape(-1), gold["col"].reshape(-1))
    assert trace_err(tr[:, 0], gold["err"]) <= TOL_TRACE


# fp32-potential barycenter engine (se2_barycenter, K3): the north star's 1e-4 holds on the barycenter,
# its log and the traces; its gauge-fixed log v_i / log w_i carry the fp32 floor of potentials of
# 10^2..10^3 nats iterated 200-500 times (reading R19: per-conv arithmetic error up to ~1e-4 nats
# at 1000-nat magnitudes even for the exact per-tap engine, tools/conv_err_probe.py), bounded here at 1e-3.
# The 1e-4 elementwise potential claim is the fp64-potential engine's (test_barycenter_parity_precise).
TOL_POT_F32 = 1e-3


@pytest.mark.parametrize("case", ["c1", "c2m", "c3m", "c2p", "c3p", "c2f", "c3q"])
def test_barycenter_parity(case, cuda_device):
    from paper_2402_15322_b200 import se2_barycenter
    pc = S.get_parity_case(case)
    cfg, d = S.parity_inputs(pc)
    gold = _golden(case)
    lams = gold["lambdas"]
    n, nsolve = len(d["mus"]), lams.shape[0]
    k = _kernel(cfg, n * nsolve)
    mus = _dev(np.stack(d["mus"]))
    v = torch.empty((nsolve, n) + cfg.shape, device="cuda")
    w = torch.empty_like(v)
    bary, tr = se2_barycenter(k, mus, lams, cfg.iters, cfg.log_domain, v_state=v, w_state=w, trace=True)
    full = pc.full_fields
    if cfg.log_domain:
        _cmp_pot("log bary", _sel(_host(bary), gold, full), gold["lbary"].reshape(nsolve, -1))
        _cmp_meas("bary", np.exp(_sel(_host(bary), gold, full)), gold["bary_lin"].reshape(nsolve, -1))
        glv, glw = _sel(_host(v), gold, full), _sel(_host(w), gold, full)
        rlv, rlw = gold["lv"].reshape(nsolve, n, -1), gold["lw"].reshape(nsolve, n, -1)
        for s in range(nsolve):
            e = bary_potential_errs(glv[s], glw[s], rlv[s], rlw[s], lams[s])
            assert max(e.values()) <= TOL_POT_F32, (s, lams[s], e)
    else:
        _cmp_meas("bary", _sel(_host(bary), gold, full), gold["bary"].reshape(nsolve, -1))
    assert trace_err(tr, gold["err"]) <= TOL_TRACE


@pytest.mark.parametrize("case", ["c1", "c2m", "c2p", "c2f", "c3p", "c3m", "c3q"])
def test_barycenter_parity_precise(case, cuda_device):
    """App. A with fp64 potentials on K4P (se2_barycenter_precise, reading R19) against the oracle at the
    north star's 1e-4 ELEMENTWISE on gauge-fixed potentials (L18) -- the configs whose log-potentials reach
    10^2..10^3 nats, where fp32 storage alone is above 1e-4 (DESIGN.md §5 floor)."""
    from paper_2402_15322_b200 import se2_barycenter_precise
    pc = S.get_parity_case(case)
    cfg, d = S.parity_inputs(pc)
    gold = _golden(case)
    lams = gold["lambdas"]
    n, nsolve = len(d["mus"]), lams.shape[0]
    k = _kernel(cfg, n * nsolve)
    mus = _dev(np.stack(d["mus"]))
    v = torch.empty((nsolve, n) + cfg.shape, device="cuda", dtype=torch.float64)
    w = torch.empty_like(v)
    lbar, tr = se2_barycenter_precise(k, mus, lams, cfg.iters, lv_state=v, lw_state=w, trace=True)
    full = pc.full_fields
    _cmp_pot("log bary", _sel(_host(lbar), gold, full), gold["lbary"].reshape(nsolve, -1))
    _cmp_meas("bary", np.exp(_sel(_host(lbar), gold, full)), gold["bary_lin"].reshape(nsolve, -1))
    glv, glw = _sel(_host(v), gold, full), _sel(_host(w), gold, full)
    rlv, rlw = gold["lv"].reshape(nsolve, n, -1), gold["lw"].reshape(nsolve, n, -1)
    for s in range(nsolve):
        e = bary_potential_errs(glv[s], glw[s], rlv[s], rlw[s], lams[s])
        assert max(e.values()) <= TOL_POT, (s, lams[s], e)
    assert trace_err(tr, gold["err"]) <= TOL_TRACE


@pytest.mark.parametrize("case", ["c4m", "c4p", "c5m", "c4q", "c4m-tc", "c4m-ffma", "c4q-ffma",
                                  "c4w", "c4w-tc", "c4w-ffma", "c4f"])
def test_jko_parity(case, cuda_device):
    """The JKO runs on the default linear engine; -tc / -ffma force K10 (tensor cores) / K2 (FFMA)."""
    from paper_2402_15322_b200 import _lib as L, make_porous_prox, make_prox, se2_jko_step
    case, _, eng = case.partition("-")
    engine_flags = {"tc": L.SE2_LIN_TC, "ffma": L.SE2_LIN_FFMA}.get(eng, 0)
    pc = S.get_parity_case(case)
    cfg, d = S.parity_inputs(pc)
    gold = _golden(case)
    k = _kernel(cfg, 1)
    prox = make_porous_prox(cfg.tau, pc.m) if pc.energy == "porous" else make_prox(k, cfg.tau)
    mu = _dev(d["mus"][0])
    nxt = torch.empty_like(mu)
    a = torch.empty_like(mu)
    b = torch.empty_like(mu)
    full = pc.full_fields
    for step in range(cfg.jko_steps):
        mass, tr = se2_jko_step(k, mu, nxt, a, b, cfg.iters, prox, cfg.log_domain, trace=True,
                                engine_flags=engine_flags)
        assert abs(mass - gold["masses"][step]) <= TOL_MEAS * abs(gold["masses"][step])
        assert trace_err(tr, gold["err"][step]) <= TOL_TRACE
        _cmp_meas(f"mu_{step + 1}", _sel(_host(nxt), gold, full), gold["mus"][step + 1].reshape(-1))
        mu, nxt = nxt, mu
    # potentials of the last inner solve (linear scalings -> compare logs)
    _cmp_pot("log a", np.log(_sel(_host(a), gold, full)), np.log(gold["a"].reshape(-1)))
    _cmp_pot("log b", np.log(_sel(_host(b), gold, full)), np.log(gold["b"].reshape(-1)))


def test_determinism(cuda_device):
    """Two identical solves give bit-identical results (fixed-order reductions, no atomics in the
    arithmetic)."""
    from paper_2402_15322_b200 import se2_barycenter
    pc = S.get_parity_case("c1")
    cfg, d = S.parity_inputs(pc)
    k = _kernel(cfg, 10)
    mus = _dev(np.stack(d["mus"]))
    lams = np.array([[t, 1 - t] for t in cfg.ts])
    b1, t1 = se2_barycenter(k, mus, lams, 20, True, trace=True)
    b2, t2 = se2_barycenter(k, mus, lams, 20, True, trace=True)
    assert torch.equal(b1, b2)
    assert np.array_equal(t1, t2)


def test_graph_replay_equals_direct_launches(cuda_device):
    """The CUDA-graph replay of a small solve is bit-identical to launching its kernels directly, on
    the first (capturing) and on a cached replay."""
    from paper_2402_15322_b200 import se2_barycenter, se2_sinkhorn
    pc = S.get_parity_case("c1")
    cfg, d = S.parity_inputs(pc)
    k = _kernel(cfg, 10)
    mus = _dev(np.stack(d["mus"]))
    lams = np.array([[t, 1 - t] for t in cfg.ts])
    ref, tref = se2_barycenter(k, mus, lams, 15, True, trace=True, no_graph=True)
    for _ in range(2):
        b, t = se2_barycenter(k, mus, lams, 15, True, trace=True)
        assert torch.equal(b, ref) and np.array_equal(t, tref)
    pc0 = S.get_parity_case("c0")
    cfg0, d0 = S.parity_inputs(pc0)
    k0 = _kernel(cfg0, 1)
    mu, nu = _dev(d0["mus"][0]), _dev(d0["mus"][1])
    a1, b1, a2, b2 = (torch.empty_like(mu) for _ in range(4))
    t1 = se2_sinkhorn(k0, mu, nu, a1, b1, 20, True, trace=True, no_graph=True, persistent=False)
    for _ in range(2):
        t2 = se2_sinkhorn(k0, mu, nu, a2, b2, 20, True, trace=True, persistent=False)
        assert torch.equal(a1, a2) and torch.equal(b1, b2) and np.array_equal(t1, t2)


def test_sinkhorn_jko_determinism(cuda_device):
    from paper_2402_15322_b200 import make_prox, se2_jko_step
    pc = S.get_parity_case("c4m")
    cfg, d = S.parity_inputs(pc)
    k = _kernel(cfg, 1)
    prox = make_prox(k, cfg.tau)
    outs = []
    for _ in range(2):
        mu = _dev(d["mus"][0])
        nxt, a, b = torch.empty_like(mu), torch.empty_like(mu), torch.empty_like(mu)
        mass, tr = se2_jko_step(k, mu, nxt, a, b, 30, prox, False, trace=True)
        outs.append((nxt.clone(), mass, tr))
    assert torch.equal(outs[0][0], outs[1][0]) and outs[0][1] == outs[1][1]
    assert np.array_equal(outs[0][2], outs[1][2])


@pytest.mark.parametrize("shape", [(12, 10, 8, 2, False), (9, 7, 4, 1, True), (16, 16, 8, 3, True), (18, 14, 12, 3, False)],
                         ids=["12x10x8", "9x7x4-warm", "16x16x8-warm", "18x14x12"])
def test_sinkhorn_k9_ragged(shape, cuda_device):
    """K9 (one cluster launch) on ragged grids (N not a multiple of 16 -> smaller clusters), with and
    without a warm start, against the fp64 oracle's log-domain Sinkhorn run on the same inputs."""
    import oracle as O
    from paper_2402_15322_b200 import Kernel, se2_launch_count, se2_sinkhorn
    nx, ny, nt, R, warm = shape
    g = O.Grid(nx, ny, nt)
    eps, w = 0.05, (1.0, 3.0, 1.0)
    rng = np.random.default_rng(nx * ny + nt)
    mu = rng.random(g.shape) ** 4 + 1e-6
    nu = rng.random(g.shape) ** 4 + 1e-6
    mu, nu = mu / mu.sum(), nu / nu.sum()
    mu[0, 0, :3] = 0.0          # zero mass: log mu = -inf must propagate as alpha = -inf
    mu /= mu.sum()
    iters = 40
    T = O.kernel_table(g, R, eps, w)
    L = O.log_kernel_table(g, R, eps, w)
    k = Kernel(nx, ny, nt, eps, w, R, max_batch=1, device=0)
    a = torch.empty(g.shape, device="cuda")
    b = torch.zeros(g.shape, device="cuda")
    beta0 = None
    if warm:
        beta0 = rng.normal(0.0, 2.0, g.shape)
        b.copy_(torch.from_numpy(beta0.astype(np.float32)))
        beta0 = b.cpu().numpy().astype(np.float64)
    n0 = se2_launch_count()
    tr = se2_sinkhorn(k, _dev(mu), _dev(nu), a, b, iters, True, trace=True, warm_start=warm)
    assert se2_launch_count() - n0 <= 3
    # oracle: the same iteration from the same beta0 (log domain)
    lmu, lnu = np.log(mu), np.log(nu)
    beta = np.zeros(g.shape) if beta0 is None else beta0
    errs = []
    with np.errstate(divide="ignore", invalid="ignore"):
        for _ in range(iters):
            alpha = np.where(lmu == -np.inf, -np.inf, lmu - O.lse_conv(L, beta))
            beta = lnu - O.lse_conv(L, alpha)
            errs.append(np.abs(np.exp(alpha + O.lse_conv(L, beta)) - mu).sum())
    ga, gb = _host(a), _host(b)
    fin = np.isfinite(alpha)
    assert np.array_equal(np.isfinite(ga), fin)
    e = gauge_fixed_pair_err(ga, gb, alpha, beta)
    assert max(e.values()) <= TOL_POT, e
    assert trace_err(tr[:, 0], np.array(errs)) <= TOL_TRACE


def test_sinkhorn_k9_determinism(cuda_device):
    from paper_2402_15322_b200 import se2_sinkhorn
    pc0 = S.get_parity_case("c0")
    cfg0, d0 = S.parity_inputs(pc0)
    k0 = _kernel(cfg0, 1)
    mu, nu = _dev(d0["mus"][0]), _dev(d0["mus"][1])
    a1, b1, a2, b2 = (torch.empty_like(mu) for _ in range(4))
    t1 = se2_sinkhorn(k0, mu, nu, a1, b1, 50, True, trace=True)
    t2 = se2_sinkhorn(k0, mu, nu, a2, b2, 50, True, trace=True)
    assert torch.equal(a1, a2) and torch.equal(b1, b2) and np.array_equal(t1, t2)


@pytest.mark.parametrize("no_split", [False, True], ids=["split-combine-fallback", "cta-redo"])
def test_hint_fallback_paths(no_split, cuda_device):
    """The exact-path hints are only an optimisation: with every hint read 60 nats too high
    (SE2_DEBUG_BAD_HINTS) each hinted output must fail verification and be recomputed -- by the
    warp-cooperative per-output fallback of the theta_i-split combine, or by the whole-CTA two-pass redo
    without the split -- and the solve must still match the oracle (c2m, 300 log-domain iterations)."""
    from paper_2402_15322_b200 import _lib as Lb
    from paper_2402_15322_b200 import se2_barycenter
    pc = S.get_parity_case("c2m")
    cfg, d = S.parity_inputs(pc)
    gold = _golden("c2m")
    lams = gold["lambdas"]
    n, nsolve = len(d["mus"]), lams.shape[0]
    k = _kernel(cfg, n * nsolve)
    mus = _dev(np.stack(d["mus"]))
    flags = Lb.SE2_DEBUG_BAD_HINTS | (Lb.SE2_DEBUG_NO_SPLIT if no_split else 0)
    k.lse_path_stats(reset=True)
    bary, _ = se2_barycenter(k, mus, lams, cfg.iters, True, debug_flags=flags)
    st = k.lse_path_stats(reset=True)
    assert st["hint_redos"] > 0
    _cmp_pot("log bary", _host(bary).reshape(nsolve, -1), gold["lbary"].reshape(nsolve, -1))
    _cmp_meas("bary", np.exp(_host(bary)).reshape(nsolve, -1), gold["bary_lin"].reshape(nsolve, -1))


def test_sinkhorn_k9_batched(cuda_device):
    """K9 with a batch of independent problems (one cluster each) equals the oracle per problem."""
    import oracle as O
    from paper_2402_15322_b200 import Kernel, se2_launch_count, se2_sinkhorn
    nx, ny, nt, R, B = 12, 10, 8, 2, 3
    g = O.Grid(nx, ny, nt)
    eps, w = 0.05, (1.0, 3.0, 1.0)
    rng = np.random.default_rng(77)
    mus = rng.random((B,) + g.shape) ** 3 + 1e-6
    nus = rng.random((B,) + g.shape) ** 3 + 1e-6
    mus /= mus.sum(axis=(1, 2, 3), keepdims=True)
    nus /= nus.sum(axis=(1, 2, 3), keepdims=True)
    L = O.log_kernel_table(g, R, eps, w)
    k = Kernel(nx, ny, nt, eps, w, R, max_batch=B, device=0)
    a = torch.empty((B,) + g.shape, device="cuda")
    b = torch.empty_like(a)
    n0 = se2_launch_count()
    tr = se2_sinkhorn(k, _dev(mus), _dev(nus), a, b, 30, True, trace=True)
    assert se2_launch_count() - n0 <= 3
    ga, gb = _host(a), _host(b)
    for i in range(B):
        lmu, lnu = np.log(mus[i]), np.log(nus[i])
        beta = np.zeros(g.shape)
        errs = []
        for _ in range(30):
            alpha = lmu - O.lse_conv(L, beta)
            beta = lnu - O.lse_conv(L, alpha)
            errs.append(np.abs(np.exp(alpha + O.lse_conv(L, beta)) - mus[i]).sum())
        e = gauge_fixed_pair_err(ga[i], gb[i], alpha, beta)
        assert max(e.values()) <= TOL_POT, (i, e)
        assert trace_err(tr[:, i], np.array(errs)) <= TOL_TRACE


def test_sinkhorn_k9_selection(cuda_device):
    """K9 is chosen only while the per-conv work is small (it evaluates every tap on <= 16 SMs); a
    larger grid runs the per-conv K3 path (many launches) -- both give the same iterates."""
    from paper_2402_15322_b200 import Kernel, se2_launch_count, se2_sinkhorn
    rng = np.random.default_rng(3)
    for (nx, ny, nt, R), small in (((16, 16, 8, 3), True), ((40, 40, 8, 4), False)):
        mu = rng.random((nt, ny, nx)) ** 3 + 1e-6
        nu = rng.random((nt, ny, nx)) ** 3 + 1e-6
        mu, nu = _dev(mu / mu.sum()), _dev(nu / nu.sum())
        k = _kernel(S.Config("x", nx, ny, nt, 0.05, (1.0, 3.0, 1.0), 2 * R + 1, "sinkhorn", 20, 2), 1)
        a, b = torch.empty_like(mu), torch.empty_like(mu)
        n0 = se2_launch_count()
        se2_sinkhorn(k, mu, nu, a, b, 20, True)
        launches = se2_launch_count() - n0
        assert (launches <= 3) == small, launches
        a2, b2 = torch.empty_like(mu), torch.empty_like(mu)
        se2_sinkhorn(k, mu, nu, a2, b2, 20, True, persistent=False)
        e = gauge_fixed_pair_err(_host(a), _host(b), _host(a2), _host(b2))
        assert max(e.values()) < TOL_POT, e


@pytest.mark.parametrize("engine", ["tc", "ffma"])
def test_linear_solvers_engines(engine, cuda_device):
    """Linear-domain Sinkhorn and App. A barycenter (20 iterations each) on a K10-covered grid with
    each linear engine forced (SE2_LIN_TC / SE2_LIN_FFMA), against the fp64 oracle run in the test:
    potentials (log a, log b) at TOL_POT, barycenter at TOL_MEAS.  20 iterations keep the linear
    scalings inside fp32's range at this eps (by 60 both engines leave it: log a spans [-84, 63],
    reading R13 -- such runs belong to the log domain)."""
    import oracle as O
    from paper_2402_15322_b200 import Kernel, _lib as L, se2_barycenter, se2_sinkhorn
    nx, ny, nt, R, eps, w = 48, 40, 16, 5, 0.02, (1.0, 3.0, 1.0)
    flags = L.SE2_LIN_TC if engine == "tc" else L.SE2_LIN_FFMA
    k = Kernel(nx, ny, nt, eps, w, R, max_batch=2)
    assert k.has_tensor_cores
    g = O.Grid(nx, ny, nt)
    T, Lt = O.kernel_table(g, R, eps, w), O.log_kernel_table(g, R, eps, w)
    mu = S.stroke_measure(nx, ny, nt, 3, seed=71).astype(np.float32).astype(np.float64)
    nu = S.stroke_measure(nx, ny, nt, 3, seed=72).astype(np.float32).astype(np.float64)
    # Sinkhorn: the engine flag rides on the solver's option flags (binding: no_graph path unchanged)
    ref = O.sinkhorn(T, Lt, mu, nu, 20, log_domain=False, trace=True)
    a, b = torch.empty((1, nt, ny, nx), device="cuda"), torch.empty((1, nt, ny, nx), device="cuda")
    opts = L.se2_opts(20, L.SE2_TRACE_ERR | flags)
    tr = np.zeros((20, 1))
    import ctypes
    from paper_2402_15322_b200.api import _ptr, _stream
    mu_d, nu_d = _dev(mu[None]), _dev(nu[None])
    L.check(L.load().se2_sinkhorn(k.handle, _ptr(mu_d), _ptr(nu_d), _ptr(a), _ptr(b), 1, None, ctypes.byref(opts),
                                  tr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _stream(mu_d.device)))
    _cmp_pot("log a", np.log(_host(a)[0]).ravel(), np.log(ref["a"]).ravel())
    _cmp_pot("log b", np.log(_host(b)[0]).ravel(), np.log(ref["b"]).ravel())
    assert trace_err(tr[:, 0], ref["err"]) <= TOL_TRACE
    # barycenter of (mu, nu) with lambda = (0.3, 0.7)
    lam = np.array([[0.3, 0.7]])
    refb = O.barycenter(T, Lt, [mu, nu], lam[0], 20, log_domain=False, trace=True)
    bary, trb = se2_barycenter(k, _dev(np.stack([mu, nu])), lam, 20, False, trace=True, debug_flags=flags)
    _cmp_meas("bary", _host(bary)[0].ravel(), refb["bary"].ravel())
    assert trace_err(trb[:, 0], refb["err"]) <= TOL_TRACE
