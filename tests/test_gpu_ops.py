"""GPU parity of the individual hot-path operators against the fp64 oracle (-m gpu).

Kernel tabulation (A1), linear conv (A2), exact LSE conv (A3), the fused scaling-update epilogues
(A4, A5, A6 pieces) and the marginal-error reduction (A7), on every config grid (full oracle
field where it finishes in seconds, sampled outputs at the full c3/c4 sizes) plus ragged / odd /
degenerate shapes.  All calls go through the C ABI (paper_2402_15322_b200 binding).
"""
import zlib

import numpy as np
import pytest
import torch

from paper_2402_15322_b200 import _lib as L

import oracle as O
import se2_synth as S
from gpu_util import measure_err, potential_err

pytestmark = pytest.mark.gpu

TOL_CONV = 1e-5     # fp32 sums of positive terms vs fp64 (relative, elementwise): K2 (FFMA)
TOL_CONV_TC = 3e-5  # K10 (tensor cores, 3-pass BF16 split): per-term split error <= 3 * 2^-18 plus the
                    # truncating fp32 accumulation of two input rows' chain (2 S K/16 steps <= 124 at R 15,
                    # <= 124 * 2^-23); reading R18 in DESIGN.md
TOL_LSE = 1e-5      # |d ly| / max(1, |ly|), plus the fp32 forward error of a log-sum-exp (lse_abs_tol)
U32 = 2.0 ** -24    # fp32 unit roundoff


def lse_abs_tol(lv, Lt):
    """fp32 forward-error term of ly = m + log sum exp(L + lv - m): the three roundings of L + lv, of the
    shifted exponent and of m + log s each cost up to u |T| absolute, T <= max|lv| + max|L| the largest
    exponent magnitude -- an output near 0 of a 2000-nat field cannot be better than ~1e-4 absolute in
    fp32, whatever the engine."""
    fin = np.isfinite(lv)
    return 3.0 * U32 * (float(np.max(np.abs(lv[fin]))) + float(np.max(np.abs(Lt))))


def _kernel(nx, ny, nt, eps, w, R, batch=1):
    from paper_2402_15322_b200 import Kernel
    return Kernel(nx, ny, nt, eps, w, R, max_batch=batch, device=0)


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def _host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy().astype(np.float64)


CFG_GRIDS = [(c.name, c.nx, c.ny, c.ntheta, c.eps, c.w, c.R) for c in S.CONFIGS]
ODD_GRIDS = [
    ("ragged", 37, 23, 12, 0.02, (1.0, 3.0, 1.0), 5),      # ragged tiles
    ("nt6", 19, 21, 6, 0.03, (1.0, 3.0, 1.0), 4),          # ntheta % 4 != 0: a partial theta quad
    ("nt2", 17, 13, 2, 0.05, (1.0, 2.0, 1.0), 2),          # half-turn only: one partial quad
    ("r15", 40, 36, 8, 0.003, (1.0, 3.0, 1.0), 15),        # the largest supported support (31 x 31)
    ("nt128", 12, 10, 128, 0.05, (1.0, 3.0, 1.0), 1),      # the largest orientation count of K3
    ("nt136", 9, 8, 136, 0.05, (1.0, 3.0, 1.0), 1),        # beyond it: the log domain runs on K4
    ("thin", 5, 70, 8, 0.05, (1.0, 2.0, 1.5), 3),
    ("r0", 33, 33, 8, 0.05, (1.0, 3.0, 1.0), 0),           # theta-only convolution
    ("nt1", 40, 24, 1, 0.01, (1.0, 2.0, 1.0), 6),          # plain anisotropic Gaussian
    ("wide", 9, 9, 4, 0.5, (1.0, 1.0, 1.0), 7),            # support wider than the grid
]


# grids K10 (tensor cores) covers: nt % 16 == 0, nx <= 256, theta band <= 8 when nt > 32
TC_GRIDS = [
    ("tc-ragged", 37, 53, 32, 0.01, (1.0, 3.0, 1.0), 7),    # N = 48 (nx padded), last 8-row group partial
    ("tc-r15", 72, 44, 16, 0.003, (1.0, 3.0, 1.0), 15),     # the largest support, nt 16 (window = all)
    ("tc-nt64", 100, 40, 64, 0.003, (1.0, 3.0, 1.0), 9),    # the 32-orientation window of the band
    ("tc-nt48", 256, 12, 48, 0.003, (1.0, 3.0, 1.0), 3),    # N = 256, wrapped theta window (6 chunks)
    ("tc-r0", 64, 16, 16, 0.01, (1.0, 3.0, 1.0), 0),        # theta-only convolution
    ("tc-thin", 16, 5, 32, 0.02, (1.0, 2.0, 1.5), 2),       # fewer rows than one group
]


@pytest.mark.parametrize("mode", ["auto", "rows", "classic"])
@pytest.mark.parametrize("case", TC_GRIDS, ids=lambda c: c[0])
def test_conv_tc_parity(case, mode, cuda_device, monkeypatch):
    """K10 forced on grids it covers, against the fp64 oracle (full fields), at TOL_CONV_TC.  auto: the
    geometry K10 picks (narrow 16-row x 8-orientation tiles for nt >= 32, balanced mode on these grids:
    pieces of tiles over the SMs); rows: the rows-per-CTA mode (SE2_TC_PIECES=0 at kernel build);
    classic: the 8-row x 16-orientation geometry with the 32-wide window (SE2_TC_NAR=0)."""
    if mode == "rows":
        monkeypatch.setenv("SE2_TC_PIECES", "0")
    if mode == "classic":
        monkeypatch.setenv("SE2_TC_NAR", "0")
    name, nx, ny, nt, eps, w, R = case
    assert _kernel(nx, ny, nt, eps, w, R, 2).has_tensor_cores
    _conv_check(name, nx, ny, nt, eps, w, R, False, batch=2, full=True, extra_flags=L.SE2_LIN_TC)


@pytest.mark.parametrize("case", CFG_GRIDS + ODD_GRIDS, ids=lambda c: c[0])
def test_kernel_stats(case, cuda_device):
    name, nx, ny, nt, eps, w, R = case
    k = _kernel(nx, ny, nt, eps, w, R)
    st = k.stats()
    T = O.kernel_table(O.Grid(nx, ny, nt), R, eps, w)
    T32 = T.astype(np.float32)
    assert st["box_taps"] == nt * (2 * R + 1) ** 2
    assert st["nnz_taps"] == int(np.count_nonzero(T32)) // nt
    band = 0
    for to in range(nt):
        for ti in range(nt):
            if np.any(T32[to, ti] != 0):
                kk = (to - ti) % nt
                if 2 * kk >= nt:
                    kk -= nt
                band = max(band, abs(kk))
    assert st["theta_band"] == band


def _conv_check(name, nx, ny, nt, eps, w, R, log_domain, batch=2, full=True, lse_exact=False, log_span=200.0,
                extra_flags=0):
    k = _kernel(nx, ny, nt, eps, w, R, batch)
    g = O.Grid(nx, ny, nt)
    shape = (batch, nt, ny, nx)
    if log_domain:
        rng = np.random.default_rng(zlib.crc32(name.encode()))
        v = rng.uniform(-log_span / 2, log_span / 2, size=shape).astype(np.float32)
        Lt = O.log_kernel_table(g, R, eps, w)
    else:
        v = S.random_positive_field(shape, seed=zlib.crc32(name.encode()), log_range=30.0)
        Tt = O.kernel_table(g, R, eps, w)
    from paper_2402_15322_b200 import se2_conv
    y = _host(se2_conv(k, _dev(v), log_domain=log_domain, lse_exact=lse_exact, extra_flags=extra_flags))
    if full:
        ref = O.lse_conv(Lt, v.astype(np.float64)) if log_domain else O.conv(Tt, v.astype(np.float64))
        got = y
    else:
        N = nx * ny * nt
        idx = S.sample_indices(N, 400, seed=3)
        ref, got = [], []
        for b in range(batch):
            for f in idx:
                to, rem = divmod(int(f), nx * ny)
                iy, ix = divmod(rem, nx)
                if log_domain:
                    ref.append(O.lse_conv_point(Lt, v[b].astype(np.float64), to, iy, ix))
                else:
                    ref.append(O.conv_point(Tt, v[b].astype(np.float64), to, iy, ix))
                got.append(y[b, to, iy, ix])
        ref, got = np.array(ref), np.array(got)
    if log_domain:
        g_, r_ = np.asarray(got, dtype=np.float64), np.asarray(ref, dtype=np.float64)
        both = (g_ == -np.inf) & (r_ == -np.inf)
        d = np.where(both, 0.0, np.abs(g_ - r_))
        bound = TOL_LSE * np.maximum(1.0, np.abs(np.where(both, 0.0, r_))) + lse_abs_tol(v, Lt)
        e = float(np.max(d / bound))
        assert e <= 1.0, (name, e, potential_err(got, ref))
    else:
        e = float(np.max(np.abs(got - ref) / np.abs(ref)))
        tc = not (extra_flags & L.SE2_LIN_FFMA) and (
            k.uses_tensor_cores or (bool(extra_flags & L.SE2_LIN_TC) and k.has_tensor_cores))
        assert e < (TOL_CONV_TC if tc else TOL_CONV), (name, tc, e)


# the c4 kernel (eps 0.003, w (1,3,1), R 15, nt 64: fp32 band +-5) on a ragged reduced window
NAR_GRID = (60, 45, 64, 0.003, (1.0, 3.0, 1.0), 15)


@pytest.mark.parametrize("field", ["smooth", "range80", "zeros", "negative"])
@pytest.mark.parametrize("mode", ["auto", "rows"])
def test_conv_tc_narrow_window(field, mode, cuda_device, monkeypatch):
    """K10's narrow geometry decides per tile between the 16-orientation window (the |to - ti| = 5 taps of
    the c4 kernel dropped, proven <= 2^-30 of every output from the split kernel's row statistics) and
    the 32-orientation window.  smooth (log range 20 nats): every tile narrow; range80 (e^U(-40, 40) per
    entry): the bound fails, tiles go wide; zeros (a few zero rows): the tiles whose outputs may vanish go
    wide; negative (one negative entry): its window's tiles go wide.  Every case against the fp64 oracle at
    TOL_CONV_TC (relative, elementwise; absolute against the field's scale for the signed input)."""
    if mode == "rows":
        monkeypatch.setenv("SE2_TC_PIECES", "0")
    from paper_2402_15322_b200 import se2_conv
    nx, ny, nt, eps, w, R = NAR_GRID
    batch = 2
    k = _kernel(nx, ny, nt, eps, w, R, batch)
    assert k.has_tensor_cores
    shape = (batch, nt, ny, nx)
    seed = zlib.crc32(field.encode())
    v = S.random_positive_field(shape, seed=seed, log_range=80.0 if field == "range80" else 20.0)
    if field == "zeros":
        v[0, :, 20:23, :] = 0.0
        v[1, 5, 40, :] = 0.0
    if field == "negative":
        v[1, 30, 10, 7] = -0.5
    k.tc_tile_stats(reset=True)
    y = _host(se2_conv(k, _dev(v), extra_flags=L.SE2_LIN_TC))
    st = k.tc_tile_stats(reset=True)
    ref = O.conv(O.kernel_table(O.Grid(nx, ny, nt), R, eps, w), v.astype(np.float64))
    if field == "negative":
        e = float(np.max(np.abs(y - ref) / np.max(np.abs(ref), axis=(2, 3), keepdims=True)))
    else:
        e = float(np.max(np.abs(y - ref) / np.abs(ref)))
    assert e < TOL_CONV_TC, (field, e, st)
    assert st["tiles"] > 0, st
    if field == "smooth":
        assert st["wide"] == 0, st
    elif field == "range80":
        assert st["wide"] > 0, st
    else:
        assert 0 < st["wide"] < st["tiles"], st


def test_conv_tc_balanced_batch3(cuda_device):
    """K10's balanced mode with 3 fields: CTA runs of chain units cross tile and field boundaries, tiles
    split into up to 3 pieces; full fields against the oracle."""
    nx, ny, nt, eps, w, R = 72, 90, 32, 0.01, (1.0, 3.0, 1.0), 7
    assert _kernel(nx, ny, nt, eps, w, R, 3).has_tensor_cores
    _conv_check("tc-batch3", nx, ny, nt, eps, w, R, False, batch=3, full=True, extra_flags=L.SE2_LIN_TC)


@pytest.mark.parametrize("case", CFG_GRIDS + ODD_GRIDS, ids=lambda c: c[0])
@pytest.mark.parametrize("engine", ["linear", "linear-ffma", "linear-tc", "log"])
def test_conv_parity(case, engine, cuda_device):
    """linear: the default engine (K10 on the tensor cores where its cost model picks it, else K2);
    linear-ffma: K2 forced (SE2_LIN_FFMA); linear-tc: K10 forced (SE2_LIN_TC) on every grid it covers
    (nt % 16 == 0, nx <= 256); log: K3."""
    name, nx, ny, nt, eps, w, R = case
    big = nx * ny * nt > 200000
    flags = {"linear-ffma": L.SE2_LIN_FFMA, "linear-tc": L.SE2_LIN_TC}.get(engine, 0)
    _conv_check(name, nx, ny, nt, eps, w, R, engine == "log", batch=1 if big else 2, full=not big, extra_flags=flags)


@pytest.mark.parametrize("case", CFG_GRIDS[:3] + ODD_GRIDS, ids=lambda c: c[0])
@pytest.mark.parametrize("span", [20.0, 2000.0], ids=["ffma-path", "exact-path"])
@pytest.mark.parametrize("lse_exact", [False, True], ids=["K3", "K4"])
def test_lse_engines(case, span, lse_exact, cuda_device):
    """Both log-domain engines against the oracle: a narrow log range keeps every channel on K3's
    FFMA path, a 2000-nat range forces its per-tap fallback; K4 is the all-exact engine."""
    name, nx, ny, nt, eps, w, R = case
    _conv_check(name + f"-{span}", nx, ny, nt, eps, w, R, True, batch=2, full=True, lse_exact=lse_exact,
                log_span=span)


def test_lse_paths_exercised(cuda_device):
    from paper_2402_15322_b200 import se2_conv
    k = _kernel(64, 64, 32, 0.01, (1.0, 4.0, 2.0), 7)
    rng = np.random.default_rng(1)
    k.lse_path_stats(reset=True)
    se2_conv(k, _dev(rng.uniform(-5, 5, (32, 64, 64))), log_domain=True)
    s1 = k.lse_path_stats(reset=True)
    assert s1["active"] > 0 and s1["ffma"] == s1["active"] and s1["active"] < s1["visited"]   # pruned + all FFMA
    se2_conv(k, _dev(rng.uniform(-1000, 1000, (32, 64, 64))), log_domain=True)
    s2 = k.lse_path_stats(reset=True)
    assert s2["ffma"] < s2["active"]                                                            # fallback used


@pytest.mark.parametrize("grid", [(64, 64, 32, 0.01, (1.0, 4.0, 2.0), 7), (37, 45, 12, 0.005, (1.0, 3.0, 1.0), 10)],
                         ids=["c2grid", "ragged"])
def test_lse_tilted_path(grid, cuda_device):
    """Steep but smooth log fields (20-40 nats per pixel plus curvature and noise) overflow the plain
    shifted path's 100-nat window range; K3's gradient-tilted FFMA path must take them, exactly."""
    from paper_2402_15322_b200 import se2_conv
    nx, ny, nt, eps, w, R = grid
    k = _kernel(nx, ny, nt, eps, w, R, 2)
    rng = np.random.default_rng(7)
    X, Y = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
    lv = np.empty((2, nt, ny, nx))
    for b in range(2):
        for t in range(nt):
            gx, gy = rng.uniform(-40, 40, 2)
            lv[b, t] = gx * X + gy * Y + 0.02 * (X - nx / 2) ** 2 + rng.uniform(-3, 3, (ny, nx)) + 50 * t
    lv = lv.astype(np.float32)
    k.lse_path_stats(reset=True)
    y = _host(se2_conv(k, _dev(lv), log_domain=True))
    ps = k.lse_path_stats(reset=True)
    assert ps["tilted"] > 0, ps
    ref = O.lse_conv(O.log_kernel_table(O.Grid(nx, ny, nt), R, eps, w), lv.astype(np.float64))
    assert potential_err(y, ref) < TOL_LSE


def test_conv_zero_and_neginf_inputs(cuda_device):
    from paper_2402_15322_b200 import se2_conv
    k = _kernel(20, 20, 8, 0.05, (1, 3, 1), 3)
    z = torch.zeros(8, 20, 20, device="cuda")
    assert torch.count_nonzero(se2_conv(k, z)).item() == 0
    ninf = torch.full((8, 20, 20), -float("inf"), device="cuda")
    out = se2_conv(k, ninf, log_domain=True)
    assert torch.all(out == -float("inf")).item()
    # a single finite log value reproduces the log kernel column
    lv = ninf.clone()
    lv[2, 10, 10] = 1.5
    out = _host(se2_conv(k, lv, log_domain=True))
    L = O.log_kernel_table(O.Grid(20, 20, 8), 3, 0.05, (1, 3, 1))
    np.testing.assert_allclose(out[:, 7:14, 7:14], L[:, 2] + 1.5, rtol=2e-6, atol=2e-5)
    assert np.all(out[:, :7, :] == -np.inf)


def test_invalid_arguments_raise(cuda_device):
    from paper_2402_15322_b200 import SE2Error, se2_conv
    from paper_2402_15322_b200 import Kernel
    with pytest.raises(SE2Error):
        Kernel(16, 16, 8, -1.0, (1, 1, 1), 3)
    with pytest.raises(SE2Error):
        Kernel(16, 16, 8, 0.1, (1, 1, 1), 16)        # radius > 15 unsupported
    k = _kernel(16, 16, 8, 0.05, (1, 3, 1), 3, batch=1)
    x = torch.ones(2, 8, 16, 16, device="cuda")
    with pytest.raises(SE2Error):
        se2_conv(k, x)                                 # batch 2 > max_batch 1
    with pytest.raises(TypeError):
        se2_conv(k, torch.ones(8, 16, 16))             # host tensor: no CPU fallback


@pytest.mark.parametrize("log_domain", [False, True], ids=["linear", "log"])
def test_fused_epilogues(log_domain, cuda_device):
    from paper_2402_15322_b200 import _lib as L, make_prox, se2_conv_update
    nx, ny, nt, eps, w, R = 40, 36, 16, 0.02, (1.0, 3.0, 1.0), 5
    k = _kernel(nx, ny, nt, eps, w, R, 2)
    g = O.Grid(nx, ny, nt)
    shape = (2, nt, ny, nx)
    v = S.random_positive_field(shape, seed=21, log_range=20.0).astype(np.float64)
    tgt = S.random_positive_field(shape, seed=22, lo=1e-6, hi=1e-3).astype(np.float64)
    Kv = O.conv(O.kernel_table(g, R, eps, w), v)
    if log_domain:
        xin, tin = np.log(v), np.log(tgt)
    else:
        xin, tin = v, tgt
    xin32, tin32 = xin.astype(np.float32), tin.astype(np.float32)
    # reference computed from the fp32-rounded inputs the GPU sees
    if log_domain:
        Kv = np.exp(O.lse_conv(O.log_kernel_table(g, R, eps, w), xin32.astype(np.float64)))
    else:
        Kv = O.conv(O.kernel_table(g, R, eps, w), xin32.astype(np.float64))
    t64 = tin32.astype(np.float64)
    tol_lin = TOL_CONV_TC if k.uses_tensor_cores else TOL_CONV
    out = torch.empty(shape, device="cuda")
    se2_conv_update(k, _dev(xin32), _dev(tin32), out, L.SE2_EPI_DIVIDE, log_domain)
    got = _host(out)
    if log_domain:
        assert potential_err(got, t64 - np.log(Kv)) < TOL_LSE
    else:
        assert measure_err(got, t64 / Kv) < tol_lin
    se2_conv_update(k, _dev(xin32), _dev(tin32), out, L.SE2_EPI_MULTIPLY, log_domain)
    got = _host(out)
    if log_domain:
        assert potential_err(got, t64 + np.log(Kv)) < TOL_LSE
    else:
        assert measure_err(got, t64 * Kv) < tol_lin
    # JKO prox: b = z^{-tau/(eps+tau)} exp(-tau V/(eps+tau)), V = |x - c|^2 (R10)
    tau = 1e-3
    prox = make_prox(k, tau)
    se2_conv_update(k, _dev(xin32), None, out, L.SE2_EPI_PROX, log_domain, prox=prox)
    got = _host(out)
    V = O.jko_potential(g)
    p = tau / (eps + tau)
    ref_log = -p * np.log(Kv) - p * V
    if log_domain:
        assert potential_err(got, ref_log) < TOL_LSE
    else:
        assert potential_err(np.log(got), ref_log) < TOL_LSE


@pytest.mark.parametrize("log_domain", [False, True], ids=["linear", "log"])
def test_marginal_error(log_domain, cuda_device):
    from paper_2402_15322_b200 import se2_marginal_error
    nx, ny, nt, eps, w, R = 28, 28, 16, 0.02, (1.0, 3.0, 1.0), 5
    k = _kernel(nx, ny, nt, eps, w, R, 2)
    g = O.Grid(nx, ny, nt)
    shape = (2, nt, ny, nx)
    a = S.random_positive_field(shape, seed=31, lo=0.5, hi=2.0)
    b = S.random_positive_field(shape, seed=32, lo=0.5, hi=2.0)
    mu = S.random_positive_field(shape, seed=33, lo=0.0, hi=1.0)
    if log_domain:
        a_in, b_in = np.log(a), np.log(b)
    else:
        a_in, b_in = a, b
    got = se2_marginal_error(k, _dev(a_in), _dev(b_in), _dev(mu), log_domain)
    Kb = O.conv(O.kernel_table(g, R, eps, w), b.astype(np.float64))
    ref = [O.marginal_error(a[i].astype(np.float64), Kb[i], mu[i].astype(np.float64)) for i in range(2)]
    np.testing.assert_allclose(got, ref, rtol=1e-5)


def test_bary_pieces(cuda_device):
    from paper_2402_15322_b200 import se2_bary_logmean, se2_bary_update
    N = 1000
    rng = np.random.default_rng(5)
    ld = rng.normal(size=(3, N)).astype(np.float32)
    lam = np.array([0.2, 0.0, 0.8])
    lbar = torch.empty(N, device="cuda")
    se2_bary_logmean(_dev(ld), lam, N, lbar)
    ref = lam[0] * ld[0].astype(np.float64) + lam[2] * ld[2]
    np.testing.assert_allclose(_host(lbar), ref, rtol=1e-6, atol=1e-6)
    lv = rng.normal(size=(3, N)).astype(np.float32)
    lv_t = _dev(lv)
    se2_bary_update(lv_t, _dev(ld), lbar, 3, N)
    np.testing.assert_allclose(_host(lv_t), lv + (ref[None] - ld), rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("log_domain", [False, True, "tc", "ffma"], ids=["linear", "log", "linear-tc", "linear-ffma"])
@pytest.mark.parametrize("grid", [(28, 28, 16, 0.02, (1.0, 3.0, 1.0), 5), (37, 23, 12, 0.02, (1.0, 3.0, 1.0), 5)],
                         ids=["c1grid", "ragged"])
def test_transport_cost(grid, log_domain, cuda_device):
    """linear-tc / linear-ffma force K10 (tensor cores, cost-table weights) / K2 on the linear path."""
    from paper_2402_15322_b200 import se2_transport_cost
    nx, ny, nt, eps, w, R = grid
    engine = log_domain if isinstance(log_domain, str) else None
    flags = {"tc": L.SE2_LIN_TC, "ffma": L.SE2_LIN_FFMA}.get(engine, 0)
    log_domain = log_domain is True
    k = _kernel(nx, ny, nt, eps, w, R, 2)
    if engine == "tc" and not k.has_tensor_cores:
        pytest.skip("grid not covered by K10 (ntheta % 16 != 0)")
    g = O.Grid(nx, ny, nt)
    shape = (2, nt, ny, nx)
    a = S.random_positive_field(shape, seed=41, log_range=10.0)
    b = S.random_positive_field(shape, seed=42, log_range=10.0)
    ain, bin_ = (np.log(a), np.log(b)) if log_domain else (a, b)
    got = se2_transport_cost(k, _dev(ain), _dev(bin_), log_domain, engine_flags=flags)
    Tc = O.cost_table(g, R, eps, w)
    ref = [O.transport_cost(Tc, a[i].astype(np.float64), b[i].astype(np.float64)) for i in range(2)]
    np.testing.assert_allclose(got, ref, rtol=2e-5)


@pytest.mark.parametrize("case", CFG_GRIDS[:4] + [g for g in ODD_GRIDS if g[0] in ("ragged", "nt6", "r15", "r0", "wide")],
                         ids=lambda c: c[0])
@pytest.mark.parametrize("span", [20.0, 2000.0, 30000.0])
def test_conv_precise(case, span, cuda_device):
    """K4P (fp64 potentials, exact exponents): elementwise ABSOLUTE error <= 2e-6 nats against the fp64 oracle
    on the same fp64 input -- even for 2000-nat fields, where every fp32 engine is limited to ~1e-4
    (lse_abs_tol).  -inf entries (zero mass) included.  span 20: the factored FFMA path; 2000: the exact path
    with grid-aligned exponents; 30000 (windows beyond 2^14 log2 units): its TwoSum form."""
    from paper_2402_15322_b200 import se2_conv_precise
    name, nx, ny, nt, eps, w, R = case
    k = _kernel(nx, ny, nt, eps, w, R, 2)
    rng = np.random.default_rng(zlib.crc32((name + str(span)).encode()))
    v = rng.uniform(-span / 2, span / 2, size=(2, nt, ny, nx))
    v[0, 0, 0, :3] = -np.inf
    y = _host(se2_conv_precise(k, torch.from_numpy(v).cuda()))
    ref = O.lse_conv(O.log_kernel_table(O.Grid(nx, ny, nt), R, eps, w), v)
    fin = np.isfinite(ref)
    assert np.array_equal(np.isfinite(y), fin)
    d = np.abs(y[fin] - ref[fin])
    assert d.max() <= 2e-6 * np.maximum(1.0, np.abs(ref[fin]) / 1000.0).max(), (name, d.max())


@pytest.mark.parametrize("mode", ["groups1", "groups3", "groups8", "exact-only"])
@pytest.mark.parametrize("span", [20.0, 400.0])
def test_conv_precise_modes(mode, span, cuda_device, monkeypatch):
    """K4P's theta_i split (SE2_K4P_GROUPS: partial (shift, fp64 sum) per output, exact combine) and the
    per-tap path alone (SE2_K4P_EXACT: no factored channels) against the fp64 oracle on c1's grid with a
    batch of 3 fields: the same 2e-6-nat bound whichever way the channels are dealt."""
    from paper_2402_15322_b200 import se2_conv_precise
    if mode == "exact-only":
        monkeypatch.setenv("SE2_K4P_EXACT", "1")
    else:
        monkeypatch.setenv("SE2_K4P_GROUPS", mode[len("groups"):])
    nx, ny, nt, eps, w, R = 28, 28, 16, 0.02, (1.0, 3.0, 1.0), 5
    k = _kernel(nx, ny, nt, eps, w, R, 3)
    rng = np.random.default_rng(zlib.crc32((mode + str(span)).encode()))
    # a smooth potential (planes per orientation) plus noise: window ranges below and above the 80-nat
    # factored-path limit depending on span
    yy, xx = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    v = np.stack([np.stack([span * (0.01 * (xx * np.cos(t) + yy * np.sin(t))) + rng.uniform(-span / 20, span / 20,
                                                                                         (ny, nx))
                            for t in np.linspace(0, 2 * np.pi, nt, endpoint=False)]) for _ in range(3)])
    y = _host(se2_conv_precise(k, torch.from_numpy(v).cuda()))
    ref = O.lse_conv(O.log_kernel_table(O.Grid(nx, ny, nt), R, eps, w), v)
    d = np.abs(y - ref)
    assert d.max() <= 2e-6 * max(1.0, np.abs(ref).max() / 1000.0), (mode, span, d.max())
