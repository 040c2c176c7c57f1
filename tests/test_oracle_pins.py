"""Pins of the fp64 oracle against what the paper and the mathematics fix (no GPU).

Each test names the oracle part it pins and the passage / closed form it uses.  A plausible
mistake in the oracle (dropped term, wrong sign or index, transposed operand) fails at least one:
  group law / inverse / half-angle / rho_b  -> worked values + homogeneous matrices + symmetry
  kernel table orientation (to vs ti, sign of dx) -> pairwise dense matrix from the group law
  conv gather/scatter                        -> dense matrix, adjoint identity, Dirac, separable case
  Sinkhorn                                   -> textbook dense Sinkhorn, exact column marginal, closed forms
  barycenter                                 -> closed forms (lambda=(1,0), identical inputs), invariant
                                                sum_i lambda_i log v_i = 0, fixed-point marginals
  JKO                                        -> tau = 0 closed form, prox stationarity, mass
"""
import json
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "group_law.json")


def _gold():
    with open(GOLD) as f:
        return json.load(f)


def _hom(g):
    x, y, t = g
    return np.array([[np.cos(t), -np.sin(t), x], [np.sin(t), np.cos(t), y], [0, 0, 1.0]])


# ---------------------------------------------------------------- group law ----------
def test_group_law_worked_values():
    G = _gold()
    for c in G["products"]:
        np.testing.assert_allclose(O.se2_mul(c["g1"], c["g2"]), c["expect"], atol=1e-12)
    for c in G["inverses"]:
        np.testing.assert_allclose(O.se2_inv(c["g"]), c["expect"], atol=1e-12)
    for c in G["relative"]:
        np.testing.assert_allclose(O.se2_mul(O.se2_inv(c["g1"]), c["g2"]), c["expect"], atol=1e-12)
    for c in G["half_angle"]:
        np.testing.assert_allclose(O.half_angle(c["g"]), c["expect"], atol=1e-12)
    for c in G["rho_b"]:
        assert abs(O.rho_b(c["g"], c["w"]) - c["expect"]) < 1e-12


def test_group_axioms_and_matrix_representation():
    rng = np.random.default_rng(1)
    g = np.stack([rng.uniform(-2, 2, 1000), rng.uniform(-2, 2, 1000), rng.uniform(-np.pi, np.pi, 1000)], -1)
    h = np.roll(g, 1, axis=0)
    k = np.roll(g, 7, axis=0)
    lhs = O.se2_mul(O.se2_mul(g, h), k)
    rhs = O.se2_mul(g, O.se2_mul(h, k))
    d = lhs - rhs
    d[:, 2] = O.wrap_angle(d[:, 2])
    assert np.abs(d).max() < 1e-12
    e = np.zeros(3)
    np.testing.assert_allclose(O.se2_mul(g, e), g, atol=1e-12)
    gi = O.se2_mul(g, O.se2_inv(g))
    gi[:, 2] = O.wrap_angle(gi[:, 2])
    assert np.abs(gi).max() < 1e-12
    for i in range(50):
        M = _hom(g[i]) @ _hom(h[i])
        p = O.se2_mul(g[i], h[i])
        np.testing.assert_allclose(_hom(p), M, atol=1e-12)


# ---------------------------------------------------------------- rho_b --------------
def test_rho_b_special_cases_and_symmetry():
    w = (1.3, 3.7, 0.9)
    for th in np.linspace(-np.pi, np.pi - 1e-9, 17):
        assert abs(O.rho_b([0, 0, th], w) - w[2] * abs(th)) < 1e-12
    for x in (-0.7, 0.2, 1.5):
        assert abs(O.rho_b([x, 0, 0], w) - w[0] * abs(x)) < 1e-12
        assert abs(O.rho_b([0, x, 0], w) - w[1] * abs(x)) < 1e-12
    assert O.rho_b([0, 0, 0], w) == 0.0
    rng = np.random.default_rng(2)
    g = np.stack([rng.uniform(-1, 1, 500), rng.uniform(-1, 1, 500), rng.uniform(-3.1, 3.1, 500)], -1)
    np.testing.assert_allclose(O.rho_b(g, w), O.rho_b(O.se2_inv(g), w), atol=1e-12)
    # half-angle coordinates are odd under inversion: b(g^{-1}) = -b(g)
    np.testing.assert_allclose(O.half_angle(O.se2_inv(g)), -O.half_angle(g), atol=1e-12)
    # mid-angle identity: (b1, b2) = R_{-theta/2} (x, y)
    b = O.half_angle(g)
    c, s = np.cos(g[:, 2] / 2), np.sin(g[:, 2] / 2)
    np.testing.assert_allclose(b[:, 0], c * g[:, 0] + s * g[:, 1], atol=1e-12)


def test_zeta():
    assert O.spatial_anisotropy((1, 3, 1)) == 3.0
    assert O.spatial_anisotropy((4, 1, 2)) == 4.0


# ---------------------------------------------------------------- kernel table ------------------
def test_kernel_table_values_and_symmetry():
    g = O.Grid(8, 8, 8)
    eps, R = 0.05, 3
    T = O.kernel_table(g, R, eps, (1, 1, 1))
    assert T[0, 0, R, R] == 1.0                                    # K(e) = 1
    for dx in range(-R, R + 1):                                    # K(dx,0,0; 1,1,1) = exp(-dx^2/eps)
        assert abs(T[0, 0, R, R + dx] - np.exp(-(dx / 8.0) ** 2 / eps)) < 1e-15
    T = O.kernel_table(g, R, eps, (1, 3, 1))
    # inversion symmetry W[to,ti](d) = W[ti,to](-d)  (K = K^T)
    np.testing.assert_allclose(T, np.flip(np.transpose(T, (1, 0, 2, 3)), axis=(2, 3)), rtol=1e-12, atol=0)
    # quarter-turn covariance W[to+nt/4, ti+nt/4](R_{pi/2} d) = W[to,ti](d)
    Tr = np.roll(T, (2, 2), axis=(0, 1))           # index (to+2, ti+2)
    # R_{pi/2}(dx, dy) = (-dy, dx):  Tr[to, ti, dy', dx'] with dx' = -dy, dy' = dx
    rot = np.transpose(T, (0, 1, 3, 2))[:, :, :, ::-1]   # rot[.., dy', dx'] = T[.., dy=-dx', dx=dy']
    np.testing.assert_allclose(Tr, rot, rtol=1e-12, atol=1e-300)
    L = O.log_kernel_table(g, R, eps, (1, 3, 1))
    np.testing.assert_allclose(np.exp(L), T, rtol=1e-13)


# ---------------------------------------------------------------- convolution -------------------
@pytest.mark.parametrize("w", [(1, 3, 1), (1, 1, 1), (2, 0.5, 3)])
def test_conv_equals_dense_group_law_matrix(w):
    """Brute force: K[g,h] = exp(-rho_b(h^{-1} g)^2 / eps) pair by pair from the group law (no table)."""
    g = O.Grid(8, 6, 8)
    eps, R = 0.07, 2
    T = O.kernel_table(g, R, eps, w)
    K = O.dense_kernel_matrix(g, R, eps, w)
    rng = np.random.default_rng(3)
    v = rng.random((2,) + g.shape)
    y = O.conv(T, v)
    yd = np.stack([(K @ vv.reshape(-1)).reshape(g.shape) for vv in v])
    np.testing.assert_allclose(y, yd, rtol=1e-13)
    ya = O.conv_adjoint(T, v)
    yda = np.stack([(K.T @ vv.reshape(-1)).reshape(g.shape) for vv in v])
    np.testing.assert_allclose(ya, yda, rtol=1e-13)
    np.testing.assert_allclose(O.conv_numpy(T, v), yd, rtol=1e-13)
    # K = K^T: gather equals scatter
    np.testing.assert_allclose(y, ya, rtol=1e-12)
    # <K a, b> = <a, K^T b>
    a, b = v[0], v[1]
    assert abs(np.sum(O.conv(T, a) * b) - np.sum(a * O.conv_adjoint(T, b))) < 1e-12 * abs(np.sum(O.conv(T, a) * b))


def test_conv_dirac_linearity_point():
    g = O.Grid(9, 9, 4)
    R = 2
    T = O.kernel_table(g, R, 0.1, (1, 2, 1))
    v = np.zeros(g.shape)
    v[1, 4, 4] = 1.0
    y = O.conv(T, v)
    # Dirac at h = (4,4,theta_1) reproduces the kernel column y(g) = K(h^{-1} g)
    for to in range(4):
        np.testing.assert_allclose(y[to, 2:7, 2:7], T[to, 1], rtol=1e-14)
    assert np.count_nonzero(y) == 4 * 25
    rng = np.random.default_rng(4)
    u, w_ = rng.random(g.shape), rng.random(g.shape)
    np.testing.assert_allclose(O.conv(T, 2 * u - 3 * w_), 2 * O.conv(T, u) - 3 * O.conv(T, w_), rtol=1e-12, atol=1e-14)
    yy = O.conv(T, u)
    for (to, iy, ix) in [(0, 0, 0), (3, 8, 8), (2, 4, 1)]:
        assert abs(O.conv_point(T, u, to, iy, ix) - yy[to, iy, ix]) < 1e-14


def test_conv_ntheta1_is_separable_gaussian():
    """N_theta = 1: K(x) = exp(-(w1^2 dx^2 + w2^2 dy^2)/eps), the textbook separable Gaussian of
    convolutional Wasserstein distances: two 1-D passes."""
    g = O.Grid(12, 10, 1)
    R, eps, w = 3, 0.02, (1.0, 2.0, 1.0)
    T = O.kernel_table(g, R, eps, w)
    rng = np.random.default_rng(5)
    v = rng.random(g.shape)
    d = np.arange(-R, R + 1)
    kx = np.exp(-(w[0] * d / 12.0) ** 2 / eps)
    ky = np.exp(-(w[1] * d / 10.0) ** 2 / eps)
    t = np.zeros_like(v)
    for j, dx in enumerate(d):   # x pass with zero padding
        src = np.zeros_like(v)
        if dx >= 0:
            src[..., dx:] = v[..., :12 - dx]
        else:
            src[..., :12 + dx] = v[..., -dx:]
        t += kx[j] * src
    y = np.zeros_like(v)
    for j, dy in enumerate(d):
        src = np.zeros_like(v)
        if dy >= 0:
            src[..., dy:, :] = t[..., :10 - dy, :]
        else:
            src[..., :10 + dy, :] = t[..., -dy:, :]
        y += ky[j] * src
    np.testing.assert_allclose(O.conv(T, v), y, rtol=1e-13)


def test_conv_quarter_turn_equivariance():
    """Left-invariance of the kernel (Lemma 3.1): K commutes with the lattice
    permutation of a rotation by pi/2 about the window centre."""
    g = O.Grid(10, 10, 8)
    T = O.kernel_table(g, 3, 0.03, (1, 3, 1))
    rng = np.random.default_rng(6)
    v = rng.random(g.shape)
    np.testing.assert_allclose(O.conv(T, O.quarter_turn(v)), O.quarter_turn(O.conv(T, v)), rtol=1e-12)
    v4 = O.quarter_turn(O.quarter_turn(O.quarter_turn(O.quarter_turn(v))))
    assert np.array_equal(v4, v)


def test_lse_conv_matches_linear_and_shift():
    g = O.Grid(8, 8, 8)
    T = O.kernel_table(g, 3, 0.05, (1, 3, 1))
    L = O.log_kernel_table(g, 3, 0.05, (1, 3, 1))
    rng = np.random.default_rng(7)
    v = rng.uniform(0.1, 2.0, g.shape)
    np.testing.assert_allclose(O.lse_conv(L, np.log(v)), np.log(O.conv(T, v)), rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(O.lse_conv_adjoint(L, np.log(v)), np.log(O.conv_adjoint(T, v)), rtol=1e-13, atol=1e-13)
    lv = np.log(v)
    np.testing.assert_allclose(O.lse_conv(L, lv + 123.4), O.lse_conv(L, lv) + 123.4, rtol=1e-13)
    # huge dynamic range where the linear form would overflow: the shift still holds exactly
    lw = rng.uniform(-800, 800, g.shape)
    a = O.lse_conv(L, lw)
    assert np.all(np.isfinite(a))
    np.testing.assert_allclose(O.lse_conv(L, lw - 500.0), a - 500.0, rtol=1e-13)
    # all -inf input -> -inf
    assert np.all(O.lse_conv(L, np.full(g.shape, -np.inf)) == -np.inf)
    y = O.lse_conv(L, lw)
    assert abs(O.lse_conv_point(L, lw, 5, 2, 7) - y[5, 2, 7]) < 1e-12


# ---------------------------------------------------------------- Sinkhorn ----------
def _dense_sinkhorn(K, mu, nu, iters):
    b = np.ones_like(nu)
    for _ in range(iters):
        a = mu / (K @ b)
        b = nu / (K.T @ a)
    return a, b


def test_sinkhorn_matches_textbook_dense():
    g = O.Grid(6, 6, 4)
    R, eps, w = 2, 0.05, (1, 2, 1)
    T = O.kernel_table(g, R, eps, w)
    L = O.log_kernel_table(g, R, eps, w)
    K = O.dense_kernel_matrix(g, R, eps, w)
    rng = np.random.default_rng(8)
    mu = rng.random(g.shape) + 0.05
    mu /= mu.sum()
    nu = rng.random(g.shape) + 0.05
    nu /= nu.sum()
    a, b = _dense_sinkhorn(K, mu.reshape(-1), nu.reshape(-1), 30)
    r = O.sinkhorn(T, L, mu, nu, 30, log_domain=False)
    np.testing.assert_allclose(r["a"].reshape(-1), a, rtol=1e-11)
    np.testing.assert_allclose(r["b"].reshape(-1), b, rtol=1e-11)
    rl = O.sinkhorn(T, L, mu, nu, 30, log_domain=True)
    np.testing.assert_allclose(rl["alpha"], np.log(r["a"]), rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(rl["beta"], np.log(r["b"]), rtol=1e-11, atol=1e-11)
    # after every b-update the second marginal is exact
    np.testing.assert_allclose(r["col"], nu, rtol=1e-12)
    np.testing.assert_allclose(rl["col"], nu, rtol=1e-11)
    # error trace is the L1 row-marginal violation and matches between domains
    np.testing.assert_allclose(r["err"], rl["err"], rtol=1e-8, atol=1e-15)
    assert abs(r["err"][-1] - np.abs(r["row"] - mu).sum()) < 1e-15
    # convergence: marginal error decreases to ~0 on this well-conditioned instance
    T2 = O.kernel_table(g, R, 1.0, w)
    r2 = O.sinkhorn(T2, None, mu, nu, 200, log_domain=False)
    assert r2["err"][-1] < 1e-9 and r2["err"][-1] < r2["err"][0]


def test_sinkhorn_circulant_fixed_point():
    """1x1xNt grid, mu = nu uniform: K is circulant with row sum s, so after one iteration
    a = 1/(Nt s) and b = 1 (b = nu / K^T a = (1/Nt) / (s/(Nt s)) = 1) -- a fixed point."""
    g = O.Grid(1, 1, 8)
    T = O.kernel_table(g, 0, 0.5, (1, 1, 1))
    L = O.log_kernel_table(g, 0, 0.5, (1, 1, 1))
    s = T[0, :, 0, 0].sum()
    mu = np.full(g.shape, 1 / 8)
    for log in (False, True):
        r = O.sinkhorn(T, L, mu, mu, 3, log_domain=log)
        a = np.exp(r["alpha"]) if log else r["a"]
        b = np.exp(r["beta"]) if log else r["b"]
        np.testing.assert_allclose(a, 1 / (8 * s), rtol=1e-13)
        np.testing.assert_allclose(b, 1.0, rtol=1e-13)
        assert r["err"][-1] < 1e-15


def test_sinkhorn_two_diracs():
    """Two Diracs within the support: the only coupling is delta x delta; marginal error 0."""
    g = O.Grid(6, 6, 4)
    T = O.kernel_table(g, 2, 0.05, (1, 2, 1))
    L = O.log_kernel_table(g, 2, 0.05, (1, 2, 1))
    mu = np.zeros(g.shape)
    mu[0, 2, 2] = 1
    nu = np.zeros(g.shape)
    nu[1, 3, 4] = 1
    r = O.sinkhorn(T, L, mu, nu, 2, log_domain=True)
    assert r["err"][-1] < 1e-14
    np.testing.assert_allclose(r["row"], mu, atol=1e-15)
    np.testing.assert_allclose(r["col"], nu, atol=1e-15)


def test_sinkhorn_quarter_turn_equivariance():
    """Corollary 4.1: pushing both marginals forward permutes the scalings."""
    g = O.Grid(8, 8, 8)
    T = O.kernel_table(g, 2, 0.05, (1, 3, 1))
    L = O.log_kernel_table(g, 2, 0.05, (1, 3, 1))
    rng = np.random.default_rng(9)
    mu = rng.random(g.shape) + 0.1
    mu /= mu.sum()
    nu = rng.random(g.shape) + 0.1
    nu /= nu.sum()
    r = O.sinkhorn(T, L, mu, nu, 15, log_domain=True)
    rq = O.sinkhorn(T, L, O.quarter_turn(mu), O.quarter_turn(nu), 15, log_domain=True)
    np.testing.assert_allclose(rq["alpha"], O.quarter_turn(r["alpha"]), rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(rq["err"], r["err"], rtol=1e-9)


# ---------------------------------------------------------------- barycenter (App. A) -----------
def _small_bary_setup(seed=10, eps=0.05):
    g = O.Grid(8, 8, 8)
    T = O.kernel_table(g, 2, eps, (1, 3, 1))
    L = O.log_kernel_table(g, 2, eps, (1, 3, 1))
    rng = np.random.default_rng(seed)
    mus = []
    for _ in range(3):
        m = rng.random(g.shape) ** 4 + 1e-3
        mus.append(m / m.sum())
    return g, T, L, mus


def test_barycenter_lambda_one_closed_form():
    """lambda = (1, 0): v_1 stays 1 and mu = K(mu_1 / K 1) at every iteration (App. A)."""
    g, T, L, mus = _small_bary_setup()
    expect = O.conv(T, mus[0] / O.conv(T, np.ones(g.shape)))
    for log in (False, True):
        for iters in (1, 5):
            r = O.barycenter(T, L, mus[:2], [1.0, 0.0], iters, log_domain=log)
            np.testing.assert_allclose(r["bary"], expect, rtol=1e-11)
    # n = 1 is the same closed form; identical inputs under any lambda as well
    r = O.barycenter(T, L, mus[:1], [1.0], 4, log_domain=False)
    np.testing.assert_allclose(r["bary"], expect, rtol=1e-12)
    r = O.barycenter(T, L, [mus[0], mus[0]], [0.3, 0.7], 4, log_domain=True)
    np.testing.assert_allclose(r["bary"], expect, rtol=1e-11)


def test_barycenter_invariants_and_fixed_point():
    """sum_i lambda_i log v_i = 0 holds at every iteration (it is invariant under the v-update since
    log mu = sum_i lambda_i log d_i); at convergence w_i K v_i = mu_i and d_i = mu for all i."""
    g, T, L, mus = _small_bary_setup()
    lam = np.array([0.2, 0.5, 0.3])
    for iters in (1, 3):
        r = O.barycenter(T, L, mus, lam, iters, log_domain=True)
        assert np.abs(np.tensordot(lam, r["lv"], axes=1)).max() < 1e-11
    g, T, L, mus = _small_bary_setup(eps=0.3)
    r = O.barycenter(T, L, mus, lam, 400, log_domain=True)
    for i in range(3):
        row = np.exp(r["lw"][i] + O.lse_conv(L, r["lv"][i]))
        np.testing.assert_allclose(row, mus[i], rtol=1e-6)
        d = np.exp(r["lv"][i] + O.lse_conv(L, r["lw"][i]))
        np.testing.assert_allclose(d, r["bary"], rtol=1e-6)
    assert r["err"][-1] < 1e-6 * 3
    assert abs(r["bary"].sum() - 1.0) < 1e-6
    rl = O.barycenter(T, L, mus, lam, 20, log_domain=False)
    rg = O.barycenter(T, L, mus, lam, 20, log_domain=True)
    np.testing.assert_allclose(rl["bary"], rg["bary"], rtol=1e-10)
    np.testing.assert_allclose(rl["err"], rg["err"], rtol=1e-7)


def test_barycenter_quarter_turn_equivariance():
    g, T, L, mus = _small_bary_setup()
    lam = [0.25, 0.75]
    r = O.barycenter(T, L, mus[:2], lam, 10, log_domain=True)
    rq = O.barycenter(T, L, [O.quarter_turn(m) for m in mus[:2]], lam, 10, log_domain=True)
    np.testing.assert_allclose(rq["bary"], O.quarter_turn(r["bary"]), rtol=1e-10)


# ---------------------------------------------------------------- JKO ---------------
def test_jko_tau_zero_is_entropic_blur():
    g = O.Grid(8, 8, 8)
    T = O.kernel_table(g, 2, 0.05, (1, 3, 1))
    L = O.log_kernel_table(g, 2, 0.05, (1, 3, 1))
    rng = np.random.default_rng(11)
    mu = rng.random(g.shape) + 0.01
    mu /= mu.sum()
    blur = O.conv(T, mu / O.conv(T, np.ones(g.shape)))
    for log in (False, True):
        r = O.jko(T, L, mu, g, eps=0.05, tau=0.0, steps=1, iters=3, log_domain=log)
        np.testing.assert_allclose(r["mus"][1], blur / blur.sum(), rtol=1e-12)
        np.testing.assert_allclose(r["masses"][0], blur.sum(), rtol=1e-12)


def test_jko_prox_stationarity_mass_equivariance():
    g = O.Grid(8, 8, 8)
    eps, tau = 0.05, 0.02
    T = O.kernel_table(g, 2, eps, (1, 3, 1))
    L = O.log_kernel_table(g, 2, eps, (1, 3, 1))
    rng = np.random.default_rng(12)
    mu = rng.random(g.shape) + 0.05
    mu /= mu.sum()
    V = O.jko_potential(g)
    # run the inner loop by hand for the final (b, z) and check the KL-prox stationarity
    # (tau/eps)(log s + V) + log(s/z) = 0 with s = b z  (R10)
    r = O.jko(T, L, mu, g, eps=eps, tau=tau, steps=1, iters=300, log_domain=False)
    b = np.ones(g.shape)
    for _ in range(300):
        a = mu / O.conv(T, b)
        z = O.conv_adjoint(T, a)
        b = z ** (-tau / (eps + tau)) * np.exp(-tau * V / (eps + tau))
    s = b * z
    res = (tau / eps) * (np.log(s) + V) + np.log(s / z)
    assert np.abs(res).max() < 1e-12
    np.testing.assert_allclose(r["mus"][1], s / s.sum(), rtol=1e-12)
    # the first marginal of the plan converges to mu_k; the plan mass to 1
    assert r["err"][0][-1] < 1e-9
    assert abs(r["masses"][0] - 1.0) < 1e-8
    rl = O.jko(T, L, mu, g, eps=eps, tau=tau, steps=2, iters=40, log_domain=True)
    rn = O.jko(T, L, mu, g, eps=eps, tau=tau, steps=2, iters=40, log_domain=False)
    np.testing.assert_allclose(rl["mus"], rn["mus"], rtol=1e-10)
    rq = O.jko(T, L, O.quarter_turn(mu), g, eps=eps, tau=tau, steps=2, iters=40, log_domain=False)
    np.testing.assert_allclose(rq["mus"][2], O.quarter_turn(rn["mus"][2]), rtol=1e-10)


# ---------------------------------------------------------------- porous-medium prox --
def test_porous_prox_stationarity_and_brute_force():
    """KL-prox of F = cell/(m-1) sum (s/cell)^m: the stationarity residual vanishes, it agrees with a
    direct scalar minimisation of the per-site objective, tau -> 0 gives s = z, z = 0 gives s = 0."""
    from scipy.optimize import minimize_scalar
    eps, tau, m, cell = 0.003, 1e-3, 5.0, 1e-3
    rng = np.random.default_rng(13)
    z = np.concatenate([[0.0, 1e-8, 1e-4], rng.uniform(1e-5, 0.5, 20)])
    s = O.porous_prox(z, eps, tau, m, cell)
    assert s[0] == 0.0
    pos = z > 0
    C = tau * m / (eps * (m - 1)) * cell ** (1 - m)
    res = C * s[pos] ** (m - 1) + np.log(s[pos] / z[pos])
    assert np.abs(res).max() < 1e-12
    assert np.all(s[pos] <= z[pos])
    for zi, si in zip(z[pos][:8], s[pos][:8]):
        f = lambda x: (tau / eps) * cell / (m - 1) * (x / cell) ** m + x * np.log(x / zi) - x + zi
        r = minimize_scalar(f, bounds=(1e-300, zi), method="bounded", options={"xatol": 1e-18})
        assert abs(r.x - si) <= 1e-6 * si
    np.testing.assert_allclose(O.porous_prox(z, eps, 1e-24, m, cell), z, rtol=1e-9)   # tau -> 0
    # monotone in z
    zz = np.linspace(1e-6, 1, 200)
    assert np.all(np.diff(O.porous_prox(zz, eps, tau, m, cell)) > 0)


def test_jko_porous_mass_equivariance():
    g = O.Grid(8, 8, 8)
    eps, tau = 0.05, 0.02
    T = O.kernel_table(g, 2, eps, (1, np.sqrt(10), np.sqrt(2)))
    L = O.log_kernel_table(g, 2, eps, (1, np.sqrt(10), np.sqrt(2)))
    rng = np.random.default_rng(14)
    mu = rng.random(g.shape) ** 3 + 0.01
    mu /= mu.sum()
    r = O.jko(T, L, mu, g, eps, tau, 1, 300, False, energy="porous", m=5.0)
    assert r["err"][0][-1] < 1e-9
    assert abs(r["masses"][0] - 1.0) < 1e-8
    rl = O.jko(T, L, mu, g, eps, tau, 2, 30, True, energy="porous", m=5.0, trace=False)
    rn = O.jko(T, L, mu, g, eps, tau, 2, 30, False, energy="porous", m=5.0, trace=False)
    np.testing.assert_allclose(rl["mus"], rn["mus"], rtol=1e-10)
    rq = O.jko(T, L, O.quarter_turn(mu), g, eps, tau, 2, 30, False, energy="porous", m=5.0, trace=False)
    np.testing.assert_allclose(rq["mus"][2], O.quarter_turn(rn["mus"][2]), rtol=1e-10)
    r0 = O.jko(T, L, mu, g, eps, 0.0, 1, 3, False, energy="porous", m=5.0, trace=False)
    blur = O.conv(T, mu / O.conv(T, np.ones(g.shape)))
    np.testing.assert_allclose(r0["mus"][1], blur / blur.sum(), rtol=1e-12)


# ---------------------------------------------------------------- transport cost -------
def test_transport_cost_two_diracs_and_dense():
    """Two Diracs: the only coupling is delta x delta, so <pi, c> = rho_b(h^{-1} g)^2 exactly (group law);
    random scalings: equals the dense double sum a K c b."""
    g = O.Grid(8, 8, 8)
    R, eps, w = 3, 0.05, (1, 3, 1)
    T = O.kernel_table(g, R, eps, w)
    L = O.log_kernel_table(g, R, eps, w)
    Tc = O.cost_table(g, R, eps, w)
    mu = np.zeros(g.shape)
    mu[1, 3, 2] = 1
    nu = np.zeros(g.shape)
    nu[2, 5, 4] = 1
    r = O.sinkhorn(T, L, mu, nu, 3, log_domain=False, trace=False)
    ge, he = g.element(1, 3, 2), g.element(2, 5, 4)
    expect = O.rho_b(O.se2_mul(O.se2_inv(he), ge), w) ** 2
    assert abs(O.transport_cost(Tc, r["a"], r["b"]) - expect) < 1e-12 * expect
    K = O.dense_kernel_matrix(g, R, eps, w)
    N = K.shape[0]
    E = g.element(*np.meshgrid(np.arange(8), np.arange(8), np.arange(8), indexing="ij")).reshape(-1, 3)
    C = O.rho_b(O.se2_mul(O.se2_inv(E[None, :, :]), E[:, None, :]), w) ** 2
    rng = np.random.default_rng(15)
    a, b = rng.random(g.shape), rng.random(g.shape)
    dense = a.reshape(-1) @ ((K * C) @ b.reshape(-1))
    assert abs(O.transport_cost(Tc, a, b) - dense) < 1e-12 * dense


# ---------------------------------------------------------------- units of V and of the Haar cell --
def test_jko_potential_units_baseline_formula():
    """BASELINE configs[4]: V(x, theta) = |x - c|^2 / 256^2 in PIXEL units on the 256 x 256 grid, c the
    grid centre, pixel centres at i + 1/2 (reading R10).  Hand-computed values at lattice points
    ((i + 1/2 - 128)^2 + (j + 1/2 - 128)^2) / 65536: a [0,1]-vs-pixel slip (factor 65536), a centre at
    128 - 1/2, or a missing half-cell offset each change them."""
    g = O.Grid(256, 256, 4)
    V = O.jko_potential(g)
    # (i, j) -> exact value (all dyadic rationals, representable in fp64)
    cases = {
        (0, 0): 32512.5 / 65536.0,          # 127.5^2 * 2
        (128, 128): 0.5 / 65536.0,          # 0.5^2 * 2
        (127, 128): 0.5 / 65536.0,          # (-0.5)^2 + 0.5^2
        (255, 0): 32512.5 / 65536.0,
        (200, 64): 9288.5 / 65536.0,        # 72.5^2 + (-63.5)^2 = 5256.25 + 4032.25
        (10, 250): 28812.5 / 65536.0,       # (-117.5)^2 + 122.5^2 = 13806.25 + 15006.25
    }
    for (i, j), want in cases.items():
        for k in range(4):                   # V does not depend on theta
            assert V[k, j, i] == want, ((i, j, k), V[k, j, i], want)
    # a window cut from the 256 lattice (cell 1/256) centres V on the window: same formula in pixels
    gw = O.Grid(100, 92, 2, 1.0 / 256.0, 1.0 / 256.0)
    Vw = O.jko_potential(gw)
    assert Vw[0, 0, 0] == ((0.5 - 50.0) ** 2 + (0.5 - 46.0) ** 2) / 65536.0


def test_haar_cell_units():
    """Haar measure of one cell dx dy dtheta on [0,1]^2 x [0, 2pi): the cells partition the window,
    so N cells have total measure 2 pi (a 1/ntheta-for-2pi/ntheta slip gives 1, a pixel-unit slip
    nx ny 2pi); the c4 lattice's cell is 2 pi / (256 * 256 * 64) = pi / 2^21."""
    for (nx, ny, nt) in [(256, 256, 64), (28, 28, 16), (37, 23, 12)]:
        g = O.Grid(nx, ny, nt)
        assert abs(O.haar_cell(g) * nx * ny * nt - 2.0 * np.pi) < 1e-12
    assert O.haar_cell(O.Grid(256, 256, 64)) == np.pi / 2.0 ** 21
    # a window of the 256 lattice keeps its cell
    assert O.haar_cell(O.Grid(100, 92, 64, 1.0 / 256.0, 1.0 / 256.0)) == np.pi / 2.0 ** 21


def test_full_field_loops_equal_point_definition():
    """The full-field C loops (x innermost, vectorised) add each output's terms in the definition's order
    (theta_i, dy, dx), so they equal the one-output definitions oracle_conv_point / oracle_lse_point BIT
    FOR BIT; ragged grids with the box wider than the window, -inf inputs, and log ranges beyond the
    fp64 exp underflow (the skipped exp(x <= -746) terms are exactly 0)."""
    rng = np.random.default_rng(21)
    for (nx, ny, nt, R) in [(11, 7, 4, 3), (5, 9, 3, 4), (16, 12, 8, 2)]:
        g = O.Grid(nx, ny, nt)
        T = O.kernel_table(g, R, 0.05, (1.0, 3.0, 1.0))
        L = O.log_kernel_table(g, R, 0.05, (1.0, 3.0, 1.0))
        v = rng.random(g.shape)
        lv = rng.uniform(-1500.0, 1500.0, g.shape)
        lv[0, 0, :2] = -np.inf
        lv[:, 1, :] = -np.inf
        y, ly = O.conv(T, v), O.lse_conv(L, lv)
        for to in range(nt):
            for iy in range(ny):
                for ix in range(nx):
                    assert y[to, iy, ix] == O.conv_point(T, v, to, iy, ix)
                    p = O.lse_conv_point(L, lv, to, iy, ix)
                    assert ly[to, iy, ix] == p or (np.isnan(p) and np.isnan(ly[to, iy, ix])), (to, iy, ix)
        # adjoint scatter loops: K = K^T to rounding
        np.testing.assert_allclose(O.conv_adjoint(T, v), y, rtol=1e-13)
        la = O.lse_conv_adjoint(L, lv)
        fin = np.isfinite(ly)
        assert np.array_equal(np.isfinite(la), fin)
        np.testing.assert_allclose(la[fin], ly[fin], rtol=1e-13, atol=1e-10)
