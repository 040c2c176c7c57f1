"""ORACLE -- TEST INFRASTRUCTURE ONLY.  fp64 reference of the SE(2) entropic-OT hot path.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
may import this module.  It never imports paper_2402_15322_b200.

Every function cites the passage it follows (P:n = PAPER.md line n).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from typing import Dict, List, Optional, Sequence

import numpy as np

__all__ = [
    "wrap_angle", "se2_mul", "se2_inv", "half_angle", "rho_b", "spatial_anisotropy",
    "Grid", "kernel_table", "log_kernel_table", "dense_kernel_matrix",
    "conv", "conv_adjoint", "lse_conv", "lse_conv_adjoint", "conv_point", "lse_conv_point",
    "conv_numpy", "sinkhorn", "barycenter", "jko", "jko_potential", "marginal_error",
    "quarter_turn", "oracle_threads", "DIV_FLOOR", "porous_prox", "haar_cell", "cost_table", "transport_cost",
]

DIV_FLOOR = 1e-30      # division guard (reading R9)
TWO_PI = 2.0 * np.pi


# ----------------------------------------------------------------------------------------------
# Group law and distance approximation
# ----------------------------------------------------------------------------------------------

def wrap_angle(t):
    """R / 2piZ represented in [-pi, pi) -- the paper's small-angle convention (P:249, P:628 fn)."""
    return np.mod(np.asarray(t, dtype=np.float64) + np.pi, TWO_PI) - np.pi


def se2_mul(g1, g2):
    """(x,y,th)(x',y',th') = (x + x'cos th - y' sin th, y + x' sin th + y' cos th, th + th')."""
    g1 = np.asarray(g1, dtype=np.float64)
    g2 = np.asarray(g2, dtype=np.float64)
    x, y, t = g1[..., 0], g1[..., 1], g1[..., 2]
    xp, yp, tp = g2[..., 0], g2[..., 1], g2[..., 2]
    c, s = np.cos(t), np.sin(t)
    return np.stack([x + xp * c - yp * s, y + xp * s + yp * c, wrap_angle(t + tp)], axis=-1)


def se2_inv(g):
    """g^{-1} = (-R^{-1} x, R^{-1})."""
    g = np.asarray(g, dtype=np.float64)
    x, y, t = g[..., 0], g[..., 1], g[..., 2]
    c, s = np.cos(t), np.sin(t)
    # R^{-1} = R(-t): (x c + y s, -x s + y c)
    return np.stack([-(x * c + y * s), -(-x * s + y * c), wrap_angle(-t)], axis=-1)


def half_angle(g):
    """Half-angle coordinates b(g) (eq. equ:logcomp), theta in the small-angle convention."""
    g = np.asarray(g, dtype=np.float64)
    x, y, t = g[..., 0], g[..., 1], wrap_angle(g[..., 2])
    c, s = np.cos(t / 2.0), np.sin(t / 2.0)
    return np.stack([x * c + y * s, -x * s + y * c, t], axis=-1)


def rho_b(g, w):
    """rho_b(g) = sqrt((w1 b1)^2 + (w2 b2)^2 + (w3 b3)^2)  (eq. eq:rhob)."""
    b = half_angle(g)
    w = np.asarray(w, dtype=np.float64)
    return np.sqrt((w[0] * b[..., 0]) ** 2 + (w[1] * b[..., 1]) ** 2 + (w[2] * b[..., 2]) ** 2)


def spatial_anisotropy(w):
    """zeta = max(w1,w2)/min(w1,w2)  (eq. equ:spatial_anisotropy)."""
    return max(w[0], w[1]) / min(w[0], w[1])


# ----------------------------------------------------------------------------------------------
# Lattice and Gibbs kernel (readings R1-R4)
# ----------------------------------------------------------------------------------------------

class Grid:
    """nx x ny x ntheta lattice on [0,1]^2 x [0, 2pi): cell centres x_i = (i + 1/2)/nx,
    theta_k = 2 pi k / ntheta.  Field arrays are [ntheta][ny][nx].
    hx, hy: cell sizes (default 1/nx, 1/ny, reading R1); a window cut from a finer lattice keeps its
    cell, x_i = (i + 1/2) hx on [0, nx hx]."""

    def __init__(self, nx: int, ny: int, ntheta: int, hx: float = 0.0, hy: float = 0.0):
        self.nx, self.ny, self.ntheta = int(nx), int(ny), int(ntheta)
        self.hx = float(hx) if hx else 1.0 / self.nx
        self.hy = float(hy) if hy else 1.0 / self.ny

    @property
    def shape(self):
        return (self.ntheta, self.ny, self.nx)

    def x(self, i):
        return (np.asarray(i, dtype=np.float64) + 0.5) * self.hx

    def y(self, j):
        return (np.asarray(j, dtype=np.float64) + 0.5) * self.hy

    def theta(self, k):
        return TWO_PI * np.asarray(k, dtype=np.float64) / self.ntheta

    def element(self, k, j, i):
        return np.stack(np.broadcast_arrays(self.x(i), self.y(j), self.theta(k)), axis=-1)


def _relative_rho2(grid: Grid, R: int, w):
    """rho_b(h^{-1} g)^2 for every (theta_g, theta_h, dy, dx) of the box, with g, h actual
    lattice elements (h at the window centre, g displaced by (dx, dy) cells)."""
    nt = grid.ntheta
    S = 2 * R + 1
    ci, cj = grid.nx // 2, grid.ny // 2
    to, ti, dy, dx = np.meshgrid(np.arange(nt), np.arange(nt), np.arange(-R, R + 1),
                                 np.arange(-R, R + 1), indexing="ij")
    g = grid.element(to, cj + dy, ci + dx)
    h = grid.element(ti, cj + 0 * dy, ci + 0 * dx)
    rel = se2_mul(se2_inv(h), g)
    r = rho_b(rel, w)
    return (r * r).reshape(nt, nt, S, S)


def kernel_table(grid: Grid, R: int, eps: float, w) -> np.ndarray:
    """T[to, ti, dy+R, dx+R] = K(h^{-1} g) = exp(-rho_b(h^{-1}g)^2 / eps)  (P:591-596 with d := rho_b,
    p = 2, App. A line 'K_eps <- exp(-rho_b^2/eps)').  Every box entry is exact in fp64."""
    return np.exp(-_relative_rho2(grid, R, w) / eps)


def log_kernel_table(grid: Grid, R: int, eps: float, w) -> np.ndarray:
    """L = -rho_b^2 / eps (log of kernel_table, evaluated directly, never via log(exp))."""
    return -_relative_rho2(grid, R, w) / eps


def cost_table(grid: Grid, R: int, eps: float, w) -> np.ndarray:
    """Tc = K * c with c = rho_b^2 (P:186-195 with d := rho_b, p = 2): the kernel of the transport cost."""
    r2 = _relative_rho2(grid, R, w)
    return np.exp(-r2 / eps) * r2


def transport_cost(Tc, a, b) -> float:
    """<pi, c> = sum_{g,h} a(g) K(g,h) c(g,h) b(h) for the plan pi = a K b (R11), i.e.
    sum_g a(g) (Tc * b)(g) -- the plan is never materialised."""
    return float(np.sum(np.asarray(a, dtype=np.float64) * conv(Tc, b)))


def dense_kernel_matrix(grid: Grid, R: int, eps: float, w) -> np.ndarray:
    """Brute-force N x N matrix K[g, h] = exp(-rho_b(h^{-1} g)^2/eps) for all lattice pairs within the
    spatial box, computed pair by pair from the group law -- no table, no convolution.
    Row/column index = (k*ny + j)*nx + i.  For tiny grids only."""
    nt, ny, nx = grid.shape
    k, j, i = np.meshgrid(np.arange(nt), np.arange(ny), np.arange(nx), indexing="ij")
    E = grid.element(k, j, i).reshape(-1, 3)
    J = j.reshape(-1)
    I = i.reshape(-1)
    N = E.shape[0]
    g = np.repeat(E[:, None, :], N, axis=1)
    h = np.repeat(E[None, :, :], N, axis=0)
    rel = se2_mul(se2_inv(h), g)
    Kd = np.exp(-rho_b(rel, w) ** 2 / eps)
    box = (np.abs(J[:, None] - J[None, :]) <= R) & (np.abs(I[:, None] - I[None, :]) <= R)
    return np.where(box, Kd, 0.0)


# ----------------------------------------------------------------------------------------------
# Group convolution: plain C loops (oracle/se2_conv_ref.c), fp64
# ----------------------------------------------------------------------------------------------

_HERE = os.path.dirname(os.path.abspath(__file__))


def _host_has_avx2() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            flags = f.read()
        return " avx2" in flags and " fma" in flags
    except OSError:
        return False


# x86-64-v3 (AVX2) build where the host has it: the x loops vectorise 4-wide.  Same source, same
# operations per output (contraction off), so both builds give bit-identical results.
_MARCH = ["-march=x86-64-v3"] if _host_has_avx2() else []
_LIB_PATH = os.path.join(_HERE, "libse2oracle_v3.so" if _MARCH else "libse2oracle.so")
_lib = None
_lib_lock = threading.Lock()


def build_oracle_lib(force: bool = False) -> str:
    """Compile oracle/se2_conv_ref.c with gcc (fp64, OpenMP).  Building the checker is not using it."""
    src = os.path.join(_HERE, "se2_conv_ref.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", *_MARCH, "-fopenmp", "-fPIC", "-shared", "-std=c99",
                               "-fno-fast-math", "-ffp-contract=off", "-o", tmp, src, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lib_lock:
        if _lib is None:
            build_oracle_lib()
            lib = ctypes.CDLL(_LIB_PATH)
            P = ctypes.POINTER(ctypes.c_double)
            ci = ctypes.c_int
            for name in ("oracle_conv_gather", "oracle_conv_scatter_adjoint", "oracle_lse_gather"):
                getattr(lib, name).argtypes = [ci, ci, ci, ci, P, P, P]
                getattr(lib, name).restype = None
            lib.oracle_lse_scatter_adjoint.argtypes = [ci, ci, ci, ci, P, P, P, P]
            lib.oracle_lse_scatter_adjoint.restype = None
            for name in ("oracle_conv_point", "oracle_lse_point"):
                getattr(lib, name).argtypes = [ci, ci, ci, ci, P, P, ci, ci, ci]
                getattr(lib, name).restype = ctypes.c_double
            _lib = lib
    return _lib


def oracle_threads() -> int:
    """Number of OpenMP threads the C loops use (OMP_NUM_THREADS, else all cores)."""
    v = os.environ.get("OMP_NUM_THREADS")
    return int(v) if v else (os.cpu_count() or 1)


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _prep(T, v):
    T = np.ascontiguousarray(T, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    nt = T.shape[0]
    S = T.shape[2]
    R = (S - 1) // 2
    assert T.shape == (nt, nt, S, S) and v.shape[-3] == nt
    return T, v, nt, R


def _batched(fn, T, v, *extra):
    T, v, nt, R = _prep(T, v)
    ny, nx = v.shape[-2], v.shape[-1]
    flat = v.reshape(-1, nt, ny, nx)
    out = np.empty_like(flat)
    for b in range(flat.shape[0]):
        src = np.ascontiguousarray(flat[b])
        dst = np.empty_like(src)
        fn(nx, ny, nt, R, _p(T), _p(src), _p(dst), *[_p(np.empty_like(src)) for _ in extra])
        out[b] = dst
    return out.reshape(v.shape)


def conv(T, v):
    """(K v)(g) = sum_h K(h^{-1}g) v(h): gather form.  v: [..., nt, ny, nx]."""
    return _batched(_load().oracle_conv_gather, T, v)


def conv_adjoint(T, a):
    """(K^T a)(h) = sum_g K(h^{-1}g) a(g): written as a scatter over g."""
    return _batched(_load().oracle_conv_scatter_adjoint, T, a)


def lse_conv(L, lv):
    """log (K exp(lv)) = LSE_h (L(g,h) + lv(h)), exact two-pass.  Same iterate as conv in logs (R7)."""
    return _batched(_load().oracle_lse_gather, L, lv)


def lse_conv_adjoint(L, la):
    """log (K^T exp(la)) as an exact two-pass scatter."""
    return _batched(_load().oracle_lse_scatter_adjoint, L, la, "scratch")


def conv_point(T, v, to, iy, ix) -> float:
    """One output sample of conv(T, v) (for sampled parity at full size)."""
    T, v, nt, R = _prep(T, v)
    ny, nx = v.shape[-2], v.shape[-1]
    return _load().oracle_conv_point(nx, ny, nt, R, _p(T), _p(v), int(to), int(iy), int(ix))


def lse_conv_point(L, lv, to, iy, ix) -> float:
    L, lv, nt, R = _prep(L, lv)
    ny, nx = lv.shape[-2], lv.shape[-1]
    return _load().oracle_lse_point(nx, ny, nt, R, _p(L), _p(lv), int(to), int(iy), int(ix))


def conv_numpy(T, v):
    """Pure-numpy gather conv (slice per (to, ti, dy, dx)) -- an independent second implementation
    used only to cross-check the C loops on small grids."""
    T = np.asarray(T, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    nt, _, S, _ = T.shape
    R = (S - 1) // 2
    ny, nx = v.shape[-2:]
    y = np.zeros(v.shape, dtype=np.float64)
    for to in range(nt):
        for ti in range(nt):
            for dy in range(-R, R + 1):
                for dx in range(-R, R + 1):
                    t = T[to, ti, dy + R, dx + R]
                    # y[to, iy, ix] += t * v[ti, iy - dy, ix - dx]
                    ys0, ys1 = max(0, dy), min(ny, ny + dy)
                    xs0, xs1 = max(0, dx), min(nx, nx + dx)
                    if ys1 <= ys0 or xs1 <= xs0:
                        continue
                    y[..., to, ys0:ys1, xs0:xs1] += t * v[..., ti, ys0 - dy:ys1 - dy, xs0 - dx:xs1 - dx]
    return y


# ----------------------------------------------------------------------------------------------
# Scaling algorithms (App. A, JKO P:224-234)
# ----------------------------------------------------------------------------------------------

def marginal_error(a, Kb, mu) -> float:
    """L1 violation of the first marginal: sum |a * (K b) - mu|  (reading R8)."""
    return float(np.sum(np.abs(np.asarray(a) * np.asarray(Kb) - np.asarray(mu))))


def _log(x):
    with np.errstate(divide="ignore"):
        return np.log(np.asarray(x, dtype=np.float64))


def _ldiv(lt, ly):
    """log of t / y: lt - ly, with log(0 / y) = -inf for every y (the linear guard maps 0/0 to 0, R9)."""
    with np.errstate(invalid="ignore"):
        return np.where(lt == -np.inf, -np.inf, lt - ly)


def sinkhorn(T, L, mu, nu, iters: int, log_domain: bool, trace: bool = True) -> Dict:
    """Sinkhorn iterations a = mu / K b, b = nu / K^T a with b^(0) = 1  (R5).

    Linear domain: divisions guarded at DIV_FLOOR (R9).  Log domain (R7): alpha = log a,
    beta = log b, alpha = log mu - LSE(L + beta), beta = log nu - LSE^T(L + alpha).
    err[l] = sum |a (K b) - mu| after the l-th b-update (R8).
    Returns a, b (or alpha, beta), row = a*Kb, col = b*K^T a, err trace.
    """
    mu = np.asarray(mu, dtype=np.float64)
    nu = np.asarray(nu, dtype=np.float64)
    err = []
    if not log_domain:
        b = np.ones_like(mu)
        Kb = conv(T, b)                      # K b of the current b (reused by the trace and the next a)
        for _ in range(iters):
            a = mu / np.maximum(Kb, DIV_FLOOR)
            Kta = conv_adjoint(T, a)
            b = nu / np.maximum(Kta, DIV_FLOOR)
            Kb = conv(T, b)
            if trace:
                err.append(marginal_error(a, Kb, mu))
        return dict(a=a, b=b, row=a * Kb, col=b * conv_adjoint(T, a), err=np.array(err))
    lmu, lnu = _log(mu), _log(nu)
    beta = np.zeros_like(mu)
    lKb = lse_conv(L, beta)
    for _ in range(iters):
        alpha = _ldiv(lmu, lKb)
        beta = _ldiv(lnu, lse_conv_adjoint(L, alpha))
        lKb = lse_conv(L, beta)
        if trace:
            err.append(float(np.sum(np.abs(np.exp(alpha + lKb) - mu))))
    return dict(alpha=alpha, beta=beta, row=np.exp(alpha + lKb),
                col=np.exp(beta + lse_conv_adjoint(L, alpha)), err=np.array(err))


def barycenter(T, L, mus: Sequence[np.ndarray], lambdas, iters: int, log_domain: bool,
               trace: bool = True) -> Dict:
    """App. A, followed verbatim:
        v_i, w_i <- 1
        for j: mu <- 1; for i: w_i <- mu_i / (K*v_i); d_i <- v_i (K*w_i); mu <- mu d_i^lambda_i
               for i: v_i <- v_i mu / d_i
        return mu
    lambda_i = 0 terms are skipped (d^0 = 1, R6).  Log domain: same iterates in logs (R7).
    err[j] = sum_i lambda_i sum|w_i (K v_i) - mu_i| after the v-update (R8); errs_i per input.
    """
    lam = np.asarray(lambdas, dtype=np.float64)
    n = len(mus)
    mus = [np.asarray(m, dtype=np.float64) for m in mus]
    err, errs = [], []
    if not log_domain:
        v = [np.ones_like(mus[0]) for _ in range(n)]
        w = [np.ones_like(mus[0]) for _ in range(n)]
        Kv = [conv(T, v[i]) for i in range(n)]      # K v_i of the current v_i (trace + next w-update)
        for _ in range(iters):
            mubar = np.ones_like(mus[0])
            d = [None] * n
            for i in range(n):
                w[i] = mus[i] / np.maximum(Kv[i], DIV_FLOOR)
                d[i] = v[i] * conv(T, w[i])
                if lam[i] != 0.0:
                    mubar = mubar * d[i] ** lam[i]
            for i in range(n):
                v[i] = v[i] * mubar / np.maximum(d[i], DIV_FLOOR)
                Kv[i] = conv(T, v[i])
            if trace:
                e = [float(np.sum(np.abs(w[i] * Kv[i] - mus[i]))) for i in range(n)]
                errs.append(e)
                err.append(float(np.dot(lam, e)))
        return dict(bary=mubar, v=np.stack(v), w=np.stack(w), err=np.array(err), errs=np.array(errs))
    lmus = [_log(m) for m in mus]
    lv = [np.zeros_like(mus[0]) for _ in range(n)]
    lw = [np.zeros_like(mus[0]) for _ in range(n)]
    lKv = [lse_conv(L, lv[i]) for i in range(n)]
    for _ in range(iters):
        lbar = np.zeros_like(mus[0])
        ld = [None] * n
        for i in range(n):
            lw[i] = _ldiv(lmus[i], lKv[i])
            ld[i] = lv[i] + lse_conv(L, lw[i])
            if lam[i] != 0.0:
                lbar = lbar + lam[i] * ld[i]
        for i in range(n):
            lv[i] = lv[i] + lbar - ld[i]
            lKv[i] = lse_conv(L, lv[i])
        if trace:
            e = [float(np.sum(np.abs(np.exp(lw[i] + lKv[i]) - mus[i]))) for i in range(n)]
            errs.append(e)
            err.append(float(np.dot(lam, e)))
    return dict(lbary=lbar, bary=np.exp(lbar), lv=np.stack(lv), lw=np.stack(lw), err=np.array(err),
                errs=np.array(errs))


def jko_potential(grid: Grid) -> np.ndarray:
    """V(x, theta) = |x - c|^2 with c the window centre, in [0,1]^2 units (BASELINE configs[4]:
    |x - c|^2 / 256^2 in pixel units on the 256 grid); broadcast over theta (R10)."""
    X = grid.x(np.arange(grid.nx))[None, None, :]
    Y = grid.y(np.arange(grid.ny))[None, :, None]
    cx, cy = 0.5 * grid.nx * grid.hx, 0.5 * grid.ny * grid.hy
    V = (X - cx) ** 2 + (Y - cy) ** 2
    return np.broadcast_to(V, grid.shape).copy()


def haar_cell(grid: Grid) -> float:
    """Haar measure of one lattice cell, dx dy dtheta with the [0,1]^2 x [0,2pi) window (R1)."""
    return grid.hx * grid.hy * (TWO_PI / grid.ntheta)


def porous_prox(z, eps: float, tau: float, m: float, cell: float):
    """KL-prox of the porous-medium energy F(mu) = 1/(m-1) int mu^m dH, mu a density w.r.t.
    the Haar measure, discretised with masses s on cells of measure `cell` (density s/cell):
        s = argmin_s (tau/eps) F(s) + KL(s | z),   F(s) = cell/(m-1) sum (s/cell)^m.
    Stationarity per site: (tau m / (eps (m-1))) (s/cell)^{m-1} + log(s/z) = 0.  With u = log s:
        g(u) = C e^{(m-1) u} + u - log z = 0,  C = tau m / (eps (m-1)) cell^{1-m},
    g convex and increasing, root <= log z: Newton from u = log z (monotone), bisection fallback on
    [log z - 50, log z].  s = 0 where z = 0."""
    z = np.asarray(z, dtype=np.float64)
    C = tau * m / (eps * (m - 1.0)) * cell ** (1.0 - m)
    out = np.zeros_like(z)
    pos = z > 0
    lz = np.log(z[pos])
    u = lz.copy()
    for _ in range(200):
        ex = C * np.exp((m - 1.0) * u)
        du = (ex + u - lz) / ((m - 1.0) * ex + 1.0)
        u = u - du
        if np.all(np.abs(du) <= 1e-15 * (1.0 + np.abs(u))):
            break
    bad = ~np.isfinite(u) | (np.abs(C * np.exp((m - 1.0) * u) + u - lz) > 1e-12 * (1 + np.abs(lz)))
    if np.any(bad):
        lo, hi = lz[bad] - 50.0, lz[bad].copy()
        for _ in range(200):
            mid = 0.5 * (lo + hi)
            gm = C * np.exp((m - 1.0) * mid) + mid - lz[bad]
            hi = np.where(gm > 0, mid, hi)
            lo = np.where(gm > 0, lo, mid)
        u[bad] = 0.5 * (lo + hi)
    out[pos] = np.exp(u)
    return out


def jko(T, L, mu0, grid: Grid, eps: float, tau: float, steps: int, iters: int, log_domain: bool,
        trace: bool = True, energy: str = "entropy_potential", m: float = 5.0) -> Dict:
    """Entropic JKO time-marching (eq. equ:GF_JKO) solved with the scaling iterations
    (eq. equ:scaling_iterations): F1 = marginal constraint mu_k (prox = mu_k),
    F2 = tau F with F(s) = sum s (log s - 1) + sum V s (entropy + linear potential, BASELINE
    configs[4]).  KL-prox (reading R10):  prox(z) = z^{eps/(eps+tau)} exp(-tau V/(eps+tau)),
    hence b = prox(z)/z = z^{-tau/(eps+tau)} exp(-tau V/(eps+tau)).
    Per step k: b <- 1; for l: a = mu_k / K b; z = K^T a; b = prox(z)/z.
    Then s = b z, mass_k = sum s, mu_{k+1} = s / mass_k.
    """
    V = jko_potential(grid)
    p = tau / (eps + tau)
    q = tau / (eps + tau)
    cell = haar_cell(grid)
    porous = energy == "porous"
    mu = np.asarray(mu0, dtype=np.float64)
    masses, errs, mus = [], [], [mu]
    for _k in range(steps):
        err = []
        if not log_domain:
            b = np.ones_like(mu)
            Kb = conv(T, b)
            for _l in range(iters):
                a = mu / np.maximum(Kb, DIV_FLOOR)
                z = np.maximum(conv_adjoint(T, a), DIV_FLOOR)
                if porous:
                    b = porous_prox(z, eps, tau, m, cell) / z            # b = prox(z)/z
                else:
                    b = z ** (-p) * np.exp(-q * V)
                if _l + 1 < iters or trace:
                    Kb = conv(T, b)
                if trace:
                    err.append(marginal_error(a, Kb, mu))
            s = b * z
        else:
            lmu = _log(mu)
            beta = np.zeros_like(mu)
            lKb = lse_conv(L, beta)
            for _l in range(iters):
                alpha = _ldiv(lmu, lKb)
                lz = lse_conv_adjoint(L, alpha)
                if porous:
                    beta = np.log(porous_prox(np.exp(lz), eps, tau, m, cell)) - lz
                else:
                    beta = -p * lz - q * V
                if _l + 1 < iters or trace:
                    lKb = lse_conv(L, beta)
                if trace:
                    err.append(float(np.sum(np.abs(np.exp(alpha + lKb) - mu))))
            s = np.exp(beta + lz)
        mass = float(s.sum())
        masses.append(mass)
        errs.append(err)
        mu = s / mass
        mus.append(mu)
    last = dict(a=a, b=b) if not log_domain else dict(alpha=alpha, beta=beta)
    return dict(mus=np.stack(mus), masses=np.array(masses), err=np.array(errs), **last)


# ----------------------------------------------------------------------------------------------
# Grid-exact left action used by the equivariance pins (Lemma 3.1)
# ----------------------------------------------------------------------------------------------

def quarter_turn(f):
    """Push-forward of a field by the rotation by +pi/2 about the window centre (a lattice
    permutation when nx == ny and 4 | ntheta): (i, j, k) -> (n-1-j, i, k + nt/4)."""
    f = np.asarray(f)
    nt, ny, nx = f.shape[-3:]
    assert nx == ny and nt % 4 == 0
    out = np.empty_like(f)
    k = np.arange(nt)
    # out[k + nt/4, i, n-1-j]  (layout [theta][y][x]:  new x = n-1-j, new y = i)
    for kk in range(nt):
        src = f[..., kk, :, :]                     # [y=j][x=i]
        # new[y'=i][x'=n-1-j] = src[j][i]  ->  new = rot90 of src
        new = np.empty_like(src)
        new[..., :, :] = np.flip(np.swapaxes(src, -1, -2), axis=-1)
        out[..., (kk + nt // 4) % nt, :, :] = new
    return out
