"""ORACLE -- TEST INFRASTRUCTURE ONLY.  fp64 reference of the lifting / projection pipeline that
turns images and orientation fields into measures on the SE(2) grid and back.

Only tests/, __graft_entry__.smoke() and bench.py may import this module.  It never imports
paper_2402_15322_b200.  Citations: P:n = PAPER.md line n.

* orientation score transform (eq. `eq:lift`): U(g) = int psi(g^{-1} . x) f(x) dx, g = (b, theta),
  g^{-1} . x = R_theta^{-1}(x - b); discretely U(b, theta_j) = sum_x psi_j(x - b) f(x) with
  psi_j(d) = psi(R_{theta_j}^{-1} d), zero padding outside the image;
* cake wavelets (P:288 and App. B P:1036-1038 defer the exact formulas to the literature; they
  "smoothly approximate indicator functions supported on cones" in the Fourier domain and
  sum_theta psi^_theta ~ 1 on a disk of radius rho0 near Nyquist, eq. `eq:fastreco` P:1025-1030 --
  reading R15 in DESIGN.md): a degree-k cardinal B-spline in the angle times a radial window,
      psi^_j(omega) = B_k( wrap(arg omega - theta_j - pi/2) / s_theta ) W(|omega|),   s_theta = 2 pi / N,
      W(rho) = 1 for rho <= c pi,  exp(-(rho - c pi)^2 / (2 ((1 - c) pi / 2)^2)) beyond,  psi^_j(0) = 1 / N,
  on the L x L DFT lattice omega = 2 pi (k1, k2) / L of the filter support; the spatial filter is
  psi_j(d) = L^-2 sum_omega psi^_j(omega) e^{i omega . d}.  The wedge of theta_j is centred at
  theta_j + pi/2 so that a line of orientation theta_j (whose spectrum is perpendicular to it) lands
  in bin j.  sum_j B_k(. - j) = 1 gives sum_j psi^_j = W exactly.  The real part of the score is used:
  the split into max(U, 0) and max(-U, 0) needs real values (R15);
* projection (eq. `eq:proj`): P(U) = sum_j U(., theta_j) (the theta measure is absorbed in the
  bank normalisation sum_j psi^_j = W);
* positive-part measures (eq. `eq:tildeW-v1`; Step 2 of P:808-809): U^+ = max(U, 0) / m^+,
  U^- = max(-U, 0) / m^-, m^+- the masses;
* signed recombination (eq. `eq:final`) and the "dominant positive response, normalised"
  (P:820): b = max(m^+ P(U^+) - m^- P(U^-), 0) / sum;
* orientation-field lift (eq. `equ:lifting_vector_field`): U(x, theta_k) = |v(x)| iff
  d_S1(psi(x), theta_k) < pi/N; the boundary case d = pi/N goes to the lower bin (the paper's strict
  inequality leaves it unassigned -- reading R16); normalised to mass 1;
* reconstruction (eq. `equ:reconstruction_vector_field`): |v| = sum_k U(x, theta_k),
  psi* = theta_argmax (ties -> smallest k).
"""
from __future__ import annotations

import numpy as np

__all__ = ["bspline", "radial_window", "cake_hat", "cake_bank", "lift_image", "split_signed", "project", "project_signed",
           "bin_of_angle", "lift_field", "reconstruct_field", "quarter_turn_image"]

TWO_PI = 2.0 * np.pi


def bspline(x, degree: int):
    """Centred cardinal B-spline of the given degree (support [-(k+1)/2, (k+1)/2]) by the Cox-de Boor
    recursion  B_k(x) = [ (x + (k+1)/2) B_{k-1}(x + 1/2) + ((k+1)/2 - x) B_{k-1}(x - 1/2) ] / k,
    B_0 = the box [-1/2, 1/2) (stable and non-negative, unlike the truncated-power sum)."""
    x = np.asarray(x, dtype=np.float64)
    k = int(degree)
    if k == 0:
        return np.where((x >= -0.5) & (x < 0.5), 1.0, 0.0)
    h = (k + 1) / 2.0
    return ((x + h) * bspline(x + 0.5, k - 1) + (h - x) * bspline(x - 0.5, k - 1)) / k


def radial_window(rho, radial_cut: float):
    """W(rho): 1 on the disk rho <= c pi, Gaussian taper (sigma = (1 - c) pi / 2) beyond."""
    rho = np.asarray(rho, dtype=np.float64)
    r0 = radial_cut * np.pi
    sig = (1.0 - radial_cut) * np.pi / 2.0
    return np.where(rho <= r0, 1.0, np.exp(-(rho - r0) ** 2 / (2.0 * sig * sig)))


def _wrap(a):
    return (np.asarray(a) + np.pi) % TWO_PI - np.pi


def cake_hat(ntheta: int, size: int, degree: int = 3, radial_cut: float = 0.8) -> np.ndarray:
    """psi^_j(omega) on the L x L lattice, array [N][k2][k1] (k = -(L-1)/2 .. (L-1)/2; k1 <-> omega_x)."""
    assert size % 2 == 1 and ntheta >= degree + 1
    L = size
    k = np.arange(L) - (L - 1) // 2
    wy, wx = np.meshgrid(TWO_PI * k / L, TWO_PI * k / L, indexing="ij")
    rho = np.hypot(wx, wy)
    W = radial_window(rho, radial_cut)
    phi = np.arctan2(wy, wx)
    s = TWO_PI / ntheta
    out = np.empty((ntheta, L, L))
    for j in range(ntheta):
        th = TWO_PI * j / ntheta
        out[j] = bspline(_wrap(phi - th - np.pi / 2) / s, degree) * W
    c = (L - 1) // 2
    out[:, c, c] = 1.0 / ntheta            # DC split uniformly (W(0) = 1)
    return out


def cake_bank(ntheta: int, size: int, degree: int = 3, radial_cut: float = 0.8) -> np.ndarray:
    """Complex spatial filters psi_j(d) = L^-2 sum_omega psi^_j(omega) e^{i omega.d}, array [N][dy][dx]
    for d in [-R, R]^2, by the explicit double sum (no FFT)."""
    H = cake_hat(ntheta, size, degree, radial_cut)
    L = size
    k = np.arange(L) - (L - 1) // 2
    w = TWO_PI * k / L
    d = k.astype(np.float64)                          # spatial offsets -R..R
    Ex = np.exp(1j * np.outer(d, w))                  # [dx][k1] = e^{i w_k1 dx}
    Ey = np.exp(1j * np.outer(d, w))                  # [dy][k2]
    # psi[j, dy, dx] = L^-2 sum_{k2,k1} H[j,k2,k1] Ey[dy,k2] Ex[dx,k1]
    return np.einsum("jab,ya,xb->jyx", H, Ey, Ex) / (L * L)


def lift_image(f, bank_real) -> np.ndarray:
    """U[j, y, x] = sum_{dy,dx} psi_j(dy, dx) f[y + dy, x + dx] (correlation, zero padding; eq. lift).
    f: [..., ny, nx]; bank_real: [N][L][L]."""
    f = np.asarray(f, dtype=np.float64)
    B = np.asarray(bank_real, dtype=np.float64)
    N, L, _ = B.shape
    R = (L - 1) // 2
    ny, nx = f.shape[-2:]
    fp = np.zeros(f.shape[:-2] + (ny + 2 * R, nx + 2 * R))
    fp[..., R:R + ny, R:R + nx] = f
    U = np.zeros(f.shape[:-2] + (N, ny, nx))
    for j in range(N):
        acc = np.zeros(f.shape[:-2] + (ny, nx))
        for a in range(L):
            for b in range(L):
                acc += B[j, a, b] * fp[..., a:a + ny, b:b + nx]
        U[..., j, :, :] = acc
    return U


def split_signed(U, floor_rel: float = 0.0):
    """(U^+, U^-, m^+, m^-): positive and negative parts, each normalised to mass 1 (eq. tildeW-v1,
    P:808-809); m^+- are the parts' masses before normalisation.  floor_rel > 0 adds floor_rel * max(part)
    to every site of a part before normalising (the configs' input recipe "plus a 1e-6 floor",
    B:configs; keeps the log-domain App. A iteration away from empty windows -- reading R17).  A part
    with zero mass is returned as zeros."""
    U = np.asarray(U, dtype=np.float64)
    out = []
    masses = []
    for part in (np.maximum(U, 0.0), np.maximum(-U, 0.0)):
        ax = (-3, -2, -1)
        m = part.sum(axis=ax)
        mx = part.max(axis=ax)
        n = part.shape[-3] * part.shape[-2] * part.shape[-1]
        fl = floor_rel * mx
        tot = m + fl * n
        x = (part + fl[..., None, None, None]) / np.where(tot > 0, tot, 1.0)[..., None, None, None]
        out.append(np.where((m > 0)[..., None, None, None], x, 0.0))
        masses.append(m)
    return out[0], out[1], masses[0], masses[1]


def project(U) -> np.ndarray:
    """P(U) = sum_j U(., theta_j)  (eq. proj)."""
    return np.asarray(U, dtype=np.float64).sum(axis=-3)


def project_signed(Up, Un, mp, mn):
    """b = max(m^+ P(U^+) - m^- P(U^-), 0) normalised to sum 1 (eq. final + P:820); returns (b, mass
    before normalisation)."""
    mp = np.asarray(mp, dtype=np.float64)
    mn = np.asarray(mn, dtype=np.float64)
    b = mp[..., None, None] * project(Up) - mn[..., None, None] * project(Un)
    b = np.maximum(b, 0.0)
    s = b.sum(axis=(-2, -1))
    return b / np.where(s > 0, s, 1.0)[..., None, None], s


def bin_of_angle(angle, ntheta: int):
    """theta bin of an orientation angle (rad): the k with d_S1(angle, theta_k) < pi/N, the lower bin at
    d = pi/N exactly (R16).  fp64: t = angle * N / (2 pi) (angle wrapped into [0, 2pi) first),
    k = ceil(t - 1/2) mod N."""
    a = np.asarray(angle, dtype=np.float64)
    a = np.mod(a, TWO_PI)
    t = a * ntheta / TWO_PI
    return (np.ceil(t - 0.5).astype(np.int64)) % ntheta


def lift_field(angle, mag, ntheta: int):
    """(U, mass): U[k, y, x] = |v(x, y)| on the bin of psi(x, y), 0 elsewhere, normalised to mass 1
    (eq. equ:lifting_vector_field).  angle, mag: [..., ny, nx]."""
    mag = np.asarray(mag, dtype=np.float64)
    k = bin_of_angle(angle, ntheta)
    U = np.zeros(mag.shape[:-2] + (ntheta,) + mag.shape[-2:])
    for kk in range(ntheta):
        U[..., kk, :, :] = np.where(k == kk, mag, 0.0)
    s = U.sum(axis=(-3, -2, -1))
    return U / np.where(s > 0, s, 1.0)[..., None, None, None], s


def reconstruct_field(U, threshold: float = 0.0):
    """(angle, mag): |v| = sum_k U(., theta_k), psi* = theta of the first maximum over k
    (eq. equ:reconstruction_vector_field); sites with |v| < threshold (or all-zero) get (0, 0)."""
    U = np.asarray(U, dtype=np.float64)
    N = U.shape[-3]
    mag = U.sum(axis=-3)
    k = np.argmax(U, axis=-3)                          # first maximum
    ang = TWO_PI * k / N
    keep = (mag >= threshold) & (mag > 0)
    return np.where(keep, ang, 0.0), np.where(keep, mag, 0.0)


def quarter_turn_image(f):
    """Rotation of an image by +pi/2 about the window centre, the spatial part of oracle.quarter_turn:
    the pixel (x = i, y = j) moves to (n-1-j, i)."""
    f = np.asarray(f)
    assert f.shape[-1] == f.shape[-2]
    return np.flip(np.swapaxes(f, -1, -2), axis=-1)
