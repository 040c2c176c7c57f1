"""Pins of the lifting / projection oracle (oracle/se2_lift.py) against what the paper and the
mathematics fix -- closed forms, exact identities, invariants.  CPU only."""
import math

import numpy as np
import pytest

import oracle as O
from oracle import se2_lift as LF

TWO_PI = 2 * np.pi


# ---- cardinal B-splines (the angular profile) -------------------------------------------------

def test_bspline_worked_values():
    # cubic: B(0) = 2/3, B(+-1) = 1/6, B(+-2) = 0;  quadratic: B(0) = 3/4, B(+-1) = 1/8;  linear: hat
    assert LF.bspline(0.0, 3) == pytest.approx(2 / 3, abs=1e-15)
    assert LF.bspline(1.0, 3) == pytest.approx(1 / 6, abs=1e-15)
    assert LF.bspline(-1.0, 3) == pytest.approx(1 / 6, abs=1e-15)
    assert LF.bspline(2.0, 3) == pytest.approx(0.0, abs=1e-15)
    assert LF.bspline(0.0, 2) == pytest.approx(3 / 4, abs=1e-15)
    assert LF.bspline(1.0, 2) == pytest.approx(1 / 8, abs=1e-15)
    assert LF.bspline(0.25, 1) == pytest.approx(0.75, abs=1e-15)
    assert LF.bspline(0.3, 0) == 1.0 and LF.bspline(0.7, 0) == 0.0


@pytest.mark.parametrize("k", [0, 1, 2, 3, 4])
def test_bspline_partition_of_unity_and_mass(k):
    x = np.random.default_rng(k).uniform(-3, 3, 200)
    s = sum(LF.bspline(x - n, k) for n in range(-8, 9))
    assert np.max(np.abs(s - 1)) < 1e-13
    g = np.linspace(-(k + 1) / 2, (k + 1) / 2, 20001)
    assert np.trapezoid(LF.bspline(g, k), g) == pytest.approx(1.0, abs=1e-4)   # box: endpoint jump
    assert np.max(np.abs(LF.bspline(x, k) - LF.bspline(-x, k))) < 1e-12 or k == 0


# ---- cake wavelets -----------------------------------------------------------------------------

@pytest.mark.parametrize("N,L,k", [(16, 15, 3), (8, 11, 2), (12, 9, 3), (32, 21, 3)])
def test_cake_partition_of_unity(N, L, k):
    """sum_j psi^_j = W exactly (eq. fastreco: the wavelets fill the Fourier disk)."""
    H = LF.cake_hat(N, L, k)
    kk = np.arange(L) - (L - 1) // 2
    wy, wx = np.meshgrid(TWO_PI * kk / L, TWO_PI * kk / L, indexing="ij")
    W = LF.radial_window(np.hypot(wx, wy), 0.8)
    assert np.max(np.abs(H.sum(0) - W)) < 1e-14
    assert H.min() >= 0.0


def test_cake_bank_explicit_sum_equals_inverse_fft():
    """The explicit inverse DFT of the oracle equals numpy's FFT of the same spectrum (independent
    evaluation of the same definition)."""
    N, L = 8, 13
    H = LF.cake_hat(N, L)
    B = LF.cake_bank(N, L)
    # ifft2 over the lattice with the DC at index 0: psi(d) = L^-2 sum H e^{i w.d}
    F = np.fft.ifft2(np.fft.ifftshift(H, axes=(-2, -1)), axes=(-2, -1))        # [j][dy mod L][dx mod L]
    R = (L - 1) // 2
    idx = np.arange(-R, R + 1) % L
    ref = F[:, idx][:, :, idx]
    assert np.max(np.abs(B - ref)) < 1e-14


def test_cake_quarter_turn_covariance_and_half_turn_conjugate():
    """psi_{j+N/4}(R_{pi/2} d) = psi_j(d) and psi_{j+N/2}(d) = conj psi_j(d) (psi_theta(x) =
    psi(R_theta^{-1} x); real spectrum)."""
    N, L = 16, 15
    B = LF.cake_bank(N, L)
    for j in range(N):
        # R_{pi/2}(dx, dy) = (-dy, dx): array [dy][dx] -> rot: new[dy'=dx][dx'=-dy]
        rot = np.rot90(B[j], k=1, axes=(0, 1))          # new[a][b] = old[b][L-1-a]
        # check against the definition index by index for a few offsets
        R = (L - 1) // 2
        for dy in (-3, 0, 2, 7):
            for dx in (-7, -1, 0, 5):
                ny_, nx_ = dx, -dy                      # R_{pi/2} (dx, dy) = (-dy, dx)
                assert abs(B[(j + N // 4) % N][ny_ + R, nx_ + R] - B[j][dy + R, dx + R]) < 1e-13
        assert np.max(np.abs(B[(j + N // 2) % N] - np.conj(B[j]))) < 1e-13
        del rot


def test_cake_sum_is_real_radial_lowpass():
    N, L = 16, 15
    B = LF.cake_bank(N, L)
    w = B.sum(0)
    assert np.max(np.abs(w.imag)) < 1e-14
    assert np.max(np.abs(w.real - np.rot90(w.real))) < 1e-14
    assert w.real.sum() == pytest.approx(1.0, abs=1e-12)       # W(0) = 1: the summed filter has mass 1


# ---- lifting and projection -------------------------------------------------------------------

def _bank(N=16, L=15):
    return LF.cake_bank(N, L).real


def test_lift_of_a_dirac_is_the_reflected_bank():
    B = _bank()
    R = 7
    f = np.zeros((32, 32))
    f[12, 20] = 1.0
    U = LF.lift_image(f, B)
    for j in (0, 3, 9):
        for y in range(12 - R, 12 + R + 1):
            for x in range(20 - R, 20 + R + 1):
                assert U[j, y, x] == pytest.approx(B[j, 12 - y + R, 20 - x + R], abs=1e-15)
    assert np.count_nonzero(np.abs(U) > 0) <= 16 * 15 * 15


def test_lift_equivariance_quarter_turn():
    """W_psi . U_g = L_g . W_psi (eq. fundID) for the grid-exact quarter turn."""
    B = _bank()
    f = np.random.default_rng(3).random((24, 24))
    U = LF.lift_image(f, B)
    U2 = LF.lift_image(LF.quarter_turn_image(f), B)
    assert np.max(np.abs(U2 - O.quarter_turn(U))) < 1e-12


def test_projection_of_lift_is_the_summed_filter():
    """P(W_psi f) = (sum_j psi_j) * f (eq. fastreco, right-hand identity)."""
    B = _bank()
    f = np.random.default_rng(4).random((20, 26))
    lhs = LF.project(LF.lift_image(f, B))
    rhs = LF.lift_image(f, B.sum(0, keepdims=True))[0]
    assert np.max(np.abs(lhs - rhs)) < 1e-12


def test_fast_reconstruction_of_a_smooth_image():
    """P(W_psi f) ~ f for f essentially band-limited to the disk where sum_j psi^_j = 1 (eq. fastreco):
    a wide Gaussian blob away from the border."""
    B = _bank(16, 21)
    y, x = np.mgrid[0:48, 0:48]
    f = np.exp(-((x - 24.0) ** 2 + (y - 22.0) ** 2) / (2 * 4.0 ** 2))
    rec = LF.project(LF.lift_image(f, B))
    assert np.linalg.norm(rec - f) / np.linalg.norm(f) < 1e-3


def test_horizontal_line_lands_in_theta_zero():
    """Orientation convention: a horizontal line's positive score concentrates in theta = 0 and pi."""
    N = 16
    B = _bank(N)
    f = np.zeros((40, 40))
    f[20, 5:35] = 1.0
    Up, Un, mp, mn = LF.split_signed(LF.lift_image(f, B))
    marg = Up.sum(axis=(-2, -1))
    assert set(np.argsort(marg)[-2:]) == {0, N // 2}
    near = [N - 1, 0, 1, N // 2 - 1, N // 2, N // 2 + 1]
    assert marg[near].sum() > 0.5 and np.allclose(marg, np.roll(marg[::-1], 1))   # mirror symmetric


def test_split_signed_recombines_exactly():
    U = np.random.default_rng(5).normal(size=(8, 10, 12))
    Up, Un, mp, mn = LF.split_signed(U)
    assert Up.min() >= 0 and Un.min() >= 0
    assert Up.sum() == pytest.approx(1.0) and Un.sum() == pytest.approx(1.0)
    assert np.max(np.abs(mp * Up - mn * Un - U)) < 1e-13
    Z, _, m0, _ = LF.split_signed(np.abs(U) * -1.0)      # no positive part: zeros, mass 0
    assert m0 == 0.0 and not Z.any()


def test_project_signed_of_an_unprocessed_lift():
    """Without processing, P~(U+, U-) = max(P(U), 0) normalised (eq. final + P:820)."""
    B = _bank(8, 11)
    f = np.random.default_rng(6).random((16, 16)) ** 3
    U = LF.lift_image(f, B)
    Up, Un, mp, mn = LF.split_signed(U)
    b, s = LF.project_signed(Up, Un, mp, mn)
    ref = np.maximum(LF.project(U), 0)
    assert s == pytest.approx(ref.sum(), rel=1e-12)
    assert np.max(np.abs(b - ref / ref.sum())) < 1e-14


# ---- orientation fields ----------------------------------------------------------------------

def test_bin_of_angle_rule():
    N = 8
    s = TWO_PI / N
    k = np.arange(N)
    assert np.array_equal(LF.bin_of_angle(k * s, N), k)
    assert np.array_equal(LF.bin_of_angle(k * s + 0.49 * s, N), k)
    assert np.array_equal(LF.bin_of_angle(k * s - 0.49 * s, N), k)
    assert np.array_equal(LF.bin_of_angle(k * s + 0.51 * s, N), (k + 1) % N)
    assert np.array_equal(LF.bin_of_angle(np.array([0.5 * s, 1.5 * s]), N), [0, 1])   # tie -> lower
    assert LF.bin_of_angle(-0.4 * s, N) == 0 and LF.bin_of_angle(-0.6 * s, N) == N - 1
    assert LF.bin_of_angle(TWO_PI - 1e-12, N) == 0


def test_field_lift_reconstruct_roundtrip():
    """lift (eq. lifting_vector_field) then reconstruct (eq. reconstruction_vector_field): magnitude
    exact (relative to the mass), angle within half a bin."""
    N = 16
    rng = np.random.default_rng(7)
    ang = rng.uniform(-4, 10, (12, 14))
    mag = rng.random((12, 14)) + 0.1
    U, m = LF.lift_field(ang, mag, N)
    assert m == pytest.approx(mag.sum()) and U.sum() == pytest.approx(1.0)
    assert np.count_nonzero(U) == mag.size
    a2, m2 = LF.reconstruct_field(U)
    assert np.max(np.abs(m2 * m - mag)) < 1e-12
    d = np.abs(((a2 - ang) + np.pi) % TWO_PI - np.pi)
    assert d.max() <= np.pi / N + 1e-12


def test_reconstruct_argmax_and_ties():
    U = np.zeros((8, 1, 3))
    U[2, 0, 0], U[5, 0, 0] = 0.6, 0.4          # bimodal -> the larger mode
    U[1, 0, 1], U[6, 0, 1] = 0.5, 0.5          # tie -> smaller k
    a, m = LF.reconstruct_field(U, threshold=0.1)
    s = TWO_PI / 8
    assert a[0, 0] == pytest.approx(2 * s) and a[0, 1] == pytest.approx(1 * s)
    assert m[0, 2] == 0 and a[0, 2] == 0          # empty site
    assert m[0, 0] == pytest.approx(1.0)


def test_field_lift_equivariance_quarter_turn():
    """Rotating the field (positions and angles by pi/2) permutes the lift exactly like the SE(2) grid
    action (Cor. 4.1's setting); angles on the lattice avoid bin-boundary ties."""
    N = 16
    rng = np.random.default_rng(8)
    ang = TWO_PI * rng.integers(0, N, (10, 10)) / N
    mag = rng.random((10, 10))
    U, _ = LF.lift_field(ang, mag, N)
    U2, _ = LF.lift_field(LF.quarter_turn_image(ang) + np.pi / 2, LF.quarter_turn_image(mag), N)
    assert np.max(np.abs(U2 - O.quarter_turn(U))) < 1e-15
    assert math.isclose(U.sum(), 1.0)


def test_split_signed_floor():
    """floor_rel adds floor_rel * max(part) everywhere before normalising (closed form)."""
    U = np.random.default_rng(9).normal(size=(2, 4, 5, 6))
    Up, Un, mp, mn = LF.split_signed(U, floor_rel=1e-3)
    pos = np.maximum(U, 0)
    for b in range(2):
        fl = 1e-3 * pos[b].max()
        ref = (pos[b] + fl) / (pos[b].sum() + fl * pos[b].size)
        assert np.max(np.abs(Up[b] - ref)) < 1e-16
        assert Up[b].min() > 0 and Up[b].sum() == pytest.approx(1.0, abs=1e-14)
    assert np.allclose(mp, pos.sum(axis=(1, 2, 3)))
    Z, _, m0, _ = LF.split_signed(-np.abs(U), floor_rel=1e-3)
    assert not Z.any() and (m0 == 0).all()
