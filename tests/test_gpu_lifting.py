"""GPU parity of the lifting / projection pipeline against the fp64 oracle
(oracle/se2_lift.py), through the C ABI (paper_2402_15322_b200.lifting).

Tolerances: tables and scores are fp32 sums of fp32-rounded filter values, compared with
|d| <= 1e-5 * (sum_d |psi_j(d)|) * max|f| (the fp32 rounding bound of the correlation); measures
elementwise relative to max with the R12 floor; integer decisions (theta bins, argmax) bit-exact,
taken in the same precision on both sides (fp64 bins from the same fp32 angles; argmax on the same
fp32 values)."""
import numpy as np
import pytest
import torch

import oracle as O
from oracle import se2_lift as LF
from gpu_util import measure_err, potential_err

pytestmark = pytest.mark.gpu


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def _host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy().astype(np.float64)


def _smooth_image(ny, nx, seed):
    """Seeded synthetic 'digit-like' image: a few Gaussian strokes (stands in for the paper's MNIST /
    QuickDraw images, P:830 -- never reproduced)."""
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:ny, 0:nx].astype(np.float64)
    f = np.zeros((ny, nx))
    for _ in range(3):
        p0 = rng.uniform([0.2 * nx, 0.2 * ny], [0.8 * nx, 0.8 * ny])
        p1 = rng.uniform([0.2 * nx, 0.2 * ny], [0.8 * nx, 0.8 * ny])
        for s in np.linspace(0, 1, 4 * max(nx, ny)):
            c = (1 - s) * p0 + s * p1
            f += np.exp(-((x - c[0]) ** 2 + (y - c[1]) ** 2) / (2 * 1.0 ** 2))
    return f / f.max()


@pytest.mark.parametrize("N,L,k,cut", [(16, 15, 3, 0.8), (8, 11, 2, 0.7), (12, 9, 0, 0.9), (32, 21, 3, 0.8)])
def test_cake_table_parity(N, L, k, cut, cuda_device):
    from paper_2402_15322_b200 import Cake
    c = Cake(N, L, k, cut)
    got = c.table().astype(np.float64)
    ref = LF.cake_bank(N, L, k, cut).real
    assert np.max(np.abs(got - ref)) <= 2e-7 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("ny,nx,batch,N,L", [(28, 28, 2, 16, 15), (37, 29, 3, 8, 11), (64, 48, 1, 32, 21),
                                             (5, 7, 1, 4, 9), (41, 35, 2, 6, 31), (20, 18, 1, 8, 33)])
def test_lift_image_parity(ny, nx, batch, N, L, cuda_device):
    from paper_2402_15322_b200 import Cake, se2_lift_image
    c = Cake(N, L)
    B = LF.cake_bank(N, L).real
    f = np.stack([_smooth_image(ny, nx, s) for s in range(batch)]).astype(np.float32).astype(np.float64)
    U = _host(se2_lift_image(c, _dev(f)))
    ref = LF.lift_image(f, B)
    bound = 1e-5 * np.abs(B).sum(axis=(1, 2)).max() * np.abs(f).max()
    assert np.max(np.abs(U - ref)) <= bound


def test_lift_image_full_size_sampled(cuda_device):
    """The largest grid of the configs (256 x 256, 64 orientations), sampled outputs against the oracle's
    per-output correlation."""
    from paper_2402_15322_b200 import Cake, se2_lift_image
    N, L = 64, 21
    c = Cake(N, L)
    B = LF.cake_bank(N, L).real
    f = _smooth_image(256, 256, 11).astype(np.float32).astype(np.float64)
    U = _host(se2_lift_image(c, _dev(f)))[0]
    R = (L - 1) // 2
    fp = np.zeros((256 + 2 * R, 256 + 2 * R))
    fp[R:-R, R:-R] = f
    rng = np.random.default_rng(1)
    bound = 1e-5 * np.abs(B).sum(axis=(1, 2)).max()
    for _ in range(3000):
        j, y, x = rng.integers(N), rng.integers(256), rng.integers(256)
        ref = np.sum(B[j] * fp[y:y + L, x:x + L])
        assert abs(U[j, y, x] - ref) <= bound


def test_split_project_parity(cuda_device):
    from paper_2402_15322_b200 import Cake, se2_lift_image, se2_project, se2_project_signed, se2_split_signed
    N, L = 16, 15
    c = Cake(N, L)
    f = np.stack([_smooth_image(30, 26, s) for s in (3, 4)])
    Ud = se2_lift_image(c, _dev(f))
    U = _host(Ud)                                  # both sides split the same fp32 values
    Up, Un, m = se2_split_signed(c, Ud)
    rp, rn, mp, mn = LF.split_signed(U)
    assert np.allclose(m[:, 0], mp, rtol=1e-12, atol=0) and np.allclose(m[:, 1], mn, rtol=1e-12, atol=0)
    assert measure_err(_host(Up), rp) <= 1e-6 and measure_err(_host(Un), rn) <= 1e-6
    assert np.array_equal(_host(Up) > 0, rp > 0) and np.array_equal(_host(Un) > 0, rn > 0)
    P = _host(se2_project(c, Ud))
    assert np.max(np.abs(P - LF.project(U))) <= 1e-6 * np.abs(U).sum(axis=1).max()
    img, tot = se2_project_signed(c, Up, Un, m)
    rb, rs = LF.project_signed(_host(Up), _host(Un), m[:, 0], m[:, 1])
    assert np.allclose(tot, rs, rtol=1e-6)
    assert measure_err(_host(img), rb) <= 1e-5
    assert abs(_host(img).sum(axis=(1, 2)) - 1).max() < 1e-5


def test_split_floor_parity(cuda_device):
    from paper_2402_15322_b200 import Cake, se2_split_signed
    c = Cake(8, 9)
    U = np.random.default_rng(12).normal(size=(3, 8, 11, 13)).astype(np.float32)
    Up, Un, m = se2_split_signed(c, _dev(U), floor_rel=1e-3)
    rp, rn, mp, mn = LF.split_signed(U.astype(np.float64), floor_rel=1e-3)
    assert measure_err(_host(Up), rp) <= 1e-6 and measure_err(_host(Un), rn) <= 1e-6
    assert np.allclose(m[:, 0], mp, rtol=1e-12) and np.allclose(m[:, 1], mn, rtol=1e-12)


def test_split_zero_mass_part(cuda_device):
    from paper_2402_15322_b200 import Cake, se2_split_signed
    c = Cake(8, 9)
    U = -np.abs(np.random.default_rng(2).normal(size=(1, 8, 6, 5))) - 0.1
    Up, Un, m = se2_split_signed(c, _dev(U))
    assert m[0, 0] == 0.0 and not _host(Up).any()
    assert abs(_host(Un).sum() - 1) < 1e-5


@pytest.mark.parametrize("N", [4, 8, 16, 64])
def test_orientation_field_parity(N, cuda_device):
    """Bins bit-exact (fp64 decision from the same fp32 angles), including exact bin boundaries,
    values to fp32 rounding; reconstruction argmax / magnitude."""
    from paper_2402_15322_b200 import Cake, se2_lift_field, se2_reconstruct_field
    c = Cake(N, 9, 3 if N >= 4 else 0)
    rng = np.random.default_rng(N)
    ny, nx = 19, 23
    ang = rng.uniform(-7, 13, (2, ny, nx)).astype(np.float32)
    s = 2 * np.pi / N
    nb = min(N, nx)
    ang[0, 0, :nb] = (np.arange(nb) * s + 0.5 * s).astype(np.float32)      # boundaries (as rounded to fp32)
    ang[0, 1, :nb] = (np.arange(nb) * s).astype(np.float32)                # centres
    mag = (rng.random((2, ny, nx)) + 0.05).astype(np.float32)
    mag[1, 3, 4] = 0.0
    U, tot = se2_lift_field(c, _dev(ang), _dev(mag))
    ref, rs = LF.lift_field(ang.astype(np.float64), mag.astype(np.float64), N)
    Ug = _host(U)
    assert np.array_equal(Ug > 0, ref > 0)                                   # same bins
    assert np.allclose(tot, rs, rtol=1e-12)
    assert measure_err(Ug, ref) <= 1e-6
    a2, m2 = se2_reconstruct_field(c, U, threshold=0.0)
    ra, rm = LF.reconstruct_field(Ug, 0.0)                                    # same fp32 values
    assert np.array_equal(_host(a2) == 0, ra == 0)
    assert np.max(np.abs(_host(a2) - ra)) < 1e-6
    assert np.max(np.abs(_host(m2) - rm)) <= 1e-6 * rm.max()


def test_reconstruct_threshold_and_ties(cuda_device):
    from paper_2402_15322_b200 import Cake, se2_reconstruct_field
    c = Cake(8, 5, 1)
    U = np.zeros((1, 8, 1, 3), dtype=np.float32)
    U[0, 2, 0, 0], U[0, 5, 0, 0] = 0.6, 0.4
    U[0, 1, 0, 1], U[0, 6, 0, 1] = 0.05, 0.05
    a, m = se2_reconstruct_field(c, _dev(U), threshold=0.2)
    a, m = _host(a)[0, 0], _host(m)[0, 0]
    assert a[0] == pytest.approx(2 * 2 * np.pi / 8, abs=1e-6) and m[0] == pytest.approx(1.0, abs=1e-6)
    assert a[1] == 0 and m[1] == 0 and a[2] == 0 and m[2] == 0
    a, m = se2_reconstruct_field(c, _dev(U), threshold=0.0)
    assert _host(a)[0, 0, 1] == pytest.approx(2 * np.pi / 8, abs=1e-6)       # tie -> smaller k


def test_interpolate_images_pipeline(cuda_device):
    """Steps 1-4 of P:802-820 end to end on a small grid against the oracle pipeline (oracle lifts,
    oracle log-domain barycenters, oracle recombination), same settings."""
    from paper_2402_15322_b200 import Cake, Kernel, interpolate_images
    ny = nx = 20
    N, L, R, eps, w, iters = 8, 9, 3, 0.05, (1.0, 3.0, 1.0), 30
    ts = [0.0, 0.5, 1.0]
    f0, f1 = _smooth_image(ny, nx, 21), _smooth_image(ny, nx, 22)
    f0, f1 = (f.astype(np.float32).astype(np.float64) for f in (f0, f1))
    c = Cake(N, L)
    k = Kernel(nx, ny, N, eps, w, R, max_batch=2 * len(ts))
    b, mass = interpolate_images(k, c, _dev(f0), _dev(f1), ts, iters)
    # oracle pipeline
    B = LF.cake_bank(N, L).real
    U = LF.lift_image(np.stack([f0, f1]), B)
    Up, Un, mp, mn = LF.split_signed(U, floor_rel=1e-6)
    g = O.Grid(nx, ny, N)
    T, Lt = O.kernel_table(g, R, eps, w), O.log_kernel_table(g, R, eps, w)
    ref = []
    for t in ts:
        lam = np.array([1 - t, t])
        bp = O.barycenter(T, Lt, [Up[0], Up[1]], lam, iters, log_domain=True, trace=False)["bary"]
        bn = O.barycenter(T, Lt, [Un[0], Un[1]], lam, iters, log_domain=True, trace=False)["bary"]
        mpt, mnt = (1 - t) * mp[0] + t * mp[1], (1 - t) * mn[0] + t * mn[1]
        rb, _ = LF.project_signed(bp, bn, mpt, mnt)
        ref.append(rb)
    ref = np.stack(ref)
    got = _host(b)
    assert np.isfinite(got).all() and got.min() >= 0
    assert np.abs(got.sum(axis=(1, 2)) - 1).max() < 1e-5
    assert measure_err(got, ref) <= 1e-4
