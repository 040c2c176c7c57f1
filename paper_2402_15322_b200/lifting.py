"""Lifting and projection: binding of the se2_cake / se2_lift_* / se2_project*
entry points of include/se2ot.h (argument marshalling only) and the paper's image-interpolation
pipeline built from them (Steps 1-4):

    1. lift f0, f1 to orientation scores U_k = W_psi f_k          (se2_lift_image, eq. lift)
    2. split into normalised measures U_k^+, U_k^-                 (se2_split_signed, eq. tildeW-v1)
    3. SE(2) barycenters Phi_t(U_0^+-, U_1^+-), same OT settings   (se2_barycenter, App. A)
    4. b_t = max(m^+ P(U_t^+) - m^- P(U_t^-), 0) / sum             (se2_project_signed, eq. final + P:820)

Orientation fields: se2_lift_field / se2_reconstruct_field.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib as L
from ._lib import check
from .api import Kernel, _ptr, _stream, se2_barycenter


def _check_dev(t: torch.Tensor, name: str, device: int, numel: Optional[int] = None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (the lifting path has no CPU fallback)")
    if t.dtype != torch.float32 or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous float32 tensor")
    if t.device.index != device:
        raise ValueError(f"{name} is on {t.device}, the lifting context on cuda:{device}")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name} must have {numel} elements, has {t.numel()}")


class Cake:
    """Lifting context: the cake-wavelet bank Re psi_j (reading R15) on the device + reduction scratch."""

    def __init__(self, ntheta: int, size: int, spline_degree: int = 3, radial_cut: float = 0.8, device: int = 0):
        lib = L.load()
        h = ctypes.c_void_p()
        check(lib.se2_cake_build(int(ntheta), int(size), int(spline_degree), float(radial_cut), int(device),
                                 ctypes.byref(h)))
        self._h = h
        self.ntheta, self.size, self.device = int(ntheta), int(size), int(device)
        self.spline_degree, self.radial_cut = int(spline_degree), float(radial_cut)

    @property
    def handle(self):
        if self._h is None:
            raise RuntimeError("lifting context closed")
        return self._h

    def table(self) -> np.ndarray:
        """The fp32 bank Re psi_j(dy, dx) as [ntheta][size][size] (host copy)."""
        out = np.empty((self.ntheta, self.size, self.size), dtype=np.float32)
        check(L.load().se2_cake_get(self.handle, out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), None, None))
        return out

    def close(self):
        if getattr(self, "_h", None) is not None:
            L.load().se2_cake_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def se2_lift_image(c: Cake, f: torch.Tensor, U: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Orientation scores U[b][j][y][x] of images f[b][y][x] (eq. lift)."""
    ny, nx = f.shape[-2:]
    batch = f.numel() // (nx * ny)
    _check_dev(f, "f", c.device)
    if U is None:
        U = torch.empty((batch, c.ntheta, ny, nx), device=f.device, dtype=torch.float32)
    _check_dev(U, "U", c.device, batch * c.ntheta * nx * ny)
    check(L.load().se2_lift_image(c.handle, _ptr(f), _ptr(U), nx, ny, batch, _stream(f.device)))
    return U


def se2_split_signed(c: Cake, U: torch.Tensor, floor_rel: float = 0.0) -> Tuple[torch.Tensor, torch.Tensor, np.ndarray]:
    """(U+, U-, masses[batch][2]) with U+- normalised positive / negative parts (eq. tildeW-v1);
    floor_rel adds floor_rel * max(part) to every site before normalising (R17)."""
    _check_dev(U, "U", c.device)
    n = c.ntheta * U.shape[-1] * U.shape[-2]
    batch = U.numel() // n
    Up, Un = torch.empty_like(U), torch.empty_like(U)
    m = np.zeros((batch, 2), dtype=np.float64)
    check(L.load().se2_split_signed(c.handle, _ptr(U), _ptr(Up), _ptr(Un), n, batch, float(floor_rel),
                                    m.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _stream(U.device)))
    return Up, Un, m


def se2_project(c: Cake, U: torch.Tensor) -> torch.Tensor:
    """P(U) = sum_j U(., theta_j) (eq. proj)."""
    _check_dev(U, "U", c.device)
    ny, nx = U.shape[-2:]
    batch = U.numel() // (c.ntheta * nx * ny)
    img = torch.empty((batch, ny, nx), device=U.device, dtype=torch.float32)
    check(L.load().se2_project(c.handle, _ptr(U), _ptr(img), nx, ny, batch, _stream(U.device)))
    return img


def se2_project_signed(c: Cake, Up: torch.Tensor, Un: torch.Tensor, masses) -> Tuple[torch.Tensor, np.ndarray]:
    """(b, mass): b = max(m+ P(U+) - m- P(U-), 0) / sum (eq. final + P:820)."""
    _check_dev(Up, "Up", c.device)
    _check_dev(Un, "Un", c.device, Up.numel())
    ny, nx = Up.shape[-2:]
    batch = Up.numel() // (c.ntheta * nx * ny)
    m = np.ascontiguousarray(np.asarray(masses, dtype=np.float64).reshape(batch, 2))
    img = torch.empty((batch, ny, nx), device=Up.device, dtype=torch.float32)
    tot = np.zeros(batch, dtype=np.float64)
    check(L.load().se2_project_signed(c.handle, _ptr(Up), _ptr(Un), m.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                      _ptr(img), nx, ny, batch, tot.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                      _stream(Up.device)))
    return img, tot


def se2_lift_field(c: Cake, angle: torch.Tensor, mag: torch.Tensor) -> Tuple[torch.Tensor, np.ndarray]:
    """(U, mass): the 0-th order B-spline lift of an orientation field (eq. lifting_vector_field; R16)."""
    _check_dev(angle, "angle", c.device)
    _check_dev(mag, "mag", c.device, angle.numel())
    ny, nx = angle.shape[-2:]
    batch = angle.numel() // (nx * ny)
    U = torch.empty((batch, c.ntheta, ny, nx), device=angle.device, dtype=torch.float32)
    tot = np.zeros(batch, dtype=np.float64)
    check(L.load().se2_lift_field(c.handle, _ptr(angle), _ptr(mag), _ptr(U), nx, ny, batch,
                                  tot.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _stream(angle.device)))
    return U, tot


def se2_reconstruct_field(c: Cake, U: torch.Tensor, threshold: float = 0.0) -> Tuple[torch.Tensor, torch.Tensor]:
    """(angle, mag) = (theta of the first argmax, sum over theta) (eq. reconstruction_vector_field)."""
    _check_dev(U, "U", c.device)
    ny, nx = U.shape[-2:]
    batch = U.numel() // (c.ntheta * nx * ny)
    ang = torch.empty((batch, ny, nx), device=U.device, dtype=torch.float32)
    mag = torch.empty_like(ang)
    check(L.load().se2_reconstruct_field(c.handle, _ptr(U), _ptr(ang), _ptr(mag), nx, ny, batch, float(threshold),
                                         _stream(U.device)))
    return ang, mag


def se2_exp(x: torch.Tensor) -> torch.Tensor:
    """exp(x) elementwise in the library (log-domain barycenter -> measure)."""
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.float32 or not x.is_contiguous():
        raise TypeError("x must be a contiguous float32 CUDA tensor")
    y = torch.empty_like(x)
    check(L.load().se2_exp(_ptr(x), _ptr(y), x.numel(), _stream(x.device)))
    return y


def se2_log(x: torch.Tensor) -> torch.Tensor:
    """log(x) elementwise in the library (measures -> log-domain targets; log 0 = -inf)."""
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.float32 or not x.is_contiguous():
        raise TypeError("x must be a contiguous float32 CUDA tensor")
    y = torch.empty_like(x)
    check(L.load().se2_log(_ptr(x), _ptr(y), x.numel(), _stream(x.device)))
    return y


def interpolate_images(k: Kernel, c: Cake, f0: torch.Tensor, f1: torch.Tensor, ts: Sequence[float], iters: int,
                       log_domain: bool = True, floor_rel: float = 1e-6) -> Tuple[torch.Tensor, np.ndarray]:
    """The paper's SE(2) image interpolation b_t (Steps 1-4) for every t in ts: lift both
    images, split each score into normalised +/- measures, take the SE(2) Wasserstein barycenters of the
    + parts and of the - parts with the same OT settings and weights Lambda_t = (1 - t, t) (App. A; here
    t weights the SECOND image so that b_0 ~ f0), and recombine with the linearly interpolated masses.
    floor_rel: the configs' input floor on the +/- measures (R17; 0 leaves empty windows, on which the
    log-domain App. A iteration is undefined).
    Returns (b [len(ts)][ny][nx], masses [len(ts)])."""
    if k.ntheta != c.ntheta:
        raise ValueError("kernel and lifting context must share ntheta")
    ny, nx = f0.shape[-2:]
    if (nx, ny) != (k.nx, k.ny):
        raise ValueError("images must match the kernel grid")
    U = se2_lift_image(c, torch.stack([f0.reshape(ny, nx), f1.reshape(ny, nx)]).contiguous())
    Up, Un, m = se2_split_signed(c, U, floor_rel)
    ts = [float(t) for t in ts]
    lam = np.array([[1.0 - t, t] for t in ts])
    barys = []
    for part in (Up, Un):
        b, _ = se2_barycenter(k, part, lam, iters, log_domain)
        if log_domain:
            b = se2_exp(b)
        barys.append(b.reshape(len(ts), c.ntheta, ny, nx).contiguous())
    m = np.ascontiguousarray(m, dtype=np.float64)
    tsa = np.ascontiguousarray(ts, dtype=np.float64)
    mt = np.empty((len(ts), 2), dtype=np.float64)
    check(L.load().se2_interp_masses(m.ctypes.data, tsa.ctypes.data, len(ts), mt.ctypes.data))
    return se2_project_signed(c, barys[0], barys[1], mt)
