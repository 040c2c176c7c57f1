"""Seeded synthetic inputs for the five BASELINE.json configs (c0..c4).

This module is shared by the oracle (tests/) and the CUDA path (bench.py,
smoke, GPU tests).  It holds NO arithmetic of the method: no group law, no
distance, no kernel, no scaling step -- only the workload description and the
random measures the paper's experiments are stand-ins for (DESIGN.md
"Input recipe").

Paper workloads (PAPER.md lines):
  * P:751   64x64x16 grid on [0,1]^2 x [0,2pi)  -> spatial window [0,1]^2
  * P:773   MNIST 28x28, 16 orientations        -> c1 stroke "digits" (synthetic
            stand-in; the dataset is not in this container and is never
            reproduced)
  * P:862   orientation fields                   -> c2 random Fourier angle field
  * P:882   "dominant line structure amid randomly located smaller line
            elements"                            -> c4 strokes
Shapes / eps / weights / supports / iteration counts come from
BASELINE.json "configs".

Arrays are float32, layout [ntheta][ny][nx] (x fastest), sum 1 (computed in
fp64, then rounded to fp32 -- the fp32 values are THE input both sides use).
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Tuple

import numpy as np

__all__ = ["Config", "CONFIGS", "get_config", "stroke_measure", "orientation_field_measure",
           "config_inputs", "random_positive_field", "dirichlet_weights"]


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    nx: int
    ny: int
    ntheta: int
    eps: float
    w: Tuple[float, float, float]
    support: int            # S: spatial box is S x S, R = (S-1)//2; theta support = all bins
    problem: str            # "sinkhorn" | "barycenter" | "jko"
    iters: int              # scaling iterations per solve
    n_inputs: int
    ts: Tuple[float, ...] = ()          # barycentric interpolation weights (c1) t -> (t, 1-t)
    jko_steps: int = 0
    tau: float = 0.0
    log_domain: bool = False            # reading L12: decided from the oracle probes
    cell: float = 0.0                   # cell size in [0,1]^2 units; 0 -> 1/nx by 1/ny (reading R1).  A
                                        # window cut from a larger grid keeps that grid's cell.

    @property
    def R(self) -> int:
        return (self.support - 1) // 2

    @property
    def N(self) -> int:
        return self.nx * self.ny * self.ntheta

    @property
    def shape(self) -> Tuple[int, int, int]:
        return (self.ntheta, self.ny, self.nx)


CONFIGS: List[Config] = [
    # BASELINE.json configs[0]
    Config("c0", 16, 16, 8, 0.05, (1.0, 3.0, 1.0), 7, "sinkhorn", 100, 2, log_domain=True),
    # configs[1]
    Config("c1", 28, 28, 16, 0.02, (1.0, 3.0, 1.0), 11, "barycenter", 200, 2,
           ts=(0.0, 0.25, 0.5, 0.75, 1.0), log_domain=True),
    # configs[2]
    Config("c2", 64, 64, 32, 0.01, (1.0, 4.0, 2.0), 15, "barycenter", 300, 2, ts=(0.5,),
           log_domain=True),
    # configs[3]
    Config("c3", 128, 128, 32, 0.005, (1.0, 3.0, 1.0), 21, "barycenter", 500, 4, log_domain=True),
    # configs[4]
    Config("c4", 256, 256, 64, 0.003, (1.0, 3.0, 1.0), 31, "jko", 200, 1, jko_steps=20,
           tau=1e-3, log_domain=False),
]


def get_config(name: str) -> Config:
    for c in CONFIGS:
        if c.name == name:
            return c
    raise KeyError(name)


def _bezier(p: np.ndarray, t: np.ndarray):
    """Cubic Bezier points and derivatives (control points p: 4x2, t: n)."""
    t = t[:, None]
    u = 1.0 - t
    pts = (u ** 3) * p[0] + 3 * (u ** 2) * t * p[1] + 3 * u * (t ** 2) * p[2] + (t ** 3) * p[3]
    der = 3 * (u ** 2) * (p[1] - p[0]) + 6 * u * t * (p[2] - p[1]) + 3 * (t ** 2) * (p[3] - p[2])
    return pts, der


def stroke_measure(nx: int, ny: int, ntheta: int, n_strokes: int, seed: int,
                   sigma_px: float = 1.0, kappa: float = 4.0, floor: float = 1e-6) -> np.ndarray:
    """Rasterised random cubic-Bezier strokes (BASELINE configs[0]):

    each curve sample c with tangent angle phi adds
        exp(-|x - c|^2 / (2 sigma^2)) * exp(kappa (cos(theta_k - phi) - 1))
    at pixel centres x = (i + 1/2, j + 1/2) px; then s <- s / max(s) + floor;
    normalised to sum 1.  theta_k = 2 pi k / ntheta.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    xs = np.arange(nx) + 0.5
    ys = np.arange(ny) + 0.5
    th = 2.0 * np.pi * np.arange(ntheta) / ntheta
    s = np.zeros((ntheta, ny, nx), dtype=np.float64)
    lo = np.array([0.15 * nx, 0.15 * ny])
    hi = np.array([0.85 * nx, 0.85 * ny])
    for _ in range(n_strokes):
        p = lo + (hi - lo) * rng.random((4, 2))
        tt = np.linspace(0.0, 1.0, 65)
        pts, _ = _bezier(p, tt)
        length = float(np.sum(np.linalg.norm(np.diff(pts, axis=0), axis=1)))
        n = max(8, int(math.ceil(4.0 * length)))
        t = (np.arange(n) + 0.5) / n
        pts, der = _bezier(p, t)
        phi = np.mod(np.arctan2(der[:, 1], der[:, 0]), 2.0 * np.pi)
        h = int(math.ceil(8.0 * sigma_px))   # blob window: exp(-32) ~ 1e-14 relative at the edge
        for (cx, cy), ph in zip(pts, phi):
            x0, x1 = max(0, int(cx) - h), min(nx, int(cx) + h + 1)
            y0, y1 = max(0, int(cy) - h), min(ny, int(cy) + h + 1)
            gx = np.exp(-((xs[x0:x1] - cx) ** 2) / (2 * sigma_px ** 2))
            gy = np.exp(-((ys[y0:y1] - cy) ** 2) / (2 * sigma_px ** 2))
            vm = np.exp(kappa * (np.cos(th - ph) - 1.0))
            s[:, y0:y1, x0:x1] += vm[:, None, None] * gy[None, :, None] * gx[None, None, :]
    s = s / s.max() + floor
    s = s / s.sum()
    return s.astype(np.float32)


def orientation_field_measure(nx: int, ny: int, ntheta: int, seed: int, n_modes: int = 8,
                              kappa: float = 8.0) -> np.ndarray:
    """Planar orientation field (BASELINE configs[2]): theta0(x) = sum_j A_j cos(2 pi k_j.x / n + phi_j),
    k_j in {-3..3}^2 \\ 0, A_j ~ U(0,1) rad, phi_j ~ U(0, 2pi); mass 1/(nx ny) per pixel times a
    von Mises (kappa) in theta centred on theta0(x), normalised over theta per pixel."""
    rng = np.random.Generator(np.random.PCG64(seed))
    ks = [(a, b) for a in range(-3, 4) for b in range(-3, 4) if (a, b) != (0, 0)]
    idx = rng.choice(len(ks), size=n_modes, replace=False)
    amp = rng.random(n_modes)
    ph = 2.0 * np.pi * rng.random(n_modes)
    X, Y = np.meshgrid(np.arange(nx) + 0.5, np.arange(ny) + 0.5, indexing="xy")
    th0 = np.zeros((ny, nx))
    for j in range(n_modes):
        kx, ky = ks[idx[j]]
        th0 += amp[j] * np.cos(2.0 * np.pi * (kx * X / nx + ky * Y / ny) + ph[j])
    th = 2.0 * np.pi * np.arange(ntheta) / ntheta
    vm = np.exp(kappa * (np.cos(th[:, None, None] - th0[None]) - 1.0))
    vm = vm / vm.sum(axis=0, keepdims=True)
    m = vm / (nx * ny)
    m = m / m.sum()
    return m.astype(np.float32)


def dirichlet_weights(n: int, seed: int) -> np.ndarray:
    """Random barycentric weights on the simplex (c3: Dirichlet(1,...,1)), fp64."""
    rng = np.random.Generator(np.random.PCG64(seed))
    lam = rng.dirichlet(np.ones(n))
    lam = lam / lam.sum()
    return lam


def random_positive_field(shape, seed: int, lo: float = 0.1, hi: float = 1.0,
                          log_range: Optional[float] = None) -> np.ndarray:
    """Generic seeded positive fp32 field for operator-level parity tests.
    If log_range is given, returns values exp(U(-log_range/2, log_range/2)) (wide dynamic range)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if log_range is not None:
        return np.exp(rng.uniform(-log_range / 2, log_range / 2, size=shape)).astype(np.float32)
    return rng.uniform(lo, hi, size=shape).astype(np.float32)


def config_inputs(cfg: Config):
    """The seeded inputs of a config (seed = 1000*cfg_index + input_index).

    returns dict with "mus": list of fp32 [ntheta][ny][nx] arrays, and per-problem extras:
      sinkhorn  : mus = [mu, nu]
      barycenter: mus = [mu_1..mu_n], "lambdas": list of fp64 weight vectors (one per solve)
      jko       : mus = [mu_0], "tau", "V_center_px"
    """
    ci = int(cfg.name[1:])
    base = 1000 * ci
    out = {}
    if cfg.name == "c0":
        out["mus"] = [stroke_measure(cfg.nx, cfg.ny, cfg.ntheta, 2, base + i) for i in range(2)]
    elif cfg.name == "c1":
        out["mus"] = [stroke_measure(cfg.nx, cfg.ny, cfg.ntheta, 3, base + i) for i in range(2)]
        out["lambdas"] = [np.array([t, 1.0 - t]) for t in cfg.ts]
    elif cfg.name == "c2":
        out["mus"] = [orientation_field_measure(cfg.nx, cfg.ny, cfg.ntheta, base + i) for i in range(2)]
        out["lambdas"] = [np.array([0.5, 0.5])]
    elif cfg.name == "c3":
        out["mus"] = [stroke_measure(cfg.nx, cfg.ny, cfg.ntheta, 6, base + i, sigma_px=1.5)
                      for i in range(4)]
        out["lambdas"] = [dirichlet_weights(4, base + 99)]
    elif cfg.name == "c4":
        out["mus"] = [stroke_measure(cfg.nx, cfg.ny, cfg.ntheta, 10, base)]
        out["tau"] = cfg.tau
        out["V_center_px"] = (cfg.nx / 2.0, cfg.ny / 2.0)
    else:
        raise KeyError(cfg.name)
    return out


# ------------------------------------------------------------------------------------------------
# Parity cases (data only): the BASELINE configs at full size (whole runs where the oracle finishes,
# prefixes where it cannot) and reduced-size analogues with ragged tiles that run to the full
# iteration count.  tests/golden/make_golden.py computes the expected values with oracle/ only.
# ------------------------------------------------------------------------------------------------

@dataclasses.dataclass(frozen=True)
class ParityCase:
    name: str
    base: str                  # BASELINE config it derives from
    nx: int
    ny: int
    ntheta: int
    R: int
    iters: int
    jko_steps: int = 0
    full_fields: bool = True   # store whole fields (else sampled entries)
    energy: str = "entropy_potential"   # JKO energy: BASELINE configs[4], or the paper's porous medium
    m: float = 5.0                      # porous-medium exponent
    w: Optional[Tuple[float, float, float]] = None   # metric override
    cell: float = 0.0                   # cell size override (0: 1/nx by 1/ny)


PARITY_CASES: List[ParityCase] = [
    ParityCase("c0", "c0", 16, 16, 8, 3, 100),
    ParityCase("c1", "c1", 28, 28, 16, 5, 200),
    ParityCase("c2p", "c2", 64, 64, 32, 7, 10, full_fields=False),
    ParityCase("c2m", "c2", 40, 36, 32, 7, 300),
    ParityCase("c2f", "c2", 64, 64, 32, 7, 300, full_fields=False),   # the whole c2 run at full size
    ParityCase("c3p", "c3", 128, 128, 32, 10, 2, full_fields=False),
    ParityCase("c3q", "c3", 128, 128, 32, 10, 100, full_fields=False),  # c3 at full size, first 100 iterations
    ParityCase("c3m", "c3", 44, 40, 32, 10, 500),                       # ragged c3 analogue, the full 500
    ParityCase("c4p", "c4", 256, 256, 64, 15, 2, jko_steps=1, full_fields=False),
    ParityCase("c4q", "c4", 256, 256, 64, 15, 20, jko_steps=1, full_fields=False),  # full c4 grid, 20 inner iterations
    ParityCase("c4m", "c4", 72, 60, 16, 4, 200, jko_steps=3),
    # the headline geometry on a reduced, ragged window: a 100 x 92 window of the c4 lattice (cells of
    # 1/256, so R = 15, ntheta = 64, eps = 0.003, w = (1,3,1) give exactly the c4 kernel), 3 JKO steps x
    # 200 inner iterations; V centred on the window
    ParityCase("c4w", "c4", 100, 92, 64, 15, 200, jko_steps=3, full_fields=False, cell=1.0 / 256.0),
    # the full c4 grid, JKO step 0: all 200 inner iterations (sampled)
    ParityCase("c4f", "c4", 256, 256, 64, 15, 200, jko_steps=1, full_fields=False),
    # NEXT #1: the paper's own gradient flow -- porous medium m = 5, w = (1, sqrt 10, sqrt 2)
    ParityCase("c5m", "c4", 64, 56, 16, 4, 100, jko_steps=2, energy="porous", m=5.0,
               w=(1.0, math.sqrt(10.0), math.sqrt(2.0))),
]


def get_parity_case(name: str) -> ParityCase:
    for c in PARITY_CASES:
        if c.name == name:
            return c
    raise KeyError(name)


def parity_inputs(pc: ParityCase):
    """Config of the case (a Config with the case's grid / radius / iteration counts) and its inputs,
    generated exactly like the base config's (same seeds, same recipe) on the case's grid."""
    base = get_config(pc.base)
    cfg = dataclasses.replace(base, name=base.name, nx=pc.nx, ny=pc.ny, ntheta=pc.ntheta,
                              support=2 * pc.R + 1, iters=pc.iters,
                              jko_steps=pc.jko_steps if pc.jko_steps else base.jko_steps,
                              w=pc.w if pc.w is not None else base.w, cell=pc.cell)
    return cfg, config_inputs(cfg)


def sample_indices(N: int, count: int, seed: int) -> np.ndarray:
    """Seeded sample of flat field indices (always includes the first and last entries)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    idx = np.unique(np.concatenate([[0, N - 1], rng.choice(N, size=min(count, N), replace=False)]))
    return idx.astype(np.int64)
