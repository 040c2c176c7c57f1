"""Helpers shared by the GPU parity tests (test-side only)."""
import numpy as np


def potential_err(g, r):
    """max |g - r| / max(1, |r|)  -- the north-star metric for (log-)potentials (reading R12)."""
    g = np.asarray(g, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    both_ninf = (g == -np.inf) & (r == -np.inf)
    d = np.where(both_ninf, 0.0, np.abs(g - r))
    return float(np.max(d / np.maximum(1.0, np.abs(np.where(both_ninf, 0.0, r)))))


def measure_err(g, r, floor_rel=1e-6):
    """max |g - r| / max(|r|, floor_rel * max|r|)  -- relative error on transported measures (R12)."""
    g = np.asarray(g, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    fl = floor_rel * np.max(np.abs(r))
    return float(np.max(np.abs(g - r) / np.maximum(np.abs(r), fl)))


def trace_err(g, r, abs_floor=1e-3):
    """Error-trace agreement |e_gpu - e_ref| / (e_ref + abs_floor); with the 1e-3 threshold of the
    tests this is |d| <= 1e-3 e_ref + 1e-6: fp32 cannot resolve an L1 marginal error below ~1e-7
    (sum of N roundoffs of mass-1 measures) while fp64 reaches 1e-17 (reading R12)."""
    g = np.asarray(g, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    return float(np.max(np.abs(g - r) / (np.abs(r) + abs_floor)))
