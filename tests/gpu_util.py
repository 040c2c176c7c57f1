"""Helpers shared by the GPU parity tests (test-side only).

Metrics (SURVEY.md ledger L18, reading R12):
  potentials (alpha = log a, beta, log v_i, log w_i): ELEMENTWISE max |g - r| / max(1, |r|), after the
      gauge fix below where a gauge exists;
  measures (marginals, barycenters, mu_{k+1}): max |g - r| / max(|r|, 1e-6 max |r|);
  error traces: |e_g - e_r| <= 1e-4 e_r + 1e-5.
"""
import numpy as np


def _pair(g, r):
    g = np.asarray(g, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    both_ninf = (g == -np.inf) & (r == -np.inf)
    return np.where(both_ninf, 0.0, g), np.where(both_ninf, 0.0, r)


def potential_err(g, r):
    """max_x |g(x) - r(x)| / max(1, |r(x)|)  -- elementwise relative error of a (log-)potential (L18).
    Entries that are -inf on both sides (zero mass) agree; -inf on one side only is an infinite error."""
    g, r = _pair(g, r)
    return float(np.max(np.abs(g - r) / np.maximum(1.0, np.abs(r))))


def potential_err_sup(g, r):
    """max |g - r| / max(1, max |r|)  -- sup-norm relative error (reported for information only)."""
    g, r = _pair(g, r)
    return float(np.max(np.abs(g - r)) / max(1.0, float(np.max(np.abs(r)))))


def gauge_mean(x):
    """Mean of the finite entries (the additive gauge component of a log-potential)."""
    x = np.asarray(x, dtype=np.float64)
    f = np.isfinite(x)
    return float(x[f].mean()) if f.any() else 0.0


def gauge_fixed_pair_err(ga, gb, ra, rb):
    """Sinkhorn potentials (alpha, beta) carry the gauge (alpha + c, beta - c) (the plan a K b is
    invariant).  Each side is fixed by its own mean of alpha: compare alpha - m and beta + m
    elementwise, and the gauge components m themselves (relative to max(1, |m_ref|))."""
    mg, mr = gauge_mean(ga), gauge_mean(ra)
    ga = np.asarray(ga, dtype=np.float64) - mg
    ra = np.asarray(ra, dtype=np.float64) - mr
    gb = np.asarray(gb, dtype=np.float64) + mg
    rb = np.asarray(rb, dtype=np.float64) + mr
    return dict(alpha=potential_err(ga, ra), beta=potential_err(gb, rb),
                gauge=abs(mg - mr) / max(1.0, abs(mr)))


def bary_potential_errs(glv, glw, rlv, rlw, lambdas):
    """App. A potentials log v_i, log w_i of one solve ([n][...] each).  (v_i, w_i) -> (c_i v_i, w_i / c_i)
    leaves every d_i and the barycenter unchanged; the iteration keeps sum_i lambda_i log c_i = 0, so
    only the lambda_i = 0 inputs carry a free (non-contracting) gauge mode.  Per input: log v_i - m_i and
    log w_i + m_i elementwise (m_i = mean of log v_i), and m_i itself for every input with lambda_i > 0
    (the lambda_i = 0 inputs are exempt from that one comparison only)."""
    out = dict(lv=0.0, lw=0.0, gauge=0.0)
    for i, lam in enumerate(np.asarray(lambdas, dtype=np.float64)):
        mg, mr = gauge_mean(glv[i]), gauge_mean(rlv[i])
        out["lv"] = max(out["lv"], potential_err(np.asarray(glv[i], dtype=np.float64) - mg,
                                                 np.asarray(rlv[i], dtype=np.float64) - mr))
        out["lw"] = max(out["lw"], potential_err(np.asarray(glw[i], dtype=np.float64) + mg,
                                                 np.asarray(rlw[i], dtype=np.float64) + mr))
        if lam != 0.0:
            out["gauge"] = max(out["gauge"], abs(mg - mr) / max(1.0, abs(mr)))
    return out


def measure_err(g, r, floor_rel=1e-6):
    """max |g - r| / max(|r|, floor_rel * max|r|)  -- relative error on transported measures (R12)."""
    g = np.asarray(g, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    fl = floor_rel * np.max(np.abs(r))
    return float(np.max(np.abs(g - r) / np.maximum(np.abs(r), fl)))


def trace_err(g, r, rel=1e-4, abs_floor=1e-5):
    """Error-trace agreement, scaled so that <= 1 passes: max |e_g - e_r| / (rel e_r + abs_floor), i.e.
    |d| <= 1e-4 e_ref + 1e-5 (L18): fp32 cannot resolve an L1 marginal error below ~1e-6 while fp64
    reaches 1e-17."""
    g = np.asarray(g, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    return float(np.max(np.abs(g - r) / (rel * np.abs(r) + abs_floor)))
