"""Python binding of the se2ot C ABI with the same names (include/se2ot.h).

Argument marshalling only (torch CUDA tensors -> device pointers, the current CUDA stream); no
arithmetic of the method happens here.  Tensors must be float32, contiguous, on the kernel's
device, layout [batch][ntheta][ny][nx].
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib as L
from ._lib import check


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _check_field(t: torch.Tensor, k: "Kernel", name: str, batch: Optional[int] = None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (the SE(2) OT path has no CPU fallback)")
    if t.dtype != torch.float32 or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous float32 tensor")
    if t.device.index != k.device:
        raise ValueError(f"{name} is on {t.device}, kernel on cuda:{k.device}")
    if t.numel() % k.N != 0:
        raise ValueError(f"{name} numel {t.numel()} is not a multiple of N={k.N}")
    if batch is not None and t.numel() != batch * k.N:
        raise ValueError(f"{name} must hold {batch} fields")


class Kernel:
    """Owns an se2_kernel (device Gibbs-kernel tables + scratch).  se2_kernel_build."""

    def __init__(self, nx: int, ny: int, ntheta: int, eps: float, w: Sequence[float], radius: int,
                 max_batch: int = 1, device: int = 0, hx: float = 0.0, hy: float = 0.0):
        lib = L.load()
        self.nx, self.ny, self.ntheta = int(nx), int(ny), int(ntheta)
        self.eps, self.w, self.radius = float(eps), tuple(float(v) for v in w), int(radius)
        self.max_batch, self.device = int(max_batch), int(device)
        self.N = self.nx * self.ny * self.ntheta
        self.hx = float(hx) if hx else 1.0 / self.nx      # cell sizes (R1); a window of a finer
        self.hy = float(hy) if hy else 1.0 / self.ny      # lattice keeps that lattice's cell
        h = ctypes.c_void_p()
        g = L.se2_grid(self.nx, self.ny, self.ntheta, float(hx), float(hy))
        m = L.se2_metric(*self.w)
        st = lib.se2_kernel_build(ctypes.byref(g), ctypes.byref(m), self.eps, self.radius, self.max_batch,
                                  self.device, ctypes.byref(h))
        check(st)
        self._h = h

    @property
    def handle(self):
        return self._h

    def stats(self) -> dict:
        s = L.se2_kernel_stats()
        check(L.load().se2_kernel_stats_get(self._h, ctypes.byref(s)))
        return dict(box_taps=s.box_taps, nnz_taps=s.nnz_taps, theta_band=s.theta_band, radius=s.radius,
                    zeta=s.zeta, table_bytes=s.table_bytes, tensor_cores=int(s.tensor_cores),
                    nnz_normal_taps=s.nnz_normal_taps)

    @property
    def uses_tensor_cores(self) -> bool:
        """True when linear convs run on the tensor-core engine (K10) by default."""
        return self.stats()["tensor_cores"] == 1

    @property
    def has_tensor_cores(self) -> bool:
        """True when K10 covers this grid (default or forced with SE2_LIN_TC)."""
        return self.stats()["tensor_cores"] != 0

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            L.load().se2_kernel_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # instrumentation
    def lse_path_stats(self, reset: bool = True) -> dict:
        """K3 counters: (tile-quad, theta_i) pairs active after pruning / on the FFMA path / visited."""
        a, f, v, t, h = (ctypes.c_int64() for _ in range(5))
        check(L.load().se2_lse_path_stats(self._h, ctypes.byref(a), ctypes.byref(f), ctypes.byref(v),
                                          ctypes.byref(t), ctypes.byref(h), 1 if reset else 0))
        return dict(active=a.value, ffma=f.value, visited=v.value, tilted=t.value, hint_redos=h.value)

    def lse_row_stats(self, reset: bool = True) -> dict:
        """K3 exact-path rows of taps (warp, theta_i, dy) evaluated / visited after row pruning."""
        live, vis = ctypes.c_int64(), ctypes.c_int64()
        check(L.load().se2_lse_row_stats(self._h, ctypes.byref(live), ctypes.byref(vis), 1 if reset else 0))
        return dict(live=live.value, visited=vis.value)

    def precise_path_stats(self, reset: bool = True) -> dict:
        """K4P: channels on the factored FFMA path / channels visited."""
        f, c, r = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check(L.load().se2_precise_path_stats(self._h, ctypes.byref(f), ctypes.byref(c), ctypes.byref(r),
                                              1 if reset else 0))
        return dict(ffma=f.value, channels=c.value, hint_redos=r.value)

    def tc_tile_stats(self, reset: bool = True) -> dict:
        """K10 narrow geometry: tiles computed / tiles on the wide (32-orientation) window."""
        t, w = ctypes.c_int64(), ctypes.c_int64()
        check(L.load().se2_tc_tile_stats(self._h, ctypes.byref(t), ctypes.byref(w), 1 if reset else 0))
        return dict(tiles=t.value, wide=w.value)

    def guard_stats(self, reset: bool = False) -> dict:
        """Division-guard clamps (R9) and porous prox non-convergences since the last solve
        started (se2_guard_stats)."""
        d, p = ctypes.c_int64(), ctypes.c_int64()
        check(L.load().se2_guard_stats(self._h, ctypes.byref(d), ctypes.byref(p), 1 if reset else 0))
        return dict(div_clamps=d.value, prox_noconv=p.value)

    def timing_enable(self, on: bool = True):
        check(L.load().se2_timing_enable(self._h, 1 if on else 0))

    def timing_get(self):
        n = ctypes.c_int64()
        ms = ctypes.c_double()
        alln = ctypes.c_int64()
        check(L.load().se2_timing_get(self._h, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(alln)))
        return n.value, ms.value, alln.value


def se2_kernel_build(nx, ny, ntheta, eps, w, radius, max_batch=1, device=0) -> Kernel:
    return Kernel(nx, ny, ntheta, eps, w, radius, max_batch, device)


def _flags(log_domain: bool, trace: bool = False, warm: bool = False, lse_exact: bool = False,
           no_graph: bool = False) -> int:
    return (L.SE2_LOG_DOMAIN if log_domain else 0) | (L.SE2_TRACE_ERR if trace else 0) | (
        L.SE2_WARM_START if warm else 0) | (L.SE2_LSE_EXACT if lse_exact else 0) | (L.SE2_NO_GRAPH if no_graph else 0)


def se2_conv(k: Kernel, x: torch.Tensor, out: Optional[torch.Tensor] = None, log_domain: bool = False,
             lse_exact: bool = False, extra_flags: int = 0) -> torch.Tensor:
    """out = K x (or log K exp(x) with log_domain).  lse_exact forces the per-tap
    log-sum-exp engine (K4) instead of the factored one (K3)."""
    _check_field(x, k, "x")
    batch = x.numel() // k.N
    if out is None:
        out = torch.empty_like(x)
    _check_field(out, k, "out", batch)
    check(L.load().se2_conv(k.handle, _ptr(x), _ptr(out), batch,
                            _flags(log_domain, lse_exact=lse_exact) | int(extra_flags), _stream(x.device)))
    return out


def make_prox(k: Kernel, tau: float, global_ny: Optional[int] = None, row_offset: int = 0) -> L.se2_prox:
    """Entropy + potential prox of the JKO step (R10): V(x) = |x - c|^2 in [0,1]^2 units, c the window
    centre, the kernel's cell sizes.  For a slab of a grid with global_ny rows whose local row 0 is
    global row `row_offset`, the centre row is global_ny / 2 - row_offset (cells)."""
    gny = k.ny if global_ny is None else int(global_ny)
    return L.se2_prox(L.SE2_PROX_ENTROPY_POTENTIAL, float(tau), k.nx / 2.0, gny / 2.0 - row_offset,
                      k.hx, k.hy, 0.0)


def make_porous_prox(tau: float, m: float) -> L.se2_prox:
    """Porous-medium prox of the paper's gradient flow, F = 1/(m-1) sum s^m."""
    if not m > 1.0:
        raise ValueError("porous-medium exponent m must be > 1")
    return L.se2_prox(L.SE2_PROX_POROUS, float(tau), 0.0, 0.0, 0.0, 0.0, float(m))


def se2_sinkhorn(k: Kernel, mu: torch.Tensor, nu: Optional[torch.Tensor], a: torch.Tensor, b: torch.Tensor,
                 iters: int, log_domain: bool, prox: Optional[L.se2_prox] = None, trace: bool = False,
                 warm_start: bool = False, lse_exact: bool = False, no_graph: bool = False,
                 persistent: bool = True) -> Optional[np.ndarray]:
    """Scaling iterations a = mu / K b, b = prox(K^T a)/K^T a.  Returns the marginal
    error trace [iters][batch] when trace=True.  persistent=False disables the one-launch cluster
    solver (K9) that small log-domain problems use otherwise."""
    _check_field(mu, k, "mu")
    batch = mu.numel() // k.N
    for name, t in (("a", a), ("b", b)):
        _check_field(t, k, name, batch)
    if nu is not None:
        _check_field(nu, k, "nu", batch)
    opts = L.se2_opts(int(iters), _flags(log_domain, trace, warm_start, lse_exact, no_graph)
                      | (0 if persistent else L.SE2_NO_PERSISTENT))
    tr = np.zeros((max(iters, 1), batch), dtype=np.float64) if trace else None
    trp = tr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if trace else None
    check(L.load().se2_sinkhorn(k.handle, _ptr(mu), _ptr(nu), _ptr(a), _ptr(b), batch,
                                ctypes.byref(prox) if prox is not None else None, ctypes.byref(opts), trp,
                                _stream(mu.device)))
    return tr[:iters] if trace else None


def se2_jko_step(k: Kernel, mu_k: torch.Tensor, mu_next: torch.Tensor, a: torch.Tensor, b: torch.Tensor,
                 iters: int, prox: L.se2_prox, log_domain: bool = False, trace: bool = False, engine_flags: int = 0):
    """One entropic JKO step (R10).  Returns (mass before normalisation, err trace).
    engine_flags: SE2_LIN_FFMA / SE2_LIN_TC to force the linear conv engine (tests, A/B)."""
    for name, t in (("mu_k", mu_k), ("mu_next", mu_next), ("a", a), ("b", b)):
        _check_field(t, k, name, 1)
    opts = L.se2_opts(int(iters), _flags(log_domain, trace) | int(engine_flags))
    mass = ctypes.c_double()
    tr = np.zeros((max(iters, 1), 1), dtype=np.float64) if trace else None
    trp = tr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if trace else None
    check(L.load().se2_jko_step(k.handle, _ptr(mu_k), _ptr(mu_next), _ptr(a), _ptr(b), ctypes.byref(prox),
                                ctypes.byref(opts), ctypes.byref(mass), trp, _stream(mu_k.device)))
    return mass.value, (tr[:iters, 0] if trace else None)


def se2_barycenter(k: Kernel, mus: torch.Tensor, lambdas, iters: int, log_domain: bool,
                   bary: Optional[torch.Tensor] = None, v_state: Optional[torch.Tensor] = None,
                   w_state: Optional[torch.Tensor] = None, trace: bool = False, lse_exact: bool = False,
                   no_graph: bool = False, debug_flags: int = 0, warm_start: bool = False):
    """App. A barycenter.  mus: [n][N]; lambdas: [nsolve][n] (host).  Returns
    (bary [nsolve][N] -- log mu under log_domain --, err trace [iters][nsolve] or None).
    warm_start: resume from v_state (required) instead of v_i = 1.
    debug_flags: SE2_DEBUG_* bits (diagnostics / tests only)."""
    _check_field(mus, k, "mus")
    n = mus.numel() // k.N
    lam = np.ascontiguousarray(np.atleast_2d(np.asarray(lambdas, dtype=np.float64)))
    if lam.shape[1] != n:
        raise ValueError(f"lambdas must be [nsolve][{n}]")
    nsolve = lam.shape[0]
    if bary is None:
        bary = torch.empty((nsolve, k.ntheta, k.ny, k.nx), device=mus.device, dtype=torch.float32)
    _check_field(bary, k, "bary", nsolve)
    for name, t in (("v_state", v_state), ("w_state", w_state)):
        if t is not None:
            _check_field(t, k, name, nsolve * n)
    if warm_start and v_state is None:
        raise ValueError("warm_start needs v_state")
    opts = L.se2_opts(int(iters), _flags(log_domain, trace, warm=warm_start, lse_exact=lse_exact, no_graph=no_graph)
                      | int(debug_flags))
    tr = np.zeros((max(iters, 1), nsolve), dtype=np.float64) if trace else None
    trp = tr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if trace else None
    check(L.load().se2_barycenter(k.handle, n, nsolve, _ptr(mus), lam.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                  _ptr(bary), _ptr(v_state), _ptr(w_state), ctypes.byref(opts), trp,
                                  _stream(mus.device)))
    return bary, (tr[:iters] if trace else None)


def _check_field64(t, k: Kernel, name: str, batch: Optional[int] = None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous float64 CUDA tensor (the precise path's fp64 potentials)")
    if t.numel() % k.N != 0 or (batch is not None and t.numel() != batch * k.N):
        raise ValueError(f"{name} must hold {batch if batch is not None else 'whole'} fields of N={k.N}")


def se2_conv_precise(k: Kernel, x: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """log(K exp(x)) on K4P (fp64 fields; exact exponents, ~1e-7 nats per conv)."""
    _check_field64(x, k, "x")
    batch = x.numel() // k.N
    if out is None:
        out = torch.empty_like(x)
    _check_field64(out, k, "out", batch)
    check(L.load().se2_conv_precise(k.handle, _ptr(x), _ptr(out), batch, _stream(x.device)))
    return out


def se2_barycenter_precise(k: Kernel, mus: torch.Tensor, lambdas, iters: int,
                           lbary: Optional[torch.Tensor] = None, lv_state: Optional[torch.Tensor] = None,
                           lw_state: Optional[torch.Tensor] = None, trace: bool = False, no_graph: bool = False,
                           warm_start: bool = False):
    """App. A in the log domain with fp64 potentials on K4P (reading R19).  mus: float32
    [n][N]; returns (log mu [nsolve][N] float64, err trace [iters][nsolve] or None)."""
    _check_field(mus, k, "mus")
    n = mus.numel() // k.N
    lam = np.ascontiguousarray(np.atleast_2d(np.asarray(lambdas, dtype=np.float64)))
    if lam.shape[1] != n:
        raise ValueError(f"lambdas must be [nsolve][{n}]")
    nsolve = lam.shape[0]
    if lbary is None:
        lbary = torch.empty((nsolve, k.ntheta, k.ny, k.nx), device=mus.device, dtype=torch.float64)
    _check_field64(lbary, k, "lbary", nsolve)
    for name, t in (("lv_state", lv_state), ("lw_state", lw_state)):
        if t is not None:
            _check_field64(t, k, name, nsolve * n)
    if warm_start and lv_state is None:
        raise ValueError("warm_start needs lv_state")
    opts = L.se2_opts(int(iters), _flags(True, trace, warm=warm_start, no_graph=no_graph))
    tr = np.zeros((max(iters, 1), nsolve), dtype=np.float64) if trace else None
    check(L.load().se2_barycenter_precise(k.handle, n, nsolve, _ptr(mus),
                                          lam.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _ptr(lbary),
                                          _ptr(lv_state), _ptr(lw_state), ctypes.byref(opts),
                                          tr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if trace else None,
                                          _stream(mus.device)))
    return lbary, (tr[:iters] if trace else None)


def se2_marginal_error(k: Kernel, a: torch.Tensor, b: torch.Tensor, mu: torch.Tensor, log_domain: bool) -> np.ndarray:
    """err_i = sum |a_i K b_i - mu_i| (R8)."""
    _check_field(mu, k, "mu")
    batch = mu.numel() // k.N
    _check_field(a, k, "a", batch)
    _check_field(b, k, "b", batch)
    out = np.zeros(batch, dtype=np.float64)
    check(L.load().se2_marginal_error(k.handle, _ptr(a), _ptr(b), _ptr(mu), batch, _flags(log_domain),
                                      out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _stream(mu.device)))
    return out


def se2_transport_cost(k: Kernel, a: torch.Tensor, b: torch.Tensor, log_domain: bool,
                       engine_flags: int = 0) -> np.ndarray:
    """<pi, rho_b^2> of the plan pi = a K b (one conv with the cost table; NEXT #2).
    engine_flags: SE2_LIN_FFMA / SE2_LIN_TC to force the linear conv engine (tests, A/B)."""
    _check_field(a, k, "a")
    batch = a.numel() // k.N
    _check_field(b, k, "b", batch)
    out = np.zeros(batch, dtype=np.float64)
    check(L.load().se2_transport_cost(k.handle, _ptr(a), _ptr(b), batch, _flags(log_domain) | int(engine_flags),
                                      out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _stream(a.device)))
    return out


def se2_conv_update(k: Kernel, x: torch.Tensor, target: Optional[torch.Tensor], out: torch.Tensor, op: int,
                    log_domain: bool, prox: Optional[L.se2_prox] = None,
                    slab: Optional[L.se2_slab] = None) -> torch.Tensor:
    """Fused conv + scaling update (step-level entry point used by the multi-GPU driver).  slab: the
    rows this rank owns and the neighbours' peer-mapped arrays that receive its boundary rows
    (se2_conv_update_slab)."""
    _check_field(x, k, "x")
    batch = x.numel() // k.N
    _check_field(out, k, "out", batch)
    if target is not None:
        _check_field(target, k, "target", batch)
    pr = ctypes.byref(prox) if prox is not None else None
    if slab is None:
        check(L.load().se2_conv_update(k.handle, _ptr(x), _ptr(target), _ptr(out), batch, int(op), pr,
                                       _flags(log_domain), _stream(x.device)))
    else:
        check(L.load().se2_conv_update_slab(k.handle, _ptr(x), _ptr(target), _ptr(out), batch, int(op), pr,
                                            _flags(log_domain), ctypes.byref(slab), _stream(x.device)))
    return out


def se2_bary_logmean(ld: torch.Tensor, lambdas, N: int, lbar: torch.Tensor) -> torch.Tensor:
    lam = np.ascontiguousarray(np.asarray(lambdas, dtype=np.float64).reshape(-1))
    n = lam.shape[0]
    check(L.load().se2_bary_logmean(n, N, _ptr(ld), lam.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                    _ptr(lbar), _stream(ld.device)))
    return lbar


def se2_bary_update(lv: torch.Tensor, ld: torch.Tensor, lbar: torch.Tensor, n: int, N: int):
    check(L.load().se2_bary_update(n, N, _ptr(lv), _ptr(ld), _ptr(lbar), _stream(lv.device)))


def se2_bary_reduce_update(partial_ptrs: torch.Tensor, n_local: int, N: int, lv: Optional[torch.Tensor],
                           ld: Optional[torch.Tensor], lbar: Optional[torch.Tensor]):
    """lbar = sum_r partials[r] (rank order), lv_i += lbar - ld_i: the sharded barycenter's allreduce fused
    with the v-update.  partial_ptrs: int64 CUDA tensor of nranks device pointers (peer buffers)."""
    if not (isinstance(partial_ptrs, torch.Tensor) and partial_ptrs.is_cuda and partial_ptrs.dtype == torch.int64):
        raise TypeError("partial_ptrs must be an int64 CUDA tensor of device pointers")
    dev = partial_ptrs.device
    check(L.load().se2_bary_reduce_update(partial_ptrs.numel(), _ptr(partial_ptrs), int(n_local), int(N), _ptr(lv),
                                          _ptr(ld), _ptr(lbar), _stream(dev)))


def se2_sum(x: torch.Tensor) -> float:
    out = ctypes.c_double()
    check(L.load().se2_sum(_ptr(x), x.numel(), ctypes.byref(out), _stream(x.device)))
    return out.value


def se2_sum_rows(x: torch.Tensor, row0: int, rows: int) -> float:
    """Sum of rows [row0, row0+rows) of every plane of x ([..., ny, nx], contiguous)."""
    ny, nx = x.shape[-2], x.shape[-1]
    planes = x.numel() // (ny * nx)
    out = ctypes.c_double()
    check(L.load().se2_sum_rows(_ptr(x), planes, ny, nx, int(row0), int(rows), ctypes.byref(out), _stream(x.device)))
    return out.value


def se2_scale_rows(x: torch.Tensor, row0: int, rows: int, factor: float):
    ny, nx = x.shape[-2], x.shape[-1]
    planes = x.numel() // (ny * nx)
    check(L.load().se2_scale_rows(_ptr(x), planes, ny, nx, int(row0), int(rows), float(factor), _stream(x.device)))


def se2_launch_count() -> int:
    return int(L.load().se2_launch_count())
