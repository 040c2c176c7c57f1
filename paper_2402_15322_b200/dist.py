"""Multi-GPU binding (se2_comm / se2_dist of include/se2ot.h).  Argument marshalling only: the loops,
the halo exchanges and the allreduces run inside libse2ot (NCCL between processes, or the loopback
transport between host threads of one process for the one-GPU tests).

B:north_star: "independent barycenter inputs ... go per GPU, with an NCCL allreduce over NVLink for the
barycenter log-mean, and a single large grid is split into spatial slabs with NVLink halo exchange".
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib as L
from .api import Kernel, _check_field, _flags, _ptr, _stream

check = L.check


class Comm:
    """A communicator (se2_comm).  Build it with `from_process_group` (one process per GPU, NCCL) or
    `loopback` (n ranks as host threads of one process)."""

    def __init__(self, handle: ctypes.c_void_p):
        self._h = handle
        n, r = ctypes.c_int32(), ctypes.c_int32()
        check(L.load().se2_comm_info(self._h, ctypes.byref(n), ctypes.byref(r)))
        self.nranks, self.rank = n.value, r.value

    @property
    def handle(self):
        return self._h

    @classmethod
    def single(cls, device: int = 0) -> "Comm":
        h = ctypes.c_void_p()
        check(L.load().se2_comm_init(None, 1, 0, int(device), ctypes.byref(h)))
        return cls(h)

    @classmethod
    def from_process_group(cls, device: int, group=None) -> "Comm":
        """NCCL communicator over the ranks of a torch.distributed group: rank 0 creates the unique id,
        torch.distributed broadcasts it (the plumbing), se2_comm_init builds the communicator."""
        import torch.distributed as dist
        ws = dist.get_world_size(group)
        rank = dist.get_rank(group)
        if ws == 1:
            return cls.single(device)
        buf = ctypes.create_string_buffer(128)
        if rank == 0:
            check(L.load().se2_comm_unique_id(buf))
        obj = [bytes(buf.raw)]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        h = ctypes.c_void_p()
        check(L.load().se2_comm_init(obj[0], ws, rank, int(device), ctypes.byref(h)))
        return cls(h)

    @classmethod
    def nccl_one_rank(cls, device: int = 0) -> "Comm":
        """A REAL one-rank NCCL communicator (unique id + ncclCommInitRank): the solvers run their collectives
        on it, so the NCCL transport can be exercised on one GPU."""
        buf = ctypes.create_string_buffer(128)
        check(L.load().se2_comm_unique_id(buf))
        h = ctypes.c_void_p()
        check(L.load().se2_comm_init(bytes(buf.raw), 1, 0, int(device), ctypes.byref(h)))
        return cls(h)

    @classmethod
    def loopback(cls, nranks: int, device: int = 0) -> List["Comm"]:
        arr = (ctypes.c_void_p * nranks)()
        check(L.load().se2_comm_init_loopback(int(nranks), int(device), arr))
        return [cls(ctypes.c_void_p(arr[i])) for i in range(nranks)]

    def split(self, color: int, key: int) -> "Comm":
        """Collective over this communicator: the ranks with the same color, ordered by key."""
        h = ctypes.c_void_p()
        check(L.load().se2_comm_split(self._h, int(color), int(key), ctypes.byref(h)))
        return Comm(h)

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        """In-place sum over the ranks (float32 or float64 CUDA tensor) on the current stream."""
        if t.dtype not in (torch.float32, torch.float64) or not t.is_cuda or not t.is_contiguous():
            raise TypeError("allreduce_ needs a contiguous float32/float64 CUDA tensor")
        check(L.load().se2_comm_allreduce(self._h, _ptr(t), t.numel(), 1 if t.dtype == torch.float64 else 0,
                                          _stream(t.device)))
        return t

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            L.load().se2_comm_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def slab_rows(ny: int, nslabs: int, index: int, R: int):
    """Rows of slab `index` of a grid of ny rows in nslabs contiguous slabs (sizes differ by <= 1):
    (row0, rows, halo_top, halo_bot) with halo R toward each neighbour and 0 at the global edges."""
    base, rem = divmod(ny, nslabs)
    row0 = index * base + min(index, rem)
    rows = base + (1 if index < rem else 0)
    top = R if index > 0 else 0
    bot = R if index + 1 < nslabs else 0
    return row0, rows, top, bot


class Dist:
    """One rank's decomposition (se2_dist): `reduce` -- the ranks whose inputs form the same barycenters,
    `slabs` -- the row slabs of the same fields (rank order = row order), and this rank's halo rows."""

    def __init__(self, reduce: Optional[Comm] = None, slabs: Optional[Comm] = None, halo_top: int = 0,
                 halo_bot: int = 0):
        self.reduce, self.slabs = reduce, slabs
        self.s = L.se2_dist(reduce.handle if reduce is not None else None, slabs.handle if slabs is not None else None,
                            int(halo_top), int(halo_bot))


def slab_kernel(nx: int, ny: int, ntheta: int, eps: float, w: Sequence[float], radius: int, nslabs: int, index: int,
                max_batch: int = 1, device: int = 0):
    """Kernel of slab `index` of an nx x ny x ntheta grid: the local grid (halo + owned + halo rows) with
    the GLOBAL cell sizes (R1), output window = the owned rows.  Returns (kernel, row0, rows, top, bot)."""
    row0, rows, top, bot = slab_rows(ny, nslabs, index, radius)
    k = Kernel(nx, top + rows + bot, ntheta, eps, w, radius, max_batch=max_batch, device=device,
               hx=1.0 / nx, hy=1.0 / ny)
    check(L.load().se2_kernel_set_window(k.handle, top, top + rows))
    return k, row0, rows, top, bot


def local_rows(x: np.ndarray, row0: int, rows: int, top: int, bot: int) -> np.ndarray:
    """The local array of a slab (halo + owned + halo rows) cut from a global [..., ny, nx] array."""
    return np.ascontiguousarray(x[..., row0 - top:row0 + rows + bot, :])


def se2_jko_step_dist(k: Kernel, d: Dist, mu_k: torch.Tensor, mu_next: torch.Tensor, a: torch.Tensor, b: torch.Tensor,
                      iters: int, prox: L.se2_prox, log_domain: bool, trace: bool = False, engine_flags: int = 0,
                      no_graph: bool = False):
    """One entropic JKO step on this rank's slab (R10).  Returns (mass over all slabs,
    error trace [iters] or None)."""
    for name, t in (("mu_k", mu_k), ("mu_next", mu_next), ("a", a), ("b", b)):
        _check_field(t, k, name, 1)
    opts = L.se2_opts(int(iters), _flags(log_domain, trace, no_graph=no_graph) | int(engine_flags))
    mass = ctypes.c_double()
    tr = np.zeros(max(iters, 1), dtype=np.float64) if trace else None
    check(L.load().se2_jko_step_dist(k.handle, ctypes.byref(d.s), _ptr(mu_k), _ptr(mu_next), _ptr(a), _ptr(b),
                                     ctypes.byref(prox), ctypes.byref(opts), ctypes.byref(mass),
                                     tr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if trace else None,
                                     _stream(mu_k.device)))
    return mass.value, (tr[:iters] if trace else None)


def se2_barycenter_dist(k: Kernel, d: Dist, mus: torch.Tensor, lambdas, iters: int,
                        bary: Optional[torch.Tensor] = None, v_state: Optional[torch.Tensor] = None,
                        w_state: Optional[torch.Tensor] = None, trace: bool = False, warm_start: bool = False,
                        no_graph: bool = False):
    """App. A (log domain) with this rank's inputs mus [n][N_local] and their weights lambdas [nsolve][n]
    (a share of weights that sum to 1 over the `reduce` ranks).  Returns (log mu [nsolve][N_local],
    trace [iters][nsolve] or None)."""
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
    opts = L.se2_opts(int(iters), _flags(True, trace, warm=warm_start, no_graph=no_graph))
    tr = np.zeros((max(iters, 1), nsolve), dtype=np.float64) if trace else None
    check(L.load().se2_barycenter_dist(k.handle, ctypes.byref(d.s), n, nsolve, _ptr(mus),
                                       lam.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _ptr(bary), _ptr(v_state),
                                       _ptr(w_state), ctypes.byref(opts),
                                       tr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if trace else None,
                                       _stream(mus.device)))
    return bary, (tr[:iters] if trace else None)


def se2_barycenter_precise_dist(k: Kernel, d: Dist, mus: torch.Tensor, lambdas, iters: int,
                                lbary: Optional[torch.Tensor] = None, lv_state: Optional[torch.Tensor] = None,
                                lw_state: Optional[torch.Tensor] = None, trace: bool = False,
                                warm_start: bool = False, no_graph: bool = False):
    """App. A with fp64 potentials (K4P, reading R19) and this rank's inputs mus [n][N] (float32), weights
    lambdas [nsolve][n] (a share of weights that sum to 1 over the `reduce` ranks) and, with `d.slabs`, this
    rank's row slab of every input (fp64 halo exchanges of w_i / v_i).  Returns (log mu [nsolve][N_local]
    float64, trace [iters][nsolve] or None)."""
    from .api import _check_field64
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
    opts = L.se2_opts(int(iters), _flags(True, trace, warm=warm_start, no_graph=no_graph))
    tr = np.zeros((max(iters, 1), nsolve), dtype=np.float64) if trace else None
    check(L.load().se2_barycenter_precise_dist(k.handle, ctypes.byref(d.s), n, nsolve, _ptr(mus),
                                               lam.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _ptr(lbary),
                                               _ptr(lv_state), _ptr(lw_state), ctypes.byref(opts),
                                               tr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if trace else None,
                                               _stream(mus.device)))
    return lbary, (tr[:iters] if trace else None)
