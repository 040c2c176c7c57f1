"""Multi-GPU drivers of the scaling loop: one process per GPU, torch.distributed for the exchanges.

Two decompositions of the north star (B:north_star "independent barycenter inputs ... go per GPU,
with an NCCL allreduce over NVLink for the barycenter log-mean, and a single large grid is split
into spatial slabs with NVLink halo exchange"):

* `ShardedBarycenter` -- App. A with the n inputs distributed over the ranks.  The only
  exchange per iteration is the allreduce of the partial weighted log-mean
  `sum_{i on rank} lambda_i log d_i` (NCCL on GPUs).
* `SlabJKO` -- the entropic JKO step (reading R10) with the grid's rows split into slabs;
  before every convolution each rank exchanges R boundary rows with its neighbours (send/recv), the
  conv runs on the slab extended by its halo (zero rows at the global edges), and the plan mass is
  allreduced once per JKO step.

The per-rank arithmetic goes through an `ops` backend: `CudaOps` (this library's kernels; the
product path) or, in the CPU tests only, a backend built on the oracle (tests/test_parallel_gloo.py),
so the decomposition logic is tested with the gloo backend without a GPU.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np
import torch
import torch.distributed as dist


def partition(n: int, world: int, rank: int):
    """Contiguous block partition of range(n) over `world` ranks (sizes differ by at most 1)."""
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


class CudaOps:
    """Per-rank arithmetic on the GPU through the se2ot C ABI."""

    def __init__(self, kernel, log_domain: bool):
        from . import api
        self.api = api
        self.k = kernel
        self.log = log_domain

    # slab: optional se2_slab (the owned rows + the neighbours' peer arrays receiving the boundary rows)
    def divide(self, x, target, out, slab=None):     # out = target / K x   (log: target - LSE x)
        from ._lib import SE2_EPI_DIVIDE
        return self.api.se2_conv_update(self.k, x, target, out, SE2_EPI_DIVIDE, self.log, slab=slab)

    def multiply(self, x, target, out, slab=None):   # out = target * K x   (log: target + LSE x)
        from ._lib import SE2_EPI_MULTIPLY
        return self.api.se2_conv_update(self.k, x, target, out, SE2_EPI_MULTIPLY, self.log, slab=slab)

    def prox(self, x, out, prox, slab=None):         # out = prox(K x) / K x   (JKO, R10)
        from ._lib import SE2_EPI_PROX
        return self.api.se2_conv_update(self.k, x, None, out, SE2_EPI_PROX, self.log, prox=prox, slab=slab)

    def log_of(self, x):                    # elementwise log (log 0 = -inf), a new tensor
        from .lifting import se2_log
        return se2_log(x.contiguous())

    def reduce_update(self, sources, lv, ld, lbar, n):
        """lbar = sum over ranks of the partial log-means (rank order), lv_i += lbar - ld_i: one kernel
        (se2_bary_reduce_update).  sources: an int64 device tensor of peer pointers (P2PExchange) or a
        list of gathered tensors (GatherExchange)."""
        if isinstance(sources, torch.Tensor):
            table = sources
        else:
            table = torch.tensor([t.data_ptr() for t in sources], dtype=torch.int64, device=lbar.device)
        N = lbar.numel()
        self.api.se2_bary_reduce_update(table, n, N, lv if n > 0 else None, ld if n > 0 else None, lbar)

    def logmean(self, ld, lambdas, out):    # out = sum_i lambda_i ld_i  (lambda_i = 0 skipped)
        return self.api.se2_bary_logmean(ld, lambdas, self.k.N, out)

    def bary_update(self, lv, ld, lbar, n):  # lv_i += lbar - ld_i
        return self.api.se2_bary_update(lv, ld, lbar, n, self.k.N)

    def sum_rows(self, x, row0: int, rows: int) -> float:   # sum over rows [row0, row0+rows) of all planes
        return self.api.se2_sum_rows(x, row0, rows)

    def scale_rows(self, x, row0: int, rows: int, factor: float):
        self.api.se2_scale_rows(x, row0, rows, factor)


class GatherExchange:
    """Peer partial log-means by `dist.all_gather` into local copies (any backend: the gloo CPU tests,
    or NCCL as the baseline transport); double-buffered by iteration parity like P2PExchange."""

    def __init__(self, like: torch.Tensor, group=None):
        self.group = group
        self.ws = dist.get_world_size(group) if dist.is_initialized() else 1
        self.slots = [torch.empty_like(like), torch.empty_like(like)]

    def slot(self, parity: int) -> torch.Tensor:
        return self.slots[parity]

    def sources(self, parity: int):
        mine = self.slots[parity]
        if self.ws == 1:
            return [mine]
        out = [torch.empty_like(mine) for _ in range(self.ws)]
        dist.all_gather(out, mine, group=self.group)
        return out


class P2PExchange:
    """Peer partial log-means read in place over NVLink: every rank owns a symmetric-memory buffer
    [2][N] (torch SymmetricMemory: peer-mapped allocations), double-buffered by iteration parity; one
    device barrier per iteration makes the slot of that parity complete on every rank, then the fused
    reduce + update kernel reads all ranks' slots through the device pointer table.  A fast rank can
    only overwrite a slot after the next iteration's barrier, i.e. after every rank finished reading
    it (the reads precede that barrier on each rank's stream)."""

    def __init__(self, like: torch.Tensor, group=None):
        import torch.distributed._symmetric_memory as symm_mem
        self.group = group if group is not None else dist.group.WORLD
        shape = tuple(like.shape)
        self.buf = symm_mem.empty((2,) + shape, dtype=torch.float32, device=like.device)
        self.hdl = symm_mem.rendezvous(self.buf, self.group)
        base = self.buf.data_ptr() - int(self.hdl.buffer_ptrs[self.hdl.rank])   # offset inside the allocation
        n = like.numel()
        self.tables = [torch.tensor([int(p) + base + parity * n * 4 for p in self.hdl.buffer_ptrs], dtype=torch.int64,
                                    device=like.device) for parity in (0, 1)]

    def slot(self, parity: int) -> torch.Tensor:
        return self.buf[parity]

    def sources(self, parity: int) -> torch.Tensor:
        self.hdl.barrier(channel=parity)
        return self.tables[parity]


class ShardedBarycenter:
    """App. A barycenter with inputs sharded over the ranks of the default process group.

    mus_local: [n_local][N] this rank's inputs; lambdas_local: their weights (the full weight vector
    sums to 1 over all ranks).  Log domain (R7, R13).  After `run`, `lbar` holds log mu on every rank.
    """

    def __init__(self, ops, mus_local: torch.Tensor, lambdas_local: Sequence[float], group=None,
                 exchange: str = "nccl"):
        """exchange: "nccl" (allreduce of the partial log-mean, then the update), "p2p" (peer buffers
        read in place by the fused reduce + update kernel, P2PExchange) or "gather" (all_gather copies
        into the same fused kernel; the CPU tests)."""
        self.ops = ops
        self.group = group
        self.n = mus_local.shape[0]
        self.lam = np.asarray(lambdas_local, dtype=np.float64)
        self.lmu = ops.log_of(mus_local) if mus_local.numel() else mus_local.clone()
        self.lv = torch.zeros_like(mus_local)
        self.lw = torch.zeros_like(mus_local)
        self.ld = torch.empty_like(mus_local)
        self.lbar = torch.empty(tuple(mus_local.shape[1:]), dtype=mus_local.dtype, device=mus_local.device)
        self.xch = None
        if exchange == "p2p":
            self.xch = P2PExchange(self.lbar, group)
        elif exchange == "gather":
            self.xch = GatherExchange(self.lbar, group)
        elif exchange != "nccl":
            raise ValueError(f"unknown exchange {exchange!r}")
        self.parity = 0

    def iterate(self, iters: int):
        if self.xch is not None:
            return self._iterate_fused(iters)
        for _ in range(iters):
            if self.n > 0:
                self.ops.divide(self.lv, self.lmu, self.lw)        # w_i = mu_i / K v_i
                self.ops.multiply(self.lw, self.lv, self.ld)       # d_i = v_i K w_i
                self.ops.logmean(self.ld, self.lam, self.lbar)     # partial sum_i lambda_i log d_i
            else:
                self.lbar.zero_()
            if dist.is_initialized() and dist.get_world_size(self.group) > 1:
                dist.all_reduce(self.lbar, op=dist.ReduceOp.SUM, group=self.group)   # log mu
            if self.n > 0:
                self.ops.bary_update(self.lv, self.ld, self.lbar, self.n)            # v_i <- v_i mu / d_i
        return self.lbar

    def _iterate_fused(self, iters: int):
        for _ in range(iters):
            slot = self.xch.slot(self.parity)
            if self.n > 0:
                self.ops.divide(self.lv, self.lmu, self.lw)        # w_i = mu_i / K v_i
                self.ops.multiply(self.lw, self.lv, self.ld)       # d_i = v_i K w_i
                self.ops.logmean(self.ld, self.lam, slot)          # this rank's partial sum_i lambda_i log d_i
            else:
                slot.zero_()
            src = self.xch.sources(self.parity)                    # every rank's partial of this parity
            self.ops.reduce_update(src, self.lv, self.ld, self.lbar, self.n)   # log mu; v_i <- v_i mu / d_i
            self.parity ^= 1
        return self.lbar


class SlabJKO:
    """Entropic JKO steps (R10) with the grid's rows split into slabs over the ranks.

    The local arrays are [nt][rows + 2R][nx]: owned rows are [R, R + rows), the R halo rows on each
    side hold the neighbours' boundary rows (zero at the global edges = the conv's zero padding).
    `ops` must wrap a kernel built for the local grid (nx, rows + 2R, nt) and prox factories must shift
    the potential's centre row by the slab offset.
    """

    def __init__(self, ops, mu_local_owned: torch.Tensor, R: int, prox, group=None, exchange: str = "nccl"):
        """exchange: "nccl" (halo rows by send/recv before each conv) or "p2p" (each conv's epilogue
        writes its boundary rows straight into the neighbours' halo rows in symmetric memory, one
        device barrier after each conv; se2_conv_update_slab)."""
        self.ops = ops
        self.R = R
        self.prox = prox
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        nt, rows, nx = mu_local_owned.shape
        self.rows = rows
        self.mu = self._ext(mu_local_owned)
        self.p2p = exchange == "p2p"
        if exchange not in ("nccl", "p2p"):
            raise ValueError(f"unknown exchange {exchange!r}")
        if self.world > 1 and R > 0:
            # a slab thinner than the halo would send rows it does not own (x[:, R:2R] reaches into its own
            # bottom halo): every rank must own at least R rows
            rows_all = [None] * self.world
            dist.all_gather_object(rows_all, int(rows), group=group)
            if min(rows_all) < R:
                raise ValueError(f"slab decomposition needs >= R = {R} rows per rank, got {rows_all}")
        if self.p2p:
            self._setup_p2p()
        else:
            self.a = torch.zeros_like(self.mu)
            self.b = torch.zeros_like(self.mu)

    def _setup_p2p(self):
        import torch.distributed._symmetric_memory as symm_mem
        from . import _lib as L
        group = self.group if self.group is not None else dist.group.WORLD
        rows_all = [None] * self.world
        dist.all_gather_object(rows_all, self.rows, group=group)
        nt, nyl, nx = self.mu.shape
        R = self.R
        shape = (nt, max(rows_all) + 2 * R, nx)   # symmetric allocations have one size; each rank uses a prefix
        n_local = nt * nyl * nx
        self._sym, self._hdl, arrays, ptrs = [], [], [], []
        for _ in range(2):   # a, b
            buf = symm_mem.empty(shape, dtype=torch.float32, device=self.mu.device)
            buf.zero_()
            hdl = symm_mem.rendezvous(buf, group)
            off = buf.data_ptr() - int(hdl.buffer_ptrs[hdl.rank])
            self._sym.append(buf)
            self._hdl.append(hdl)
            arrays.append(buf.view(-1)[:n_local].view(nt, nyl, nx))
            ptrs.append([int(p) + off for p in hdl.buffer_ptrs])
        self.a, self.b = arrays
        self._slabs = []
        for k in range(2):
            sl = L.se2_slab(R, R + self.rows, R, None, 0, 0, None, 0, 0)
            if self.rank > 0:                       # my first R owned rows -> the upper rank's bottom halo
                ru = rows_all[self.rank - 1]
                sl.up, sl.up_shift, sl.ny_up = ptrs[k][self.rank - 1], ru, ru + 2 * R
            if self.rank < self.world - 1:          # my last R owned rows -> the lower rank's top halo
                rd = rows_all[self.rank + 1]
                sl.dn, sl.dn_shift, sl.ny_dn = ptrs[k][self.rank + 1], self.rows, rd + 2 * R
            self._slabs.append(sl)

    def _ext(self, owned):
        nt, rows, nx = owned.shape
        out = torch.zeros((nt, rows + 2 * self.R, nx), dtype=owned.dtype, device=owned.device)
        out[:, self.R:self.R + rows] = owned
        return out

    def owned(self, x):
        return x[:, self.R:self.R + self.rows]

    def halo_exchange(self, x):
        """Fill x's halo rows from the neighbours' boundary rows (zeros at the global edges)."""
        R = self.R
        if R == 0:
            return
        if self.world == 1:
            x[:, :R].zero_()
            x[:, R + self.rows:].zero_()
            return
        up, down = self.rank - 1, self.rank + 1
        send_up = x[:, R:2 * R].contiguous()                       # my first R owned rows -> rank-1
        send_down = x[:, self.rows:self.rows + R].contiguous()     # my last R owned rows  -> rank+1
        recv_up = torch.zeros_like(send_up)                         # rank-1's last rows -> my top halo
        recv_down = torch.zeros_like(send_down)                     # rank+1's first rows -> my bottom halo
        ops = []
        if up >= 0:
            ops.append(dist.P2POp(dist.isend, send_up, up, self.group))
            ops.append(dist.P2POp(dist.irecv, recv_up, up, self.group))
        if down < self.world:
            ops.append(dist.P2POp(dist.isend, send_down, down, self.group))
            ops.append(dist.P2POp(dist.irecv, recv_down, down, self.group))
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        x[:, :R] = recv_up
        x[:, R + self.rows:] = recv_down

    def step(self, iters: int):
        """One JKO step: b <- 1; iters x (a = mu / K b ; b = prox(K a) / K a); s = b K a; normalise."""
        self.b.fill_(1.0)
        if self.p2p:
            # halo rows of b start as the neighbours' b (= 1) or the zero padding at the global edges; after
            # that the neighbours' epilogues fill them (ordered by the device barrier after each conv: a
            # rank's next conv, which reads its halos, runs after every rank's previous conv finished)
            R = self.R
            if R > 0 and self.rank == 0:
                self.b[:, :R].zero_()
            if R > 0 and self.rank == self.world - 1:
                self.b[:, R + self.rows:].zero_()
            for _ in range(iters):
                self.ops.divide(self.b, self.mu, self.a, slab=self._slabs[0])
                self._hdl[0].barrier(channel=0)
                self.ops.prox(self.a, self.b, self.prox, slab=self._slabs[1])
                self._hdl[1].barrier(channel=0)
        for _ in range(0 if self.p2p else iters):
            self.halo_exchange(self.b)
            self.ops.divide(self.b, self.mu, self.a)
            self.halo_exchange(self.a)
            self.ops.prox(self.a, self.b, self.prox)
        # s = b * K a (the last prox's input), then mu_{k+1} = s / sum s over all slabs
        self.ops.multiply(self.a, self.b, self.mu)                  # mu <- b * K a = s (halo rows junk)
        local = self.ops.sum_rows(self.mu, self.R, self.rows)
        mass = torch.tensor([local], dtype=torch.float64)
        if self.world > 1:
            if dist.get_backend(self.group) == "nccl":
                mass = mass.cuda()
            dist.all_reduce(mass, op=dist.ReduceOp.SUM, group=self.group)
        m = float(mass.item())
        self.ops.scale_rows(self.mu, self.R, self.rows, 1.0 / m)
        return m
