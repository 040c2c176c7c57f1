"""Multi-process (world_size 2, gloo, CPU) tests of the multi-GPU decompositions in
paper_2402_15322_b200/parallel.py.  The per-rank arithmetic is supplied by an oracle-backed ops
object (test-side only), so what is tested here is the decomposition itself: the input partition and
the log-mean allreduce of the sharded barycenter, and the slab partition, halo exchange, shifted
potential and mass allreduce of the slab JKO -- against the unsharded oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2402_15322_b200.parallel import ShardedBarycenter, SlabJKO, partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleOps:
    """fp64 CPU arithmetic from the oracle, with the CudaOps interface."""

    def __init__(self, T, L, log, eps=None, global_ny=None, nx=None):
        self.T, self.L, self.log = T, L, log
        self.eps, self.gny, self.nx = eps, global_ny, nx

    def _conv(self, x):
        return O.lse_conv(self.L, x.numpy()) if self.log else O.conv(self.T, x.numpy())

    def divide(self, x, target, out):
        y = self._conv(x)
        t = target.numpy()
        out.copy_(torch.from_numpy(np.where(t == -np.inf, -np.inf, t - y) if self.log
                                   else t / np.maximum(y, O.DIV_FLOOR)))

    def multiply(self, x, target, out):
        y = self._conv(x)
        out.copy_(torch.from_numpy(target.numpy() + y if self.log else target.numpy() * y))

    def prox(self, x, out, prox):
        tau, row_off = prox
        z = np.maximum(O.conv(self.T, x.numpy()), O.DIV_FLOOR)
        nt, ny_loc, nx = z.shape
        X = (np.arange(nx) + 0.5) / self.nx
        Y = (np.arange(ny_loc) + row_off + 0.5) / self.gny
        V = (X[None, None, :] - 0.5) ** 2 + (Y[None, :, None] - 0.5) ** 2
        p = tau / (self.eps + tau)
        out.copy_(torch.from_numpy(z ** (-p) * np.exp(-p * V)))

    def log_of(self, x):
        with np.errstate(divide="ignore"):
            return torch.from_numpy(np.log(x.numpy()))

    def reduce_update(self, sources, lv, ld, lbar, n):
        acc = np.zeros(lbar.shape)
        for t in sources:                       # rank order
            acc = acc + t.numpy()
        lbar.copy_(torch.from_numpy(acc))
        if n > 0:
            lv += lbar[None] - ld

    def logmean(self, ld, lam, out):
        acc = np.zeros(out.shape)
        for i, l in enumerate(lam):
            if l != 0.0:
                acc = acc + l * ld[i].numpy()
        out.copy_(torch.from_numpy(acc))

    def bary_update(self, lv, ld, lbar, n):
        lv += lbar[None] - ld

    def sum_rows(self, x, row0, rows):
        return float(x[..., row0:row0 + rows, :].sum())

    def scale_rows(self, x, row0, rows, f):
        x[..., row0:row0 + rows, :] *= f


def _bary_fused_worker(rank, world, port, q):
    """The fused reduce + update exchange (GatherExchange transport, the P2P driver's sequence)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = O.Grid(12, 10, 8)
        T = O.kernel_table(g, 2, 0.05, (1, 3, 1))
        L = O.log_kernel_table(g, 2, 0.05, (1, 3, 1))
        rng = np.random.default_rng(0)
        mus = [rng.random(g.shape) ** 3 + 1e-3 for _ in range(3)]
        mus = [m / m.sum() for m in mus]
        lam = np.array([0.2, 0.5, 0.3])
        lo, hi = partition(3, world, rank)
        local = torch.from_numpy(np.stack(mus[lo:hi])) if hi > lo else torch.zeros((0,) + g.shape, dtype=torch.float64)
        drv = ShardedBarycenter(OracleOps(T, L, True), local, lam[lo:hi], exchange="gather")
        lbar = drv.iterate(12).numpy().copy()
        ref = O.barycenter(T, L, mus, lam, 12, log_domain=True, trace=False)["lbary"]
        errs = [None] * world
        dist.all_gather_object(errs, float(np.max(np.abs(lbar - ref))))
        if rank == 0:
            q.put(max(errs))
    finally:
        dist.destroy_process_group()


def _bary_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = O.Grid(12, 10, 8)
        T = O.kernel_table(g, 2, 0.05, (1, 3, 1))
        L = O.log_kernel_table(g, 2, 0.05, (1, 3, 1))
        rng = np.random.default_rng(0)
        mus = [rng.random(g.shape) ** 3 + 1e-3 for _ in range(3)]
        mus = [m / m.sum() for m in mus]
        lam = np.array([0.2, 0.5, 0.3])
        lo, hi = partition(3, world, rank)
        drv = ShardedBarycenter(OracleOps(T, L, True), torch.from_numpy(np.stack(mus[lo:hi])), lam[lo:hi])
        lbar = drv.iterate(12).numpy().copy()
        if rank == 0:
            ref = O.barycenter(T, L, mus, lam, 12, log_domain=True, trace=False)["lbary"]
            q.put(float(np.max(np.abs(lbar - ref))))
    finally:
        dist.destroy_process_group()


def _slab_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, nt, R, eps, tau = 12, 11, 8, 2, 0.05, 0.02
        g = O.Grid(nx, ny, nt)
        T = O.kernel_table(g, R, eps, (1, 3, 1))      # cell sizes of the GLOBAL grid (R1)
        rng = np.random.default_rng(1)
        mu = rng.random(g.shape) + 0.05
        mu /= mu.sum()
        r0, r1 = partition(ny, world, rank)
        ops = OracleOps(T, None, False, eps=eps, global_ny=ny, nx=nx)
        drv = SlabJKO(ops, torch.from_numpy(mu[:, r0:r1].copy()), R, prox=(tau, r0 - R))
        masses = [drv.step(15) for _ in range(2)]
        owned = drv.owned(drv.mu).numpy().copy()
        full = [None] * world
        dist.all_gather_object(full, (r0, r1, owned))
        if rank == 0:
            out = np.zeros(g.shape)
            for a, b, o in full:
                out[:, a:b] = o
            ref = O.jko(T, None, mu, g, eps, tau, 2, 15, log_domain=False, trace=False)
            q.put((float(np.max(np.abs(out - ref["mus"][2]) / ref["mus"][2])),
                   float(np.max(np.abs(np.array(masses) - ref["masses"])))))
    finally:
        dist.destroy_process_group()


def _run(worker, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    mp.start_processes(worker, args=(world, port, q), nprocs=world, join=True, start_method="spawn")
    return q.get()


def test_partition():
    for n in (1, 3, 4, 7, 256):
        for w in (1, 2, 3, 8):
            parts = [partition(n, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_sharded_barycenter_gloo():
    err = _run(_bary_worker)
    assert err < 1e-10, err


def test_slab_jko_gloo():
    rel, dmass = _run(_slab_worker)
    assert rel < 1e-10 and dmass < 1e-12, (rel, dmass)


def _thin_slab_worker(rank, world, port, q):
    """4 ranks on 6 rows with R = 2: ranks own 2, 2, 1, 1 rows -- thinner than the halo, rejected on every rank."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, nt, R = 8, 6, 4, 2
        g = O.Grid(nx, ny, nt)
        T = O.kernel_table(g, R, 0.05, (1, 3, 1))
        mu = np.full(g.shape, 1.0 / (nx * ny * nt))
        r0, r1 = partition(ny, world, rank)
        ops = OracleOps(T, None, False, eps=0.05, global_ny=ny, nx=nx)
        try:
            SlabJKO(ops, torch.from_numpy(mu[:, r0:r1].copy()), R, prox=(0.02, r0 - R))
            msg = "accepted"
        except ValueError as e:
            msg = str(e)
        msgs = [None] * world
        dist.all_gather_object(msgs, msg)
        if rank == 0:
            q.put(msgs)
    finally:
        dist.destroy_process_group()


def test_slab_jko_rejects_slabs_thinner_than_the_halo_gloo():
    msgs = _run(_thin_slab_worker, world=4)
    assert all("rows per rank" in m for m in msgs), msgs


def _empty_rank_worker(rank, world, port, q):
    """3 ranks, 2 inputs: rank 2 owns none and still takes part in the allreduce."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = O.Grid(10, 8, 4)
        T = O.kernel_table(g, 2, 0.1, (1, 2, 1))
        L = O.log_kernel_table(g, 2, 0.1, (1, 2, 1))
        rng = np.random.default_rng(3)
        mus = [rng.random(g.shape) + 0.05 for _ in range(2)]
        mus = [m / m.sum() for m in mus]
        lam = np.array([0.6, 0.4])
        lo, hi = partition(2, world, rank)
        local = torch.from_numpy(np.stack(mus[lo:hi])) if hi > lo else torch.zeros((0,) + g.shape, dtype=torch.float64)
        drv = ShardedBarycenter(OracleOps(T, L, True), local, lam[lo:hi])
        lbar = drv.iterate(6).numpy().copy()
        ref = O.barycenter(T, L, mus, lam, 6, log_domain=True, trace=False)["lbary"]
        err = float(np.max(np.abs(lbar - ref)))
        errs = [None] * world
        dist.all_gather_object(errs, err)
        if rank == 0:
            q.put(max(errs))
    finally:
        dist.destroy_process_group()


def test_sharded_barycenter_rank_without_inputs_gloo():
    assert _run(_empty_rank_worker, world=3) < 1e-10


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_barycenter_fused_exchange_gloo(world):
    """The fused exchange sequence (slot per parity, gather of every rank's partial, one reduce + update
    per iteration), ranks 2 and 4 (4 > 3 inputs: one rank owns none)."""
    assert _run(_bary_fused_worker, world=world) < 1e-10
