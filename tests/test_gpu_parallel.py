"""The multi-GPU drivers (parallel.py) on one GPU with the CUDA ops backend, against the oracle
(world size 1: the same code path minus the collectives; the exchanges themselves are covered by
tests/test_parallel_gloo.py)."""
import numpy as np
import pytest
import torch

import oracle as O
from gpu_util import measure_err, potential_err

pytestmark = pytest.mark.gpu


def test_sharded_barycenter_single_rank(cuda_device):
    from paper_2402_15322_b200 import Kernel
    from paper_2402_15322_b200.parallel import CudaOps, ShardedBarycenter
    nx, ny, nt, R, eps, w = 40, 36, 16, 5, 0.02, (1.0, 3.0, 1.0)
    g = O.Grid(nx, ny, nt)
    rng = np.random.default_rng(0)
    mus = [(rng.random(g.shape) ** 3 + 1e-3).astype(np.float32) for _ in range(3)]
    mus = [(m / m.sum()).astype(np.float32) for m in mus]
    lam = np.array([0.2, 0.5, 0.3])
    k = Kernel(nx, ny, nt, eps, w, R, max_batch=3)
    drv = ShardedBarycenter(CudaOps(k, True), torch.from_numpy(np.stack(mus)).cuda(), lam)
    lbar = drv.iterate(30).cpu().numpy().astype(np.float64)
    ref = O.barycenter(O.kernel_table(g, R, eps, w), O.log_kernel_table(g, R, eps, w),
                       [m.astype(np.float64) for m in mus], lam, 30, log_domain=True, trace=False)
    assert potential_err(lbar, ref["lbary"]) < 1e-4
    assert measure_err(np.exp(lbar), ref["bary"]) < 1e-4


@pytest.mark.parametrize("engine", ["default", "tc"])
def test_slab_jko_single_rank(engine, cuda_device, monkeypatch):
    """engine tc: K10 made the default linear engine of the slab kernels (SE2_TC_DEFAULT=1 at build)."""
    if engine == "tc":
        monkeypatch.setenv("SE2_TC_DEFAULT", "1")
    from paper_2402_15322_b200 import Kernel, make_prox
    from paper_2402_15322_b200.parallel import CudaOps, SlabJKO
    nx, ny, nt, R, eps, tau = 48, 40, 16, 4, 0.003, 1e-3
    g = O.Grid(nx, ny, nt)
    rng = np.random.default_rng(1)
    mu = (rng.random(g.shape) + 0.05)
    mu = (mu / mu.sum()).astype(np.float32)
    # slab kernel: the grid plus R halo rows on each side, global cell sizes (R1)
    k = Kernel(nx, ny + 2 * R, nt, eps, (1, 3, 1), R, hx=1.0 / nx, hy=1.0 / ny)
    assert k.uses_tensor_cores == (engine == "tc")
    prox = make_prox(k, tau, global_ny=ny, row_offset=-R)
    drv = SlabJKO(CudaOps(k, False), torch.from_numpy(mu).cuda(), R, prox)
    masses = [drv.step(50) for _ in range(2)]
    out = drv.owned(drv.mu).cpu().numpy().astype(np.float64)
    ref = O.jko(O.kernel_table(g, R, eps, (1, 3, 1)), None, mu.astype(np.float64), g, eps, tau, 2, 50,
                log_domain=False, trace=False)
    assert measure_err(out, ref["mus"][2]) < 1e-4
    np.testing.assert_allclose(masses, ref["masses"], rtol=1e-4)


def test_bary_reduce_update_kernel(cuda_device):
    """se2_bary_reduce_update on simulated peers (three local buffers behind a device pointer table):
    lbar = sum in rank order, lv_i += lbar - ld_i."""
    from paper_2402_15322_b200.api import se2_bary_reduce_update
    rng = np.random.default_rng(5)
    N, n = 1000, 2
    parts = [torch.from_numpy(rng.normal(size=N).astype(np.float32)).cuda() for _ in range(3)]
    table = torch.tensor([p.data_ptr() for p in parts], dtype=torch.int64, device="cuda")
    lv0 = rng.normal(size=(n, N)).astype(np.float32)
    ld = rng.normal(size=(n, N)).astype(np.float32)
    lv = torch.from_numpy(lv0.copy()).cuda()
    lbar = torch.empty(N, device="cuda")
    se2_bary_reduce_update(table, n, N, lv, torch.from_numpy(ld).cuda(), lbar)
    torch.cuda.synchronize()
    ref = (parts[0].cpu().numpy() + parts[1].cpu().numpy()) + parts[2].cpu().numpy()   # float32, rank order
    assert np.array_equal(lbar.cpu().numpy(), ref)
    assert np.allclose(lv.cpu().numpy(), lv0 + (ref[None] - ld), rtol=0, atol=1e-6)
    se2_bary_reduce_update(table, 0, N, None, None, lbar)          # a rank without inputs
    assert np.array_equal(lbar.cpu().numpy(), ref)


def _one_rank_group():
    import socket
    import torch.distributed as dist
    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    return dist


@pytest.mark.parametrize("exchange", ["p2p", "gather"])
def test_sharded_barycenter_fused_exchange_single_rank(exchange, cuda_device):
    """The fused exchange on a 1-rank NCCL group: symmetric-memory slots + device barrier + the
    reduce/update kernel (p2p), or all_gather copies into the same kernel (gather), against the oracle."""
    from paper_2402_15322_b200 import Kernel
    from paper_2402_15322_b200.parallel import CudaOps, ShardedBarycenter
    _one_rank_group()
    nx, ny, nt, R, eps, w = 40, 36, 16, 5, 0.02, (1.0, 3.0, 1.0)
    g = O.Grid(nx, ny, nt)
    rng = np.random.default_rng(0)
    mus = [(rng.random(g.shape) ** 3 + 1e-3).astype(np.float32) for _ in range(3)]
    mus = [(m / m.sum()).astype(np.float32) for m in mus]
    lam = np.array([0.2, 0.5, 0.3])
    k = Kernel(nx, ny, nt, eps, w, R, max_batch=3)
    drv = ShardedBarycenter(CudaOps(k, True), torch.from_numpy(np.stack(mus)).cuda(), lam, exchange=exchange)
    lbar = drv.iterate(30).cpu().numpy().astype(np.float64)
    ref = O.barycenter(O.kernel_table(g, R, eps, w), O.log_kernel_table(g, R, eps, w),
                       [m.astype(np.float64) for m in mus], lam, 30, log_domain=True, trace=False)
    assert potential_err(lbar, ref["lbary"]) < 1e-4
    assert measure_err(np.exp(lbar), ref["bary"]) < 1e-4


@pytest.mark.parametrize("engine", ["default", "tc"])
@pytest.mark.parametrize("split", [(21,), (13, 11)], ids=["2-slabs", "3-slabs"])
def test_slab_jko_peer_halos_simulated_ranks(split, engine, cuda_device, monkeypatch):
    """se2_conv_update_slab: each slab's conv stores its owned rows and writes its boundary rows straight
    into the neighbours' halo rows (what peer-mapped memory gives across GPUs).  Here the slabs of 2 or
    3 'ranks' live on one GPU and run one after the other on one stream (stream order stands in for the
    cross-rank barrier -- no kernel waits on another); 2 JKO steps x 50 iterations against the
    unsharded oracle."""
    if engine == "tc":      # K10 as the slab kernels' default engine: its epilogue writes the peer halos
        monkeypatch.setenv("SE2_TC_DEFAULT", "1")
    from paper_2402_15322_b200 import Kernel, make_prox
    from paper_2402_15322_b200 import _lib as Lb
    from paper_2402_15322_b200.api import se2_conv_update, se2_sum_rows, se2_scale_rows
    nx, ny, nt, R, eps, tau, w = 48, 40, 16, 4, 0.003, 1e-3, (1.0, 3.0, 1.0)
    g = O.Grid(nx, ny, nt)
    rng = np.random.default_rng(1)
    mu = (rng.random(g.shape) + 0.05)
    mu = (mu / mu.sum()).astype(np.float32)
    cuts = [0] + list(np.cumsum(split)) + [ny]
    slabs = [(cuts[i], cuts[i + 1]) for i in range(len(cuts) - 1)]
    S = len(slabs)
    ks, proxes, A, B, M = [], [], [], [], []
    for r0, r1 in slabs:
        rows = r1 - r0
        k = Kernel(nx, rows + 2 * R, nt, eps, w, R, hx=1.0 / nx, hy=1.0 / ny)
        ks.append(k)
        proxes.append(make_prox(k, tau, global_ny=ny, row_offset=r0 - R))
        A.append(torch.zeros((nt, rows + 2 * R, nx), device="cuda"))
        B.append(torch.zeros((nt, rows + 2 * R, nx), device="cuda"))
        m = torch.zeros((nt, rows + 2 * R, nx), device="cuda")
        m[:, R:R + rows] = torch.from_numpy(mu[:, r0:r1]).cuda()
        M.append(m)

    def slab_struct(i, arrs):
        r0, r1 = slabs[i]
        rows = r1 - r0
        s = Lb.se2_slab(R, R + rows, R, None, 0, 0, None, 0, 0)
        if i > 0:                       # my top owned rows -> the upper slab's bottom halo
            rows_up = slabs[i - 1][1] - slabs[i - 1][0]
            s.up, s.up_shift, s.ny_up = arrs[i - 1].data_ptr(), rows_up, rows_up + 2 * R
        if i < S - 1:                   # my bottom owned rows -> the lower slab's top halo
            s.dn, s.dn_shift, s.ny_dn = arrs[i + 1].data_ptr(), rows, slabs[i + 1][1] - slabs[i + 1][0] + 2 * R
        return s

    sa = [slab_struct(i, A) for i in range(S)]
    sb = [slab_struct(i, B) for i in range(S)]
    masses = []
    for _ in range(2):
        for i in range(S):
            B[i].fill_(1.0)
        B[0][:, :R] = 0.0
        B[-1][:, B[-1].shape[1] - R:] = 0.0
        for _ in range(50):
            for i in range(S):
                se2_conv_update(ks[i], B[i], M[i], A[i], Lb.SE2_EPI_DIVIDE, False, slab=sa[i])
            for i in range(S):
                se2_conv_update(ks[i], A[i], None, B[i], Lb.SE2_EPI_PROX, False, prox=proxes[i], slab=sb[i])
        for i in range(S):      # s = b K a on the owned rows (no halo writes)
            r0, r1 = slabs[i]
            se2_conv_update(ks[i], A[i], B[i], M[i], Lb.SE2_EPI_MULTIPLY, False,
                            slab=Lb.se2_slab(R, R + r1 - r0, 0, None, 0, 0, None, 0, 0))
        tot = sum(se2_sum_rows(M[i], R, slabs[i][1] - slabs[i][0]) for i in range(S))
        for i in range(S):
            se2_scale_rows(M[i], R, slabs[i][1] - slabs[i][0], 1.0 / tot)
        masses.append(tot)
    out = np.concatenate([M[i][:, R:R + slabs[i][1] - slabs[i][0]].cpu().numpy() for i in range(S)], axis=1)
    ref = O.jko(O.kernel_table(g, R, eps, w), None, mu.astype(np.float64), g, eps, tau, 2, 50,
                log_domain=False, trace=False)
    assert measure_err(out.astype(np.float64), ref["mus"][2]) < 1e-4
    np.testing.assert_allclose(masses, ref["masses"], rtol=1e-4)


@pytest.mark.parametrize("engine", ["default", "tc"])
def test_slab_jko_p2p_single_rank(engine, cuda_device, monkeypatch):
    """SlabJKO with the peer-memory halo path (symmetric memory slabs, se2_conv_update_slab, a device
    barrier after each conv) on a 1-rank NCCL group, against the oracle; tc: K10 as the slab engine."""
    if engine == "tc":
        monkeypatch.setenv("SE2_TC_DEFAULT", "1")
    from paper_2402_15322_b200 import Kernel, make_prox
    from paper_2402_15322_b200.parallel import CudaOps, SlabJKO
    _one_rank_group()
    nx, ny, nt, R, eps, tau = 48, 40, 16, 4, 0.003, 1e-3
    g = O.Grid(nx, ny, nt)
    rng = np.random.default_rng(1)
    mu = (rng.random(g.shape) + 0.05)
    mu = (mu / mu.sum()).astype(np.float32)
    k = Kernel(nx, ny + 2 * R, nt, eps, (1, 3, 1), R, hx=1.0 / nx, hy=1.0 / ny)
    assert k.uses_tensor_cores == (engine == "tc")
    prox = make_prox(k, tau, global_ny=ny, row_offset=-R)
    drv = SlabJKO(CudaOps(k, False), torch.from_numpy(mu).cuda(), R, prox, exchange="p2p")
    masses = [drv.step(50) for _ in range(2)]
    out = drv.owned(drv.mu).cpu().numpy().astype(np.float64)
    ref = O.jko(O.kernel_table(g, R, eps, (1, 3, 1)), None, mu.astype(np.float64), g, eps, tau, 2, 50,
                log_domain=False, trace=False)
    assert measure_err(out, ref["mus"][2]) < 1e-4
    np.testing.assert_allclose(masses, ref["masses"], rtol=1e-4)
