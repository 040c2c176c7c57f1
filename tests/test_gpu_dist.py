"""The multi-GPU solvers behind the C ABI (se2_jko_step_dist, se2_barycenter_dist; -m gpu).

One GPU is all this pool has, so the multi-rank cases run their ranks as host threads of one process
with the loopback transport (se2_comm_init_loopback): every halo exchange / allreduce is a stream-
ordered device copy or reduction ordered by CUDA events and host rendezvous -- no kernel waits on
another rank's kernel -- and the slab / shard logic is exactly the code the NCCL transport drives.
Expected values: the fp64 oracle on the whole grid (tests/ may call oracle/).
"""
import threading

import numpy as np
import pytest
import torch

import oracle as O
import se2_synth as S
from gpu_util import bary_potential_errs, measure_err, potential_err, trace_err

pytestmark = pytest.mark.gpu


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def _host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy().astype(np.float64)


def _run_ranks(n, fn):
    """fn(rank) in n host threads, each on its own CUDA stream; re-raises the first failure."""
    out, errs = [None] * n, []

    def body(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                out[r] = fn(r)
                s.synchronize()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in ts), "rank thread hung"
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("engine", ["default", "tc"])
def test_jko_dist_one_rank_is_jko_step(engine, cuda_device):
    """With one rank (no communicators) the distributed step IS se2_jko_step: bit-identical outputs."""
    from paper_2402_15322_b200 import Kernel, _lib as L, make_prox, se2_jko_step
    from paper_2402_15322_b200.dist import Dist, se2_jko_step_dist
    pc = S.get_parity_case("c4m")
    cfg, d = S.parity_inputs(pc)
    flags = L.SE2_LIN_TC if engine == "tc" else 0
    k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=1)
    prox = make_prox(k, cfg.tau)
    mu = _dev(d["mus"][0])
    outs = []
    for dist in (False, True):
        nxt, a, b = torch.empty_like(mu), torch.empty_like(mu), torch.empty_like(mu)
        if dist:
            mass, tr = se2_jko_step_dist(k, Dist(), mu, nxt, a, b, 40, prox, False, trace=True, engine_flags=flags)
        else:
            mass, tr = se2_jko_step(k, mu, nxt, a, b, 40, prox, False, trace=True, engine_flags=flags)
        outs.append((nxt, a, b, mass, tr))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    assert torch.equal(outs[0][2], outs[1][2])
    assert outs[0][3] == outs[1][3] and np.array_equal(outs[0][4], outs[1][4])


@pytest.mark.parametrize("nslabs,engine", [(2, "ffma"), (3, "ffma"), (2, "tc"), (4, "tc")])
def test_jko_dist_slabs_loopback(nslabs, engine, cuda_device):
    """The c4 decomposition: one JKO flow with the grid's rows split into slabs (owned-row convs, R-row
    halo exchange after every conv, mass / trace summed over slabs) against the fp64 oracle on the whole
    grid: 2 JKO steps x 40 inner iterations at the c4 eps / tau."""
    from paper_2402_15322_b200 import _lib as L, make_prox
    from paper_2402_15322_b200.dist import Comm, Dist, local_rows, se2_jko_step_dist, slab_kernel
    nx, ny, nt, R, eps, tau, w = 40, 44, 16, 4, 0.003, 1e-3, (1.0, 3.0, 1.0)
    flags = L.SE2_LIN_TC if engine == "tc" else L.SE2_LIN_FFMA
    g = O.Grid(nx, ny, nt)
    mu0 = S.stroke_measure(nx, ny, nt, 3, seed=77).astype(np.float64)
    ref = O.jko(O.kernel_table(g, R, eps, w), None, mu0, g, eps, tau, 2, 40, log_domain=False, trace=True)
    comms = Comm.loopback(nslabs)

    def rank(r):
        k, row0, rows, top, bot = slab_kernel(nx, ny, nt, eps, w, R, nslabs, r)
        prox = make_prox(k, tau, global_ny=ny, row_offset=row0 - top)
        d = Dist(slabs=comms[r], halo_top=top, halo_bot=bot)
        mu = _dev(local_rows(mu0, row0, rows, top, bot))
        nxt, a, b = torch.empty_like(mu), torch.empty_like(mu), torch.empty_like(mu)
        masses, trs = [], []
        for _ in range(2):
            m, tr = se2_jko_step_dist(k, d, mu, nxt, a, b, 40, prox, False, trace=True, engine_flags=flags)
            masses.append(m)
            trs.append(tr)
            mu, nxt = nxt, mu
        return row0, rows, top, _host(mu)[:, top:top + rows], masses, trs

    res = _run_ranks(nslabs, rank)
    out = np.zeros(g.shape)
    for row0, rows, top, own, masses, trs in res:
        out[:, row0:row0 + rows] = own
        np.testing.assert_allclose(masses, ref["masses"], rtol=1e-4)     # every rank sees the global mass
        for s in range(2):
            assert trace_err(trs[s], ref["err"][s]) <= 1.0
    assert measure_err(out, ref["mus"][2]) <= 1e-4


@pytest.mark.parametrize("nslabs", [2, 8])
def test_jko_dist_slabs_headline_geometry(nslabs, cuda_device):
    """The north star's c4 split at the HEADLINE geometry and length: the full 256x256x64 grid (R 15, eps 0.003),
    JKO step 0 with all 200 inner iterations, rows split into 2 / 8 slabs (8: the 8-GPU layout, 32 owned rows +
    15-row halos) over the loopback transport, default engine (K10 on every slab), against the whole-grid fp64
    oracle's golden c4f (sampled entries of mu_1 and both potentials, the mass, the 200-entry error trace)."""
    import os
    from paper_2402_15322_b200 import make_prox
    from paper_2402_15322_b200.dist import Comm, Dist, local_rows, se2_jko_step_dist, slab_kernel
    from gpu_util import potential_err
    path = os.path.join(os.path.dirname(__file__), "golden", "c4f.npz")
    if not os.path.exists(path):
        pytest.skip("golden c4f.npz not generated: run tests/golden/make_golden.py c4f")
    gold = dict(np.load(path))
    pc = S.get_parity_case("c4f")
    cfg, d = S.parity_inputs(pc)
    mu0 = d["mus"][0]
    comms = Comm.loopback(nslabs)

    def rank(r):
        k, row0, rows, top, bot = slab_kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, nslabs, r)
        assert k.uses_tensor_cores
        prox = make_prox(k, cfg.tau, global_ny=cfg.ny, row_offset=row0 - top)
        dd = Dist(slabs=comms[r], halo_top=top, halo_bot=bot)
        mu = _dev(local_rows(mu0, row0, rows, top, bot))
        nxt, a, b = torch.empty_like(mu), torch.empty_like(mu), torch.empty_like(mu)
        m, tr = se2_jko_step_dist(k, dd, mu, nxt, a, b, cfg.iters, prox, False, trace=True)
        own = slice(top, top + rows)
        res = (row0, rows, _host(nxt)[:, own], _host(a)[:, own], _host(b)[:, own], m, tr)
        k.close()
        return res

    res = _run_ranks(nslabs, rank)
    shape = (cfg.ntheta, cfg.ny, cfg.nx)
    mu1, a, b = np.zeros(shape), np.zeros(shape), np.zeros(shape)
    for row0, rows, o_mu, o_a, o_b, m, tr in res:
        mu1[:, row0:row0 + rows], a[:, row0:row0 + rows], b[:, row0:row0 + rows] = o_mu, o_a, o_b
        assert abs(m - gold["masses"][0]) <= 1e-4 * abs(gold["masses"][0])     # every rank sees the global mass
        assert trace_err(tr, gold["err"][0]) <= 1.0
    idx = gold["sample_idx"]
    assert measure_err(mu1.reshape(-1)[idx], gold["mus"][1].reshape(-1)) <= 1e-4
    assert potential_err(np.log(a.reshape(-1)[idx]), np.log(gold["a"].reshape(-1))) <= 1e-4
    assert potential_err(np.log(b.reshape(-1)[idx]), np.log(gold["b"].reshape(-1))) <= 1e-4


def test_barycenter_dist_one_rank_is_barycenter(cuda_device):
    from paper_2402_15322_b200 import Kernel, se2_barycenter
    from paper_2402_15322_b200.dist import Dist, se2_barycenter_dist
    pc = S.get_parity_case("c1")
    cfg, d = S.parity_inputs(pc)
    lams = np.stack(d["lambdas"])
    k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=10)
    mus = _dev(np.stack(d["mus"]))
    b1, t1 = se2_barycenter(k, mus, lams, 30, True, trace=True)
    b2, t2 = se2_barycenter_dist(k, Dist(), mus, lams, 30, trace=True)
    assert torch.equal(b1, b2) and np.array_equal(t1, t2)


@pytest.mark.parametrize("layout", ["inputs2", "inputs4", "inputs2xslabs2"])
def test_barycenter_dist_loopback(layout, cuda_device):
    """App. A with the 4 inputs of a c3-like problem sharded over ranks (allreduce of the weighted
    log-mean per iteration) and, for inputs2xslabs2, every input's grid split into 2 row slabs as well
    (c3's 8-GPU 'one input per GPU pair' layout at 4 ranks) -- against the fp64 oracle, 30 iterations."""
    from paper_2402_15322_b200.dist import Comm, Dist, local_rows, se2_barycenter_dist, slab_kernel
    nx, ny, nt, R, eps, w = 36, 40, 16, 6, 0.01, (1.0, 3.0, 1.0)
    g = O.Grid(nx, ny, nt)
    mus = [S.stroke_measure(nx, ny, nt, 3, seed=300 + i, sigma_px=1.5).astype(np.float64) for i in range(4)]
    lam = np.array([0.1, 0.4, 0.2, 0.3])
    iters = 30
    ref = O.barycenter(O.kernel_table(g, R, eps, w), O.log_kernel_table(g, R, eps, w), mus, lam, iters,
                       log_domain=True, trace=True)
    nin = {"inputs2": 2, "inputs4": 4, "inputs2xslabs2": 2}[layout]
    nsl = 2 if layout == "inputs2xslabs2" else 1
    world = Comm.loopback(nin * nsl)
    per = 4 // nin

    def rank(r):
        ii, si = r // nsl, r % nsl                      # input group, slab
        reduce = world[r].split(si, ii) if nin > 1 else None     # ranks with the same slab
        slabs = world[r].split(1000 + ii, si) if nsl > 1 else None   # ranks with the same inputs
        k, row0, rows, top, bot = slab_kernel(nx, ny, nt, eps, w, R, nsl, si, max_batch=per)
        d = Dist(reduce=reduce, slabs=slabs, halo_top=top, halo_bot=bot)
        sel = list(range(ii * per, (ii + 1) * per))
        m = _dev(np.stack([local_rows(mus[i], row0, rows, top, bot) for i in sel]))
        v = torch.empty((1, per) + tuple(m.shape[1:]), device="cuda")
        wst = torch.empty_like(v)
        bary, tr = se2_barycenter_dist(k, d, m, lam[sel][None], iters, v_state=v, w_state=wst, trace=True)
        return (row0, rows, top, sel, _host(bary)[0][:, top:top + rows], _host(v)[0][:, :, top:top + rows],
                _host(wst)[0][:, :, top:top + rows], tr)

    res = _run_ranks(nin * nsl, rank)
    lbar = np.zeros(g.shape)
    lv = np.zeros((4,) + g.shape)
    lw = np.zeros((4,) + g.shape)
    for row0, rows, top, sel, b, v, wv, tr in res:
        lbar[:, row0:row0 + rows] = b                 # identical on every input rank of the slab
        for j, i in enumerate(sel):
            lv[i][:, row0:row0 + rows] = v[j]
            lw[i][:, row0:row0 + rows] = wv[j]
        assert trace_err(tr[:, 0], ref["err"]) <= 1.0
    assert measure_err(np.exp(lbar), ref["bary"]) <= 1e-4
    assert potential_err(lbar, ref["lbary"]) <= 1e-4
    e = bary_potential_errs(lv, lw, ref["lv"], ref["lw"], lam)
    assert max(e.values()) <= 1e-4, e


def test_barycenter_precise_dist_one_rank_is_precise(cuda_device):
    """One rank (no communicator): se2_barycenter_precise_dist IS se2_barycenter_precise, bit for bit."""
    from paper_2402_15322_b200 import Kernel, se2_barycenter_precise
    from paper_2402_15322_b200.dist import Dist, se2_barycenter_precise_dist
    pc = S.get_parity_case("c1")
    cfg, d = S.parity_inputs(pc)
    lams = np.stack(d["lambdas"])
    k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=10)
    mus = _dev(np.stack(d["mus"]))
    b1, t1 = se2_barycenter_precise(k, mus, lams, 30, trace=True)
    b2, t2 = se2_barycenter_precise_dist(k, Dist(), mus, lams, 30, trace=True)
    assert torch.equal(b1, b2) and np.array_equal(t1, t2)


@pytest.mark.parametrize("layout", ["inputs2", "inputs4", "slabs2", "inputs2xslabs2", "slabs3"])
def test_barycenter_precise_dist_loopback(layout, cuda_device):
    """The fp64-potential barycenter with the 4 inputs of a c3-like problem sharded over ranks (fp64
    allreduce of the weighted log-mean per iteration) and/or every input's grid split into row slabs (fp64
    halo exchanges of w_i / v_i; inputs2xslabs2 is c3's 8-GPU 'one input per GPU pair' layout at 4 ranks)
    against the fp64 oracle at the north star's 1e-4 ELEMENTWISE on gauge-fixed potentials, 120 iterations."""
    from paper_2402_15322_b200.dist import Comm, Dist, local_rows, se2_barycenter_precise_dist, slab_kernel
    nx, ny, nt, R, eps, w = 36, 40, 16, 6, 0.01, (1.0, 3.0, 1.0)
    g = O.Grid(nx, ny, nt)
    mus = [S.stroke_measure(nx, ny, nt, 3, seed=300 + i, sigma_px=1.5).astype(np.float64) for i in range(4)]
    lam = np.array([0.1, 0.4, 0.2, 0.3])
    iters = 120
    ref = O.barycenter(O.kernel_table(g, R, eps, w), O.log_kernel_table(g, R, eps, w), mus, lam, iters,
                       log_domain=True, trace=True)
    nin = {"inputs2": 2, "inputs4": 4, "slabs2": 1, "inputs2xslabs2": 2, "slabs3": 1}[layout]
    nsl = {"slabs2": 2, "inputs2xslabs2": 2, "slabs3": 3}.get(layout, 1)
    world = Comm.loopback(nin * nsl)
    per = 4 // nin

    def rank(r):
        ii, si = r // nsl, r % nsl                                    # input group, slab
        reduce = world[r].split(si, ii) if nin > 1 else None          # ranks with the same slab
        slabs = world[r].split(1000 + ii, si) if nsl > 1 else None    # ranks with the same inputs
        k, row0, rows, top, bot = slab_kernel(nx, ny, nt, eps, w, R, nsl, si, max_batch=per)
        sel = list(range(ii * per, (ii + 1) * per))
        m = _dev(np.stack([local_rows(mus[i], row0, rows, top, bot) for i in sel]))
        v = torch.empty((1, per) + tuple(m.shape[1:]), device="cuda", dtype=torch.float64)
        wst = torch.empty_like(v)
        lb, tr = se2_barycenter_precise_dist(k, Dist(reduce=reduce, slabs=slabs, halo_top=top, halo_bot=bot), m,
                                             lam[sel][None], iters, lv_state=v, lw_state=wst, trace=True)
        return (row0, rows, sel, _host(lb)[0][:, top:top + rows], _host(v)[0][:, :, top:top + rows],
                _host(wst)[0][:, :, top:top + rows], tr)

    res = _run_ranks(nin * nsl, rank)
    lbar = np.zeros(g.shape)
    lv = np.zeros((4,) + g.shape)
    lw = np.zeros((4,) + g.shape)
    for row0, rows, sel, lb, v, wv, tr in res:
        lbar[:, row0:row0 + rows] = lb                # identical on every input rank of the slab
        assert trace_err(tr[:, 0], ref["err"]) <= 1.0
        for j, i in enumerate(sel):
            lv[i][:, row0:row0 + rows] = v[j]
            lw[i][:, row0:row0 + rows] = wv[j]
    assert potential_err(lbar, ref["lbary"]) <= 1e-4
    assert measure_err(np.exp(lbar), ref["bary"]) <= 1e-4
    e = bary_potential_errs(lv, lw, ref["lv"], ref["lw"], lam)
    assert max(e.values()) <= 1e-4, e


@pytest.mark.parametrize("engine", ["ffma", "tc", "log"])
def test_conv_output_window(engine, cuda_device):
    """se2_kernel_set_window: the conv computes exactly the window rows of the full conv (rows outside are
    input-only halos and are not written)."""
    from paper_2402_15322_b200 import Kernel, _lib as L, se2_conv
    nx, ny, nt, R, eps, w = 48, 40, 16, 5, 0.01, (1.0, 3.0, 1.0)
    k = Kernel(nx, ny, nt, eps, w, R, max_batch=2)
    lo, hi = 7, 29
    L.check(L.load().se2_kernel_set_window(k.handle, lo, hi))
    g = O.Grid(nx, ny, nt)
    rng = np.random.default_rng(3)
    log = engine == "log"
    x = rng.uniform(-20, 0, (2, nt, ny, nx)) if log else np.exp(rng.uniform(-10, 0, (2, nt, ny, nx)))
    x32 = x.astype(np.float32)
    out = torch.full((2, nt, ny, nx), 12345.0, device="cuda")
    flags = {"ffma": L.SE2_LIN_FFMA, "tc": L.SE2_LIN_TC}.get(engine, 0)
    se2_conv(k, _dev(x32), out, log_domain=log, extra_flags=flags)
    got = _host(out)
    ref = (O.lse_conv(O.log_kernel_table(g, R, eps, w), x32.astype(np.float64)) if log
           else O.conv(O.kernel_table(g, R, eps, w), x32.astype(np.float64)))
    assert np.all(got[:, :, :lo] == 12345.0) and np.all(got[:, :, hi:] == 12345.0)
    if log:
        assert np.max(np.abs(got[:, :, lo:hi] - ref[:, :, lo:hi])) < 1e-4
    else:
        assert np.max(np.abs(got[:, :, lo:hi] / ref[:, :, lo:hi] - 1)) < 3e-5


def test_nccl_transport_one_rank(cuda_device):
    """The NCCL transport itself on one GPU: a REAL one-rank NCCL communicator (ncclGetUniqueId +
    ncclCommInitRank through the dlopen'ed entry points), its allreduce (fp32 / fp64: a one-rank sum is the
    identity), ncclCommSplit, and the sharded barycenter solvers running their per-iteration log-mean
    allreduce on it -- inside the CUDA graph of a small solve too.  The multi-rank exchange logic is the
    loopback tests'; this pins the NCCL calls (symbols, datatypes, stream, in-place buffers, capture)."""
    from paper_2402_15322_b200 import Kernel, se2_barycenter, se2_barycenter_precise
    from paper_2402_15322_b200.dist import Comm, Dist, se2_barycenter_dist, se2_barycenter_precise_dist
    comm = Comm.nccl_one_rank(0)
    assert (comm.nranks, comm.rank) == (1, 0)
    x32 = torch.arange(100003, dtype=torch.float32, device="cuda") * 0.25
    x64 = torch.arange(4099, dtype=torch.float64, device="cuda") / 3.0
    r32, r64 = x32.clone(), x64.clone()
    comm.allreduce_(x32)
    comm.allreduce_(x64)
    torch.cuda.synchronize()
    assert torch.equal(x32, r32) and torch.equal(x64, r64)
    sub = comm.split(0, 0)
    assert (sub.nranks, sub.rank) == (1, 0)
    sub.allreduce_(x32)
    torch.cuda.synchronize()
    assert torch.equal(x32, r32)
    pc = S.get_parity_case("c1")
    cfg, d = S.parity_inputs(pc)
    lams = np.stack(d["lambdas"])
    k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=10)
    mus = _dev(np.stack(d["mus"]))
    # the allreduce path sums partial log-means and then updates (two kernels) where the one-rank path fuses
    # them: equal up to fp32 rounding of the log-mean, not bit for bit
    b1, t1 = se2_barycenter(k, mus, lams, 30, True, trace=True)
    b2, t2 = se2_barycenter_dist(k, Dist(reduce=sub), mus, lams, 30, trace=True)
    assert measure_err(np.exp(_host(b2)), np.exp(_host(b1))) < 2e-3   # the fp32 potentials' rounding floor (R19)
    assert trace_err(t2, t1) < 1.0
    p1, u1 = se2_barycenter_precise(k, mus, lams, 30, trace=True)
    p2, u2 = se2_barycenter_precise_dist(k, Dist(reduce=comm), mus, lams, 30, trace=True)
    assert potential_err(_host(p2), _host(p1)) < 1e-6
    assert trace_err(u2, u1) < 1.0
    k.close()
    sub.close()
    comm.close()
