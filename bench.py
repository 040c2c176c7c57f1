"""Benchmark of the SE(2) entropic-OT hot path (BASELINE.json metric: Sinkhorn iters/s on the SE(2)
grid + group-conv fraction of roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--workload c4]

Workload (default c4, the largest config, which fits one GPU): the entropic JKO gradient flow on
the 256x256x64 grid, eps = 0.003, w = (1,3,1), support 31x31x64, tau = 1e-3.  One step = one JKO
step = 200 inner scaling iterations (2 group convolutions each, fused prox / division / error
epilogues) + the normalisation of mu_{k+1}.  value = inner Sinkhorn iterations per second summed
of the one flow.  Multi-GPU (torchrun, N ranks): the SAME flow with the grid's rows split into N slabs
(se2_jko_step_dist: owned-row convs, R-row NCCL halo exchange after every conv) -> "scaling": "strong";
independent per-GPU flows are reported as the extra key "replicas".

Timing: W untimed warm-up steps; then K steps, each bracketed by CUDA events on the launching
stream, with an L2 flush (write of a 256 MiB buffer, outside the events) before each step; barrier
+ synchronize around the timed region; the max over ranks is reported.  `e2e` repeats the step
through the same C-ABI call with the step's input copied from pinned HOST memory and the result
copied back inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOADS = {
    "c4": "c4: entropic JKO gradient flow on 256x256x64 SE(2) grid ([0,1]^2 x [0,2pi)), eps=0.003, "
          "w=(1,3,1), support 31x31x64, tau=1e-3, V=|x-c|^2; one step = one JKO step = 200 inner "
          "scaling iterations (2 group convs each) + normalisation; linear-domain fp32",
}


def _tc_executed_flop(cfg, R, batch=1, band=5, wide_frac=0.0):
    """MMA flops K10 executes per launch (3 BF16 passes, N = nx rounded up to 16): the 'executed' rate next
    to the algorithmic one.  Mirrors conv_tc.cu's geometry choice (tc_geom / conv_tc_decide):
      * narrow geometry (nt >= 32, band <= 12): 16-row x 8-orientation M tiles, K = 16 (one K-step) on
        tiles whose bound holds and K = 32 on the rest (wide_frac of the tiles, from se2_tc_tile_stats);
      * classic (nt = 16): 8-row x 16-orientation tiles, K = all orientations;
    the balanced mode (tiles' chain units spread evenly over 148 CTAs) when its per-SM chain is below 0.95
    of the row-count mode's, else tc_rows_out's output rows per CTA (max_batch = batch)."""
    npad = (cfg.nx + 15) // 16 * 16
    nar = cfg.ntheta // 8 >= 4 and band <= 12
    kr = 16 if nar else 8
    nblk = cfg.ntheta // (128 // kr)
    S_ = 2 * R + 1
    ksteps = (1.0 - wide_frac) * 1 + wide_frac * 2 if nar else min(cfg.ntheta // 8, 4) // 2
    per_row = S_ * ksteps * 3 * 2.0 * 128 * npad * 16

    def chain(y0, rows):
        return min(cfg.ny - 1, y0 + rows - 1 + R) - max(0, y0 - R) + 1

    best, rows_out = None, kr
    for rows in range(kr, kr // 2 - 1, -1):
        ctas = -(-cfg.ny // rows) * nblk * batch
        cost = -(-ctas // 148) * min(cfg.ny, rows + 2 * R)
        if best is None or cost < best:
            best, rows_out = cost, rows
    ug = sum(chain(y0, kr) for y0 in range(0, cfg.ny, kr))
    lmax = max(chain(y0, kr) for y0 in range(0, cfg.ny, kr))
    q = max(-(-batch * nblk * ug // 148), (lmax + 1) // 2)
    if q < 0.95 * best:                      # balanced mode
        return batch * nblk * ug * per_row
    total = sum(chain(y0, rows_out) for y0 in range(0, cfg.ny, rows_out))
    return total * nblk * batch * per_row


def _conv_roofline(k, cfg, st, achieved, conv_avg_ms, flop_per_conv, n_conv, conv_ms, dev_ms, ffma_peak, sm_max,
                   peaks, peak_src, clocks, workload):
    """Roofline object of the dominant kernel (the linear group conv): K10 on the tensor cores when the
    kernel uses it, else K2 on the FP32 pipes.  achieved = ALGORITHMIC flops (2 nnz per output) / the
    average launch time measured with CUDA events on the launching stream."""
    common = {"achieved": achieved, "unit": "TFLOP/s", "flop_per_launch": flop_per_conv, "conv_launches": n_conv,
              "conv_avg_ms": conv_avg_ms, "conv_share_of_step": conv_ms / dev_ms if dev_ms else None}
    traffic_all = {}
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic_all = json.load(f)
    if k.uses_tensor_cores:
        peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1590.0)))
        ts = k.tc_tile_stats(reset=False)
        tc_wide = ts["wide"] / ts["tiles"] if ts["tiles"] else 0.0
        executed = _tc_executed_flop(cfg, cfg.R, band=st["theta_band"], wide_frac=tc_wide) / (conv_avg_ms / 1000.0) / 1e12
        return {"bound": "tensor", "kernel": "conv_tc_kernel (tcgen05 BF16, 3-pass split) + tc_split_input_kernel",
                "peak": peak, "frac": achieved / peak, "traffic": traffic_all.get(f"{workload}_conv_tc_bytes_per_launch"),
                "peak_source": f"MEASURED_PEAKS.json bf16_tflops_sustained ({peak_src}; the kernel runs inside a "
                               f"long step); dense BF16 is the dtype the MMAs execute",
                "executed_mma_tflops": executed,
                "executed_frac": executed / float(peaks.get("bf16_tflops", peak)),
                "executed_frac_vs_nominal": executed / (148 * 4096 * 2 * sm_max * 1e6 / 1e12),
                "executed_frac_note": "executed MMA rate / the BURST bf16 peak (cuBLAS 8192^3 best of 10); "
                                      "executed_frac_vs_nominal: / 148 SM x 4096 BF16 MAC/cycle x 2 x sm_max_mhz",
                "executed_note": "3 BF16 passes (hi.hi + hi.lo + lo.hi) over the 16-orientation window of each "
                                 "16-row x 8-orientation M tile (32 on tiles whose bound fails) and its 16 + 2R "
                                 "input rows: executed / algorithmic = "
                                 f"{_tc_executed_flop(cfg, cfg.R, band=st['theta_band'], wide_frac=tc_wide) / flop_per_conv:.2f}",
                "tc_tiles_wide_frac": tc_wide,
                "vs_ffma_roofline": achieved / ffma_peak, **common}
    return {"bound": "alu", "kernel": "conv_linear_kernel<15> (fp32 FFMA)", "peak": ffma_peak,
            "frac": achieved / ffma_peak, "traffic": traffic_all.get(f"{workload}_conv_linear_bytes_per_launch"),
            "peak_source": f"148 SM x 128 FP32 lanes x 2 flop x {sm_max:.0f} MHz (clock from "
                           f"MEASURED_PEAKS.json, {peak_src}); FFMA has no measured peak",
            "peak_at_run_clock": (148 * 128 * 2 * clocks["sm_mhz"] * 1e6 / 1e12) if clocks.get("sm_mhz") else None,
            **common}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (profiling recipe)."""

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _taps_1d(n, R):
    """sum over outputs i in [0,n) of #{j in [0,n): |i-j| <= R} (zero padding)."""
    i = np.arange(n)
    return int(np.sum(np.minimum(i + R, n - 1) - np.maximum(i - R, 0) + 1))


def cpu_oracle_sample(cfg, seconds_hint=15.0):
    """Time the oracle (as it stands) on a bounded sample of the workload: one group convolution over
    the first `rows` rows of the grid (its own zero-padded window), scaled to one full inner
    iteration (2 convs on the full grid) by the exact box-tap ratio.  Returns (iters/s, desc, threads)."""
    import oracle as O
    import se2_synth as S
    rows = 64 if cfg.ny >= 64 else cfg.ny
    g = O.Grid(cfg.nx, rows, cfg.ntheta)
    T = O.kernel_table(g, cfg.R, cfg.eps, cfg.w)
    v = S.random_positive_field((cfg.ntheta, rows, cfg.nx), seed=5).astype(np.float64)
    t0 = time.perf_counter()
    O.conv(T, v)
    dt = time.perf_counter() - t0
    taps_s = _taps_1d(cfg.nx, cfg.R) * _taps_1d(rows, cfg.R)
    taps_f = _taps_1d(cfg.nx, cfg.R) * _taps_1d(cfg.ny, cfg.R)
    t_iter = 2.0 * dt * taps_f / taps_s
    desc = (f"oracle fp64 conv (C loops, OpenMP) over rows 0-{rows - 1} of the {cfg.nx}x{cfg.ny}x{cfg.ntheta} "
            f"grid ({dt:.2f} s), scaled by the exact box-tap ratio to one inner iteration (2 convs)")
    return 1.0 / t_iter, desc, O.oracle_threads(), dt


def run_reference(args):
    ws, rank, _ = _dist_env()
    if rank != 0:
        return 0
    import se2_synth as S
    cfg = S.get_config(args.workload)
    vals = []
    for i in range(args.warmup + args.steps):
        v, desc, threads, dt = cpu_oracle_sample(cfg)
        if i >= args.warmup:
            vals.append(v)
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": "Sinkhorn iters/s on SE(2) grid", "value": value, "unit": "iters/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * cfg.iters / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.workload]},
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": threads, "kind": "oracle",
                         "sample": desc + " -- a PROJECTION of the oracle's iteration rate from that timed sample, "
                                          "not a timed full iteration"},
        "projected": True,
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_sweep(device: int):
    """Every BASELINE config solved once end to end on this GPU (after one warm-up solve), timed with
    CUDA events: iterations/s of the whole config (c1: all five t-values batched), conv time share,
    and for the log-domain configs the K3 path mix (pruned / FFMA / per-tap fallback pairs)."""
    import torch

    import se2_synth as S
    from paper_2402_15322_b200 import Kernel, make_prox, se2_barycenter, se2_jko_step, se2_sinkhorn
    out = {}
    for cfg in S.CONFIGS:
        d = S.config_inputs(cfg)
        n = len(d["mus"])
        lams = np.atleast_2d(np.stack(d["lambdas"])) if "lambdas" in d else None
        batch = n * (lams.shape[0] if lams is not None else 1)
        k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=max(batch, 1), device=device)
        mus = torch.from_numpy(np.stack(d["mus"])).cuda()

        def solve():
            if cfg.problem == "sinkhorn":
                a = torch.empty_like(mus[0])
                b = torch.empty_like(mus[0])
                se2_sinkhorn(k, mus[0].contiguous(), mus[1].contiguous(), a, b, cfg.iters, cfg.log_domain, trace=True)
                return cfg.iters
            if cfg.problem == "barycenter":
                se2_barycenter(k, mus, lams, cfg.iters, cfg.log_domain, trace=True)
                return cfg.iters
            prox = make_prox(k, cfg.tau)
            mu, nxt = mus[0].clone(), torch.empty_like(mus[0])
            a, b = torch.empty_like(mu), torch.empty_like(mu)
            se2_jko_step(k, mu, nxt, a, b, cfg.iters, prox, cfg.log_domain, trace=True)
            return cfg.iters

        solve()                      # warm-up (captures the CUDA graph of small solves)
        torch.cuda.synchronize()
        k.lse_path_stats(reset=True)
        k.lse_row_stats(reset=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        it = solve()                 # timed: as a user runs it (graph replay for small problems)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        ps = k.lse_path_stats(reset=True)
        rs = k.lse_row_stats(reset=True)
        k.timing_enable(True)        # instrumented re-run (direct launches) for the conv time share
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        solve()
        t1.record()
        torch.cuda.synchronize()
        ms_instr = t0.elapsed_time(t1)
        nconv, conv_ms, _ = k.timing_get()
        k.timing_enable(False)
        st = k.stats()
        rec = {"problem": cfg.problem, "grid": f"{cfg.nx}x{cfg.ny}x{cfg.ntheta}", "fields_per_conv": batch,
               "iters": it, "ms": ms, "iters_per_s": it / (ms / 1000.0), "domain": "log" if cfg.log_domain else "linear",
               "conv_share": conv_ms / ms_instr if ms_instr else None, "conv_avg_ms": conv_ms / max(nconv, 1),
               "graph": bool(batch * cfg.N <= (1 << 21))}
        if not cfg.log_domain:
            flop = 2.0 * cfg.N * st["nnz_taps"] * (batch if cfg.problem != "jko" else 1)
            rec["conv_tflops"] = flop / (rec["conv_avg_ms"] / 1000.0) / 1e12
        else:
            rec["k3_pairs"] = ps
            rec["k3_active_frac"] = ps["active"] / max(ps["visited"], 1)
            rec["k3_ffma_frac_of_active"] = ps["ffma"] / max(ps["active"], 1)
            rec["k3_exact_rows_live_frac"] = rs["live"] / max(rs["visited"], 1)
        if cfg.problem == "barycenter" and cfg.log_domain:
            # the fp64-potential engine (K4P): the one whose potentials meet the north star's 1e-4
            # elementwise (tests/test_gpu_parity.py::test_barycenter_parity_precise; R19)
            from paper_2402_15322_b200 import se2_barycenter_precise
            se2_barycenter_precise(k, mus, lams, cfg.iters, trace=True)
            torch.cuda.synchronize()
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            p0.record()
            se2_barycenter_precise(k, mus, lams, cfg.iters, trace=True)
            p1.record()
            torch.cuda.synchronize()
            pms = p0.elapsed_time(p1)
            rec["precise_fp64_potentials"] = {"ms": pms, "iters_per_s": cfg.iters / (pms / 1000.0),
                                              "engine": "K4P exact log-domain conv, fp64 potentials"}
            rec["engine"] = "K3 (fp32 potentials)"
        out[cfg.name] = rec
        k.close()
        if cfg.name == "c0":
            # c0's "replicas" unit: 64 independent c0 problems (seeds 0..63) in ONE K9 launch, one thread-block
            # cluster per problem (the batched mode of the one-launch solver): problems x iterations / s
            B = 64
            kb = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=B, device=device)
            mu_b = torch.from_numpy(np.stack([S.stroke_measure(cfg.nx, cfg.ny, cfg.ntheta, 2, seed=5000 + 2 * i)
                                              for i in range(B)]).astype(np.float32)).cuda()
            nu_b = torch.from_numpy(np.stack([S.stroke_measure(cfg.nx, cfg.ny, cfg.ntheta, 2, seed=5001 + 2 * i)
                                              for i in range(B)]).astype(np.float32)).cuda()
            a_b, b_b = torch.empty_like(mu_b), torch.empty_like(mu_b)
            se2_sinkhorn(kb, mu_b, nu_b, a_b, b_b, cfg.iters, True, trace=True)
            torch.cuda.synchronize()
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            q0.record()
            se2_sinkhorn(kb, mu_b, nu_b, a_b, b_b, cfg.iters, True, trace=True)
            q1.record()
            torch.cuda.synchronize()
            qms = q0.elapsed_time(q1)
            out["c0_batched64"] = {"problems": B, "iters": cfg.iters, "ms": qms,
                                   "problem_iters_per_s": B * cfg.iters / (qms / 1000.0),
                                   "engine": "K9, one cluster per problem in one launch"}
            kb.close()
    return out


def next_rows(device: int):
    """The SURVEY §8f NEXT rows built beyond the scaling loop, each measured (CUDA events, after a
    warm-up) at a paper-sized workload:
      #1 porous-medium JKO (m = 5, w = (1, sqrt 10, sqrt 2)) on the c4 grid, one JKO step of
         200 inner iterations -> inner iterations/s;
      #2 transport cost <pi, rho_b^2> of a c4 plan (one conv with the cost table) -> ms and TFLOP/s;
      #3 lifting: the orientation-score correlation of a 256 x 256 image at 64 orientations (21 x 21
         cake wavelets) -> ms and TFLOP/s (2 N L^2 flop) vs the FFMA peak, and the whole image
         interpolation (Steps 1-4) on c1's 28 x 28 x 16 grid for 5 t-values x 200 iterations."""
    import math

    import torch

    import se2_synth as S
    from paper_2402_15322_b200 import (Cake, Kernel, interpolate_images, make_porous_prox, make_prox, se2_jko_step,
                                       se2_lift_image, se2_sinkhorn, se2_transport_cost)

    def timed(fn, reps=1):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    out = {}
    peak = 148 * 128 * 2 * 1.965e9 / 1e12
    cfg = S.get_config("c4")
    d = S.config_inputs(cfg)
    w5 = (1.0, math.sqrt(10.0), math.sqrt(2.0))
    k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, w5, cfg.R, max_batch=1, device=device)
    mu = torch.from_numpy(d["mus"][0]).cuda()
    nxt, a, b = torch.empty_like(mu), torch.empty_like(mu), torch.empty_like(mu)
    prox = make_porous_prox(cfg.tau, 5.0)
    ms = timed(lambda: se2_jko_step(k, mu, nxt, a, b, cfg.iters, prox, log_domain=False, trace=False))
    out["porous_jko_c4"] = {"workload": "porous-medium JKO step (m = 5, w = (1, sqrt 10, sqrt 2)) on 256x256x64, "
                                        "200 inner iterations", "ms_per_step": ms,
                            "inner_iters_per_s": cfg.iters / (ms / 1000.0)}
    k.close()
    k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=1, device=device)
    se2_jko_step(k, mu, nxt, a, b, cfg.iters, make_prox(k, cfg.tau), log_domain=False, trace=False)
    ms = timed(lambda: se2_transport_cost(k, a, b, False), reps=5)
    flop = 2.0 * cfg.N * k.stats()["nnz_taps"]
    engine = "K10 (tensor cores, cost-table weights)" if k.uses_tensor_cores else "K2 (FFMA)"
    out["transport_cost_c4"] = {"workload": "<pi, rho_b^2> of the c4 JKO plan (one cost-table conv + dot)",
                                "engine": engine, "ms": ms, "tflops": flop / (ms / 1000.0) / 1e12,
                                "algorithmic_vs_ffma_peak": flop / (ms / 1000.0) / 1e12 / peak}
    k.close()
    c = Cake(64, 21, device=device)
    y, x = np.mgrid[0:256, 0:256]
    img = torch.from_numpy(np.exp(-((x - 128.0) ** 2 + (y - 100.0) ** 2) / 800.0).astype(np.float32)).cuda()
    U = torch.empty((1, 64, 256, 256), device="cuda")
    ms = timed(lambda: se2_lift_image(c, img, U), reps=10)
    flop = 2.0 * 64 * 256 * 256 * 21 * 21
    out["lift_image_256"] = {"workload": "orientation score of a 256x256 image, 64 cake wavelets 21x21", "ms": ms,
                             "tflops": flop / (ms / 1000.0) / 1e12, "frac_of_ffma_peak": flop / (ms / 1000.0) / 1e12 / peak}
    c.close()
    c1 = S.get_config("c1")
    c = Cake(c1.ntheta, 15, device=device)
    kk = Kernel(c1.nx, c1.ny, c1.ntheta, c1.eps, c1.w, c1.R, max_batch=10, device=device)
    rng = np.random.default_rng(5)
    f0, f1 = (torch.from_numpy(rng.random((28, 28)).astype(np.float32) ** 4).cuda() for _ in range(2))
    ts = [0.0, 0.25, 0.5, 0.75, 1.0]
    ms = timed(lambda: interpolate_images(kk, c, f0, f1, ts, c1.iters))
    out["interpolate_images_c1"] = {"workload": "image interpolation (lift, +/- split, 2 x 5 barycenters of 200 "
                                                "log-domain iterations, signed projection) on 28x28x16", "ms": ms}
    kk.close()
    c.close()
    return out


def sharded_barycenter(ws: int, rank: int, local: int, world, iters: int = 500):
    """c3's barycenter (4 inputs, 128x128x32, log domain) through se2_barycenter_dist: the inputs sharded
    over the ranks (NCCL allreduce of the partial weighted log-mean, 2 MB, every iteration) and, at 8
    ranks, each input's grid split into 2 row slabs as well ("sharded one input per GPU pair",
    B:configs[3]; halo exchange of w_i and v_i per iteration).  Strong scaling of one problem.
    Returns iterations/s (max device time over ranks, CUDA events)."""
    import torch
    import torch.distributed as dist

    import se2_synth as S
    from paper_2402_15322_b200.dist import Dist, local_rows, se2_barycenter_dist, slab_kernel
    from paper_2402_15322_b200.parallel import partition
    cfg = S.get_config("c3")
    d = S.config_inputs(cfg)
    lam = np.asarray(d["lambdas"][0])
    nin = min(ws, 4)                      # input groups
    nsl = ws // nin if ws % nin == 0 else 1
    if nin * nsl != ws:
        nin, nsl = ws, 1
    ii, si = rank // nsl, rank % nsl
    lo, hi = partition(4, nin, ii)
    reduce = world.split(si, ii) if world is not None and nin > 1 else None
    slabs = world.split(1000 + ii, si) if world is not None and nsl > 1 else None
    k, row0, rows, top, bot = slab_kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, nsl, si,
                                          max_batch=max(hi - lo, 1), device=local)
    dd = Dist(reduce=reduce, slabs=slabs, halo_top=top, halo_bot=bot)
    mus = torch.from_numpy(np.stack([local_rows(m, row0, rows, top, bot) for m in d["mus"][lo:hi]])).cuda()
    lam_local = lam[lo:hi][None]
    se2_barycenter_dist(k, dd, mus, lam_local, 2)   # warm-up (graph capture at 1 rank)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    se2_barycenter_dist(k, dd, mus, lam_local, iters)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"workload": f"c3 barycenter (4 inputs, 128x128x32, log domain) via se2_barycenter_dist: {nin} input "
                        f"group(s) x {nsl} row slab(s); NCCL allreduce of the weighted log-mean per iteration"
                        + ("; halo exchange of w_i, v_i" if nsl > 1 else ""),
            "iters": iters, "ms": ms, "iters_per_s": iters / (ms / 1000.0), "n_gpus": ws}


def sharded_barycenter_precise(ws: int, rank: int, local: int, world, iters: int = 500):
    """c3's barycenter with fp64 potentials (the engine meeting the north star's 1e-4 on potentials, R19)
    through se2_barycenter_precise_dist: the 4 inputs sharded over min(N, 4) ranks, fp64 allreduce of the
    weighted log-mean per iteration (ranks beyond 4 idle).  Returns iterations/s (max device time)."""
    import torch
    import torch.distributed as dist

    import se2_synth as S
    from paper_2402_15322_b200 import Kernel
    from paper_2402_15322_b200.dist import Dist, se2_barycenter_precise_dist
    from paper_2402_15322_b200.parallel import partition
    cfg = S.get_config("c3")
    d = S.config_inputs(cfg)
    lam = np.asarray(d["lambdas"][0])
    nin = min(ws, 4)
    sub = world.split(0 if rank < nin else 1, rank) if world is not None else None
    ms = 0.0
    if rank < nin:
        lo, hi = partition(4, nin, rank)
        k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=max(hi - lo, 1), device=local)
        dd = Dist(reduce=sub if nin > 1 else None)
        mus = torch.from_numpy(np.stack(d["mus"][lo:hi])).cuda()
        se2_barycenter_precise_dist(k, dd, mus, lam[lo:hi][None], 2)
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    if rank < nin:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        se2_barycenter_precise_dist(k, dd, mus, lam[lo:hi][None], iters)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        k.close()
    if ws > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if sub is not None:
        sub.close()
    return {"workload": f"c3 barycenter (4 inputs, 128x128x32, log domain, fp64 potentials: K4P) via "
                        f"se2_barycenter_precise_dist: inputs over {nin} rank(s), fp64 allreduce of the weighted "
                        f"log-mean per iteration", "iters": iters, "ms": ms, "iters_per_s": iters / (ms / 1000.0),
            "n_gpus_used": nin}


def c1_tvalues(ws: int, rank: int, local: int):
    """c1's five t-values distributed over the ranks (5 / 3 / 2 / 1 per GPU at 1 / 2 / 4 / 8;
    no collective), each rank solving its share of the interpolation batched, fp64 potentials (K4P).
    Returns barycenter iterations/s summed over all t-values (max device time over ranks)."""
    import torch
    import torch.distributed as dist

    import se2_synth as S
    from paper_2402_15322_b200 import Kernel, se2_barycenter_precise
    from paper_2402_15322_b200.parallel import partition
    cfg = S.get_config("c1")
    d = S.config_inputs(cfg)
    lams_all = np.atleast_2d(np.stack(d["lambdas"]))
    lo, hi = partition(lams_all.shape[0], ws, rank)
    ms = 0.0
    k = None
    if hi > lo:
        k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=2 * (hi - lo), device=local)
        mus = torch.from_numpy(np.stack(d["mus"])).cuda()
        se2_barycenter_precise(k, mus, lams_all[lo:hi], cfg.iters)
        torch.cuda.synchronize()
    dist.barrier()
    if k is not None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        se2_barycenter_precise(k, mus, lams_all[lo:hi], cfg.iters)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        k.close()
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"workload": f"c1: 5 t-values x 200 barycenter iterations (fp64 potentials), split over {ws} GPUs",
            "ms": ms, "solve_iters_per_s": lams_all.shape[0] * cfg.iters / (ms / 1000.0), "scaling": "strong"}


def replicas(ws: int, rank: int, local: int, cfg, d, steps: int = 2):
    """Every rank runs its own c4 JKO flow (independent problems, no collective): the weak-scaling extra."""
    import torch
    import torch.distributed as dist

    from paper_2402_15322_b200 import Kernel, make_prox, se2_jko_step
    k = Kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, max_batch=1, device=local)
    prox = make_prox(k, cfg.tau)
    mu = torch.from_numpy(d["mus"][0]).cuda()
    nxt, a, b = torch.empty_like(mu), torch.empty_like(mu), torch.empty_like(mu)
    se2_jko_step(k, mu, nxt, a, b, cfg.iters, prox, log_domain=False)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        se2_jko_step(k, mu, nxt, a, b, cfg.iters, prox, log_domain=False)
        mu, nxt = nxt, mu
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    k.close()
    return {"workload": f"{ws} independent c4 JKO flows (one per GPU, no collective)", "value": ws * cfg.iters * steps /
            (float(t.item()) / 1000.0), "unit": "iters/s", "scaling": "weak"}


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import se2_synth as S
    from paper_2402_15322_b200 import make_prox, se2_launch_count
    from paper_2402_15322_b200.dist import Comm, Dist, local_rows, se2_jko_step_dist, slab_kernel

    ws, rank, local = _dist_env()
    torch.cuda.set_device(local)
    world = None
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        world = Comm.from_process_group(local)
    cfg = S.get_config(args.workload)
    d = S.config_inputs(cfg)
    # the c4 grid's rows split into ws slabs (ws = 1: the whole grid; the same call path)
    k, row0, rows, top, bot = slab_kernel(cfg.nx, cfg.ny, cfg.ntheta, cfg.eps, cfg.w, cfg.R, ws, rank, 1, local)
    dd = Dist(slabs=world, halo_top=top, halo_bot=bot)
    st = k.stats()
    prox = make_prox(k, cfg.tau, global_ny=cfg.ny, row_offset=row0 - top)
    mu_local0 = local_rows(d["mus"][0], row0, rows, top, bot)
    mu = torch.from_numpy(mu_local0).cuda()
    nxt = torch.empty_like(mu)
    a = torch.empty_like(mu)
    b = torch.empty_like(mu)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    iters = cfg.iters

    def step():
        nonlocal mu, nxt
        se2_jko_step_dist(k, dd, mu, nxt, a, b, iters, prox, log_domain=False, trace=False)
        mu, nxt = nxt, mu

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    l0 = se2_launch_count()
    k.timing_enable(True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t_wall = time.perf_counter()
        for i in range(args.steps):
            flush.fill_(float(i))                      # L2 flush (outside the events)
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    n_conv, conv_ms, _ = k.timing_get()
    k.timing_enable(False)
    launches = se2_launch_count() - l0
    dev_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    if ws > 1:
        t = torch.tensor([dev_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms = float(t.item())
        dist.barrier()
    ms_per_step = dev_ms / args.steps
    value = iters * args.steps / (dev_ms / 1000.0)     # inner iterations of the one flow all ranks share

    # ---- e2e: same step through the C ABI with host buffers, H2D + D2H inside the timed region
    host_in = torch.from_numpy(mu_local0).pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    e2e_steps = max(1, min(args.steps, 3))
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        mu.copy_(host_in, non_blocking=True)
        se2_jko_step_dist(k, dd, mu, nxt, a, b, iters, prox, log_domain=False, trace=False)
        host_out.copy_(nxt, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = iters * e2e_steps / (e2e_ms / 1000.0)
    nbytes = mu.numel() * 4

    out = None
    if rank == 0:
        peaks, peak_src = _peaks()
        clocks = clk.summary()
        sm_max = float(peaks.get("sm_max_mhz", 1965.0))
        ffma_peak = 148 * 128 * 2 * sm_max * 1e6 / 1e12           # TFLOP/s
        # algorithmic work of one conv launch on this rank: 2 flop per fp32-NORMAL tap of every owned output
        flop_per_conv = 2.0 * cfg.nx * rows * cfg.ntheta * st["nnz_normal_taps"]
        conv_avg_ms = conv_ms / max(n_conv, 1)
        achieved = flop_per_conv / (conv_avg_ms / 1000.0) / 1e12
        par = (f"slabs x{ws}: one c4 JKO flow, the 256 rows split into {ws} slabs (se2_jko_step_dist: owned-row "
               f"convs, R-row NCCL halo exchange after every conv, mass allreduce per step)") if ws > 1 else \
            "1 GPU (se2_jko_step_dist with one slab == se2_jko_step)"
        out = {
            "metric": "Sinkhorn iters/s on SE(2) grid", "value": value, "unit": "iters/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 fields; linear conv on tensor cores as 3 BF16 products (hi.hi + hi.lo + lo.hi) "
                     "with fp32 accumulation" if k.uses_tensor_cores else "f32", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.workload], "inner_iters_per_step": iters,
                       "l2": "flushed before every timed step (256 MiB write, outside the step events)",
                       "parallelism": par, "rows_on_rank0": rows},
            "roofline": _conv_roofline(k, cfg, st, achieved, conv_avg_ms, flop_per_conv, n_conv, conv_ms, dev_ms,
                                       ffma_peak, sm_max, peaks, peak_src, clocks, args.workload),
            "e2e": {"value": e2e_value, "unit": "iters/s", "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes},
            "gpu_launches": int(launches),
            "clocks": clocks,
            "wall_s_timed_region": t_wall,
        }
    k.close()
    if ws > 1:
        try:
            rep = replicas(ws, rank, local, cfg, d)
        except Exception as exc:
            rep = {"error": f"{type(exc).__name__}: {exc}"}
        if rank == 0:
            out["replicas"] = rep
        try:
            c1t = c1_tvalues(ws, rank, local)
        except Exception as exc:
            c1t = {"error": f"{type(exc).__name__}: {exc}"}
        if rank == 0:
            out["c1_tvalues"] = c1t
    if not args.no_configs:
        try:
            sharded = sharded_barycenter(ws, rank, local, world)
        except Exception as exc:  # the headline must not depend on this extra measurement
            sharded = {"error": f"{type(exc).__name__}: {exc}"}
        if rank == 0:
            out["sharded_barycenter_c3"] = sharded
        try:
            sharded_p = sharded_barycenter_precise(ws, rank, local, world)
        except Exception as exc:  # the headline must not depend on this extra measurement
            sharded_p = {"error": f"{type(exc).__name__}: {exc}"}
        if rank == 0:
            out["sharded_barycenter_c3_precise"] = sharded_p
    if ws > 1:
        dist.barrier()
        world.close()
        dist.destroy_process_group()
    if rank == 0:
        if not args.no_configs:
            out["configs"] = config_sweep(local)
            try:
                out["next_rows"] = next_rows(local)
            except Exception as e:  # measurement extra: never fail the headline line
                out["next_rows"] = {"error": str(e)[:300]}
        if not args.no_cpu_baseline and ws == 1:   # the oracle baseline: rank 0 at N = 1 only
            v, desc, threads, _ = cpu_oracle_sample(cfg)
            out["cpu_baseline"] = {"value": v, "unit": "iters/s", "cores": threads, "kind": "oracle",
                                   "sample": desc + " (a PROJECTION of one inner iteration from that timed sample)"}
        print(json.dumps(out), flush=True)
        if args.manifest:
            try:
                write_manifest(args.manifest, args, cfg, d, out)
            except Exception as exc:  # the manifest is a log: it never fails the bench line
                print(f"manifest not written: {type(exc).__name__}: {exc}", file=sys.stderr)
    return 0


def write_manifest(path, args, cfg, inputs, out):
    """Run manifest (SURVEY §5 "metrics / logging"): one JSON line per bench run with the config, the input
    seeds and the SHA-256 of every seeded input array and of the library that ran, the GPU, the SM clock
    samples of the timed region and the headline numbers.  Appended, never read back by the bench."""
    import dataclasses
    import hashlib
    import platform

    import torch

    import paper_2402_15322_b200 as pkg
    from paper_2402_15322_b200 import _lib

    def sha(b):
        return hashlib.sha256(b).hexdigest()

    ci = int(cfg.name[1:])
    lib = os.path.join(os.path.dirname(os.path.abspath(pkg.__file__)), "libse2ot.so")
    prop = torch.cuda.get_device_properties(torch.cuda.current_device())
    man = {
        "time_utc": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
        "argv": sys.argv[1:],
        "config": dataclasses.asdict(cfg),
        "seeds": {f"mu[{i}]": 1000 * ci + i for i in range(len(inputs["mus"]))},
        "input_sha256": {f"mu[{i}]": sha(np.ascontiguousarray(m, dtype=np.float32).tobytes())
                         for i, m in enumerate(inputs["mus"])},
        "libse2ot_sha256": sha(open(lib, "rb").read()),
        "abi_version": int(_lib.load().se2_abi_version()),
        "gpu": {"name": prop.name, "sms": prop.multi_processor_count, "cc": f"{prop.major}.{prop.minor}",
                "memory_gb": round(prop.total_memory / 2 ** 30, 1)},
        "host": {"cores": os.cpu_count(), "machine": platform.machine()},
        "torch": torch.__version__, "cuda": torch.version.cuda,
        "clocks": out.get("clocks"),
        "value": out.get("value"), "unit": out.get("unit"), "n_gpus": out.get("n_gpus"),
        "ms_per_step": out.get("ms_per_step"), "e2e": out.get("e2e"),
        "roofline_frac": (out.get("roofline") or {}).get("frac"),
        "gpu_launches": out.get("gpu_launches"),
        "configs_iters_per_s": {n: c.get("iters_per_s") for n, c in (out.get("configs") or {}).items()
                                if isinstance(c, dict) and "iters_per_s" in c},
    }
    d = os.path.dirname(os.path.abspath(path))
    os.makedirs(d, exist_ok=True)
    with open(path, "a") as f:
        f.write(json.dumps(man) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config sweep (c0..c4 solves)")
    ap.add_argument("--manifest", default=os.environ.get("SE2_MANIFEST", ""),
                    help="append a run manifest (config, seeds, input / library SHA-256, GPU, clocks, results) "
                         "as one JSON line to this file")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
