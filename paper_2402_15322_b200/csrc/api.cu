// C ABI of libse2ot (include/se2ot.h): validation, kernel objects, and the scaling-loop drivers
// (Sinkhorn P:557-560, JKO P:224-234, barycenter App. A).  Host code only orders
// launches on the caller's stream; every arithmetic step runs in the CUDA kernels.
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <string>
#include <vector>

#include "se2_internal.cuh"

namespace se2 {
static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
static std::atomic<int64_t> g_launches{0};
void count_launch(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}  // namespace se2

using namespace se2;

extern "C" int64_t se2_launch_count(void);

#include "api_internal.cuh"

extern "C" {

const char* se2_last_error(void) { return g_last_error.c_str(); }
int32_t se2_abi_version(void) { return SE2OT_ABI_VERSION; }
int64_t se2_launch_count(void) { return g_launches.load(); }

se2_status se2_kernel_build(const se2_grid* grid, const se2_metric* metric, double eps, int32_t radius,
                            int32_t max_batch, int32_t device, se2_kernel* out) {
    SE2_CHECK_ARG(out != nullptr && grid != nullptr && metric != nullptr, "null argument");
    *out = nullptr;
    SE2_CHECK_ARG(grid->nx > 0 && grid->ny > 0 && grid->ntheta > 0, "grid sizes must be positive");
    SE2_CHECK_ARG(eps > 0 && isfinite(eps), "eps must be > 0");
    SE2_CHECK_ARG(metric->w1 > 0 && metric->w2 > 0 && metric->w3 > 0, "metric weights must be > 0");
    SE2_CHECK_ARG(radius >= 0, "radius must be >= 0");
    SE2_CHECK_ARG(max_batch >= 1, "max_batch must be >= 1");
    if (radius > kMaxRadius) {
        set_error("radius > 15 is not supported by the conv engines");
        return SE2_EUNSUPPORTED;
    }
    int ndev = 0;
    SE2_CUDA_TRY(cudaGetDeviceCount(&ndev));
    SE2_CHECK_ARG(device >= 0 && device < ndev, "bad device index");
    DeviceGuard g(device);

    se2_kernel_s* k = new se2_kernel_s();
    k->device = device;
    k->nx = grid->nx;
    k->ny = grid->ny;
    k->nt = grid->ntheta;
    k->R = radius;
    k->S = 2 * radius + 1;
    k->eps = eps;
    k->w1 = metric->w1;
    k->w2 = metric->w2;
    k->w3 = metric->w3;
    k->max_batch = max_batch;
    SE2_CHECK_ARG(grid->hx >= 0 && grid->hy >= 0, "cell sizes must be >= 0");
    k->hx = grid->hx > 0 ? grid->hx : 1.0 / grid->nx;
    k->hy = grid->hy > 0 ? grid->hy : 1.0 / grid->ny;
    k->extra = new KernelExtra();

    const int nquads = (k->nt + 3) / 4;
    const size_t tab = (size_t)nquads * k->nt * k->S * k->S * 4 * sizeof(float);
    const size_t tabl = (size_t)k->nt * k->nt * k->S * ((k->S + 3) / 4 * 4) * sizeof(float);
    cudaError_t e = cudaMalloc(&k->Eq, tab);
    if (e == cudaSuccess) e = cudaMalloc(&k->Lq, tab);
    if (e == cudaSuccess) e = cudaMalloc(&k->LqRow, (size_t)nquads * k->nt * k->S * kRowSegs * 4 * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&k->Wl, tabl);
    if (e == cudaSuccess) e = cudaMalloc(&k->Lth, sizeof(float) * k->nt * k->nt);
    if (e == cudaSuccess) e = cudaMalloc(&k->LseS, sizeof(float) * k->nt * k->nt);
    if (e == cudaSuccess) e = cudaMemset(k->Eq, 0, tab);
    if (e == cudaSuccess) e = cudaMemset(k->Lq, 0, tab);
    if (e == cudaSuccess) e = cudaMemset(k->Wl, 0, tabl);
    if (e != cudaSuccess) {
        set_error(std::string("table allocation: ") + cudaGetErrorString(e));
        se2_kernel_destroy(k);
        return SE2_ENOMEM;
    }
    k->table_bytes = 2 * tab + tabl + 2 * sizeof(float) * k->nt * k->nt;
    {
        const size_t nst = lse_fast_stats_floats(k, max_batch);
        cudaError_t e2 = cudaMalloc(&k->lstats, sizeof(float) * nst);
        if (e2 == cudaSuccess) e2 = cudaMalloc(&k->lse_counters, sizeof(int) * 16);
        if (e2 == cudaSuccess) e2 = cudaMalloc(&k->guard, sizeof(unsigned int) * 4);
        if (e2 == cudaSuccess) e2 = cudaMemset(k->guard, 0, sizeof(unsigned int) * 4);
        if (e2 == cudaSuccess) e2 = cudaMemset(k->lse_counters, 0, sizeof(int) * 16);
        // theta_i-split scratch for grids that give fewer than 2 CTAs per SM (at most 8 groups, 64 MB)
        {
            const int64_t N = k->N();
            size_t want = (size_t)max_batch * N * 8;
            if (want * sizeof(float) > ((size_t)64 << 20)) want = ((size_t)64 << 20) / sizeof(float);
            if (e2 == cudaSuccess) e2 = cudaMalloc(&k->split, sizeof(float) * want);
            k->split_floats = want;
        }
        if (e2 != cudaSuccess) {
            set_error(std::string("scratch allocation: ") + cudaGetErrorString(e2));
            se2_kernel_destroy(k);
            return SE2_ENOMEM;
        }
    }
    e = tabulate(k, 0);
    if (e == cudaSuccess) e = conv_tc_prepare(k);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        set_error(std::string("tabulate: ") + cudaGetErrorString(e));
        se2_kernel_destroy(k);
        return SE2_ECUDA;
    }
    *out = k;
    if (k->S > std::min(k->nx, k->ny)) {
        set_error("support box exceeds the grid");
        return SE2_WKERNEL_TOO_WIDE;
    }
    return SE2_OK;
}

se2_status se2_kernel_stats_get(se2_kernel k, se2_kernel_stats* o) {
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(o != nullptr, "null stats");
    o->box_taps = (int64_t)k->nt * k->S * k->S;
    o->nnz_taps = k->nnz_taps;
    o->theta_band = k->band;
    o->radius = k->R;
    o->zeta = std::max(k->w1, k->w2) / std::min(k->w1, k->w2);
    o->table_bytes = k->table_bytes;
    o->tensor_cores = k->tc_w == nullptr ? 0 : (k->tc_fast ? 1 : 2);
    o->nnz_normal_taps = k->nnz_normal_taps;
    return SE2_OK;
}

void se2_kernel_destroy(se2_kernel k) {
    if (!k) return;
    DeviceGuard g(k->device);
    if (k->Eq) cudaFree(k->Eq);
    if (k->Lth) cudaFree(k->Lth);
    if (k->LseS) cudaFree(k->LseS);
    if (k->Lq) cudaFree(k->Lq);
    if (k->LqRow) cudaFree(k->LqRow);
    if (k->Wl) cudaFree(k->Wl);
    if (k->Wcl) cudaFree(k->Wcl);
    if (k->Lcq) cudaFree(k->Lcq);
    if (k->lstats) cudaFree(k->lstats);
    if (k->split) cudaFree(k->split);
    if (k->tc_w) cudaFree(k->tc_w);
    if (k->tc_x) cudaFree(k->tc_x);
    se2::conv_tc_release(k);
    if (k->lse_counters) cudaFree(k->lse_counters);
    if (k->guard) cudaFree(k->guard);
    if (k->L2hi) cudaFree(k->L2hi);
    if (k->L2lo) cudaFree(k->L2lo);
    if (k->L2row) cudaFree(k->L2row);
    if (k->pstats) cudaFree(k->pstats);
    if (k->psplit) cudaFree(k->psplit);
    KernelExtra* x = extra(k);
    if (x) {
        x->clear_graphs();
        if (x->cap) cudaStreamDestroy(x->cap);
        if (x->ev_in) cudaEventDestroy(x->ev_in);
        if (x->ev_out) cudaEventDestroy(x->ev_out);
        for (Workspace* w : {&x->ws, &x->trace, &x->partial, &x->misc})
            if (w->ptr) cudaFree(w->ptr);
        delete x;
    }
    for (auto& p : k->timing.events) {
        cudaEventDestroy(p.first);
        cudaEventDestroy(p.second);
    }
    delete k;
}

se2_status se2_kernel_set_window(se2_kernel k, int32_t row_lo, int32_t row_hi) {
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(row_lo >= 0 && row_hi > row_lo && row_hi <= k->ny, "window must satisfy 0 <= lo < hi <= ny");
    DeviceGuard g(k->device);
    k->win_lo = row_lo;
    k->win_hi = (row_lo == 0 && row_hi == k->ny) ? 0 : row_hi;
    extra(k)->clear_graphs();   // captured solves used the previous geometry
    cudaError_t e = conv_tc_decide(k);
    if (e != cudaSuccess) {
        set_error(std::string("K10 geometry: ") + cudaGetErrorString(e));
        return SE2_ECUDA;
    }
    return SE2_OK;
}

se2_status se2_conv(se2_kernel k, const float* in, float* out, int32_t batch, uint32_t flags, se2_stream stream) {
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(in && out && in != out, "in/out must be distinct non-null device pointers");
    SE2_CHECK_ARG(batch >= 1 && batch <= k->max_batch, "batch out of range [1, max_batch]");
    DeviceGuard g(k->device);
    Epilogue epi;
    epi.op = EPI_STORE;
    epi.out = out;
    return run_conv(k, in, batch, flags, epi, (cudaStream_t)stream, nullptr);
}

se2_status se2_conv_update(se2_kernel k, const float* in, const float* target, float* out, int32_t batch,
                           int32_t op, const se2_prox* prox, uint32_t flags, se2_stream stream) {
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(in && out && in != out, "in/out must be distinct non-null device pointers");
    SE2_CHECK_ARG(batch >= 1 && batch <= k->max_batch, "batch out of range [1, max_batch]");
    SE2_CHECK_ARG(op == SE2_EPI_DIVIDE || op == SE2_EPI_MULTIPLY || op == SE2_EPI_PROX, "bad epilogue op");
    SE2_CHECK_ARG(op == SE2_EPI_PROX || target != nullptr, "target required");
    SE2_CHECK_ARG(op != SE2_EPI_PROX || (prox != nullptr && prox->tau >= 0 &&
                                         (prox->kind == SE2_PROX_ENTROPY_POTENTIAL ||
                                          (prox->kind == SE2_PROX_POROUS && prox->m > 1.0))),
                  "JKO prox required (entropy+potential, or porous with m > 1)");
    DeviceGuard g(k->device);
    Epilogue epi;
    epi.op = op;
    epi.target = target;
    epi.out = out;
    if (op == SE2_EPI_PROX) fill_prox(epi, k, prox);
    return run_conv(k, in, batch, flags, epi, (cudaStream_t)stream, nullptr);
}

se2_status se2_conv_update_slab(se2_kernel k, const float* in, const float* target, float* out, int32_t batch,
                                int32_t op, const se2_prox* prox, uint32_t flags, const se2_slab* slab,
                                se2_stream stream) {
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(slab != nullptr, "slab required");
    SE2_CHECK_ARG(slab->own_lo >= 0 && slab->own_hi > slab->own_lo && slab->own_hi <= k->ny && slab->halo >= 0 &&
                      slab->halo <= slab->own_hi - slab->own_lo,
                  "bad slab rows");
    SE2_CHECK_ARG(!slab->up || (slab->ny_up >= 1 && slab->up_shift + slab->own_lo + slab->halo <= slab->ny_up &&
                                slab->up_shift + slab->own_lo >= 0),
                  "bad upper halo geometry");
    SE2_CHECK_ARG(!slab->dn || (slab->ny_dn >= 1 && slab->own_hi - slab->halo - slab->dn_shift >= 0 &&
                                slab->own_hi - slab->dn_shift <= slab->ny_dn),
                  "bad lower halo geometry");
    SE2_CHECK_ARG(in && out && in != out, "in/out must be distinct non-null device pointers");
    SE2_CHECK_ARG(batch >= 1 && batch <= k->max_batch, "batch out of range [1, max_batch]");
    SE2_CHECK_ARG(op == SE2_EPI_DIVIDE || op == SE2_EPI_MULTIPLY || op == SE2_EPI_PROX, "bad epilogue op");
    SE2_CHECK_ARG(op == SE2_EPI_PROX || target != nullptr, "target required");
    SE2_CHECK_ARG(op != SE2_EPI_PROX || (prox != nullptr && prox->tau >= 0 &&
                                         (prox->kind == SE2_PROX_ENTROPY_POTENTIAL ||
                                          (prox->kind == SE2_PROX_POROUS && prox->m > 1.0))),
                  "JKO prox required (entropy+potential, or porous with m > 1)");
    DeviceGuard g(k->device);
    Epilogue epi;
    epi.op = op;
    epi.target = target;
    epi.out = out;
    if (op == SE2_EPI_PROX) fill_prox(epi, k, prox);
    epi.slab_lo = slab->own_lo;
    epi.slab_hi = slab->own_hi;
    epi.slab_halo = slab->halo;
    epi.ny_self = k->ny;
    epi.nx_self = k->nx;
    epi.halo_up = slab->up;
    epi.up_shift = slab->up_shift;
    epi.ny_up = slab->ny_up;
    epi.halo_dn = slab->dn;
    epi.dn_shift = slab->dn_shift;
    epi.ny_dn = slab->ny_dn;
    return run_conv(k, in, batch, flags, epi, (cudaStream_t)stream, nullptr);
}

// ---- Sinkhorn / JKO inner solve -------------------------------------------------------------------
static se2_status sinkhorn_impl(se2_kernel_s* k, const float* mu, const float* nu, float* a, float* b, int batch,
                                const se2_prox* prox, const se2_opts* opts, double* err_trace_host,
                                float* s_out, cudaStream_t s) {
    const bool LOG = (opts->flags & SE2_LOG_DOMAIN) != 0;
    const bool trace = (opts->flags & SE2_TRACE_ERR) != 0 && err_trace_host != nullptr;
    const bool jko = prox != nullptr && (prox->kind == SE2_PROX_ENTROPY_POTENTIAL || prox->kind == SE2_PROX_POROUS);
    const int64_t N = k->N();
    const int64_t BN = (int64_t)batch * N;
    const int iters = opts->iters;
    KernelExtra* x = extra(k);

    // workspaces first (allocation invalidates captured graphs), then the launch sequence
    // log targets (2 BN) + shift hints of the two convolutions (2 BN)
    size_t need = (size_t)(LOG ? 4 : 0) * BN * sizeof(float);
    se2_status st = ensure(x->ws, std::max<size_t>(need, 16), x);
    if (st != SE2_OK) return st;
    const int bpf = conv_blocks_per_field(k, LOG, opts->flags);
    if (trace) {
        st = ensure(x->partial, (size_t)batch * bpf * sizeof(float), x);
        if (st != SE2_OK) return st;
        st = ensure(x->trace, (size_t)std::max(iters, 1) * batch * sizeof(double), x);
        if (st != SE2_OK) return st;
    }
    // K9: the whole loop in one cluster launch when the grid fits in shared memory (c0-sized)
    const int k9c = (LOG && !jko && batch <= 64 && s_out == nullptr && iters > 0 && k->win_hi == 0 &&
                     !(opts->flags & (SE2_NO_PERSISTENT | SE2_LSE_EXACT | SE2_LSE_K3EXACT | SE2_LSE_NOTILT)))
                        ? k9_cluster_size(k) : 0;
    if (k9c > 0) {
        if (trace) {
            st = ensure(x->partial, (size_t)std::max(iters, 1) * batch * k9c * sizeof(float), x);
            if (st != SE2_OK) return st;
        }
        float* kpart = trace ? reinterpret_cast<float*>(x->partial.ptr) : nullptr;
        double* ktr = trace ? reinterpret_cast<double*>(x->trace.ptr) : nullptr;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (k->timing.on) {   // reported as one conv-engine launch (the loop has no separate convs)
            Timing& t = k->timing;
            if (t.used == t.events.size()) {
                cudaEvent_t ea, eb;
                SE2_CUDA_TRY(cudaEventCreate(&ea));
                SE2_CUDA_TRY(cudaEventCreate(&eb));
                t.events.push_back({ea, eb});
            }
            e0 = t.events[t.used].first;
            e1 = t.events[t.used].second;
            t.used++;
            t.all_launches++;
            SE2_CUDA_TRY(cudaEventRecord(e0, s));
        }
        cudaError_t ce = launch_sinkhorn_small(k, mu, nu, a, b, batch, iters, (opts->flags & SE2_WARM_START) != 0, kpart,
                                               ktr, k9c, s);
        if (ce != cudaSuccess) {
            set_error(std::string("K9 launch: ") + cudaGetErrorString(ce));
            return SE2_ECUDA;
        }
        if (e1) SE2_CUDA_TRY(cudaEventRecord(e1, s));
        if (trace && iters > 0)
            SE2_CUDA_TRY(cudaMemcpyAsync(err_trace_host, ktr, sizeof(double) * iters * batch, cudaMemcpyDeviceToHost, s));
        return SE2_OK;
    }
    float* partial = reinterpret_cast<float*>(x->partial.ptr);
    double* tr = reinterpret_cast<double*>(x->trace.ptr);
    std::vector<uint64_t> key = {1, as_key(mu), as_key(nu), as_key(a), as_key(b), (uint64_t)batch, (uint64_t)iters,
                                 (uint64_t)opts->flags, (uint64_t)trace, as_key(s_out), as_key(x->ws.ptr),
                                 as_key(partial), as_key(tr)};
    if (prox) {
        key.push_back((uint64_t)prox->kind);
        for (double v : {prox->tau, prox->cx, prox->cy, prox->hx, prox->hy, prox->m}) key.push_back(as_key(v));
    }
    auto enqueue = [&](cudaStream_t s) -> se2_status {
    se2_status st = SE2_OK;
    const float* tmu = mu;
    const float* tnu = nu;
    if (LOG) {
        float* lmu = reinterpret_cast<float*>(x->ws.ptr);
        float* lnu = lmu + BN;
        SE2_CUDA_TRY(launch_log(mu, lmu, BN, s));
        tmu = lmu;
        if (!jko) {
            SE2_CUDA_TRY(launch_log(nu, lnu, BN, s));
            tnu = lnu;
        }
    }
    if (!(opts->flags & SE2_WARM_START)) SE2_CUDA_TRY(launch_fill(b, BN, LOG ? 0.f : 1.f, s));

    // exact-path shift hints (K3): they save the max pass over S^2 taps, which only pays off for
    // wider supports (measured: c0 at R = 3 is 14% slower with hints, c1 at R = 5 8% faster)
    const bool hints = LOG && k->R >= 5;
    float* hint1 = hints ? reinterpret_cast<float*>(x->ws.ptr) + 2 * BN : nullptr;   // K b
    float* hint2 = hints ? hint1 + BN : nullptr;                                      // K a
    for (int l = 0; l < iters; ++l) {
        NvtxRange nvtx_iter("se2 iteration", l);
        // a = mu / K b   (error of the previous iterate fused: sum |a_old K b - mu|)
        Epilogue e1;
        e1.op = EPI_DIVIDE;
        e1.target = tmu;
        e1.out = a;
        e1.hint_in = (l > 0) ? hint1 : nullptr;
        e1.hint_out = hint1;
        if (trace && l > 0) {
            e1.err_a = a;
            e1.err_mu = mu;
            e1.err_partial = partial;
        }
        st = run_conv(k, b, batch, opts->flags, e1, s, nullptr);
        if (st != SE2_OK) return st;
        if (trace && l > 0) SE2_CUDA_TRY(launch_reduce_partials(partial, batch, bpf, tr + (int64_t)(l - 1) * batch, s));
        // b = prox(K^T a) / K^T a    (K^T = K)
        Epilogue e2;
        e2.out = b;
        e2.hint_in = (l > 0) ? hint2 : nullptr;
        e2.hint_out = hint2;
        if (jko) {
            e2.op = EPI_PROX;
            fill_prox(e2, k, prox);
            if (l == iters - 1) e2.out2 = s_out;
        } else {
            e2.op = EPI_DIVIDE;
            e2.target = tnu;
        }
        st = run_conv(k, a, batch, opts->flags, e2, s, nullptr);
        if (st != SE2_OK) return st;
    }
    if (trace && iters > 0) {
        Epilogue e3;
        e3.op = EPI_ERRONLY;
        e3.err_a = a;
        e3.err_mu = mu;
        e3.err_partial = partial;
        e3.hint_in = hint1;
        st = run_conv(k, b, batch, opts->flags, e3, s, nullptr);
        if (st != SE2_OK) return st;
        SE2_CUDA_TRY(launch_reduce_partials(partial, batch, bpf, tr + (int64_t)(iters - 1) * batch, s));
    }
    return SE2_OK;
    };
    st = run_graph(k, s, std::move(key), (int64_t)batch * N <= kGraphMaxElems && !(opts->flags & SE2_NO_GRAPH), enqueue);
    if (st != SE2_OK) return st;
    if (trace && iters > 0)
        SE2_CUDA_TRY(cudaMemcpyAsync(err_trace_host, tr, sizeof(double) * iters * batch, cudaMemcpyDeviceToHost, s));
    return SE2_OK;
}

se2_status se2_sinkhorn(se2_kernel k, const float* mu, const float* nu, float* a, float* b, int32_t batch,
                        const se2_prox* prox, const se2_opts* opts, double* err_trace_host, se2_stream stream) {
    NvtxRange nvtx_call("se2_sinkhorn");
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(opts != nullptr && opts->iters >= 0, "opts required, iters >= 0");
    SE2_CHECK_ARG(mu && a && b && a != b, "mu, a, b must be non-null distinct device pointers");
    const bool jko = prox != nullptr && (prox->kind == SE2_PROX_ENTROPY_POTENTIAL || prox->kind == SE2_PROX_POROUS);
    SE2_CHECK_ARG(jko || nu != nullptr, "nu required for the marginal prox");
    SE2_CHECK_ARG(prox == nullptr || prox->kind == SE2_PROX_MARGINAL ||
                      (jko && prox->tau >= 0 && (prox->kind != SE2_PROX_POROUS || prox->m > 1.0)),
                  "bad prox");
    SE2_CHECK_ARG(batch >= 1 && batch <= k->max_batch, "batch out of range [1, max_batch]");
    DeviceGuard g(k->device);
    cudaStream_t s = (cudaStream_t)stream;
    se2_status st = reset_guard(k, s);
    if (st != SE2_OK) return st;
    st = sinkhorn_impl(k, mu, nu, a, b, batch, prox, opts, err_trace_host, nullptr, s);
    if (st != SE2_OK) return st;
    const float* ps[2] = {a, b};
    const int64_t ns[2] = {(int64_t)batch * k->N(), (int64_t)batch * k->N()};
    return check_finite(k, ps, ns, 2, s);
}

se2_status se2_jko_step(se2_kernel k, const float* mu_k, float* mu_next, float* a, float* b, const se2_prox* prox,
                        const se2_opts* opts, double* mass_host, double* err_trace_host, se2_stream stream) {
    NvtxRange nvtx_call("se2_jko_step");
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(opts != nullptr && opts->iters >= 1, "opts required, iters >= 1");
    SE2_CHECK_ARG(prox != nullptr && prox->tau >= 0 &&
                      (prox->kind == SE2_PROX_ENTROPY_POTENTIAL || (prox->kind == SE2_PROX_POROUS && prox->m > 1.0)),
                  "JKO prox required (entropy+potential, or porous with m > 1)");
    SE2_CHECK_ARG(mu_k && mu_next && a && b && mu_k != mu_next, "bad pointers");
    DeviceGuard g(k->device);
    cudaStream_t s = (cudaStream_t)stream;
    se2_status st = reset_guard(k, s);
    if (st != SE2_OK) return st;
    st = sinkhorn_impl(k, mu_k, nullptr, a, b, 1, prox, opts, err_trace_host, mu_next, s);
    if (st != SE2_OK) return st;
    KernelExtra* x = extra(k);
    st = ensure(x->misc, 4096);
    if (st != SE2_OK) return st;
    double* dsum = reinterpret_cast<double*>(reinterpret_cast<char*>(x->misc.ptr) + 64);
    double* dscr = dsum + 8;
    const int64_t N = k->N();
    SE2_CUDA_TRY(launch_sum(mu_next, N, dsum, dscr, s));
    SE2_CUDA_TRY(launch_scale(mu_next, N, dsum, s));
    if (mass_host) SE2_CUDA_TRY(cudaMemcpyAsync(mass_host, dsum, sizeof(double), cudaMemcpyDeviceToHost, s));
    const float* ps[3] = {a, b, mu_next};
    const int64_t ns[3] = {N, N, N};
    return check_finite(k, ps, ns, 3, s);
}

// ---- barycenter (App. A) ----------------------------------------------------------------------
se2_status se2_barycenter(se2_kernel k, int32_t n, int32_t nsolve, const float* mus, const double* lambdas,
                          float* bary, float* v_state, float* w_state, const se2_opts* opts,
                          double* err_trace_host, se2_stream stream) {
    NvtxRange nvtx_call("se2_barycenter");
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(opts != nullptr && opts->iters >= 0, "opts required");
    SE2_CHECK_ARG(n >= 1 && nsolve >= 1, "n, nsolve >= 1");
    SE2_CHECK_ARG((int64_t)n * nsolve <= k->max_batch, "n*nsolve exceeds max_batch");
    SE2_CHECK_ARG(mus && lambdas && bary, "null pointer");
    for (int sv = 0; sv < nsolve; ++sv) {
        double sum = 0;
        for (int i = 0; i < n; ++i) {
            SE2_CHECK_ARG(lambdas[sv * n + i] >= 0 && isfinite(lambdas[sv * n + i]), "lambda must be >= 0");
            sum += lambdas[sv * n + i];
        }
        SE2_CHECK_ARG(fabs(sum - 1.0) <= 1e-9, "lambdas must lie on the simplex");
    }
    const bool warm = (opts->flags & SE2_WARM_START) != 0;
    SE2_CHECK_ARG(!warm || v_state != nullptr, "SE2_WARM_START needs v_state (the initial v_i)");
    DeviceGuard g(k->device);
    cudaStream_t s = (cudaStream_t)stream;
    const bool LOG = (opts->flags & SE2_LOG_DOMAIN) != 0;
    const bool trace = (opts->flags & SE2_TRACE_ERR) != 0 && err_trace_host != nullptr;
    const int64_t N = k->N();
    const int F = n * nsolve;
    se2_status st0 = reset_guard(k, s);
    if (st0 != SE2_OK) return st0;
    const int64_t FN = (int64_t)F * N;
    const int iters = opts->iters;
    KernelExtra* x = extra(k);
    // workspace: mu_rep [F][N] (linear), lmu_rep [F][N], v [F][N], w [F][N], d [F][N]
    size_t need = (size_t)8 * FN * sizeof(float);
    se2_status st = ensure(x->ws, need, x);
    if (st != SE2_OK) return st;
    float* mu_rep = reinterpret_cast<float*>(x->ws.ptr);
    float* lmu_rep = mu_rep + FN;
    float* v = v_state ? v_state : lmu_rep + FN;
    float* w = w_state ? w_state : lmu_rep + 2 * FN;
    float* d = lmu_rep + 3 * FN;
    float* v_lo = lmu_rep + 4 * FN;   // compensation of the running sum log v (log domain)
    const bool hints = LOG && k->R >= 5;   // see sinkhorn_impl
    float* hint1 = hints ? lmu_rep + 5 * FN : nullptr;   // shift hints of K v and K w (log domain)
    float* hint2 = hints ? lmu_rep + 6 * FN : nullptr;
    st = ensure(x->misc, 4096 + sizeof(float) * F, x);
    if (st != SE2_OK) return st;
    const int bpf = conv_blocks_per_field(k, LOG, opts->flags);
    if (trace) {
        st = ensure(x->partial, (size_t)F * bpf * sizeof(float), x);
        if (st != SE2_OK) return st;
        st = ensure(x->trace, (size_t)std::max(iters, 1) * F * sizeof(double), x);
        if (st != SE2_OK) return st;
    }
    float* partial = reinterpret_cast<float*>(x->partial.ptr);
    double* tr = reinterpret_cast<double*>(x->trace.ptr);
    float* lam_dev = reinterpret_cast<float*>(reinterpret_cast<char*>(x->misc.ptr) + 4096);
    std::vector<float> lamf(F);
    for (int i = 0; i < F; ++i) lamf[i] = (float)lambdas[i];
    SE2_CUDA_TRY(cudaMemcpyAsync(lam_dev, lamf.data(), sizeof(float) * F, cudaMemcpyHostToDevice, s));
    SE2_CUDA_TRY(cudaStreamSynchronize(s));   // lamf lives on this stack frame

    std::vector<uint64_t> key = {2, as_key(mus), as_key(bary), as_key(v), as_key(w), (uint64_t)n, (uint64_t)nsolve,
                                 (uint64_t)iters, (uint64_t)opts->flags, (uint64_t)trace, as_key(x->ws.ptr),
                                 as_key(x->misc.ptr), as_key(partial), as_key(tr)};
    auto enqueue = [&](cudaStream_t s) -> se2_status {
        se2_status st = SE2_OK;
        for (int sv = 0; sv < nsolve; ++sv)
            SE2_CUDA_TRY(cudaMemcpyAsync(mu_rep + (int64_t)sv * n * N, mus, sizeof(float) * n * N,
                                         cudaMemcpyDeviceToDevice, s));
        const float* tmu = mu_rep;
        if (LOG) {
            SE2_CUDA_TRY(launch_log(mu_rep, lmu_rep, FN, s));
            tmu = lmu_rep;
        }
        // v_i, w_i <- 1 (App. A), or resume from the caller's v_i (SE2_WARM_START; w_i is recomputed
        // from v_i by the first half-step before it is read)
        if (!warm) SE2_CUDA_TRY(launch_fill(v, FN, LOG ? 0.f : 1.f, s));
        SE2_CUDA_TRY(launch_fill(v_lo, FN, 0.f, s));
        SE2_CUDA_TRY(launch_fill(w, FN, LOG ? 0.f : 1.f, s));
        for (int j = 0; j < iters; ++j) {
            NvtxRange nvtx_iter("se2 iteration", j);
            // w_i = mu_i / K v_i   (fused: error of the previous v-update, sum |w_i K v_i - mu_i|)
            Epilogue e1;
            e1.op = EPI_DIVIDE;
            e1.target = tmu;
            e1.out = w;
            e1.hint_in = (j > 0) ? hint1 : nullptr;
            e1.hint_out = hint1;
            if (trace && j > 0) {
                e1.err_a = w;
                e1.err_mu = mu_rep;
                e1.err_partial = partial;
            }
            st = run_conv(k, v, F, opts->flags, e1, s, nullptr);
            if (st != SE2_OK) return st;
            if (trace && j > 0) SE2_CUDA_TRY(launch_reduce_partials(partial, F, bpf, tr + (int64_t)(j - 1) * F, s));
            // d_i = v_i K w_i
            Epilogue e2;
            e2.op = EPI_MULTIPLY;
            e2.target = v;
            e2.out = d;
            e2.hint_in = (j > 0) ? hint2 : nullptr;
            e2.hint_out = hint2;
            st = run_conv(k, w, F, opts->flags, e2, s, nullptr);
            if (st != SE2_OK) return st;
            // mu = prod d_i^lambda_i ;  v_i <- v_i mu / d_i
            if (LOG) {
                SE2_CUDA_TRY(launch_bary_logmean_update(n, nsolve, N, d, lam_dev, bary, v, v_lo, s));
            } else {
                SE2_CUDA_TRY(launch_bary_update_lin(n, nsolve, N, v, d, lam_dev, bary, k->guard, s));
            }
        }
        if (trace && iters > 0) {
            Epilogue e3;
            e3.op = EPI_ERRONLY;
            e3.err_a = w;
            e3.err_mu = mu_rep;
            e3.err_partial = partial;
            e3.hint_in = hint1;
            st = run_conv(k, v, F, opts->flags, e3, s, nullptr);
            if (st != SE2_OK) return st;
            SE2_CUDA_TRY(launch_reduce_partials(partial, F, bpf, tr + (int64_t)(iters - 1) * F, s));
        }
        return SE2_OK;
    };
    st = run_graph(k, s, std::move(key), FN <= kGraphMaxElems && !(opts->flags & SE2_NO_GRAPH), enqueue);
    if (st != SE2_OK) return st;
    if (trace && iters > 0) {
        std::vector<double> h((size_t)iters * F);
        SE2_CUDA_TRY(cudaMemcpyAsync(h.data(), tr, sizeof(double) * iters * F, cudaMemcpyDeviceToHost, s));
        SE2_CUDA_TRY(cudaStreamSynchronize(s));
        for (int j = 0; j < iters; ++j)
            for (int sv = 0; sv < nsolve; ++sv) {
                double e = 0;
                for (int i = 0; i < n; ++i) e += lambdas[sv * n + i] * h[(size_t)j * F + sv * n + i];
                err_trace_host[(size_t)j * nsolve + sv] = e;
            }
    }
    const float* ps[3] = {bary, v, w};
    const int64_t ns[3] = {(int64_t)nsolve * N, FN, FN};
    return check_finite(k, ps, ns, 3, s);
}

// ---- barycenter with fp64 potentials (K4P; the elementwise 1e-4 parity of reading R19) --------------
se2_status se2_conv_precise(se2_kernel k, const double* in, double* out, int32_t batch, se2_stream stream) {
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(in && out && (const void*)in != (const void*)out, "in/out must be distinct non-null device pointers");
    SE2_CHECK_ARG(batch >= 1 && batch <= k->max_batch, "batch out of range [1, max_batch]");
    DeviceGuard g(k->device);
    cudaStream_t s = (cudaStream_t)stream;
    SE2_CUDA_TRY(tabulate_precise(k, s));
    EpiP epi;
    epi.op = EPI_STORE;
    epi.out = out;
    return run_conv_precise(k, in, batch, epi, s);
}

se2_status se2_barycenter_precise(se2_kernel k, int32_t n, int32_t nsolve, const float* mus, const double* lambdas,
                                  double* lbary, double* lv_state, double* lw_state, const se2_opts* opts,
                                  double* err_trace_host, se2_stream stream) {
    NvtxRange nvtx_call("se2_barycenter_precise");
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(opts != nullptr && opts->iters >= 0, "opts required");
    SE2_CHECK_ARG(n >= 1 && nsolve >= 1, "n, nsolve >= 1");
    SE2_CHECK_ARG((int64_t)n * nsolve <= k->max_batch, "n*nsolve exceeds max_batch");
    SE2_CHECK_ARG(mus && lambdas && lbary, "null pointer");
    for (int sv = 0; sv < nsolve; ++sv) {
        double sum = 0;
        for (int i = 0; i < n; ++i) {
            SE2_CHECK_ARG(lambdas[sv * n + i] >= 0 && isfinite(lambdas[sv * n + i]), "lambda must be >= 0");
            sum += lambdas[sv * n + i];
        }
        SE2_CHECK_ARG(fabs(sum - 1.0) <= 1e-9, "lambdas must lie on the simplex");
    }
    const bool warm = (opts->flags & SE2_WARM_START) != 0;
    SE2_CHECK_ARG(!warm || lv_state != nullptr, "SE2_WARM_START needs lv_state");
    DeviceGuard g(k->device);
    cudaStream_t s = (cudaStream_t)stream;
    SE2_CUDA_TRY(tabulate_precise(k, s));
    se2_status st = reset_guard(k, s);
    if (st != SE2_OK) return st;
    const bool trace = (opts->flags & SE2_TRACE_ERR) != 0 && err_trace_host != nullptr;
    const int64_t N = k->N();
    const int F = n * nsolve;
    const int64_t FN = (int64_t)F * N;
    const int iters = opts->iters;
    KernelExtra* x = extra(k);
    // workspace: mu_rep (float) [F][N]; lmu, v, w, d (double) [F][N]
    st = ensure(x->ws, (size_t)FN * (sizeof(float) + 4 * sizeof(double)) + 64, x);
    if (st != SE2_OK) return st;
    float* mu_rep = reinterpret_cast<float*>(x->ws.ptr);
    double* lmu = reinterpret_cast<double*>(reinterpret_cast<char*>(x->ws.ptr) + ((FN * sizeof(float) + 63) / 64) * 64);
    double* v = lv_state ? lv_state : lmu + FN;
    double* w = lw_state ? lw_state : lmu + 2 * FN;
    double* d = lmu + 3 * FN;
    st = ensure(x->misc, 4096 + sizeof(double) * F, x);
    if (st != SE2_OK) return st;
    const int bpf = conv_blocks_per_field_precise(k);
    if (trace) {
        st = ensure(x->partial, (size_t)F * bpf * sizeof(float), x);
        if (st != SE2_OK) return st;
        st = ensure(x->trace, (size_t)std::max(iters, 1) * F * sizeof(double), x);
        if (st != SE2_OK) return st;
    }
    float* partial = reinterpret_cast<float*>(x->partial.ptr);
    double* tr = reinterpret_cast<double*>(x->trace.ptr);
    double* lam_dev = reinterpret_cast<double*>(reinterpret_cast<char*>(x->misc.ptr) + 4096);
    SE2_CUDA_TRY(cudaMemcpyAsync(lam_dev, lambdas, sizeof(double) * F, cudaMemcpyHostToDevice, s));
    SE2_CUDA_TRY(cudaStreamSynchronize(s));
    std::vector<uint64_t> key = {5, as_key(mus), as_key(lbary), as_key(v), as_key(w), (uint64_t)n, (uint64_t)nsolve,
                                 (uint64_t)iters, (uint64_t)opts->flags, (uint64_t)trace, as_key(x->ws.ptr),
                                 as_key(x->misc.ptr), as_key(partial), as_key(tr)};
    auto enqueue = [&](cudaStream_t s) -> se2_status {
        se2_status st = SE2_OK;
        for (int sv = 0; sv < nsolve; ++sv)
            SE2_CUDA_TRY(cudaMemcpyAsync(mu_rep + (int64_t)sv * n * N, mus, sizeof(float) * n * N,
                                         cudaMemcpyDeviceToDevice, s));
        SE2_CUDA_TRY(launch_log_f64(mu_rep, lmu, FN, s));
        if (!warm) SE2_CUDA_TRY(launch_fill_f64(v, FN, 0.0, s));
        SE2_CUDA_TRY(launch_fill_f64(w, FN, 0.0, s));
        for (int j = 0; j < iters; ++j) {
            NvtxRange nvtx_iter("se2 iteration", j);
            EpiP e1;   // w_i = mu_i / K v_i  (error of the previous v-update fused)
            e1.op = EPI_DIVIDE;
            e1.target = lmu;
            e1.out = w;
            if (trace && j > 0) {
                e1.err_a = w;
                e1.err_mu = mu_rep;
                e1.err_partial = partial;
            }
            st = run_conv_precise(k, v, F, e1, s);
            if (st != SE2_OK) return st;
            if (trace && j > 0) SE2_CUDA_TRY(launch_reduce_partials(partial, F, bpf, tr + (int64_t)(j - 1) * F, s));
            EpiP e2;   // d_i = v_i K w_i
            e2.op = EPI_MULTIPLY;
            e2.target = v;
            e2.out = d;
            st = run_conv_precise(k, w, F, e2, s);
            if (st != SE2_OK) return st;
            SE2_CUDA_TRY(launch_bary_logmean_update_f64(n, nsolve, N, d, lam_dev, lbary, v, s));
        }
        if (trace && iters > 0) {
            EpiP e3;
            e3.op = EPI_ERRONLY;
            e3.err_a = w;
            e3.err_mu = mu_rep;
            e3.err_partial = partial;
            st = run_conv_precise(k, v, F, e3, s);
            if (st != SE2_OK) return st;
            SE2_CUDA_TRY(launch_reduce_partials(partial, F, bpf, tr + (int64_t)(iters - 1) * F, s));
        }
        return SE2_OK;
    };
    st = run_graph(k, s, std::move(key), FN <= kGraphMaxElems && !(opts->flags & SE2_NO_GRAPH), enqueue);
    if (st != SE2_OK) return st;
    if (trace && iters > 0) {
        std::vector<double> h((size_t)iters * F);
        SE2_CUDA_TRY(cudaMemcpyAsync(h.data(), tr, sizeof(double) * iters * F, cudaMemcpyDeviceToHost, s));
        SE2_CUDA_TRY(cudaStreamSynchronize(s));
        for (int j = 0; j < iters; ++j)
            for (int sv = 0; sv < nsolve; ++sv) {
                double e = 0;
                for (int i = 0; i < n; ++i) e += lambdas[sv * n + i] * h[(size_t)j * F + sv * n + i];
                err_trace_host[(size_t)j * nsolve + sv] = e;
            }
    }
    se2_status st2 = ensure(x->misc, 4096 + sizeof(double) * F, x);
    if (st2 != SE2_OK) return st2;
    int* cnt = reinterpret_cast<int*>(x->misc.ptr);
    SE2_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int), s));
    SE2_CUDA_TRY(launch_count_nonfinite_f64(lbary, (int64_t)nsolve * N, cnt, s));
    SE2_CUDA_TRY(launch_count_nonfinite_f64(v, FN, cnt, s));
    SE2_CUDA_TRY(launch_count_nonfinite_f64(w, FN, cnt, s));
    int h = 0;
    SE2_CUDA_TRY(cudaMemcpyAsync(&h, cnt, sizeof(int), cudaMemcpyDeviceToHost, s));
    SE2_CUDA_TRY(cudaStreamSynchronize(s));
    if (h != 0) {
        set_error("non-finite values produced by the iteration (" + std::to_string(h) + " entries)");
        return SE2_ENONFINITE;
    }
    return SE2_OK;
}

se2_status se2_marginal_error(se2_kernel k, const float* a, const float* b, const float* mu, int32_t batch,
                              uint32_t flags, double* err_host, se2_stream stream) {
    NvtxRange nvtx_call("se2_marginal_error");
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(a && b && mu && err_host, "null pointer");
    SE2_CHECK_ARG(batch >= 1 && batch <= k->max_batch, "batch out of range [1, max_batch]");
    DeviceGuard g(k->device);
    cudaStream_t s = (cudaStream_t)stream;
    const bool LOG = (flags & SE2_LOG_DOMAIN) != 0;
    KernelExtra* x = extra(k);
    const int bpf = conv_blocks_per_field(k, LOG, flags);
    se2_status st = ensure(x->partial, (size_t)batch * bpf * sizeof(float));
    if (st != SE2_OK) return st;
    st = ensure(x->trace, (size_t)batch * sizeof(double));
    if (st != SE2_OK) return st;
    Epilogue e;
    e.op = EPI_ERRONLY;
    e.err_a = a;
    e.err_mu = mu;
    e.err_partial = reinterpret_cast<float*>(x->partial.ptr);
    st = run_conv(k, b, batch, flags, e, s, nullptr);
    if (st != SE2_OK) return st;
    double* tr = reinterpret_cast<double*>(x->trace.ptr);
    SE2_CUDA_TRY(launch_reduce_partials(e.err_partial, batch, bpf, tr, s));
    SE2_CUDA_TRY(cudaMemcpyAsync(err_host, tr, sizeof(double) * batch, cudaMemcpyDeviceToHost, s));
    SE2_CUDA_TRY(cudaStreamSynchronize(s));
    return SE2_OK;
}

se2_status se2_transport_cost(se2_kernel k, const float* a, const float* b, int32_t batch, uint32_t flags,
                              double* cost_host, se2_stream stream) {
    NvtxRange nvtx_call("se2_transport_cost");
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(a && b && cost_host, "null pointer");
    SE2_CHECK_ARG(batch >= 1 && batch <= k->max_batch, "batch out of range [1, max_batch]");
    DeviceGuard g(k->device);
    cudaStream_t s = (cudaStream_t)stream;
    const bool LOG = (flags & SE2_LOG_DOMAIN) != 0;
    if (k->Wcl == nullptr) {
        const size_t tabl = (size_t)k->nt * k->nt * k->S * ((k->S + 3) / 4 * 4) * sizeof(float);
        const size_t tab = (size_t)((k->nt + 3) / 4) * k->nt * k->S * k->S * 4 * sizeof(float);
        cudaError_t e = cudaMalloc(&k->Wcl, tabl);
        if (e == cudaSuccess) e = cudaMalloc(&k->Lcq, tab);
        if (e == cudaSuccess) e = cudaMemsetAsync(k->Wcl, 0, tabl, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(k->Lcq, 0xff, tab, s);   // NaN pattern; overwritten below
        if (e == cudaSuccess) e = tabulate_cost(k, s);
        if (e != cudaSuccess) {
            set_error(std::string("cost tables: ") + cudaGetErrorString(e));
            return SE2_ENOMEM;
        }
        // quad padding (to >= nt) must not produce NaN in the log engine: set it to -inf
        if (k->nt % 4 != 0) {
            std::vector<float> h(tab / sizeof(float));
            SE2_CUDA_TRY(cudaMemcpyAsync(h.data(), k->Lcq, tab, cudaMemcpyDeviceToHost, s));
            SE2_CUDA_TRY(cudaStreamSynchronize(s));
            for (float& v : h)
                if (v != v) v = -INFINITY;
            SE2_CUDA_TRY(cudaMemcpyAsync(k->Lcq, h.data(), tab, cudaMemcpyHostToDevice, s));
        }
        k->table_bytes += tabl + tab;
    }
    {
        cudaError_t e = conv_tc_prepare_cost(k, s);
        if (e != cudaSuccess) {
            set_error(std::string("cost table (K10 weights): ") + cudaGetErrorString(e));
            return SE2_ECUDA;
        }
    }
    KernelExtra* x = extra(k);
    Epilogue e;
    e.op = EPI_DOT;
    e.table = LOG ? k->Lcq : k->Wcl;
    const int bpf = LOG ? conv_blocks_per_field_lse(k)
                        : (conv_tc_route(k, flags, e) ? conv_blocks_per_field_tc(k) : conv_blocks_per_field_linear(k));
    se2_status st = ensure(x->partial, (size_t)batch * bpf * sizeof(float));
    if (st != SE2_OK) return st;
    st = ensure(x->trace, (size_t)batch * sizeof(double));
    if (st != SE2_OK) return st;
    e.err_a = a;
    e.err_partial = reinterpret_cast<float*>(x->partial.ptr);
    // cost = sum_x a(x) sum_y K(x,y) rho^2(x,y) b(y): one conv of b with the cost table (the log domain
    // uses the exact per-tap engine: the cost table has no theta-factored form)
    st = run_conv(k, b, batch, LOG ? (flags | SE2_LSE_EXACT) : flags, e, s, nullptr);
    if (st != SE2_OK) return st;
    double* tr = reinterpret_cast<double*>(x->trace.ptr);
    SE2_CUDA_TRY(launch_reduce_partials(e.err_partial, batch, bpf, tr, s));
    SE2_CUDA_TRY(cudaMemcpyAsync(cost_host, tr, sizeof(double) * batch, cudaMemcpyDeviceToHost, s));
    SE2_CUDA_TRY(cudaStreamSynchronize(s));
    return SE2_OK;
}

se2_status se2_bary_logmean(int32_t n, int64_t N, const float* ld, const double* lambdas, float* lbar,
                            se2_stream stream) {
    SE2_CHECK_ARG(n >= 1 && N >= 1 && ld && lambdas && lbar, "bad arguments");
    // lambdas are host values; pass them through a small device copy
    float* lam_dev = nullptr;
    SE2_CUDA_TRY(cudaMallocAsync(&lam_dev, sizeof(float) * n, (cudaStream_t)stream));
    std::vector<float> lf(n);
    for (int i = 0; i < n; ++i) lf[i] = (float)lambdas[i];
    SE2_CUDA_TRY(cudaMemcpyAsync(lam_dev, lf.data(), sizeof(float) * n, cudaMemcpyHostToDevice, (cudaStream_t)stream));
    SE2_CUDA_TRY(launch_bary_logmean(n, 1, N, ld, lam_dev, lbar, (cudaStream_t)stream));
    SE2_CUDA_TRY(cudaFreeAsync(lam_dev, (cudaStream_t)stream));
    return SE2_OK;
}

se2_status se2_bary_update(int32_t n, int64_t N, float* lv, const float* ld, const float* lbar, se2_stream stream) {
    SE2_CHECK_ARG(n >= 1 && N >= 1 && lv && ld && lbar, "bad arguments");
    SE2_CUDA_TRY(launch_bary_update_log(n, 1, N, lv, nullptr, ld, lbar, (cudaStream_t)stream));
    return SE2_OK;
}

se2_status se2_bary_reduce_update(int32_t nranks, const float* const* partials_dev, int32_t n_local, int64_t N,
                                  float* lv, const float* ld, float* lbar, se2_stream stream) {
    SE2_CHECK_ARG(nranks >= 1 && partials_dev && N >= 1 && n_local >= 0, "bad arguments");
    SE2_CHECK_ARG(n_local == 0 || (lv && ld), "lv and ld required when n_local > 0");
    SE2_CUDA_TRY(launch_bary_reduce_update(nranks, partials_dev, n_local, N, lv, ld, lbar, (cudaStream_t)stream));
    return SE2_OK;
}

se2_status se2_sum(const float* xp, int64_t n, double* out_host, se2_stream stream) {
    SE2_CHECK_ARG(xp && n >= 1 && out_host, "bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    double* d = nullptr;
    SE2_CUDA_TRY(cudaMallocAsync(&d, sizeof(double) * 512, s));
    SE2_CUDA_TRY(launch_sum(xp, n, d, d + 8, s));
    SE2_CUDA_TRY(cudaMemcpyAsync(out_host, d, sizeof(double), cudaMemcpyDeviceToHost, s));
    SE2_CUDA_TRY(cudaFreeAsync(d, s));
    SE2_CUDA_TRY(cudaStreamSynchronize(s));
    return SE2_OK;
}

se2_status se2_sum_rows(const float* xp, int32_t planes, int32_t ny, int32_t nx, int32_t row0, int32_t rows,
                        double* out_host, se2_stream stream) {
    SE2_CHECK_ARG(xp && out_host && planes >= 1 && nx >= 1 && row0 >= 0 && rows >= 0 && row0 + rows <= ny,
                  "bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    double* d = nullptr;
    SE2_CUDA_TRY(cudaMallocAsync(&d, sizeof(double) * 512, s));
    SE2_CUDA_TRY(launch_sum_rows(xp, planes, ny, nx, row0, rows, d, d + 8, s));
    SE2_CUDA_TRY(cudaMemcpyAsync(out_host, d, sizeof(double), cudaMemcpyDeviceToHost, s));
    SE2_CUDA_TRY(cudaFreeAsync(d, s));
    SE2_CUDA_TRY(cudaStreamSynchronize(s));
    return SE2_OK;
}

se2_status se2_scale_rows(float* xp, int32_t planes, int32_t ny, int32_t nx, int32_t row0, int32_t rows,
                          double factor, se2_stream stream) {
    SE2_CHECK_ARG(xp && planes >= 1 && nx >= 1 && row0 >= 0 && rows >= 0 && row0 + rows <= ny, "bad arguments");
    SE2_CUDA_TRY(launch_scale_rows(xp, planes, ny, nx, row0, rows, factor, (cudaStream_t)stream));
    return SE2_OK;
}

se2_status se2_lse_path_stats(se2_kernel k, int64_t* active_pairs, int64_t* ffma_pairs, int64_t* visited_pairs,
                              int64_t* tilted_pairs, int64_t* hint_redos, int32_t reset) {
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    DeviceGuard g(k->device);
    int h[5] = {0, 0, 0, 0, 0};
    SE2_CUDA_TRY(cudaDeviceSynchronize());
    SE2_CUDA_TRY(cudaMemcpy(h, k->lse_counters, sizeof(int) * 5, cudaMemcpyDeviceToHost));
    if (active_pairs) *active_pairs = h[0];
    if (ffma_pairs) *ffma_pairs = h[1];
    if (visited_pairs) *visited_pairs = h[2];
    if (tilted_pairs) *tilted_pairs = h[3];
    if (hint_redos) *hint_redos = h[4];
    if (reset) SE2_CUDA_TRY(cudaMemset(k->lse_counters, 0, sizeof(int) * 5));
    return SE2_OK;
}

se2_status se2_guard_stats(se2_kernel k, int64_t* div_clamps, int64_t* prox_noconv, int32_t reset) {
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    DeviceGuard g(k->device);
    unsigned int h[4] = {0, 0, 0, 0};
    SE2_CUDA_TRY(cudaDeviceSynchronize());
    SE2_CUDA_TRY(cudaMemcpy(h, k->guard, sizeof(h), cudaMemcpyDeviceToHost));
    if (div_clamps) *div_clamps = h[0];
    if (prox_noconv) *prox_noconv = h[1];
    if (reset) SE2_CUDA_TRY(cudaMemset(k->guard, 0, sizeof(h)));
    return SE2_OK;
}

se2_status se2_lse_row_stats(se2_kernel k, int64_t* rows_live, int64_t* rows_visited, int32_t reset) {
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    DeviceGuard g(k->device);
    unsigned long long h[2] = {0, 0};
    SE2_CUDA_TRY(cudaDeviceSynchronize());
    SE2_CUDA_TRY(cudaMemcpy(h, k->lse_counters + 8, sizeof(h), cudaMemcpyDeviceToHost));
    if (rows_live) *rows_live = (int64_t)h[0];
    if (rows_visited) *rows_visited = (int64_t)h[1];
    if (reset) SE2_CUDA_TRY(cudaMemset(k->lse_counters + 8, 0, sizeof(h)));
    return SE2_OK;
}

se2_status se2_precise_path_stats(se2_kernel k, int64_t* ffma_channels, int64_t* channels, int64_t* hint_redos,
                                  int32_t reset) {
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(ffma_channels != nullptr && channels != nullptr, "null output");
    DeviceGuard g(k->device);
    unsigned long long h[2] = {0, 0};
    SE2_CUDA_TRY(cudaDeviceSynchronize());
    SE2_CUDA_TRY(cudaMemcpy(h, k->lse_counters + 12, sizeof(h), cudaMemcpyDeviceToHost));
    *ffma_channels = (int64_t)h[0];
    *channels = (int64_t)h[1];
    if (hint_redos) *hint_redos = 0;   // K4P runs two-pass (a hinted variant measured no faster on c3)
    if (reset) SE2_CUDA_TRY(cudaMemset(k->lse_counters + 12, 0, sizeof(h)));
    return SE2_OK;
}

se2_status se2_tc_tile_stats(se2_kernel k, int64_t* tiles, int64_t* wide_tiles, int32_t reset) {
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(tiles != nullptr && wide_tiles != nullptr, "null output");
    DeviceGuard g(k->device);
    SE2_CUDA_TRY(cudaDeviceSynchronize());
    SE2_CUDA_TRY(se2::conv_tc_tile_counts(k, tiles, wide_tiles, reset != 0));
    return SE2_OK;
}

se2_status se2_timing_enable(se2_kernel k, int32_t on) {
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    k->timing.on = on != 0;
    k->timing.used = 0;
    k->timing.all_launches = 0;
    return SE2_OK;
}

se2_status se2_timing_get(se2_kernel k, int64_t* n_launches, double* conv_ms, int64_t* all_launches) {
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    DeviceGuard g(k->device);
    double tot = 0;
    for (size_t i = 0; i < k->timing.used; ++i) {
        SE2_CUDA_TRY(cudaEventSynchronize(k->timing.events[i].second));
        float ms = 0;
        SE2_CUDA_TRY(cudaEventElapsedTime(&ms, k->timing.events[i].first, k->timing.events[i].second));
        tot += ms;
    }
    if (n_launches) *n_launches = (int64_t)k->timing.used;
    if (conv_ms) *conv_ms = tot;
    if (all_launches) *all_launches = k->timing.all_launches;
    k->timing.used = 0;
    k->timing.all_launches = 0;
    return SE2_OK;
}

}  // extern "C"
