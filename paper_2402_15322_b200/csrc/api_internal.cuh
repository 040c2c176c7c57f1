// Internals shared by the C-ABI translation units (api.cu: single-GPU solvers; dist.cu: the
// multi-GPU solvers): device guard, grow-only workspaces, the conv dispatch with optional event
// timing, CUDA-graph replay of small solves, prox parameters and the end-of-solve checks.
#pragma once
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX 3 (resolves the tool's injection library with dlopen)

#include "se2_internal.cuh"

extern "C" int64_t se2_launch_count(void);

// NVTX ranges (SURVEY §5 "tracing"): one per C-ABI solve, per scaling iteration and per conv, pushed only
// when the process runs with SE2_NVTX=1 (read once) so the default hot loops do no extra host work.
inline bool se2_nvtx_on() {
    static const bool on = [] {
        const char* e = getenv("SE2_NVTX");
        return e && e[0] && e[0] != '0';
    }();
    return on;
}
struct NvtxRange {
    bool on;
    explicit NvtxRange(const char* name) : on(se2_nvtx_on()) {
        if (on) nvtxRangePushA(name);
    }
    NvtxRange(const char* name, int index) : on(se2_nvtx_on()) {
        if (on) {
            char buf[64];
            snprintf(buf, sizeof buf, "%s %d", name, index);
            nvtxRangePushA(buf);
        }
    }
    ~NvtxRange() {
        if (on) nvtxRangePop();
    }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

using namespace se2;

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// grow-only device workspace owned by the kernel object
struct Workspace {
    void* ptr = nullptr;
    size_t bytes = 0;
};

}  // namespace

// a captured solve (CUDA graph) keyed by everything its launches depend on
struct GraphEntry {
    std::vector<uint64_t> key;
    cudaGraphExec_t exec = nullptr;
    int64_t nlaunch = 0;
};

// extra per-kernel state not in the header struct
struct KernelExtra {
    Workspace ws;         // fields
    Workspace trace;      // device error trace
    Workspace partial;    // conv error partials
    Workspace misc;       // lambdas, counters, sums
    std::vector<GraphEntry> graphs;   // small-problem solves replayed as CUDA graphs
    cudaStream_t cap = nullptr;       // private stream for capture / replay
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    void clear_graphs() {
        for (auto& gph : graphs)
            if (gph.exec) cudaGraphExecDestroy(gph.exec);
        graphs.clear();
    }
};

static KernelExtra* extra(se2_kernel_s* k) { return reinterpret_cast<KernelExtra*>(k->extra); }

static se2_status ensure(Workspace& w, size_t bytes, KernelExtra* owner = nullptr) {
    if (w.bytes >= bytes) return SE2_OK;
    if (owner) owner->clear_graphs();   // captured graphs reference the old buffers
    if (w.ptr) cudaFree(w.ptr);
    w.ptr = nullptr;
    w.bytes = 0;
    cudaError_t e = cudaMalloc(&w.ptr, bytes);
    if (e != cudaSuccess) {
        set_error(std::string("cudaMalloc workspace: ") + cudaGetErrorString(e));
        return SE2_ENOMEM;
    }
    w.bytes = bytes;
    return SE2_OK;
}

// ---- conv dispatch with optional event timing ---------------------------------------------------
static se2_status run_conv(se2_kernel_s* k, const float* in, int batch, uint32_t flags, const Epilogue& epi_in,
                           cudaStream_t s, int* bpf) {
    const bool log_domain = (flags & SE2_LOG_DOMAIN) != 0;
    NvtxRange nvtx_conv(log_domain ? "se2 conv (log domain)" : "se2 conv (linear)");
    Epilogue epi = epi_in;
    epi.guard = k->guard;   // every conv epilogue counts its guarded divisions / prox failures
    if (k->win_hi > 0 && epi.slab_hi == 0) {   // output window: rows outside are input-only halo rows
        epi.slab_lo = k->wlo();
        epi.slab_hi = k->whi();
        epi.ny_self = k->ny;
        epi.nx_self = k->nx;
    }
    Timing& t = k->timing;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (t.on) {
        if (t.used == t.events.size()) {
            cudaEvent_t a, b;
            SE2_CUDA_TRY(cudaEventCreate(&a));
            SE2_CUDA_TRY(cudaEventCreate(&b));
            t.events.push_back({a, b});
        }
        e0 = t.events[t.used].first;
        e1 = t.events[t.used].second;
        t.used++;
        SE2_CUDA_TRY(cudaEventRecord(e0, s));
    }
    cudaError_t e;
    if (!log_domain)
        e = conv_tc_route(k, flags, epi) ? launch_conv_tc(k, in, batch, epi, s, bpf)
                                         : launch_conv_linear(k, in, batch, epi, s, bpf);
    else if ((flags & SE2_LSE_EXACT) || k->nt > 128)   // K3 holds per-channel state for <= 128 orientations
        e = launch_conv_lse(k, in, batch, epi, s, bpf);
    else
        e = launch_conv_lse_fast(k, in, batch, epi, s, bpf, k->lstats,
                                 ((flags & SE2_LSE_K3EXACT) ? 1 : ((flags & SE2_LSE_NOTILT) ? 2 : 0)) |
                                     ((flags & SE2_DEBUG_BAD_HINTS) ? 4 : 0) | ((flags & SE2_DEBUG_NO_SPLIT) ? 8 : 0),
                                 k->lse_counters,
                                 k->split, k->split_floats);
    if (e != cudaSuccess) {
        set_error(std::string("conv launch: ") + cudaGetErrorString(e));
        return SE2_ECUDA;
    }
    t.all_launches++;
    if (t.on) SE2_CUDA_TRY(cudaEventRecord(e1, s));
    return SE2_OK;
}

// Replay `enqueue` (a launch sequence on a given stream) as a CUDA graph for small problems, where the
// ~10 launches per scaling iteration are latency-bound; the graph is captured on first use and cached
// under `key`.  Work is ordered after / before the caller's stream with events.  `use` = false runs
// the sequence directly on the caller's stream (large problems, timing instrumentation on).
template <class F>
static se2_status run_graph(se2_kernel_s* k, cudaStream_t s, std::vector<uint64_t> key, bool use, F&& enqueue) {
    static const bool disabled = getenv("SE2_NO_GRAPH") != nullptr;
    if (!use || disabled || k->timing.on) return enqueue(s);
    KernelExtra* x = extra(k);
    if (!x->cap) {
        SE2_CUDA_TRY(cudaStreamCreateWithFlags(&x->cap, cudaStreamNonBlocking));
        SE2_CUDA_TRY(cudaEventCreateWithFlags(&x->ev_in, cudaEventDisableTiming));
        SE2_CUDA_TRY(cudaEventCreateWithFlags(&x->ev_out, cudaEventDisableTiming));
    }
    GraphEntry* hit = nullptr;
    for (auto& gph : x->graphs)
        if (gph.key == key) hit = &gph;
    SE2_CUDA_TRY(cudaEventRecord(x->ev_in, s));
    SE2_CUDA_TRY(cudaStreamWaitEvent(x->cap, x->ev_in, 0));
    if (!hit) {
        if (x->graphs.size() >= 8) {   // small cache: drop the oldest
            if (x->graphs.front().exec) cudaGraphExecDestroy(x->graphs.front().exec);
            x->graphs.erase(x->graphs.begin());
        }
        SE2_CUDA_TRY(cudaStreamBeginCapture(x->cap, cudaStreamCaptureModeThreadLocal));
        const int64_t l0 = se2_launch_count();
        se2_status st = enqueue(x->cap);
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamEndCapture(x->cap, &graph);
        if (st != SE2_OK) {
            if (graph) cudaGraphDestroy(graph);
            return st;
        }
        if (e != cudaSuccess) {
            set_error(std::string("graph capture: ") + cudaGetErrorString(e));
            return SE2_ECUDA;
        }
        GraphEntry ge;
        ge.key = std::move(key);
        ge.nlaunch = se2_launch_count() - l0;
        e = cudaGraphInstantiate(&ge.exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) {
            set_error(std::string("graph instantiate: ") + cudaGetErrorString(e));
            return SE2_ECUDA;
        }
        x->graphs.push_back(ge);
        hit = &x->graphs.back();
        SE2_CUDA_TRY(cudaGraphLaunch(hit->exec, x->cap));   // the capture itself executed nothing
    } else {
        SE2_CUDA_TRY(cudaGraphLaunch(hit->exec, x->cap));
        count_launch(hit->nlaunch);
    }
    SE2_CUDA_TRY(cudaEventRecord(x->ev_out, x->cap));
    SE2_CUDA_TRY(cudaStreamWaitEvent(s, x->ev_out, 0));
    return SE2_OK;
}

static uint64_t as_key(const void* p) { return (uint64_t)(uintptr_t)p; }
static uint64_t as_key(double v) {
    uint64_t u;
    memcpy(&u, &v, sizeof(u));
    return u;
}
// batch * N at or below which solves use graphs (2^21; SE2_GRAPH_MAX_LOG2 overrides it for measurements: the c4
// JKO step as one graph of 1 200 kernel nodes measured no faster than its direct launches)
static const int64_t kGraphMaxElems = (int64_t)1 << (getenv("SE2_GRAPH_MAX_LOG2") ? atoi(getenv("SE2_GRAPH_MAX_LOG2")) : 21);

static se2_status check_kernel(se2_kernel k) {
    if (!k) {
        set_error("null kernel");
        return SE2_EINVAL;
    }
    return SE2_OK;
}


static void fill_prox(Epilogue& epi, const se2_kernel_s* k, const se2_prox* prox) {
    epi.prox_kind = prox->kind;
    if (prox->kind == SE2_PROX_POROUS) {
        // C = tau m / (eps (m-1)) cell^{1-m}: the energy acts on the density s / cell, cell = dx dy dtheta
        const double cell = k->hx * k->hy * (6.283185307179586476925286766559 / k->nt);
        epi.prox_lnc = (float)(log(prox->tau * prox->m / (k->eps * (prox->m - 1.0))) + (1.0 - prox->m) * log(cell));
        epi.prox_m1 = (float)(prox->m - 1.0);
    }
    const double p = prox->tau / (k->eps + prox->tau);
    epi.prox_p = (float)p;
    epi.prox_q = (float)p;
    epi.cx = (float)prox->cx;
    epi.cy = (float)prox->cy;
    epi.hx = (float)prox->hx;
    epi.hy = (float)prox->hy;
}

// zero the guard counters at the start of a solve (stream-ordered, outside any captured graph)
static se2_status reset_guard(se2_kernel_s* k, cudaStream_t s) {
    SE2_CUDA_TRY(cudaMemsetAsync(k->guard, 0, sizeof(unsigned int) * 4, s));
    return SE2_OK;
}

// one fp64-potential log conv (K4P) with the kernel's optional per-launch timing events
static se2_status run_conv_precise(se2_kernel_s* k, const double* in, int batch, const EpiP& epi, cudaStream_t s) {
    NvtxRange nvtx_conv("se2 conv (log domain, fp64 potentials)");
    Timing& t = k->timing;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (t.on) {
        if (t.used == t.events.size()) {
            cudaEvent_t a, b;
            SE2_CUDA_TRY(cudaEventCreate(&a));
            SE2_CUDA_TRY(cudaEventCreate(&b));
            t.events.push_back({a, b});
        }
        e0 = t.events[t.used].first;
        e1 = t.events[t.used].second;
        t.used++;
        SE2_CUDA_TRY(cudaEventRecord(e0, s));
    }
    cudaError_t e = launch_conv_lse_precise(k, in, batch, epi, s, nullptr);
    if (e != cudaSuccess) {
        set_error(std::string("precise conv launch: ") + cudaGetErrorString(e));
        return SE2_ECUDA;
    }
    t.all_launches++;
    if (t.on) SE2_CUDA_TRY(cudaEventRecord(e1, s));
    return SE2_OK;
}


// End of a solve: count non-finite entries of the outputs (SE2_ENONFINITE) and read the guard counters
// of the solve: clamped divisions -> warning SE2_WGUARD_HIT (the clamp is counted and reported),
// porous prox sites without convergence -> warning SE2_WPROX_NOCONV.  Outputs stay valid on warnings.
static se2_status check_finite(se2_kernel_s* k, const float* const* ptrs, const int64_t* ns, int count,
                               cudaStream_t s) {
    KernelExtra* x = extra(k);
    se2_status st = ensure(x->misc, 4096);
    if (st != SE2_OK) return st;
    int* cnt = reinterpret_cast<int*>(x->misc.ptr);
    SE2_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int), s));
    for (int i = 0; i < count; ++i)
        if (ptrs[i]) SE2_CUDA_TRY(launch_count_nonfinite(ptrs[i], ns[i], cnt, s));
    int h = 0;
    unsigned int gh[4] = {0, 0, 0, 0};
    SE2_CUDA_TRY(cudaMemcpyAsync(&h, cnt, sizeof(int), cudaMemcpyDeviceToHost, s));
    SE2_CUDA_TRY(cudaMemcpyAsync(gh, k->guard, sizeof(gh), cudaMemcpyDeviceToHost, s));
    SE2_CUDA_TRY(cudaStreamSynchronize(s));
    if (h != 0) {
        set_error("non-finite values produced by the iteration (" + std::to_string(h) + " entries)");
        return SE2_ENONFINITE;
    }
    if (gh[1] != 0) {
        set_error("porous prox: " + std::to_string(gh[1]) + " site evaluations did not converge");
        return SE2_WPROX_NOCONV;
    }
    if (gh[0] != 0) {
        set_error("division guard clamped " + std::to_string(gh[0]) + " denominators at 1e-30");
        return SE2_WGUARD_HIT;
    }
    return SE2_OK;
}

