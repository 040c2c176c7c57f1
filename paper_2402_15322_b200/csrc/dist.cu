// Multi-GPU scaling loops behind the C ABI (B:north_star: "independent barycenter inputs ... go per GPU,
// with an NCCL allreduce over NVLink for the barycenter log-mean, and a single large grid is split into
// spatial slabs with NVLink halo exchange").  One process (or, for the loopback transport, one host
// thread) per rank.
//
//  * se2_comm: a communicator.  Production transport: NCCL (libnccl.so.2, resolved with dlopen at
//    se2_comm_init, so the library loads without it and shares the NCCL build torch already loaded).
//    Test transport: "loopback" -- n ranks as n host threads of one process on one GPU; the exchanges
//    are stream-ordered device copies / reduction kernels synchronised with CUDA events and host-side
//    rendezvous (no kernel ever waits on another rank's kernel), so the slab / shard logic runs on one
//    GPU exactly as it would on n.
//  * se2_jko_step_dist: the entropic JKO step (R10) on a row slab of the grid: every conv
//    computes only the owned rows (the kernel's output window), its epilogue packs the first / last R
//    owned rows into send buffers, and the neighbours' rows arrive in the halo rows before the next conv
//    reads them; the plan mass and the error trace are summed over the slabs.
//  * se2_barycenter_dist: App. A with the inputs sharded over the `reduce` ranks (one
//    allreduce of the partial weighted log-mean per iteration) and, optionally, each input's grid split
//    into row slabs over the `slabs` ranks (c3 on 8 GPUs: 4 inputs x 2 slabs).
#include <dlfcn.h>
#include <nccl.h>   // types and enum values only: the functions are resolved with dlopen

#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>

#include "api_internal.cuh"

namespace {

// ---------------------------------------------------------------------------------------------------
// NCCL entry points (dlopen)
// ---------------------------------------------------------------------------------------------------
struct Nccl {
    bool loaded = false;
    std::string why;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclCommSplit) CommSplit = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    decltype(&ncclCommCount) CommCount = nullptr;
    decltype(&ncclCommUserRank) CommUserRank = nullptr;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        // prefer the libnccl already mapped into the process (torch's), else the system one
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            n.why = std::string("dlopen libnccl.so.2: ") + dlerror();
            return;
        }
#define SE2_SYM(f)                                                      \
    n.f = reinterpret_cast<decltype(n.f)>(dlsym(h, "nccl" #f));          \
    if (!n.f) {                                                         \
        n.why = "libnccl lacks nccl" #f;                                \
        return;                                                         \
    }
        SE2_SYM(GetUniqueId) SE2_SYM(CommInitRank) SE2_SYM(CommDestroy) SE2_SYM(CommSplit) SE2_SYM(AllReduce)
        SE2_SYM(Send) SE2_SYM(Recv) SE2_SYM(GroupStart) SE2_SYM(GroupEnd) SE2_SYM(GetErrorString)
        SE2_SYM(CommCount) SE2_SYM(CommUserRank)
#undef SE2_SYM
        n.loaded = true;
    });
    return n;
}

#define SE2_NCCL_TRY(expr)                                                                           \
    do {                                                                                             \
        ncclResult_t _r = (expr);                                                                    \
        if (_r != ncclSuccess) {                                                                     \
            set_error(std::string(#expr) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(_r) : "?")); \
            return SE2_ENCCL;                                                                        \
        }                                                                                            \
    } while (0)

// ---------------------------------------------------------------------------------------------------
// small kernels of the exchanges
// ---------------------------------------------------------------------------------------------------
inline int grid_of(int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, 148 * 16); }

// x[plane][row0 + r][i] = src[plane][r][i] for r < rows (received halo rows into the local grid)
__global__ void unpack_rows_kernel(float* __restrict__ x, int planes, int ny, int nx, int row0, int rows,
                                   const float* __restrict__ src) {
    const int64_t n = (int64_t)planes * rows * nx;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = i / ((int64_t)rows * nx);
        const int64_t rem = i - p * rows * nx;
        x[(p * ny + row0) * nx + rem] = src[i];
    }
}

// dst[plane][r][i] = x[plane][row0 + r][i] for r < rows (boundary rows of a field not produced by a conv)
__global__ void pack_rows_kernel(const float* __restrict__ x, int planes, int ny, int nx, int row0, int rows,
                                 float* __restrict__ dst) {
    const int64_t n = (int64_t)planes * rows * nx;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = i / ((int64_t)rows * nx);
        const int64_t rem = i - p * rows * nx;
        dst[i] = x[(p * ny + row0) * nx + rem];
    }
}

// x[plane][row0 + r][i] /= *sum for r < rows (the slab's share of mu_{k+1} = s / sum s)
__global__ void scale_rows_dev_kernel(float* __restrict__ x, int planes, int ny, int nx, int row0, int rows,
                                      const double* __restrict__ sum) {
    const double inv = 1.0 / *sum;   // as launch_scale: the product in fp64, rounded once
    const int64_t n = (int64_t)planes * rows * nx;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = i / ((int64_t)rows * nx);
        const int64_t rem = i - p * rows * nx;
        float* e = x + (p * ny + row0) * nx + rem;
        *e = (float)((double)*e * inv);
    }
}

// out[i] = sum_{q < n} in[q][i] in rank order (loopback allreduce; the same order on every rank)
template <class T>
__global__ void sum_ranks_kernel(const T* const* __restrict__ in, int n, int64_t count, T* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        T t = in[0][i];
        for (int q = 1; q < n; ++q) t += in[q][i];
        out[i] = t;
    }
}

}  // namespace

// ---------------------------------------------------------------------------------------------------
// communicators
// ---------------------------------------------------------------------------------------------------
struct se2_comm_s {
    int n = 1, r = 0, device = 0;
    bool capturable = true;   // the exchanges can be recorded into a CUDA graph
    // the solvers run their collectives on this communicator: more than one rank, or a one-rank NCCL
    // communicator built from a unique id (the NCCL transport exercised on one GPU)
    bool live = false;
    virtual ~se2_comm_s() {}
    // in-place sum over the ranks (f64: doubles, else floats), identical result on every rank
    virtual se2_status allreduce(void* buf, int64_t count, bool f64, cudaStream_t s) = 0;
    // halo exchange along the rank order: send_up -> rank r-1 (which receives it as recv_dn), send_dn ->
    // rank r+1 (received as recv_up); ranks 0 / n-1 have no upper / lower neighbour (pointers ignored)
    virtual se2_status neighbours(const float* send_up, float* recv_up, const float* send_dn, float* recv_dn,
                                  int64_t count, cudaStream_t s) = 0;
    virtual se2_status split(int color, int key, se2_comm_s** out) = 0;
};

namespace {

struct NcclComm final : se2_comm_s {
    ncclComm_t c = nullptr;
    ~NcclComm() override {
        if (c && nccl().loaded) nccl().CommDestroy(c);
    }
    se2_status allreduce(void* buf, int64_t count, bool f64, cudaStream_t s) override {
        if (c == nullptr || count == 0) return SE2_OK;
        SE2_NCCL_TRY(nccl().AllReduce(buf, buf, (size_t)count, f64 ? ncclFloat64 : ncclFloat32, ncclSum, c, s));
        return SE2_OK;
    }
    se2_status neighbours(const float* send_up, float* recv_up, const float* send_dn, float* recv_dn, int64_t count,
                          cudaStream_t s) override {
        if (n == 1 || count == 0) return SE2_OK;
        SE2_NCCL_TRY(nccl().GroupStart());
        if (r > 0) {
            SE2_NCCL_TRY(nccl().Send(send_up, (size_t)count, ncclFloat32, r - 1, c, s));
            SE2_NCCL_TRY(nccl().Recv(recv_up, (size_t)count, ncclFloat32, r - 1, c, s));
        }
        if (r + 1 < n) {
            SE2_NCCL_TRY(nccl().Send(send_dn, (size_t)count, ncclFloat32, r + 1, c, s));
            SE2_NCCL_TRY(nccl().Recv(recv_dn, (size_t)count, ncclFloat32, r + 1, c, s));
        }
        SE2_NCCL_TRY(nccl().GroupEnd());
        return SE2_OK;
    }
    se2_status split(int color, int key, se2_comm_s** out) override {
        auto* m = new NcclComm();
        ncclComm_t nc = nullptr;
        ncclResult_t rr = nccl().CommSplit(c, color, key, &nc, nullptr);
        if (rr != ncclSuccess) {
            delete m;
            set_error(std::string("ncclCommSplit: ") + nccl().GetErrorString(rr));
            return SE2_ENCCL;
        }
        int cnt = 1, me = 0;
        nccl().CommCount(nc, &cnt);
        nccl().CommUserRank(nc, &me);
        m->c = nc;
        m->n = cnt;
        m->r = me;
        m->device = device;
        m->live = true;
        *out = m;
        return SE2_OK;
    }
};

// ---- loopback: n ranks as host threads of one process (tests of the multi-rank logic on one GPU) ----
struct LoopWorld {
    int n = 1;
    std::mutex mu;
    std::condition_variable cv;
    // generation-counted rendezvous that also gathers one record per rank
    struct Rec {
        const void* p0 = nullptr;
        const void* p1 = nullptr;
        cudaEvent_t ev = nullptr;
        int a = 0, b = 0;
    };
    std::vector<Rec> cur, done;
    int arrived = 0;
    uint64_t gen = 0;
    std::map<std::pair<uint64_t, int>, std::shared_ptr<LoopWorld>> subs;   // (split sequence, color)
    // events of destroyed member comms: a slower rank may still be enqueueing a wait on an event of a rank
    // that already returned from the call and destroyed its communicator, so they live as long as the world
    std::vector<cudaEvent_t> retired;
    ~LoopWorld() {
        for (auto e : retired) cudaEventDestroy(e);
    }

    std::vector<Rec> gather(int r, const Rec& rec) {
        std::unique_lock<std::mutex> lk(mu);
        if (cur.empty()) cur.resize(n);
        cur[r] = rec;
        const uint64_t g = gen;
        if (++arrived == n) {
            done = cur;
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
        return done;   // copied under the lock; the next generation's completion waits for every rank
    }
};

struct LoopComm final : se2_comm_s {
    std::shared_ptr<LoopWorld> w;
    uint64_t splits = 0;
    std::vector<cudaEvent_t> evs;
    size_t next_ev = 0;
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    void** table = nullptr;   // device pointer table (n entries)
    LoopComm() { capturable = false; }
    ~LoopComm() override {
        if (w) {
            std::lock_guard<std::mutex> lk(w->mu);
            w->retired.insert(w->retired.end(), evs.begin(), evs.end());
        } else {
            for (auto e : evs) cudaEventDestroy(e);
        }
        if (scratch) cudaFree(scratch);
        if (table) cudaFree(table);
    }
    cudaEvent_t event() {
        if (evs.size() < 8) {
            cudaEvent_t e;
            cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            evs.push_back(e);
        }
        return evs[next_ev++ % evs.size()];
    }
    se2_status allreduce(void* buf, int64_t count, bool f64, cudaStream_t s) override {
        if (n == 1 || count == 0) return SE2_OK;
        const size_t bytes = (size_t)count * (f64 ? 8 : 4);
        if (scratch_bytes < bytes) {
            if (scratch) cudaFree(scratch);
            SE2_CUDA_TRY(cudaMalloc(&scratch, bytes));
            scratch_bytes = bytes;
        }
        if (!table) SE2_CUDA_TRY(cudaMalloc(&table, sizeof(void*) * n));
        LoopWorld::Rec me;
        me.p0 = buf;
        me.ev = event();
        SE2_CUDA_TRY(cudaEventRecord(me.ev, s));
        auto all = w->gather(r, me);
        std::vector<const void*> ptrs(n);
        for (int q = 0; q < n; ++q) {
            SE2_CUDA_TRY(cudaStreamWaitEvent(s, all[q].ev, 0));
            ptrs[q] = all[q].p0;
        }
        SE2_CUDA_TRY(cudaMemcpyAsync(table, ptrs.data(), sizeof(void*) * n, cudaMemcpyHostToDevice, s));
        if (f64)
            sum_ranks_kernel<double><<<grid_of(count), 256, 0, s>>>(reinterpret_cast<const double* const*>(table), n,
                                                                    count, reinterpret_cast<double*>(scratch));
        else
            sum_ranks_kernel<float><<<grid_of(count), 256, 0, s>>>(reinterpret_cast<const float* const*>(table), n,
                                                                   count, reinterpret_cast<float*>(scratch));
        count_launch();
        SE2_CUDA_TRY(cudaGetLastError());
        // every rank must have read every buffer before any rank overwrites its own
        LoopWorld::Rec rd;
        rd.ev = event();
        SE2_CUDA_TRY(cudaEventRecord(rd.ev, s));
        auto all2 = w->gather(r, rd);
        for (int q = 0; q < n; ++q) SE2_CUDA_TRY(cudaStreamWaitEvent(s, all2[q].ev, 0));
        SE2_CUDA_TRY(cudaMemcpyAsync(buf, scratch, bytes, cudaMemcpyDeviceToDevice, s));
        // the host copy of `ptrs` is consumed by the H2D copy above before the stream moves on
        SE2_CUDA_TRY(cudaStreamSynchronize(s));
        return SE2_OK;
    }
    se2_status neighbours(const float* send_up, float* recv_up, const float* send_dn, float* recv_dn, int64_t count,
                          cudaStream_t s) override {
        if (n == 1 || count == 0) return SE2_OK;
        LoopWorld::Rec me;
        me.p0 = send_up;
        me.p1 = send_dn;
        me.ev = event();
        SE2_CUDA_TRY(cudaEventRecord(me.ev, s));
        auto all = w->gather(r, me);
        const size_t bytes = (size_t)count * sizeof(float);
        if (r > 0) {   // rank r-1's last rows -> my upper halo
            SE2_CUDA_TRY(cudaStreamWaitEvent(s, all[r - 1].ev, 0));
            SE2_CUDA_TRY(cudaMemcpyAsync(recv_up, all[r - 1].p1, bytes, cudaMemcpyDeviceToDevice, s));
        }
        if (r + 1 < n) {   // rank r+1's first rows -> my lower halo
            SE2_CUDA_TRY(cudaStreamWaitEvent(s, all[r + 1].ev, 0));
            SE2_CUDA_TRY(cudaMemcpyAsync(recv_dn, all[r + 1].p0, bytes, cudaMemcpyDeviceToDevice, s));
        }
        // the neighbours read my send buffers: they may be rewritten only after those copies
        LoopWorld::Rec rd;
        rd.ev = event();
        SE2_CUDA_TRY(cudaEventRecord(rd.ev, s));
        auto all2 = w->gather(r, rd);
        if (r > 0) SE2_CUDA_TRY(cudaStreamWaitEvent(s, all2[r - 1].ev, 0));
        if (r + 1 < n) SE2_CUDA_TRY(cudaStreamWaitEvent(s, all2[r + 1].ev, 0));
        return SE2_OK;
    }
    se2_status split(int color, int key, se2_comm_s** out) override {
        LoopWorld::Rec me;
        me.a = color;
        me.b = key;
        auto all = w->gather(r, me);
        const uint64_t seq = splits++;
        std::vector<std::pair<int, int>> members;   // (key, rank) of my color
        for (int q = 0; q < n; ++q)
            if (all[q].a == color) members.push_back({all[q].b, q});
        std::sort(members.begin(), members.end());
        auto* m = new LoopComm();
        m->n = (int)members.size();
        m->live = m->n > 1;
        for (int i = 0; i < m->n; ++i)
            if (members[i].second == r) m->r = i;
        m->device = device;
        {
            std::lock_guard<std::mutex> lk(w->mu);
            auto& sw = w->subs[{seq, color}];
            if (!sw) {
                sw = std::make_shared<LoopWorld>();
                sw->n = m->n;
            }
            m->w = sw;
        }
        *out = m;
        return SE2_OK;
    }
};

// ---------------------------------------------------------------------------------------------------
// slab geometry of a dist call
// ---------------------------------------------------------------------------------------------------
struct Slab {
    int top = 0, bot = 0;     // halo rows above / below the owned rows
    int lo = 0, hi = 0;       // owned rows [lo, hi) of the kernel grid
    bool on = false;          // more than one slab
};

se2_status slab_of(se2_kernel_s* k, const se2_dist* d, Slab* sl) {
    SE2_CHECK_ARG(d->halo_top >= 0 && d->halo_bot >= 0 && d->halo_top + d->halo_bot < k->ny, "bad halo rows");
    sl->top = d->halo_top;
    sl->bot = d->halo_bot;
    sl->lo = d->halo_top;
    sl->hi = k->ny - d->halo_bot;
    sl->on = d->slabs != nullptr && d->slabs->n > 1;
    if (sl->on) {
        const se2_comm_s* c = d->slabs;
        SE2_CHECK_ARG(sl->top == (c->r > 0 ? k->R : 0) && sl->bot == (c->r + 1 < c->n ? k->R : 0),
                      "halo rows must be R toward each neighbour slab and 0 at the global edges");
        SE2_CHECK_ARG(sl->hi - sl->lo >= k->R, "every slab must own at least R rows (its halo comes from one neighbour)");
    } else {
        SE2_CHECK_ARG(sl->top == 0 && sl->bot == 0, "halo rows without a slab communicator");
    }
    if (k->wlo() != sl->lo || k->whi() != sl->hi) {   // the kernel's output window = the owned rows
        k->win_lo = sl->lo;
        k->win_hi = (sl->lo == 0 && sl->hi == k->ny) ? 0 : sl->hi;
        extra(k)->clear_graphs();
        cudaError_t e = conv_tc_decide(k);
        if (e != cudaSuccess) {
            set_error(std::string("K10 geometry: ") + cudaGetErrorString(e));
            return SE2_ECUDA;
        }
    }
    return SE2_OK;
}

// pack pointers for an epilogue: first / last R owned rows into send_up / send_dn ([planes][R][nx])
void set_pack(Epilogue& e, const se2_kernel_s* k, const Slab& sl, const se2_comm_s* c, float* send_up,
              float* send_dn) {
    if (!sl.on) return;
    e.slab_lo = sl.lo;
    e.slab_hi = sl.hi;
    e.slab_halo = k->R;
    e.ny_self = k->ny;
    e.nx_self = k->nx;
    if (c->r > 0) {
        e.halo_up = send_up;
        e.up_shift = -sl.lo;
        e.ny_up = k->R;
    }
    if (c->r + 1 < c->n) {
        e.halo_dn = send_dn;
        e.dn_shift = sl.hi - k->R;
        e.ny_dn = k->R;
    }
}

// neighbours' boundary rows -> the halo rows of x ([planes][ny][nx]).  The send buffers hold x's first /
// last R owned rows: packed by the producing conv's epilogue (set_pack), or here when pack is set (fields
// written by elementwise kernels)
// (row_words: 4-byte words per grid row -- nx for float fields, 2 nx for fp64 fields moved as word pairs)
se2_status exchange(se2_kernel_s* k, const Slab& sl, se2_comm_s* c, float* x, int planes, float* bufs, cudaStream_t s,
                    bool pack = false, int row_words = 0) {
    if (!sl.on) return SE2_OK;
    const int nxw = row_words > 0 ? row_words : k->nx;
    const int64_t cnt = (int64_t)planes * k->R * nxw;
    float* send_up = bufs;
    float* send_dn = bufs + cnt;
    float* recv_up = bufs + 2 * cnt;
    float* recv_dn = bufs + 3 * cnt;
    if (pack) {
        if (c->r > 0) {
            pack_rows_kernel<<<grid_of(cnt), 256, 0, s>>>(x, planes, k->ny, nxw, sl.lo, k->R, send_up);
            count_launch();
        }
        if (c->r + 1 < c->n) {
            pack_rows_kernel<<<grid_of(cnt), 256, 0, s>>>(x, planes, k->ny, nxw, sl.hi - k->R, k->R, send_dn);
            count_launch();
        }
        SE2_CUDA_TRY(cudaGetLastError());
    }
    se2_status st = c->neighbours(send_up, recv_up, send_dn, recv_dn, cnt, s);
    if (st != SE2_OK) return st;
    if (sl.top > 0) {
        unpack_rows_kernel<<<grid_of(cnt), 256, 0, s>>>(x, planes, k->ny, nxw, 0, sl.top, recv_up);
        count_launch();
    }
    if (sl.bot > 0) {
        unpack_rows_kernel<<<grid_of(cnt), 256, 0, s>>>(x, planes, k->ny, nxw, sl.hi, sl.bot, recv_dn);
        count_launch();
    }
    SE2_CUDA_TRY(cudaGetLastError());
    return SE2_OK;
}

bool any_multi(const se2_dist* d) {
    return (d->slabs && d->slabs->n > 1) || (d->reduce && d->reduce->live);
}
bool all_capturable(const se2_dist* d) {
    return (!d->slabs || d->slabs->n == 1 || d->slabs->capturable) && (!d->reduce || !d->reduce->live || d->reduce->capturable);
}

}  // namespace

// ---------------------------------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------------------------------
extern "C" {

se2_status se2_comm_unique_id(uint8_t* id_out) {
    SE2_CHECK_ARG(id_out != nullptr, "null id");
    Nccl& n = nccl();
    if (!n.loaded) {
        set_error(n.why);
        return SE2_ENCCL;
    }
    ncclUniqueId id;
    SE2_NCCL_TRY(n.GetUniqueId(&id));
    memcpy(id_out, &id, sizeof(id));
    return SE2_OK;
}

se2_status se2_comm_init(const uint8_t* id, int32_t nranks, int32_t rank, int32_t device, se2_comm* out) {
    SE2_CHECK_ARG(out != nullptr, "null out");
    *out = nullptr;
    SE2_CHECK_ARG(nranks >= 1 && rank >= 0 && rank < nranks && device >= 0, "bad rank / size / device");
    auto* c = new NcclComm();
    c->n = nranks;
    c->r = rank;
    c->device = device;
    SE2_CHECK_ARG(nranks == 1 || id != nullptr, "null unique id");
    if (id != nullptr) {   // nranks = 1 with an id: a real one-rank NCCL communicator
        Nccl& n = nccl();
        if (!n.loaded) {
            delete c;
            set_error(n.why);
            return SE2_ENCCL;
        }
        DeviceGuard g(device);
        ncclUniqueId uid;
        memcpy(&uid, id, sizeof(uid));
        ncclResult_t r = n.CommInitRank(&c->c, nranks, uid, rank);
        if (r != ncclSuccess) {
            delete c;
            set_error(std::string("ncclCommInitRank: ") + n.GetErrorString(r));
            return SE2_ENCCL;
        }
        c->live = true;
    }
    *out = c;
    return SE2_OK;
}

se2_status se2_comm_init_loopback(int32_t nranks, int32_t device, se2_comm* out) {
    SE2_CHECK_ARG(out != nullptr && nranks >= 1 && device >= 0, "bad arguments");
    auto w = std::make_shared<LoopWorld>();
    w->n = nranks;
    for (int r = 0; r < nranks; ++r) {
        auto* c = new LoopComm();
        c->n = nranks;
        c->live = nranks > 1;
        c->r = r;
        c->device = device;
        c->w = w;
        out[r] = c;
    }
    return SE2_OK;
}

se2_status se2_comm_split(se2_comm parent, int32_t color, int32_t key, se2_comm* out) {
    SE2_CHECK_ARG(parent != nullptr && out != nullptr && color >= 0, "bad arguments");
    *out = nullptr;
    if (parent->n == 1 && !parent->live) {
        auto* c = new NcclComm();   // a single rank: no transport needed
        c->device = parent->device;
        *out = c;
        return SE2_OK;
    }
    DeviceGuard g(parent->device);
    se2_comm_s* c = nullptr;
    se2_status st = parent->split(color, key, &c);
    if (st != SE2_OK) return st;
    *out = c;
    return SE2_OK;
}

se2_status se2_comm_info(se2_comm c, int32_t* nranks, int32_t* rank) {
    SE2_CHECK_ARG(c != nullptr, "null comm");
    if (nranks) *nranks = c->n;
    if (rank) *rank = c->r;
    return SE2_OK;
}

void se2_comm_destroy(se2_comm c) { delete c; }

se2_status se2_comm_allreduce(se2_comm c, void* buf, int64_t count, int32_t f64, se2_stream stream) {
    SE2_CHECK_ARG(c != nullptr && (buf != nullptr || count == 0) && count >= 0, "bad arguments");
    DeviceGuard g(c->device);
    return c->allreduce(buf, count, f64 != 0, (cudaStream_t)stream);
}

// ---- slab JKO -------------------------------------------------------------------------------------
se2_status se2_jko_step_dist(se2_kernel k, const se2_dist* dist, const float* mu_k, float* mu_next, float* a, float* b,
                             const se2_prox* prox, const se2_opts* opts, double* mass_host, double* err_trace_host,
                             se2_stream stream) {
    NvtxRange nvtx_call("se2_jko_step_dist");
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(dist != nullptr, "dist required (se2_jko_step for one GPU)");
    SE2_CHECK_ARG(opts != nullptr && opts->iters >= 1, "opts required, iters >= 1");
    SE2_CHECK_ARG(prox != nullptr && prox->tau >= 0 &&
                      (prox->kind == SE2_PROX_ENTROPY_POTENTIAL || (prox->kind == SE2_PROX_POROUS && prox->m > 1.0)),
                  "JKO prox required (entropy+potential, or porous with m > 1)");
    SE2_CHECK_ARG(mu_k && mu_next && a && b && mu_k != mu_next && a != b, "bad pointers");
    SE2_CHECK_ARG(!(opts->flags & SE2_WARM_START), "warm start is not supported by the slab JKO");
    DeviceGuard g(k->device);
    cudaStream_t s = (cudaStream_t)stream;
    Slab sl;
    se2_status st = slab_of(k, dist, &sl);
    if (st != SE2_OK) return st;
    st = reset_guard(k, s);
    if (st != SE2_OK) return st;
    se2_comm_s* sc = dist->slabs;
    const bool LOG = (opts->flags & SE2_LOG_DOMAIN) != 0;
    const bool trace = (opts->flags & SE2_TRACE_ERR) != 0 && err_trace_host != nullptr;
    const int iters = opts->iters;
    const int64_t N = k->N();
    KernelExtra* x = extra(k);
    const int64_t cnt = (int64_t)k->nt * k->R * k->nx;   // one direction's halo rows
    // workspace: log target (log domain), 4 halo buffers, shift hints (log domain)
    size_t need = (size_t)((LOG ? 3 : 0) * N + 4 * cnt) * sizeof(float);
    st = ensure(x->ws, std::max<size_t>(need, 16), x);
    if (st != SE2_OK) return st;
    float* lmu = reinterpret_cast<float*>(x->ws.ptr);
    float* bufs = lmu + (LOG ? N : 0);
    float* hint1 = LOG && k->R >= 5 ? bufs + 4 * cnt : nullptr;
    float* hint2 = hint1 ? hint1 + N : nullptr;
    const int bpf = conv_blocks_per_field(k, LOG, opts->flags);
    if (trace) {
        st = ensure(x->partial, (size_t)bpf * sizeof(float), x);
        if (st != SE2_OK) return st;
        st = ensure(x->trace, (size_t)iters * sizeof(double), x);
        if (st != SE2_OK) return st;
    }
    st = ensure(x->misc, 4096, x);
    if (st != SE2_OK) return st;
    float* partial = reinterpret_cast<float*>(x->partial.ptr);
    double* tr = reinterpret_cast<double*>(x->trace.ptr);
    double* dsum = reinterpret_cast<double*>(reinterpret_cast<char*>(x->misc.ptr) + 64);
    double* dscr = dsum + 8;
    std::vector<uint64_t> key = {3, as_key(mu_k), as_key(mu_next), as_key(a), as_key(b), (uint64_t)iters,
                                 (uint64_t)opts->flags, (uint64_t)trace, as_key(x->ws.ptr), as_key(partial), as_key(tr),
                                 (uint64_t)sl.lo, (uint64_t)sl.hi, (uint64_t)prox->kind};
    for (double v : {prox->tau, prox->cx, prox->cy, prox->hx, prox->hy, prox->m}) key.push_back(as_key(v));
    auto enqueue = [&](cudaStream_t s) -> se2_status {
        se2_status st = SE2_OK;
        const float* tmu = mu_k;
        if (LOG) {
            SE2_CUDA_TRY(launch_log(mu_k, lmu, N, s));
            tmu = lmu;
        }
        // b = 1 on every row: the halo rows hold the neighbours' b (= 1 as well)
        SE2_CUDA_TRY(launch_fill(b, N, LOG ? 0.f : 1.f, s));
        if (sl.on) SE2_CUDA_TRY(launch_fill(mu_next, N, 0.f, s));   // its halo rows are never written
        for (int l = 0; l < iters; ++l) {
            NvtxRange nvtx_iter("se2 iteration", l);
            Epilogue e1;   // a = mu / K b, owned rows; error of the previous iterate fused
            e1.op = EPI_DIVIDE;
            e1.target = tmu;
            e1.out = a;
            e1.hint_in = (l > 0) ? hint1 : nullptr;
            e1.hint_out = hint1;
            if (trace && l > 0) {
                e1.err_a = a;
                e1.err_mu = mu_k;
                e1.err_partial = partial;
            }
            set_pack(e1, k, sl, sc, bufs, bufs + cnt);
            st = run_conv(k, b, 1, opts->flags, e1, s, nullptr);
            if (st != SE2_OK) return st;
            if (trace && l > 0) SE2_CUDA_TRY(launch_reduce_partials(partial, 1, bpf, tr + (l - 1), s));
            st = exchange(k, sl, sc, a, k->nt, bufs, s);
            if (st != SE2_OK) return st;
            Epilogue e2;   // b = prox(K a) / K a, owned rows; s = b K a on the last iteration
            e2.op = EPI_PROX;
            e2.out = b;
            e2.hint_in = (l > 0) ? hint2 : nullptr;
            e2.hint_out = hint2;
            fill_prox(e2, k, prox);
            if (l == iters - 1) e2.out2 = mu_next;
            set_pack(e2, k, sl, sc, bufs, bufs + cnt);
            st = run_conv(k, a, 1, opts->flags, e2, s, nullptr);
            if (st != SE2_OK) return st;
            st = exchange(k, sl, sc, b, k->nt, bufs, s);
            if (st != SE2_OK) return st;
        }
        if (trace) {
            Epilogue e3;
            e3.op = EPI_ERRONLY;
            e3.err_a = a;
            e3.err_mu = mu_k;
            e3.err_partial = partial;
            e3.hint_in = hint1;
            st = run_conv(k, b, 1, opts->flags, e3, s, nullptr);
            if (st != SE2_OK) return st;
            SE2_CUDA_TRY(launch_reduce_partials(partial, 1, bpf, tr + (iters - 1), s));
        }
        // mu_{k+1} = s / sum s over every slab's owned rows (one slab: exactly se2_jko_step's reduction)
        if (!sl.on) {
            SE2_CUDA_TRY(launch_sum(mu_next, N, dsum, dscr, s));
            SE2_CUDA_TRY(launch_scale(mu_next, N, dsum, s));
            return SE2_OK;
        }
        SE2_CUDA_TRY(launch_sum_rows(mu_next, k->nt, k->ny, k->nx, sl.lo, sl.hi - sl.lo, dsum, dscr, s));
        st = sc->allreduce(dsum, 1, true, s);
        if (st != SE2_OK) return st;
        scale_rows_dev_kernel<<<grid_of((int64_t)k->nt * (sl.hi - sl.lo) * k->nx), 256, 0, s>>>(
            mu_next, k->nt, k->ny, k->nx, sl.lo, sl.hi - sl.lo, dsum);
        count_launch();
        SE2_CUDA_TRY(cudaGetLastError());
        return SE2_OK;
    };
    const bool graph = N <= kGraphMaxElems && !(opts->flags & SE2_NO_GRAPH) && !any_multi(dist);
    st = run_graph(k, s, std::move(key), graph, enqueue);
    if (st != SE2_OK) return st;
    if (trace) {
        if (sc) {
            st = sc->allreduce(tr, iters, true, s);
            if (st != SE2_OK) return st;
        }
        SE2_CUDA_TRY(cudaMemcpyAsync(err_trace_host, tr, sizeof(double) * iters, cudaMemcpyDeviceToHost, s));
    }
    if (mass_host) SE2_CUDA_TRY(cudaMemcpyAsync(mass_host, dsum, sizeof(double), cudaMemcpyDeviceToHost, s));
    const float* ps[3] = {a, b, mu_next};
    const int64_t ns[3] = {N, N, N};
    return check_finite(k, ps, ns, 3, s);
}

// ---- sharded (+ slab) barycenter, log domain ---------------------------------------------------------
se2_status se2_barycenter_dist(se2_kernel k, const se2_dist* dist, int32_t n, int32_t nsolve, const float* mus,
                               const double* lambdas, float* bary, float* v_state, float* w_state, const se2_opts* opts,
                               double* err_trace_host, se2_stream stream) {
    NvtxRange nvtx_call("se2_barycenter_dist");
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(dist != nullptr, "dist required (se2_barycenter for one GPU)");
    SE2_CHECK_ARG(opts != nullptr && opts->iters >= 0, "opts required");
    SE2_CHECK_ARG((opts->flags & SE2_LOG_DOMAIN) != 0, "the distributed barycenter runs in the log domain (R13)");
    SE2_CHECK_ARG(n >= 1 && nsolve >= 1, "n (inputs on this rank), nsolve >= 1");
    SE2_CHECK_ARG((int64_t)n * nsolve <= k->max_batch, "n*nsolve exceeds max_batch");
    SE2_CHECK_ARG(mus && lambdas && bary, "null pointer");
    for (int i = 0; i < n * nsolve; ++i)
        SE2_CHECK_ARG(lambdas[i] >= 0 && isfinite(lambdas[i]), "lambda must be >= 0 (the simplex is over all ranks)");
    const bool warm = (opts->flags & SE2_WARM_START) != 0;
    SE2_CHECK_ARG(!warm || v_state != nullptr, "SE2_WARM_START needs v_state (the initial v_i)");
    DeviceGuard g(k->device);
    cudaStream_t s = (cudaStream_t)stream;
    Slab sl;
    se2_status st = slab_of(k, dist, &sl);
    if (st != SE2_OK) return st;
    st = reset_guard(k, s);
    if (st != SE2_OK) return st;
    se2_comm_s* sc = dist->slabs;
    se2_comm_s* rc = dist->reduce;
    const bool trace = (opts->flags & SE2_TRACE_ERR) != 0 && err_trace_host != nullptr;
    const int64_t N = k->N();
    const int F = n * nsolve;
    const int64_t FN = (int64_t)F * N;
    const int iters = opts->iters;
    KernelExtra* x = extra(k);
    const int64_t cnt = (int64_t)F * k->nt * k->R * k->nx;
    // workspace: mu_rep, lmu_rep, v, w, d, v_lo, hints (2) [F][N]; 4 halo buffers
    size_t need = (size_t)(8 * FN + 4 * cnt) * sizeof(float);
    st = ensure(x->ws, need, x);
    if (st != SE2_OK) return st;
    float* mu_rep = reinterpret_cast<float*>(x->ws.ptr);
    float* lmu_rep = mu_rep + FN;
    float* v = v_state ? v_state : lmu_rep + FN;
    float* w = w_state ? w_state : lmu_rep + 2 * FN;
    float* d = lmu_rep + 3 * FN;
    float* v_lo = lmu_rep + 4 * FN;
    const bool hints = k->R >= 5;
    float* hint1 = hints ? lmu_rep + 5 * FN : nullptr;
    float* hint2 = hints ? lmu_rep + 6 * FN : nullptr;
    float* bufs = mu_rep + 8 * FN;
    st = ensure(x->misc, 4096 + sizeof(float) * F, x);
    if (st != SE2_OK) return st;
    const int bpf = conv_blocks_per_field(k, true, opts->flags);
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
    SE2_CUDA_TRY(cudaStreamSynchronize(s));
    const bool reduce = rc != nullptr && rc->live;
    std::vector<uint64_t> key = {4, as_key(mus), as_key(bary), as_key(v), as_key(w), (uint64_t)n, (uint64_t)nsolve,
                                 (uint64_t)iters, (uint64_t)opts->flags, (uint64_t)trace, as_key(x->ws.ptr),
                                 as_key(x->misc.ptr), as_key(partial), as_key(tr), (uint64_t)sl.lo, (uint64_t)sl.hi};
    auto enqueue = [&](cudaStream_t s) -> se2_status {
        se2_status st = SE2_OK;
        for (int sv = 0; sv < nsolve; ++sv)
            SE2_CUDA_TRY(cudaMemcpyAsync(mu_rep + (int64_t)sv * n * N, mus, sizeof(float) * n * N,
                                         cudaMemcpyDeviceToDevice, s));
        SE2_CUDA_TRY(launch_log(mu_rep, lmu_rep, FN, s));
        if (!warm) SE2_CUDA_TRY(launch_fill(v, FN, 0.f, s));
        SE2_CUDA_TRY(launch_fill(v_lo, FN, 0.f, s));
        SE2_CUDA_TRY(launch_fill(w, FN, 0.f, s));
        if (sl.on) SE2_CUDA_TRY(launch_fill(d, FN, 0.f, s));   // halo rows of d are never written
        if (warm) {   // the caller's v_i may lack current halo rows
            st = exchange(k, sl, sc, v, F * k->nt, bufs, s, true);
            if (st != SE2_OK) return st;
        }
        for (int j = 0; j < iters; ++j) {
            NvtxRange nvtx_iter("se2 iteration", j);
            Epilogue e1;   // w_i = mu_i / K v_i
            e1.op = EPI_DIVIDE;
            e1.target = lmu_rep;
            e1.out = w;
            e1.hint_in = (j > 0) ? hint1 : nullptr;
            e1.hint_out = hint1;
            if (trace && j > 0) {
                e1.err_a = w;
                e1.err_mu = mu_rep;
                e1.err_partial = partial;
            }
            set_pack(e1, k, sl, sc, bufs, bufs + cnt);
            st = run_conv(k, v, F, opts->flags, e1, s, nullptr);
            if (st != SE2_OK) return st;
            if (trace && j > 0) SE2_CUDA_TRY(launch_reduce_partials(partial, F, bpf, tr + (int64_t)(j - 1) * F, s));
            st = exchange(k, sl, sc, w, F * k->nt, bufs, s);
            if (st != SE2_OK) return st;
            Epilogue e2;   // d_i = v_i K w_i
            e2.op = EPI_MULTIPLY;
            e2.target = v;
            e2.out = d;
            e2.hint_in = (j > 0) ? hint2 : nullptr;
            e2.hint_out = hint2;
            st = run_conv(k, w, F, opts->flags, e2, s, nullptr);
            if (st != SE2_OK) return st;
            if (!reduce) {   // mu = prod_i d_i^lambda_i and v_i <- v_i mu / d_i, fused
                SE2_CUDA_TRY(launch_bary_logmean_update(n, nsolve, N, d, lam_dev, bary, v, v_lo, s));
            } else {         // this rank's partial sum_i lambda_i log d_i, summed over the input ranks
                SE2_CUDA_TRY(launch_bary_logmean(n, nsolve, N, d, lam_dev, bary, s));
                st = rc->allreduce(bary, (int64_t)nsolve * N, false, s);
                if (st != SE2_OK) return st;
                SE2_CUDA_TRY(launch_bary_update_log(n, nsolve, N, v, v_lo, d, bary, s));
            }
            st = exchange(k, sl, sc, v, F * k->nt, bufs, s, true);   // v's halo rows for the next K v
            if (st != SE2_OK) return st;
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
    const bool graph = FN <= kGraphMaxElems && !(opts->flags & SE2_NO_GRAPH) && !any_multi(dist);
    st = run_graph(k, s, std::move(key), graph, enqueue);
    if (st != SE2_OK) return st;
    if (trace && iters > 0) {
        // per solve: sum_i lambda_i e_i over this rank's inputs, then over the slabs and the input ranks
        std::vector<double> h((size_t)iters * F), e((size_t)iters * nsolve, 0.0);
        SE2_CUDA_TRY(cudaMemcpyAsync(h.data(), tr, sizeof(double) * iters * F, cudaMemcpyDeviceToHost, s));
        SE2_CUDA_TRY(cudaStreamSynchronize(s));
        for (int j = 0; j < iters; ++j)
            for (int sv = 0; sv < nsolve; ++sv)
                for (int i = 0; i < n; ++i) e[(size_t)j * nsolve + sv] += lambdas[sv * n + i] * h[(size_t)j * F + sv * n + i];
        SE2_CUDA_TRY(cudaMemcpyAsync(tr, e.data(), sizeof(double) * e.size(), cudaMemcpyHostToDevice, s));
        if (sc) {
            st = sc->allreduce(tr, (int64_t)e.size(), true, s);
            if (st != SE2_OK) return st;
        }
        if (rc) {
            st = rc->allreduce(tr, (int64_t)e.size(), true, s);
            if (st != SE2_OK) return st;
        }
        SE2_CUDA_TRY(cudaMemcpyAsync(err_trace_host, tr, sizeof(double) * e.size(), cudaMemcpyDeviceToHost, s));
        SE2_CUDA_TRY(cudaStreamSynchronize(s));
    }
    const float* ps[3] = {bary, v, w};
    const int64_t ns[3] = {(int64_t)nsolve * N, FN, FN};
    return check_finite(k, ps, ns, 3, s);
}

// App. A with fp64 potentials (K4P, reading R19) and this rank's inputs: per iteration the partial weighted
// log-mean sum_i lambda_i log d_i (fp64) is all-reduced over `reduce` and, with row slabs, the fp64 w_i / v_i
// boundary rows are exchanged with the neighbour slabs (packed by a row-copy kernel: the fp64 epilogue has no
// packing stores) -- c3's 8-GPU "one input per GPU pair" layout on the 1e-4 engine.
se2_status se2_barycenter_precise_dist(se2_kernel k, const se2_dist* dist, int32_t n, int32_t nsolve, const float* mus,
                                       const double* lambdas, double* lbary, double* lv_state, double* lw_state,
                                       const se2_opts* opts, double* err_trace_host, se2_stream stream) {
    NvtxRange nvtx_call("se2_barycenter_precise_dist");
    if (check_kernel(k) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(dist != nullptr, "dist required (se2_barycenter_precise for one GPU)");
    SE2_CHECK_ARG(opts != nullptr && opts->iters >= 0, "opts required");
    SE2_CHECK_ARG(n >= 1 && nsolve >= 1, "n (inputs on this rank), nsolve >= 1");
    SE2_CHECK_ARG((int64_t)n * nsolve <= k->max_batch, "n*nsolve exceeds max_batch");
    SE2_CHECK_ARG(mus && lambdas && lbary, "null pointer");
    for (int i = 0; i < n * nsolve; ++i)
        SE2_CHECK_ARG(lambdas[i] >= 0 && isfinite(lambdas[i]), "lambda must be >= 0 (the simplex is over all ranks)");
    const bool warm = (opts->flags & SE2_WARM_START) != 0;
    SE2_CHECK_ARG(!warm || lv_state != nullptr, "SE2_WARM_START needs lv_state");
    DeviceGuard g(k->device);
    cudaStream_t s = (cudaStream_t)stream;
    SE2_CUDA_TRY(tabulate_precise(k, s));
    Slab sl;
    se2_status st = slab_of(k, dist, &sl);
    if (st != SE2_OK) return st;
    st = reset_guard(k, s);
    if (st != SE2_OK) return st;
    se2_comm_s* sc = dist->slabs;
    se2_comm_s* rc = dist->reduce;
    const bool reduce = rc != nullptr && rc->live;
    const bool trace = (opts->flags & SE2_TRACE_ERR) != 0 && err_trace_host != nullptr;
    const int64_t N = k->N();
    const int F = n * nsolve;
    const int64_t FN = (int64_t)F * N;
    const int iters = opts->iters;
    KernelExtra* x = extra(k);
    // workspace: mu_rep (float) [F][N]; lmu, v, w, d (double) [F][N]; 4 halo buffers of fp64 rows
    const int64_t cnt = sl.on ? (int64_t)F * k->nt * k->R * 2 * k->nx : 0;   // 4-byte words per buffer
    st = ensure(x->ws, (size_t)FN * (sizeof(float) + 4 * sizeof(double)) + 64 + (size_t)4 * cnt * sizeof(float), x);
    if (st != SE2_OK) return st;
    float* mu_rep = reinterpret_cast<float*>(x->ws.ptr);
    double* lmu = reinterpret_cast<double*>(reinterpret_cast<char*>(x->ws.ptr) + ((FN * sizeof(float) + 63) / 64) * 64);
    double* v = lv_state ? lv_state : lmu + FN;
    double* w = lw_state ? lw_state : lmu + 2 * FN;
    double* d = lmu + 3 * FN;
    float* bufs = reinterpret_cast<float*>(lmu + 4 * FN);
    auto xchg = [&](double* f, cudaStream_t s) {   // f's halo rows <- the neighbours' boundary rows (fp64)
        return exchange(k, sl, sc, reinterpret_cast<float*>(f), F * k->nt, bufs, s, true, 2 * k->nx);
    };
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
    std::vector<uint64_t> key = {6, as_key(mus), as_key(lbary), as_key(v), as_key(w), (uint64_t)n, (uint64_t)nsolve,
                                 (uint64_t)iters, (uint64_t)opts->flags, (uint64_t)trace, as_key(x->ws.ptr),
                                 as_key(x->misc.ptr), as_key(partial), as_key(tr), (uint64_t)sl.lo, (uint64_t)sl.hi};
    auto enqueue = [&](cudaStream_t s) -> se2_status {
        se2_status st = SE2_OK;
        for (int sv = 0; sv < nsolve; ++sv)
            SE2_CUDA_TRY(cudaMemcpyAsync(mu_rep + (int64_t)sv * n * N, mus, sizeof(float) * n * N,
                                         cudaMemcpyDeviceToDevice, s));
        SE2_CUDA_TRY(launch_log_f64(mu_rep, lmu, FN, s));
        if (!warm) SE2_CUDA_TRY(launch_fill_f64(v, FN, 0.0, s));
        SE2_CUDA_TRY(launch_fill_f64(w, FN, 0.0, s));
        if (sl.on) SE2_CUDA_TRY(launch_fill_f64(d, FN, 0.0, s));   // halo rows of d are never written
        if (warm) {   // the caller's v_i may lack current halo rows
            st = xchg(v, s);
            if (st != SE2_OK) return st;
        }
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
            st = xchg(w, s);
            if (st != SE2_OK) return st;
            EpiP e2;   // d_i = v_i K w_i
            e2.op = EPI_MULTIPLY;
            e2.target = v;
            e2.out = d;
            st = run_conv_precise(k, w, F, e2, s);
            if (st != SE2_OK) return st;
            if (!reduce) {
                SE2_CUDA_TRY(launch_bary_logmean_update_f64(n, nsolve, N, d, lam_dev, lbary, v, s));
            } else {   // this rank's partial sum_i lambda_i log d_i, summed over the input ranks in fp64
                SE2_CUDA_TRY(launch_bary_logmean_f64(n, nsolve, N, d, lam_dev, lbary, s));
                st = rc->allreduce(lbary, (int64_t)nsolve * N, true, s);
                if (st != SE2_OK) return st;
                SE2_CUDA_TRY(launch_bary_update_f64(n, nsolve, N, d, lbary, v, s));
            }
            st = xchg(v, s);   // v's halo rows for the next K v
            if (st != SE2_OK) return st;
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
    const bool graph = FN <= kGraphMaxElems && !(opts->flags & SE2_NO_GRAPH) && !any_multi(dist);
    st = run_graph(k, s, std::move(key), graph, enqueue);
    if (st != SE2_OK) return st;
    if (trace && iters > 0) {
        std::vector<double> h((size_t)iters * F), e((size_t)iters * nsolve, 0.0);
        SE2_CUDA_TRY(cudaMemcpyAsync(h.data(), tr, sizeof(double) * iters * F, cudaMemcpyDeviceToHost, s));
        SE2_CUDA_TRY(cudaStreamSynchronize(s));
        for (int j = 0; j < iters; ++j)
            for (int sv = 0; sv < nsolve; ++sv)
                for (int i = 0; i < n; ++i) e[(size_t)j * nsolve + sv] += lambdas[sv * n + i] * h[(size_t)j * F + sv * n + i];
        SE2_CUDA_TRY(cudaMemcpyAsync(tr, e.data(), sizeof(double) * e.size(), cudaMemcpyHostToDevice, s));
        if (sc) {
            st = sc->allreduce(tr, (int64_t)e.size(), true, s);
            if (st != SE2_OK) return st;
        }
        if (rc) {
            st = rc->allreduce(tr, (int64_t)e.size(), true, s);
            if (st != SE2_OK) return st;
        }
        SE2_CUDA_TRY(cudaMemcpyAsync(err_trace_host, tr, sizeof(double) * e.size(), cudaMemcpyDeviceToHost, s));
        SE2_CUDA_TRY(cudaStreamSynchronize(s));
    }
    int* nbad = reinterpret_cast<int*>(x->misc.ptr);
    SE2_CUDA_TRY(cudaMemsetAsync(nbad, 0, sizeof(int), s));
    SE2_CUDA_TRY(launch_count_nonfinite_f64(lbary, (int64_t)nsolve * N, nbad, s));
    SE2_CUDA_TRY(launch_count_nonfinite_f64(v, FN, nbad, s));
    SE2_CUDA_TRY(launch_count_nonfinite_f64(w, FN, nbad, s));
    int h = 0;
    SE2_CUDA_TRY(cudaMemcpyAsync(&h, nbad, sizeof(int), cudaMemcpyDeviceToHost, s));
    SE2_CUDA_TRY(cudaStreamSynchronize(s));
    if (h != 0) {
        set_error("non-finite values produced by the iteration (" + std::to_string(h) + " entries)");
        return SE2_ENONFINITE;
    }
    return SE2_OK;
}

}  // extern "C"
