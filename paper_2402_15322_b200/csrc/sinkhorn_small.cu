// K9: the whole log-domain Sinkhorn loop of a small grid in ONE launch (P:557-560 with the
// log form of reading R7):
//     alpha = log mu - LSEconv(beta),   beta = log nu - LSEconv(alpha),   beta^(0) = 0 (b^(0) = 1)
// for l = 1..iters, plus the fused marginal-error trace e_l = sum |exp(alpha + LSEconv(beta)) - mu|
// (reading R10; the a-update of iteration l+1 computes e_l, an extra error-only pass the last one).
//
// One thread-block cluster of C CTAs (16 when the device allows non-portable clusters, else 8).
// Every CTA keeps BOTH potentials of the whole grid in shared memory (log2 units, planes padded with
// an R-wide -inf border) and owns N/C outputs; each output's log-sum-exp over all (theta_i, dy, dx)
// taps is exact (every tap, online max per tap row, K4 arithmetic) split over `split` lanes by theta_i.  A CTA publishes its new outputs to
// every CTA of the cluster with distributed-shared-memory stores (mapa + st.shared::cluster); one
// cluster barrier (release/acquire) per half-iteration orders the exchange: a half-iteration reads one
// potential and writes the other, and the barrier before it guarantees that no CTA still reads the
// buffer being written.  No HBM traffic inside the loop except the per-iteration error partials.
#include <stdlib.h>

#include "conv_common.cuh"

namespace se2 {

constexpr int kK9Threads = 512;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

struct K9Args {
    const float* mu;
    const float* nu;
    float* a;             // alpha out (natural log)
    float* b;             // beta in (warm start) / out
    const float* Lq;      // [nt/4][nt][S][S][4] L log2(e)
    float* err_partial;   // [iters][C] (trace) or null
    double* trace;        // [iters] or null
    int nx, ny, nt, iters, warm, C, split, per_cta, batch;
};

// exact log-sum-exp (log2 units) of one output over this lane's theta_i subset, combined over the
// `split` lanes of its group.  One pass, online per tap row: the row's terms are formed in registers,
// the running maximum is raised to the row maximum (rescaling the sum once per row), then the row's
// 2^(t - max) are added.  The fields are stored with an R-wide -inf border (zero padding of the
// linear kernel), so the taps need no bounds checks.
template <int R>
__device__ __forceinline__ float k9_lse2(const float* __restrict__ f, const float* __restrict__ tab, int pw, int pp,
                                         int ny, int nt, int x, int y, int part, int split) {
    constexpr int S = 2 * R + 1;
    const int dylo = max(-R, y - (ny - 1)), dyhi = min(R, y);
    float m = -INFINITY, s = 0.f, s2 = 0.f;   // two partial sums: shorter dependency chains
    for (int ti = part; ti < nt; ti += split) {
        const float* fp = f + ti * pp + x + R;          // padded column of x
        const float* tp = tab + ti * S * S + R;
        for (int dy = dylo; dy <= dyhi; ++dy) {
            const float* frow = fp + (y - dy + R) * pw;
            const float* trow = tp + (dy + R) * S;
            float t[S];
#pragma unroll
            for (int dx = -R; dx <= R; ++dx) t[dx + R] = trow[dx] + frow[-dx];
            float rm0 = t[0], rm1 = (S > 1) ? t[1] : -INFINITY;
#pragma unroll
            for (int j = 2; j < S; j += 2) {
                rm0 = fmaxf(rm0, t[j]);
                if (j + 1 < S) rm1 = fmaxf(rm1, t[j + 1]);
            }
            const float rm = fmaxf(rm0, rm1);
            if (rm > m) {
                const float sc = ex2_approx(m - rm);
                s *= sc;
                s2 *= sc;
                m = rm;
            }
            if (m != -INFINITY) {
#pragma unroll
                for (int j = 0; j < S; j += 2) {
                    s += ex2_approx(t[j] - m);
                    if (j + 1 < S) s2 += ex2_approx(t[j + 1] - m);
                }
            }
        }
    }
    s += s2;
    float mg = m;
    for (int o = 1; o < split; o <<= 1) mg = fmaxf(mg, __shfl_xor_sync(0xffffffffu, mg, o));
    const bool none = (mg == -INFINITY);   // uniform over the group; every lane still reaches the shuffles
    s = (m == -INFINITY) ? 0.f : s * ex2_approx(m - mg);
    for (int o = 1; o < split; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return none ? -INFINITY : mg + lg2_norm(s);
}

template <int R>
__global__ void __launch_bounds__(kK9Threads) sinkhorn_small_kernel(K9Args p) {
    constexpr int S = 2 * R + 1;
    extern __shared__ __align__(16) float smem[];
    const int N = p.nx * p.ny * p.nt;
    // one cluster per problem of the batch (clusters are consecutive C-block groups along x)
    const int prob = blockIdx.x / p.C;
    p.mu += (int64_t)prob * N;
    p.nu += (int64_t)prob * N;
    p.a += (int64_t)prob * N;
    p.b += (int64_t)prob * N;
    const int plane = p.nx * p.ny;
    const int pw = p.nx + 2 * R, pp = pw * (p.ny + 2 * R);   // padded plane (-inf border)
    const int NP = pp * p.nt;
    const int rank = (int)cluster_rank();
    const int o0 = rank * p.per_cta;
    const int to_lo = o0 / plane, to_hi = (o0 + p.per_cta - 1) / plane;
    const int nto = to_hi - to_lo + 1;
    float* fA = smem;                       // alpha * log2(e), whole grid, padded planes
    float* fB = fA + NP;                    // beta  * log2(e), whole grid, padded planes
    float* tab = fB + NP;                   // [nto][nt][S][S] L log2(e) of this CTA's output orientations
    float* myA = tab + nto * p.nt * S * S;  // own outputs, natural log: alpha, beta, log mu, log nu
    float* myB = myA + p.per_cta;
    float* lmu = myB + p.per_cta;
    float* lnu = lmu + p.per_cta;
    __shared__ float red[kK9Threads / 32];

    // ---- setup: tables, initial beta (whole grid), targets of the own outputs
    for (int i = threadIdx.x; i < nto * p.nt * S * S; i += kK9Threads) {
        const int tl = i / (p.nt * S * S), rem = i - tl * (p.nt * S * S);
        const int to = to_lo + tl, ti = rem / (S * S), d = rem - ti * (S * S);
        tab[i] = p.Lq[((((int64_t)(to >> 2) * p.nt + ti) * S * S) + d) * 4 + (to & 3)];
    }
    for (int i = threadIdx.x; i < NP; i += kK9Threads) {
        const int ti = i / pp, r = i - ti * pp, yy = r / pw - R, xx = r - (r / pw) * pw - R;
        const bool in = yy >= 0 && yy < p.ny && xx >= 0 && xx < p.nx;
        fA[i] = in ? 0.f : -INFINITY;
        fB[i] = in ? (p.warm ? p.b[(ti * p.ny + yy) * p.nx + xx] * kLog2e : 0.f) : -INFINITY;
    }
    for (int i = threadIdx.x; i < p.per_cta; i += kK9Threads) {
        lmu[i] = logf(p.mu[o0 + i]);
        lnu[i] = logf(p.nu[o0 + i]);
        myA[i] = 0.f;
        myB[i] = p.warm ? p.b[o0 + i] : 0.f;
    }
    __syncthreads();

    const uint32_t baseA = (uint32_t)__cvta_generic_to_shared(fA);
    const uint32_t baseB = (uint32_t)__cvta_generic_to_shared(fB);
    const int groups = kK9Threads / p.split;
    const int grp = threadIdx.x / p.split, part = threadIdx.x - grp * p.split;
    const bool trace = p.err_partial != nullptr;

    // one half-iteration: conv of `src`, update of the own outputs of `dst` (natural copy `mine`),
    // publication to every CTA.  err_slot >= 0: also accumulate the marginal error of the alpha
    // update (uses the alpha before the update); write_dst false: error-only pass.
    auto half = [&](const float* src, uint32_t dst_base, float* mine, const float* tgt, int err_slot, bool write_dst) {
        float err = 0.f;
        for (int ob = 0; ob < p.per_cta; ob += groups) {   // same trip count for every lane (shuffles)
            const int ol = ob + grp;
            const bool act = ol < p.per_cta;
            const int o = o0 + (act ? ol : 0);
            const int to = o / plane, rem = o - to * plane, y = rem / p.nx, x = rem - y * p.nx;
            const float ly2 = k9_lse2<R>(src, tab + (to - to_lo) * p.nt * S * S, pw, pp, p.ny, p.nt, x, y, part, p.split);
            if (act && part == 0) {
                const float ly = ly2 * kLn2;
                if (err_slot >= 0) err += fabsf(expf(myA[ol] + ly) - p.mu[o]);
                if (write_dst) {
                    const float t = tgt[ol];
                    const float v = (t == -INFINITY) ? -INFINITY : t - ly;
                    mine[ol] = v;
                    const float v2 = v * kLog2e;
                    const uint32_t off = 4u * (uint32_t)(to * pp + (y + R) * pw + x + R);
                    for (int r = 0; r < p.C; ++r) st_cluster_f32(map_to_rank(dst_base + off, r), v2);
                }
            }
        }
        if (err_slot >= 0) {
            const float t = block_sum<kK9Threads>(err, red);
            if (threadIdx.x == 0) p.err_partial[((int64_t)err_slot * p.batch + prob) * p.C + rank] = t;
        }
        cluster_sync_all();
    };

    cluster_sync_all();   // every CTA's shared memory is live before remote stores
    for (int l = 0; l < p.iters; ++l) {
        half(fB, baseA, myA, lmu, (trace && l > 0) ? l - 1 : -1, true);    // alpha = log mu - LSE(beta)
        half(fA, baseB, myB, lnu, -1, true);                                // beta  = log nu - LSE(alpha)
    }
    if (trace && p.iters > 0) half(fB, baseA, myA, lmu, p.iters - 1, false);

    for (int i = threadIdx.x; i < p.per_cta; i += kK9Threads) {
        p.a[o0 + i] = myA[i];
        p.b[o0 + i] = myB[i];
    }
    if (trace && rank == 0) {
        __threadfence();
        for (int l = threadIdx.x; l < p.iters; l += kK9Threads) {
            double acc = 0.0;
            for (int r = 0; r < p.C; ++r) acc += (double)p.err_partial[((int64_t)l * p.batch + prob) * p.C + r];
            p.trace[(int64_t)l * p.batch + prob] = acc;
        }
    }
}

size_t k9_smem_bytes(const se2_kernel_s* k, int C) {
    const int64_t N = k->N();
    if (C <= 0 || N % C != 0) return (size_t)-1;
    const int per_cta = (int)(N / C);
    const int plane = k->nx * k->ny;
    const int nto = (per_cta + plane - 1) / plane + 1;
    const size_t NP = (size_t)(k->nx + 2 * k->R) * (k->ny + 2 * k->R) * k->nt;
    return sizeof(float) * (2 * NP + (size_t)nto * k->nt * k->S * k->S + 4 * (size_t)per_cta);
}

template <int R>
static cudaError_t launch_k9_r(const se2_kernel_s* k, const float* mu, const float* nu, float* a, float* b,
                               int batch, int iters, bool warm, float* err_partial, double* trace, int C,
                               cudaStream_t s) {
    const size_t smem = k9_smem_bytes(k, C);
    cudaError_t e = cudaFuncSetAttribute(sinkhorn_small_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (C > 8) {
        e = cudaFuncSetAttribute(sinkhorn_small_kernel<R>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    K9Args p;
    p.mu = mu; p.nu = nu; p.a = a; p.b = b; p.Lq = k->Lq;
    p.err_partial = err_partial; p.trace = trace;
    p.nx = k->nx; p.ny = k->ny; p.nt = k->nt; p.iters = iters; p.warm = warm ? 1 : 0; p.C = C; p.batch = batch;
    p.per_cta = (int)(k->N() / C);
    // lanes per output: enough to occupy the CTA, a power of two <= 8 that divides into a warp
    int split = 1;
    while (split * 2 <= 8 && split * 2 <= k->nt && p.per_cta * split * 2 <= kK9Threads) split *= 2;
    p.split = split;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C * batch, 1, 1);
    cfg.blockDim = dim3(kK9Threads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, sinkhorn_small_kernel<R>, p);
    count_launch();
    return e;
}

// cluster size for K9 on this kernel's grid, 0 if K9 does not apply (shared memory, divisibility)
int k9_cluster_size(const se2_kernel_s* k) {
    static int max_c = -1;
    if (max_c < 0) {
        max_c = 8;
        // non-portable 16-CTA clusters: probe once
        cudaFuncAttributes fa;
        if (cudaFuncGetAttributes(&fa, sinkhorn_small_kernel<3>) == cudaSuccess &&
            cudaFuncSetAttribute(sinkhorn_small_kernel<3>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess)
            max_c = 16;
        cudaGetLastError();
    }
    if (k->R > 15) return 0;
    // K9 evaluates every box tap exactly on <= 16 SMs: it beats the per-conv K3 path (pruning, FFMA
    // factoring, all SMs) only while the per-conv work is small.  Measured (tools/k9_vs_k3.py, 100
    // iterations): 0.8 M taps/conv 1.0 vs 3.0 ms, 1.8 M 2.6 vs 3.3 ms, 8.3 M 7.4 vs 3.5 ms.
    if ((double)k->N() * k->S * k->S * k->nt > 3.0e6) return 0;
    static const int cap = getenv("SE2_K9_CLUSTER") ? atoi(getenv("SE2_K9_CLUSTER")) : 16;   // tuning
    for (int C = max_c < cap ? max_c : cap; C >= 2; C /= 2) {
        if (k->N() % C != 0) continue;
        if (k9_smem_bytes(k, C) <= (size_t)200 * 1024) return C;
    }
    return 0;
}

cudaError_t launch_sinkhorn_small(const se2_kernel_s* k, const float* mu, const float* nu, float* a, float* b,
                                  int batch, int iters, bool warm, float* err_partial, double* trace, int C,
                                  cudaStream_t s) {
    switch (k->R) {
#define SE2_CASE(r) \
    case r: return launch_k9_r<r>(k, mu, nu, a, b, batch, iters, warm, err_partial, trace, C, s);
        SE2_CASE(0) SE2_CASE(1) SE2_CASE(2) SE2_CASE(3) SE2_CASE(4) SE2_CASE(5) SE2_CASE(6) SE2_CASE(7)
        SE2_CASE(8) SE2_CASE(9) SE2_CASE(10) SE2_CASE(11) SE2_CASE(12) SE2_CASE(13) SE2_CASE(14) SE2_CASE(15)
#undef SE2_CASE
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace se2
