// K3: SE(2) group convolution in the log domain -- theta-factored, shifted FFMA log-sum-exp with an
// exact per-tap fallback and exact-bound channel pruning (reading R7).
//
//   ly[to, x] = log sum_ti sum_d exp( Lth(to,ti) + Ls(to,ti,d) + lv[ti, x - d] )
//
// Per CTA (a 32 x 16 spatial tile T, an output-orientation quad, one field) and per input
// orientation ti, with mu = min_T lv[ti] and M = max over the window (T + halo) of lv[ti]:
//   * prune  if  M + Lth + log sum_d e^{Ls}  <  LB - 30  for every to of the quad, where
//            LB(to) = max_j (Lth(to,j) + mu_j) <= ly(to, x) for all x in T (centre taps);
//            the skipped mass is < e^{-30} of the output per channel;
//   * FFMA   if  M - mu <= 100: stage v~ = exp(lv - m), m = mu + 62, and accumulate
//            S = sum_d exp(Ls + 40) v~ with fp32 FFMA; every term within e^{-25} of the channel's
//            largest term is a normal fp32 product and the sum cannot overflow (derivation in
//            DESIGN.md), then fold log S + m - 40 + Lth into the output's running (max, sum);
//   * exact  otherwise: the two-pass per-tap log-sum-exp of K4 for this channel.
// Cost of the FFMA path per tap = 1 FFMA (vs 1 MUFU.EX2 + 5 FP32 ops for the exact one).
#include "conv_common.cuh"

namespace se2 {

template <int R>
struct LseFCfg {
    static constexpr int S = 2 * R + 1;
    static constexpr int P = 4;
    static constexpr int WX = 4;
    static constexpr int NT = 32 * WX;
    static constexpr int TY = 32, TX = P * WX;   // 32 x 16 tile (>= R in both directions)
    static constexpr int WIN_H = TY + 2 * R;
    static constexpr int WIN_W = TX + 2 * R;
    static constexpr int RL = ((P + 2 * R) + 3) / 4 * 4;
    static constexpr int NEED = ((WX - 1) * P + RL) > WIN_W ? ((WX - 1) * P + RL) : WIN_W;
    static constexpr int P0 = (NEED + 3) / 4 * 4;
    static constexpr int PITCH = ((P0 / 4) % 2 == 1) ? P0 : P0 + 4;
    static constexpr int WIN = WIN_H * PITCH;
    static constexpr int FIL = S * S * 4;
    static constexpr int MAXNT = 256;
    static constexpr size_t SMEM = (size_t)(2 * WIN + 2 * FIL) * sizeof(float) + 64;
};
constexpr int kLseTileY = 32, kLseTileX = 16;

// per (field, theta, tile) min and max of lv over the 32 x 16 tile
__global__ void lse_stats_kernel(const float* __restrict__ in, int nx, int ny, int nt, int tiles_x, int tiles_y,
                                 float* __restrict__ tmin, float* __restrict__ tmax) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int ntile = tiles_x * tiles_y;
    const int64_t total = (int64_t)gridDim.y * nt * ntile;   // gridDim.y = batch
    const int b = blockIdx.y;
    if (warp >= nt * ntile) return;
    const int th = warp / ntile, t = warp % ntile;
    const int x0 = (t % tiles_x) * kLseTileX, y0 = (t / tiles_x) * kLseTileY;
    const float* src = in + ((int64_t)b * nt + th) * nx * ny;
    float mn = INFINITY, mx = -INFINITY;
    for (int i = lane; i < kLseTileY * kLseTileX; i += 32) {
        int y = y0 + i / kLseTileX, x = x0 + i % kLseTileX;
        if (y < ny && x < nx) {
            float v = src[(int64_t)y * nx + x];
            mn = fminf(mn, v);
            mx = fmaxf(mx, v);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) {
        int64_t o = ((int64_t)b * nt + th) * ntile + t;
        tmin[o] = mn;
        tmax[o] = mx;
    }
    (void)total;
}

template <int R>
__global__ void __launch_bounds__(LseFCfg<R>::NT)
conv_lse_fast_kernel(const float* __restrict__ in, const float* __restrict__ Eq, const float* __restrict__ Lq,
                     const float* __restrict__ Lth, const float* __restrict__ LseS,
                     const float* __restrict__ tmin, const float* __restrict__ tmax, int nx, int ny, int nt,
                     int tiles_x, int tiles_y, int force_exact, Epilogue epi, int* __restrict__ counters) {
    using C = LseFCfg<R>;
    extern __shared__ __align__(16) float smem[];
    float* sWin = smem;
    float* sFil = smem + 2 * C::WIN;
    float* sRed = sFil + 2 * C::FIL;
    __shared__ float sMu[C::MAXNT], sM[C::MAXNT], sCoef[C::MAXNT][4], sLB[4];
    __shared__ int sList[C::MAXNT];
    __shared__ int sNAct, sNFast;
    __shared__ float sRef;

    const int tile = blockIdx.x;
    const int qd = blockIdx.y;
    const int b = blockIdx.z;
    const int ntile = tiles_x * tiles_y;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int x0 = tx * C::TX, y0 = ty * C::TY;
    const int64_t N = (int64_t)nx * ny * nt;
    const float* vin = in + (int64_t)b * N;
    const int lane = threadIdx.x & 31;
    const int wx = threadIdx.x >> 5;
    const float NEG_INF = -INFINITY;
    const float LOW = -1e30f;   // "no term yet" sentinel of the running maxima (finite: no inf - inf)

    // ---- per-channel bounds --------------------------------------------------------------------
    for (int i = threadIdx.x; i < nt; i += C::NT) {
        const int64_t base = ((int64_t)b * nt + i) * ntile;
        sMu[i] = tmin[base + tile];
        float M = NEG_INF;
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                int yy = ty + dy, xx = tx + dx;
                if (yy >= 0 && yy < tiles_y && xx >= 0 && xx < tiles_x) M = fmaxf(M, tmax[base + yy * tiles_x + xx]);
            }
        sM[i] = M;
    }
    __syncthreads();
    if (wx < 4) {   // warp q: lower bound LB(to_q) = max_j (Lth(to_q, j) + mu_j)
        const int to = 4 * qd + wx;
        float lb = NEG_INF;
        if (to < nt)
            for (int j = lane; j < nt; j += 32) lb = fmaxf(lb, Lth[to * nt + j] + sMu[j]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lb = fmaxf(lb, __shfl_xor_sync(0xffffffffu, lb, o));
        if (lane == 0) sLB[wx] = lb;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float ref = NEG_INF;
        for (int q = 0; q < 4; ++q)
            if (4 * qd + q < nt) ref = fmaxf(ref, sLB[q]);
        if (ref == NEG_INF) {   // every channel has -inf somewhere in the tile: use an upper bound
            for (int j = 0; j < nt; ++j) ref = fmaxf(ref, sM[j] + Lth[(4 * qd) * nt + j]);
        }
        sRef = (ref == NEG_INF || ref != ref) ? 0.f : ref;
    }
    __syncthreads();
    const float ref = sRef;
    // status per channel: 0 skip, 1 FFMA path, 2 exact path; coefficient of the FFMA path
    for (int i = threadIdx.x; i < nt; i += C::NT) {
        const float M = sM[i], mu = sMu[i];
        int st = 0;
        if (M != NEG_INF) {
            bool active = false;
            for (int q = 0; q < 4; ++q) {
                const int to = 4 * qd + q;
                if (to >= nt) continue;
                const float ub = M + Lth[to * nt + i] + LseS[to * nt + i];
                if (!(ub < sLB[q] - kPruneGap)) active = true;
            }
            if (active) st = (!force_exact && mu != NEG_INF && (M - mu) <= kFastRange) ? 1 : 2;
        }
        sList[i] = st;
        if (st == 1)
            for (int q = 0; q < 4; ++q) {
                const int to = 4 * qd + q;
                const float lt = (to < nt) ? Lth[to * nt + i] : 0.f;
                // (m - kEsShift + Lth - ref) log2(e), m = mu + kShiftAbove; (mu - ref) first: both large
                sCoef[i][q] = (((mu - ref) + (kShiftAbove - kEsShift)) + lt) * kLog2e;
            }
    }
    __syncthreads();
    if (threadIdx.x == 0) {   // compact the active list: entry = channel | (path << 16)
        int n = 0, nf = 0;
        for (int i = 0; i < nt; ++i) {
            int st = sList[i];
            if (st) {
                sList[n++] = i | (st << 16);
                nf += (st == 1);
            }
        }
        sNAct = n;
        sNFast = nf;
    }
    __syncthreads();
    const int nact = sNAct;
    if (counters != nullptr && threadIdx.x == 0) {
        atomicAdd(&counters[0], nact);
        atomicAdd(&counters[1], sNFast);
        atomicAdd(&counters[2], nt);
    }

    for (int i = threadIdx.x; i < 2 * C::WIN_H; i += C::NT) {
        float* row = sWin + (i / C::WIN_H) * C::WIN + (i % C::WIN_H) * C::PITCH;
        for (int c = C::WIN_W; c < C::PITCH; ++c) row[c] = 0.f;
    }

    auto stage = [&](int a, int buf) {
        const int ent = sList[a];
        const int ti = ent & 0xffff, path = ent >> 16;
        const float* src = vin + (int64_t)ti * nx * ny;
        float* dw = sWin + buf * C::WIN;
        for (int i = threadIdx.x; i < C::WIN_H * C::WIN_W; i += C::NT) {
            int r = i / C::WIN_W, c = i - r * C::WIN_W;
            int gy = y0 - R + r, gx = x0 - R + c;
            bool ok = (gy >= 0) && (gy < ny) && (gx >= 0) && (gx < nx);
            if (ok)
                cp_async4(dw + r * C::PITCH + c, src + (int64_t)gy * nx + gx, true);
            else
                dw[r * C::PITCH + c] = NEG_INF;
        }
        const float* fsrc = (path == 1 ? Eq : Lq) + ((int64_t)qd * nt + ti) * C::FIL;
        float* df = sFil + buf * C::FIL;
        for (int i = threadIdx.x; i < C::FIL / 4; i += C::NT) cp_async16(df + 4 * i, fsrc + 4 * i);
        cp_async_commit();
    };

    float Macc[4][C::P], Sacc[4][C::P];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int p = 0; p < C::P; ++p) { Macc[q][p] = LOW; Sacc[q][p] = 0.f; }

    if (nact > 0) stage(0, 0);
    for (int a = 0; a < nact; ++a) {
        const int buf = a & 1;
        const int ent = sList[a];
        const int ti = ent & 0xffff, path = ent >> 16;
        if (a + 1 < nact) {
            stage(a + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        // transform the elements this thread staged (own cp.async copies are complete)
        {
            float* dw = sWin + buf * C::WIN;
            const float shift = (path == 1) ? (sMu[ti] + kShiftAbove) : ref;
            for (int i = threadIdx.x; i < C::WIN_H * C::WIN_W; i += C::NT) {
                int r = i / C::WIN_W, c = i - r * C::WIN_W;
                float v = dw[r * C::PITCH + c];
                float u = (v - shift) * kLog2e;
                dw[r * C::PITCH + c] = (path == 1) ? ex2_approx(u) : u;
            }
        }
        __syncthreads();
        const float* win = sWin + buf * C::WIN + wx * C::P;
        const float4* fil = reinterpret_cast<const float4*>(sFil + buf * C::FIL);
        float acc[4][C::P];
        if (path == 1) {
            // ---------------- FFMA path: S = sum_d exp(Ls + 40) * exp(lv - m)
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int p = 0; p < C::P; ++p) acc[q][p] = 0.f;
#pragma unroll 1
            for (int dy = 0; dy < C::S; ++dy) {
                const float4* rowp = reinterpret_cast<const float4*>(win + (lane - dy + 2 * R) * C::PITCH);
                float r[C::RL];
#pragma unroll
                for (int j = 0; j < C::RL / 4; ++j) {
                    float4 t = rowp[j];
                    r[4 * j + 0] = t.x; r[4 * j + 1] = t.y; r[4 * j + 2] = t.z; r[4 * j + 3] = t.w;
                }
                const float4* frow = fil + dy * C::S;
#pragma unroll
                for (int dx = 0; dx < C::S; ++dx) {
                    const float4 w = frow[dx];
#pragma unroll
                    for (int p = 0; p < C::P; ++p) {
                        const float xv = r[p - dx + 2 * R];
                        acc[0][p] = fmaf(w.x, xv, acc[0][p]);
                        acc[1][p] = fmaf(w.y, xv, acc[1][p]);
                        acc[2][p] = fmaf(w.z, xv, acc[2][p]);
                        acc[3][p] = fmaf(w.w, xv, acc[3][p]);
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float cf = sCoef[ti][q];
#pragma unroll
                for (int p = 0; p < C::P; ++p) {
                    const float t = lg2_approx(acc[q][p]) + cf;     // lg2(0) = -inf: no contribution
                    const float mx = fmaxf(Macc[q][p], t);
                    Sacc[q][p] = Sacc[q][p] * ex2_approx(Macc[q][p] - mx) + ex2_approx(t - mx);
                    Macc[q][p] = mx;
                }
            }
        } else {
            // ---------------- exact path: two passes over the taps of this channel
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int p = 0; p < C::P; ++p) acc[q][p] = Macc[q][p];
#pragma unroll 1
            for (int dy = 0; dy < C::S; ++dy) {
                const float4* rowp = reinterpret_cast<const float4*>(win + (lane - dy + 2 * R) * C::PITCH);
                float r[C::RL];
#pragma unroll
                for (int j = 0; j < C::RL / 4; ++j) {
                    float4 t = rowp[j];
                    r[4 * j + 0] = t.x; r[4 * j + 1] = t.y; r[4 * j + 2] = t.z; r[4 * j + 3] = t.w;
                }
                const float4* frow = fil + dy * C::S;
#pragma unroll
                for (int dx = 0; dx < C::S; ++dx) {
                    const float4 w = frow[dx];
#pragma unroll
                    for (int p = 0; p < C::P; ++p) {
                        const float xv = r[p - dx + 2 * R];
                        acc[0][p] = fmaxf(acc[0][p], xv + w.x);
                        acc[1][p] = fmaxf(acc[1][p], xv + w.y);
                        acc[2][p] = fmaxf(acc[2][p], xv + w.z);
                        acc[3][p] = fmaxf(acc[3][p], xv + w.w);
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int p = 0; p < C::P; ++p) {
                    const float mn = acc[q][p];      // >= Macc (LOW sentinel when nothing finite yet)
                    Sacc[q][p] *= ex2_approx(Macc[q][p] - mn);
                    Macc[q][p] = mn;
                }
#pragma unroll 1
            for (int dy = 0; dy < C::S; ++dy) {
                const float4* rowp = reinterpret_cast<const float4*>(win + (lane - dy + 2 * R) * C::PITCH);
                float r[C::RL];
#pragma unroll
                for (int j = 0; j < C::RL / 4; ++j) {
                    float4 t = rowp[j];
                    r[4 * j + 0] = t.x; r[4 * j + 1] = t.y; r[4 * j + 2] = t.z; r[4 * j + 3] = t.w;
                }
                const float4* frow = fil + dy * C::S;
#pragma unroll
                for (int dx = 0; dx < C::S; ++dx) {
                    const float4 w = frow[dx];
#pragma unroll
                    for (int p = 0; p < C::P; ++p) {
                        const float xv = r[p - dx + 2 * R];
                        Sacc[0][p] += ex2_approx((xv + w.x) - Macc[0][p]);
                        Sacc[1][p] += ex2_approx((xv + w.y) - Macc[1][p]);
                        Sacc[2][p] += ex2_approx((xv + w.z) - Macc[2][p]);
                        Sacc[3][p] += ex2_approx((xv + w.w) - Macc[3][p]);
                    }
                }
            }
        }
        __syncthreads();
    }

    float err = 0.f;
    const int gy = y0 + lane;
    if (gy < ny) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int to = 4 * qd + q;
            if (to >= nt) continue;
#pragma unroll
            for (int p = 0; p < C::P; ++p) {
                const int gx = x0 + wx * C::P + p;
                if (gx < nx) {
                    float ly = (Macc[q][p] <= LOW || !(Sacc[q][p] > 0.f))
                                   ? NEG_INF
                                   : ref + (Macc[q][p] + log2f(Sacc[q][p])) * kLn2;
                    int64_t idx = (int64_t)b * N + ((int64_t)to * ny + gy) * nx + gx;
                    err += apply_epilogue<true>(epi, idx, gx, gy, ly);
                }
            }
        }
    }
    if (epi.err_partial != nullptr) {
        float t = block_sum<C::NT>(err, sRed);
        if (threadIdx.x == 0)
            epi.err_partial[(int64_t)b * (gridDim.x * gridDim.y) + blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

template <int R>
static cudaError_t launch_lsef_r(const se2_kernel_s* k, const float* in, int batch, const Epilogue& epi,
                                 cudaStream_t s, int* bpf, float* tmin, float* tmax, int force_exact,
                                 int* counters) {
    using C = LseFCfg<R>;
    const int tiles_x = (k->nx + C::TX - 1) / C::TX;
    const int tiles_y = (k->ny + C::TY - 1) / C::TY;
    const int ntile = tiles_x * tiles_y;
    {
        const int warps = k->nt * ntile;
        dim3 g((warps * 32 + 255) / 256, batch);
        lse_stats_kernel<<<g, 256, 0, s>>>(in, k->nx, k->ny, k->nt, tiles_x, tiles_y, tmin, tmax);
        count_launch();
    }
    cudaError_t e = cudaFuncSetAttribute(conv_lse_fast_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::SMEM);
    if (e != cudaSuccess) return e;
    dim3 grid(ntile, (k->nt + 3) / 4, batch);
    if (bpf) *bpf = (int)(grid.x * grid.y);
    conv_lse_fast_kernel<R><<<grid, C::NT, C::SMEM, s>>>(in, k->Eq, k->Lq, k->Lth, k->LseS, tmin, tmax, k->nx,
                                                          k->ny, k->nt, tiles_x, tiles_y, force_exact, epi,
                                                          counters);
    count_launch();
    return cudaGetLastError();
}

size_t lse_fast_stats_floats(const se2_kernel_s* k, int batch) {
    const int tiles_x = (k->nx + kLseTileX - 1) / kLseTileX;
    const int tiles_y = (k->ny + kLseTileY - 1) / kLseTileY;
    return (size_t)batch * k->nt * tiles_x * tiles_y;
}

int conv_blocks_per_field_lse_fast(const se2_kernel_s* k) {
    const int tiles_x = (k->nx + kLseTileX - 1) / kLseTileX;
    const int tiles_y = (k->ny + kLseTileY - 1) / kLseTileY;
    return tiles_x * tiles_y * ((k->nt + 3) / 4);
}

cudaError_t launch_conv_lse_fast(const se2_kernel_s* k, const float* in, int batch, const Epilogue& epi,
                                 cudaStream_t s, int* bpf, float* tmin, float* tmax, int force_exact,
                                 int* counters) {
    if (k->nt > LseFCfg<1>::MAXNT) return cudaErrorInvalidValue;
    switch (k->R) {
#define SE2_CASE(r) \
    case r: return launch_lsef_r<r>(k, in, batch, epi, s, bpf, tmin, tmax, force_exact, counters);
        SE2_CASE(0) SE2_CASE(1) SE2_CASE(2) SE2_CASE(3) SE2_CASE(4) SE2_CASE(5) SE2_CASE(6) SE2_CASE(7)
        SE2_CASE(8) SE2_CASE(9) SE2_CASE(10) SE2_CASE(11) SE2_CASE(12) SE2_CASE(13) SE2_CASE(14) SE2_CASE(15)
#undef SE2_CASE
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace se2
