// K2: SE(2) group convolution, linear domain, fp32 FFMA.
//
//   y[b, to, y, x] = sum_{ti in band(to)} sum_{|dy|,|dx| <= R} W[to, ti, dy, dx] * v[b, ti, y-dy, x-dx]
//
// an implicit GEMM with M = (y, x), N = theta_o, K = (theta_i, dy, dx), restricted to the
// theta_i band where the fp32 table is nonzero (the taps outside the band are exactly 0 in fp32;
// inside the band every box tap is nonzero for the BASELINE configs, so no FFMA is wasted).
//
// One CTA = one output orientation theta_o x a tile of 32 rows (one per lane) x 16*WX columns
// (16 per thread, WX warps along x).  Per theta_i of the band the CTA stages, double-buffered with
// cp.async, the (32+2R) x (16 WX + 2R) input window (zero padded) and the S x S filter slice
// W[to][ti] (rows padded to a multiple of 4).  Per filter row dy each thread loads its input row
// segment (16 + 2R floats, LDS.128, conflict-free because pitch/4 is odd and lanes are rows) and
// issues 16 FFMA per tap against LDS.128 broadcasts of 4 filter taps: >= 95% of the issued
// instructions are FFMA.
#include "conv_common.cuh"

namespace se2 {

template <int R, int WX, bool TMA = false, int PP = 16>
struct LinCfg {
    static constexpr int S = 2 * R + 1;
    static constexpr int SP = (S + 3) / 4 * 4;  // filter row pitch (LDS.128 of 4 taps)
    static constexpr int P = PP;   // columns per thread
    static constexpr int NT = 32 * WX;
    static constexpr int TY = 32, TX = P * WX;
    // left halo of the staged window: R (cp.async path) or R rounded up to a multiple of 4 (TMA
    // boxes must start on a 16-byte boundary in x); smem column c <-> global column x0 - A + c
    static constexpr int A = TMA ? (R + 3) / 4 * 4 : R;
    static constexpr int WIN_H = TY + 2 * R;
    static constexpr int WIN_W = TX + R + A;
    static constexpr int RL = ((P + R + A) + 3) / 4 * 4;  // register row length (floats)
    static constexpr int NEED = ((WX - 1) * P + RL) > WIN_W ? ((WX - 1) * P + RL) : WIN_W;
    static constexpr int P0 = (NEED + 3) / 4 * 4;
    static constexpr int PITCH = ((P0 / 4) % 2 == 1) ? P0 : P0 + 4;  // pitch/4 odd -> no conflicts
    static constexpr int WIN = WIN_H * PITCH;
    static constexpr int FIL = S * SP;
    static constexpr size_t SMEM = (size_t)(2 * WIN + 2 * FIL) * sizeof(float) + 64;
    // TMA variant: window buffers padded to 128 B (TMA destination alignment) + 2 mbarriers
    static constexpr int WINA = (WIN * 4 + 127) / 128 * 32;
    static constexpr size_t SMEM_TMA = (size_t)(2 * WINA + 2 * FIL) * sizeof(float) + 64 + 128;
};

// W table layout used here: Wl[to][ti][S][SP] (dx padded with zeros to SP)
template <int R, int WX, bool TMA, int NBUF = 2, int PP = 16>
__global__ void __launch_bounds__(LinCfg<R, WX>::NT)
conv_linear_kernel(const float* __restrict__ in, const float* __restrict__ Wl, int nx, int ny, int nt,
                   int band, int tiles_x, int y_lo, int y_hi, Epilogue epi, const __grid_constant__ CUtensorMap tmap) {
    using C = LinCfg<R, WX, TMA, PP>;
    extern __shared__ __align__(128) float smem[];
    constexpr int WSTRIDE = TMA ? C::WINA : C::WIN;   // floats between the two window buffers
    float* sWin = smem;                     // [NBUF][WSTRIDE]
    float* sFil = smem + NBUF * WSTRIDE;    // [NBUF][FIL]
    float* sRed = sFil + NBUF * C::FIL;     // reduction scratch (16 floats)
    uint64_t* sBar = reinterpret_cast<uint64_t*>(sRed + 16);   // 2 mbarriers (TMA variant)

    const int tile = blockIdx.x;
    const int to = blockIdx.y;
    const int b = blockIdx.z;
    const int x0 = (tile % tiles_x) * C::TX;
    const int y0 = y_lo + (tile / tiles_x) * C::TY;   // output window [y_lo, y_hi) (slab kernels)
    const int64_t N = (int64_t)nx * ny * nt;
    const float* vin = in + (int64_t)b * N;
    const int lane = threadIdx.x & 31;
    const int wx = threadIdx.x >> 5;

    // theta_i range: [to - band, to + band] (mod nt), or all of them
    int nti = 1 + 2 * band;
    int ti0 = to - band;
    if (nti >= nt) { nti = nt; ti0 = 0; }

    // address of the __grid_constant__ tensor map taken here (param space); a lambda capture of the
    // parameter itself would copy it to local memory, which TMA cannot read
    const CUtensorMap* tmp = &tmap;
    if (TMA) {
        if (threadIdx.x == 0) {
            mbar_init(&sBar[0], 1);
            mbar_init(&sBar[1], 1);
            mbar_fence_init();
        }
        __syncthreads();
    } else {
        // zero the pitch padding columns once (never used in arithmetic; keeps initcheck clean)
        for (int i = threadIdx.x; i < 2 * C::WIN_H; i += C::NT) {
            float* row = sWin + (i / C::WIN_H) * WSTRIDE + (i % C::WIN_H) * C::PITCH;
            for (int c = C::WIN_W; c < C::PITCH; ++c) row[c] = 0.f;
        }
    }

    // stage the window of input orientation ti (with its halo; zeros outside the grid) and the filter
    // slice W[to][ti].  TMA variant: one thread issues a 3-D tensor copy of the PITCH x WIN_H box at
    // (x0 - R, y0 - R, b*nt + ti) (out-of-bounds -> zero fill) plus a 1-D bulk copy of the filter.
    auto stage = [&](int it, int buf) {
        int ti = ti0 + it;
        ti = ((ti % nt) + nt) % nt;
        const float* fsrc = Wl + ((int64_t)to * nt + ti) * C::FIL;
        float* dw = sWin + buf * WSTRIDE;
        float* df = sFil + buf * C::FIL;
        if (TMA) {
            if (threadIdx.x == 0) {
                fence_proxy_async();
                mbar_expect_tx(&sBar[buf], (uint32_t)((C::WIN_H * C::PITCH + C::FIL) * sizeof(float)));
                tma_load_3d(dw, tmp, &sBar[buf], x0 - C::A, y0 - R, b * nt + ti);
                bulk_load(df, fsrc, (uint32_t)(C::FIL * sizeof(float)), &sBar[buf]);
            }
        } else {
            const float* src = vin + (int64_t)ti * nx * ny;
            for (int i = threadIdx.x; i < C::WIN_H * C::WIN_W; i += C::NT) {
                int r = i / C::WIN_W, c = i - r * C::WIN_W;
                int gy = y0 - R + r, gx = x0 - C::A + c;
                bool ok = (gy >= 0) && (gy < ny) && (gx >= 0) && (gx < nx);
                cp_async4(dw + r * C::PITCH + c, ok ? (src + (int64_t)gy * nx + gx) : vin, ok);
            }
            for (int i = threadIdx.x; i < C::FIL / 4; i += C::NT) cp_async16(df + 4 * i, fsrc + 4 * i);
            cp_async_commit();
        }
    };

    float acc[C::P];
#pragma unroll
    for (int p = 0; p < C::P; ++p) acc[p] = 0.f;

    stage(0, 0);
    for (int it = 0; it < nti; ++it) {
        const int buf = (NBUF == 2) ? (it & 1) : 0;
        if (NBUF == 2) {
            if (it + 1 < nti) stage(it + 1, buf ^ 1);
        } else if (it > 0) {
            stage(it, 0);   // single buffer: the previous channel's readers finished at the barrier below
        }
        if (TMA) {
            mbar_wait(&sBar[buf], (uint32_t)(NBUF == 2 ? ((it >> 1) & 1) : (it & 1)));
        } else {
            if (it + 1 < nti) cp_async_wait<1>();
            else cp_async_wait<0>();
            __syncthreads();
        }
        const float* win = sWin + buf * WSTRIDE + wx * C::P;
        const float* fil = sFil + buf * C::FIL;
#pragma unroll 1
        for (int dy = 0; dy < C::S; ++dy) {
            const float4* rowp = reinterpret_cast<const float4*>(win + (lane - dy + 2 * R) * C::PITCH);
            float r[C::RL];
#pragma unroll
            for (int j = 0; j < C::RL / 4; ++j) {
                float4 t = rowp[j];
                r[4 * j + 0] = t.x; r[4 * j + 1] = t.y; r[4 * j + 2] = t.z; r[4 * j + 3] = t.w;
            }
            const float4* frow = reinterpret_cast<const float4*>(fil + dy * C::SP);
#pragma unroll
            for (int d4 = 0; d4 < C::SP / 4; ++d4) {
                const float4 w4 = frow[d4];
                const float wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int dx = 4 * d4 + e;
                    if (dx < C::S) {
#pragma unroll
                        for (int p = 0; p < C::P; ++p) acc[p] = fmaf(wv[e], r[p - dx + R + C::A], acc[p]);
                    }
                }
            }
        }
        __syncthreads();
    }

    // fused epilogue
    float err = 0.f;
    const int gy = y0 + lane;
    if (gy < y_hi) {
#pragma unroll
        for (int p = 0; p < C::P; ++p) {
            const int gx = x0 + wx * C::P + p;
            if (gx < nx) {
                int64_t idx = (int64_t)b * N + ((int64_t)to * ny + gy) * nx + gx;
                err += apply_epilogue<false>(epi, idx, gx, gy, acc[p]);
            }
        }
    }
    if (epi.err_partial != nullptr) {
        float t = block_sum<C::NT>(err, sRed);
        if (threadIdx.x == 0)
            epi.err_partial[(int64_t)b * (gridDim.x * gridDim.y) + blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

// warps along x per CTA (tile = 32 x 16*WX): 2 -> 32x32 tiles, ~42 KB smem at R = 15
constexpr int kLinWX = 2;

template <int R>
static cudaError_t launch_lin_r(const se2_kernel_s* k, const float* in, int batch, const Epilogue& epi,
                                cudaStream_t s, int* bpf) {
    using C = LinCfg<R, kLinWX, false>;
    using CT = LinCfg<R, kLinWX, true>;
    int tiles_x = (k->nx + C::TX - 1) / C::TX;
    int tiles_y = (k->wrows() + C::TY - 1) / C::TY;
    dim3 grid(tiles_x * tiles_y, k->nt, batch);
    const int ylo = k->wlo(), yhi = k->whi();
    if (bpf) *bpf = (int)(grid.x * grid.y);
    CUtensorMap tmap;
    const bool tma = make_field_tmap(&tmap, in, k->nx, k->ny, k->nt * batch, CT::PITCH, CT::WIN_H);
    cudaError_t e;
    // buffers per CTA and CTAs per SM (via smem padding).  Tuned on B200 at c4 (profiles/r01_*):
    // a single TMA buffer (20.8 KB -> 10 CTAs / 20 warps per SM; the other CTAs hide each CTA's load
    // bubble) beats double buffering at 5 CTAs / SM: 1.448 vs 1.553 ms; 32 columns per thread (one
    // warp per CTA) measured 1.516 ms.  Env overrides for experiments.
    static const int nbuf = getenv("SE2_LIN_NBUF") ? atoi(getenv("SE2_LIN_NBUF")) : 1;
    static const int occ = getenv("SE2_LIN_OCC") ? atoi(getenv("SE2_LIN_OCC")) : 0;
    if (tma && nbuf == 1) {
        size_t smem = (size_t)(CT::WINA + CT::FIL) * sizeof(float) + 64 + 128;
        if (occ > 0) {
            size_t want = (size_t)(227 * 1024) / occ - 1024;
            if (want > smem) smem = want;
        }
        e = cudaFuncSetAttribute(conv_linear_kernel<R, kLinWX, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        if (e != cudaSuccess) return e;
        conv_linear_kernel<R, kLinWX, true, 1><<<grid, CT::NT, smem, s>>>(in, epi.table ? epi.table : k->Wl, k->nx,
                                                                         k->ny, k->nt, k->band, tiles_x, ylo, yhi, epi, tmap);
    } else if (tma) {
        size_t smem = CT::SMEM_TMA;
        if (occ > 0) {
            size_t want = (size_t)(227 * 1024) / occ - 1024;
            if (want > smem) smem = want;
        }
        e = cudaFuncSetAttribute(conv_linear_kernel<R, kLinWX, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        if (e != cudaSuccess) return e;
        conv_linear_kernel<R, kLinWX, true><<<grid, CT::NT, smem, s>>>(in, epi.table ? epi.table : k->Wl, k->nx, k->ny, k->nt, k->band,
                                                                            tiles_x, ylo, yhi, epi, tmap);
    } else {
        e = cudaFuncSetAttribute(conv_linear_kernel<R, kLinWX, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)C::SMEM);
        if (e != cudaSuccess) return e;
        conv_linear_kernel<R, kLinWX, false><<<grid, C::NT, C::SMEM, s>>>(in, epi.table ? epi.table : k->Wl, k->nx, k->ny, k->nt, k->band,
                                                                         tiles_x, ylo, yhi, epi, tmap);
    }
    count_launch();
    return cudaGetLastError();
}

int conv_blocks_per_field_linear(const se2_kernel_s* k) {
    using C = LinCfg<1, kLinWX, false>;   // all radii and variants share the tile geometry
    int tiles_x = (k->nx + C::TX - 1) / C::TX;
    int tiles_y = (k->wrows() + C::TY - 1) / C::TY;
    return tiles_x * tiles_y * k->nt;
}

cudaError_t launch_conv_linear(const se2_kernel_s* k, const float* in, int batch, const Epilogue& epi,
                               cudaStream_t s, int* bpf) {
    switch (k->R) {
#define SE2_CASE(r) \
    case r: return launch_lin_r<r>(k, in, batch, epi, s, bpf);
        SE2_CASE(0) SE2_CASE(1) SE2_CASE(2) SE2_CASE(3) SE2_CASE(4) SE2_CASE(5) SE2_CASE(6) SE2_CASE(7)
        SE2_CASE(8) SE2_CASE(9) SE2_CASE(10) SE2_CASE(11) SE2_CASE(12) SE2_CASE(13) SE2_CASE(14) SE2_CASE(15)
#undef SE2_CASE
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace se2
