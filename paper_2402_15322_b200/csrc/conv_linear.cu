// K2: SE(2) group convolution, linear domain, fp32 FFMA.
//
//   y[b, to, y, x] = sum_{ti in band(to)} sum_{|dy|,|dx| <= R} W[to, ti, dy, dx] * v[b, ti, y-dy, x-dx]
//
// an implicit GEMM with M = (y, x), N = theta_o, K = (theta_i, dy, dx), restricted to the
// theta_i band where the fp32 table is nonzero (the taps outside the band are exactly 0 in fp32).
//
// CTA = 4 warps.  Tile = 32 rows (one per lane) x 32 columns (8 per thread, 4 warps along x)
// x 4 output orientations (a theta quad).  Per theta_i the CTA stages, double-buffered with
// cp.async, the (32+2R) x (32+2R) input window (zero padded) and the S x S x 4 filter block
// (theta-quad interleaved, so one LDS.128 broadcast feeds 4 orientations).  Each thread keeps
// 4 x 8 accumulators; per filter row dy it loads its input row segment (8 + 2R floats, LDS.128,
// conflict-free: pitch/4 odd) and issues S*32 FFMA against S LDS.128 filter broadcasts.
#include "conv_common.cuh"

namespace se2 {

template <int R>
struct LinCfg {
    static constexpr int S = 2 * R + 1;
    static constexpr int P = 8;    // columns per thread
    static constexpr int WX = 4;   // warps along x
    static constexpr int NT = 32 * WX;
    static constexpr int TY = 32, TX = P * WX;
    static constexpr int WIN_H = TY + 2 * R;
    static constexpr int WIN_W = TX + 2 * R;
    static constexpr int RL = ((P + 2 * R) + 3) / 4 * 4;  // register row length (floats)
    static constexpr int NEED = ((WX - 1) * P + RL) > WIN_W ? ((WX - 1) * P + RL) : WIN_W;
    static constexpr int P0 = (NEED + 3) / 4 * 4;
    static constexpr int PITCH = ((P0 / 4) % 2 == 1) ? P0 : P0 + 4;  // pitch/4 odd -> no conflicts
    static constexpr int WIN = WIN_H * PITCH;
    static constexpr int FIL = S * S * 4;
    static constexpr size_t SMEM = (size_t)(2 * WIN + 2 * FIL) * sizeof(float) + 64;
};

template <int R>
__global__ void __launch_bounds__(LinCfg<R>::NT)
conv_linear_kernel(const float* __restrict__ in, const float* __restrict__ Wq, int nx, int ny, int nt,
                   int band, int tiles_x, Epilogue epi) {
    using C = LinCfg<R>;
    extern __shared__ __align__(16) float smem[];
    float* sWin = smem;                 // [2][WIN]
    float* sFil = smem + 2 * C::WIN;    // [2][FIL]
    float* sRed = sFil + 2 * C::FIL;    // reduction scratch (16 floats)

    const int tile = blockIdx.x;
    const int qd = blockIdx.y;
    const int b = blockIdx.z;
    const int x0 = (tile % tiles_x) * C::TX;
    const int y0 = (tile / tiles_x) * C::TY;
    const int64_t N = (int64_t)nx * ny * nt;
    const float* vin = in + (int64_t)b * N;
    const int lane = threadIdx.x & 31;
    const int wx = threadIdx.x >> 5;

    // theta_i range: [4qd - band, 4qd + 3 + band] (mod nt), or all of them
    int nti = 4 + 2 * band;
    int ti0 = 4 * qd - band;
    if (nti >= nt) { nti = nt; ti0 = 0; }

    // zero the pitch padding columns once (never used in arithmetic; keeps initcheck clean)
    for (int i = threadIdx.x; i < 2 * C::WIN_H; i += C::NT) {
        float* row = sWin + (i / C::WIN_H) * C::WIN + (i % C::WIN_H) * C::PITCH;
        for (int c = C::WIN_W; c < C::PITCH; ++c) row[c] = 0.f;
    }

    auto stage = [&](int it, int buf) {
        int ti = ti0 + it;
        ti = ((ti % nt) + nt) % nt;
        const float* src = vin + (int64_t)ti * nx * ny;
        float* dw = sWin + buf * C::WIN;
        for (int i = threadIdx.x; i < C::WIN_H * C::WIN_W; i += C::NT) {
            int r = i / C::WIN_W, c = i % C::WIN_W;
            int gy = y0 - R + r, gx = x0 - R + c;
            bool ok = (gy >= 0) && (gy < ny) && (gx >= 0) && (gx < nx);
            cp_async4(dw + r * C::PITCH + c, ok ? (src + (int64_t)gy * nx + gx) : vin, ok);
        }
        const float* fsrc = Wq + ((int64_t)qd * nt + ti) * C::FIL;
        float* df = sFil + buf * C::FIL;
        for (int i = threadIdx.x; i < C::FIL / 4; i += C::NT) cp_async16(df + 4 * i, fsrc + 4 * i);
        cp_async_commit();
    };

    float acc[4][C::P];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int p = 0; p < C::P; ++p) acc[q][p] = 0.f;

    stage(0, 0);
    for (int it = 0; it < nti; ++it) {
        const int buf = it & 1;
        if (it + 1 < nti) {
            stage(it + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const float* win = sWin + buf * C::WIN + wx * C::P;
        const float4* fil = reinterpret_cast<const float4*>(sFil + buf * C::FIL);
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
        __syncthreads();
    }

    // fused epilogue
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
                    int64_t idx = (int64_t)b * N + ((int64_t)to * ny + gy) * nx + gx;
                    err += apply_epilogue<false>(epi, idx, gx, gy, acc[q][p]);
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
static cudaError_t launch_lin_r(const se2_kernel_s* k, const float* in, int batch, const Epilogue& epi,
                                cudaStream_t s, int* bpf) {
    using C = LinCfg<R>;
    cudaError_t e = cudaFuncSetAttribute(conv_linear_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::SMEM);
    if (e != cudaSuccess) return e;
    int tiles_x = (k->nx + C::TX - 1) / C::TX;
    int tiles_y = (k->ny + C::TY - 1) / C::TY;
    dim3 grid(tiles_x * tiles_y, (k->nt + 3) / 4, batch);
    if (bpf) *bpf = (int)(grid.x * grid.y);
    conv_linear_kernel<R><<<grid, C::NT, C::SMEM, s>>>(in, k->Wq, k->nx, k->ny, k->nt, k->band, tiles_x, epi);
    count_launch();
    return cudaGetLastError();
}

int conv_blocks_per_field_linear(const se2_kernel_s* k) {
    // all radii share the tile geometry
    using C = LinCfg<1>;
    int tiles_x = (k->nx + C::TX - 1) / C::TX;
    int tiles_y = (k->ny + C::TY - 1) / C::TY;
    return tiles_x * tiles_y * ((k->nt + 3) / 4);
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
