// K4: SE(2) group convolution in the log domain, exact log-sum-exp (reading R7):
//
//   ly[b, to, x] = log sum_{ti, dy, dx} exp( L[to, ti, dy, dx] + lv[b, ti, x - (dx, dy)] )
//
// i.e. log(K exp(lv)) without ever forming exp(lv): every tap is evaluated as exp2 of its exponent
// relative to a per-output running maximum, so no scaling can overflow or underflow before it
// is negligible.  Per theta_i chunk (one staged input channel) each output does two passes over
// the S x S taps: (A) the chunk maximum, (B) the rescaled exp-sum
//     s <- s * 2^(m - m') + sum 2^(t - m'),   m' = max(m, max_chunk t),   t in log2 units.
// Cost per tap and output: 1 MUFU.EX2 + 5 FP32 ops -> bounded by the MUFU pipe (16/clk/SM).
//
// Tiling as the linear engine but with 4 columns per thread (16 outputs x {m, s, chunk max}):
// CTA = 4 warps; tile = 32 rows x 16 columns x one theta quad.  All nt input orientations are
// visited (the log path has no fp32 band: far orientations can dominate when potentials vary).
#include "conv_common.cuh"

namespace se2 {

template <int R>
struct LseCfg {
    static constexpr int S = 2 * R + 1;
    static constexpr int P = 4;
    static constexpr int WX = 4;
    static constexpr int NT = 32 * WX;
    static constexpr int TY = 32, TX = P * WX;
    static constexpr int WIN_H = TY + 2 * R;
    static constexpr int WIN_W = TX + 2 * R;
    static constexpr int RL = ((P + 2 * R) + 3) / 4 * 4;
    static constexpr int NEED = ((WX - 1) * P + RL) > WIN_W ? ((WX - 1) * P + RL) : WIN_W;
    static constexpr int P0 = (NEED + 3) / 4 * 4;
    static constexpr int PITCH = ((P0 / 4) % 2 == 1) ? P0 : P0 + 4;
    static constexpr int WIN = WIN_H * PITCH;
    static constexpr int FIL = S * S * 4;
    static constexpr size_t SMEM = (size_t)(2 * WIN + 2 * FIL) * sizeof(float) + 64;
};

template <int R>
__global__ void __launch_bounds__(LseCfg<R>::NT)
conv_lse_kernel(const float* __restrict__ in, const float* __restrict__ Lq, int nx, int ny, int nt,
                int tiles_x, Epilogue epi) {
    using C = LseCfg<R>;
    extern __shared__ __align__(16) float smem[];
    float* sWin = smem;
    float* sFil = smem + 2 * C::WIN;
    float* sRed = sFil + 2 * C::FIL;

    const int tile = blockIdx.x;
    const int qd = blockIdx.y;
    const int b = blockIdx.z;
    const int x0 = (tile % tiles_x) * C::TX;
    const int y0 = (tile / tiles_x) * C::TY;
    const int64_t N = (int64_t)nx * ny * nt;
    const float* vin = in + (int64_t)b * N;
    const int lane = threadIdx.x & 31;
    const int wx = threadIdx.x >> 5;
    const float NEG_INF = -INFINITY;

    for (int i = threadIdx.x; i < 2 * C::WIN_H; i += C::NT) {
        float* row = sWin + (i / C::WIN_H) * C::WIN + (i % C::WIN_H) * C::PITCH;
        for (int c = C::WIN_W; c < C::PITCH; ++c) row[c] = NEG_INF;
    }

    auto stage = [&](int ti, int buf) {
        const float* src = vin + (int64_t)ti * nx * ny;
        float* dw = sWin + buf * C::WIN;
        for (int i = threadIdx.x; i < C::WIN_H * C::WIN_W; i += C::NT) {
            int r = i / C::WIN_W, c = i % C::WIN_W;
            int gy = y0 - R + r, gx = x0 - R + c;
            bool ok = (gy >= 0) && (gy < ny) && (gx >= 0) && (gx < nx);
            if (ok)
                cp_async4(dw + r * C::PITCH + c, src + (int64_t)gy * nx + gx, true);
            else
                dw[r * C::PITCH + c] = NEG_INF;   // log of the zero padding
        }
        const float* fsrc = Lq + ((int64_t)qd * nt + ti) * C::FIL;
        float* df = sFil + buf * C::FIL;
        for (int i = threadIdx.x; i < C::FIL / 4; i += C::NT) cp_async16(df + 4 * i, fsrc + 4 * i);
        cp_async_commit();
    };

    float m[4][C::P], s[4][C::P];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int p = 0; p < C::P; ++p) { m[q][p] = NEG_INF; s[q][p] = 0.f; }

    stage(0, 0);
    for (int ti = 0; ti < nt; ++ti) {
        const int buf = ti & 1;
        if (ti + 1 < nt) {
            stage(ti + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const float* win = sWin + buf * C::WIN + wx * C::P;
        const float4* fil = reinterpret_cast<const float4*>(sFil + buf * C::FIL);

        // pass A: chunk maximum of t = L2 + lv*log2(e)
        float cm[4][C::P];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int p = 0; p < C::P; ++p) cm[q][p] = m[q][p];
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
                    cm[0][p] = fmaxf(cm[0][p], fmaf(xv, kLog2e, w.x));
                    cm[1][p] = fmaxf(cm[1][p], fmaf(xv, kLog2e, w.y));
                    cm[2][p] = fmaxf(cm[2][p], fmaf(xv, kLog2e, w.z));
                    cm[3][p] = fmaxf(cm[3][p], fmaf(xv, kLog2e, w.w));
                }
            }
        }
        // rescale running sums to the new maxima (m = -inf while nothing finite was seen)
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int p = 0; p < C::P; ++p) {
                float mn = cm[q][p];
                float safe = (mn == NEG_INF) ? 0.f : mn;
                s[q][p] *= ex2_approx(m[q][p] - safe);
                m[q][p] = safe;   // stored shift (0 when all -inf so far; s stays 0)
                cm[q][p] = mn;
            }
        // pass B: s += 2^(t - m)
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
                    s[0][p] += ex2_approx(fmaf(xv, kLog2e, w.x) - m[0][p]);
                    s[1][p] += ex2_approx(fmaf(xv, kLog2e, w.y) - m[1][p]);
                    s[2][p] += ex2_approx(fmaf(xv, kLog2e, w.z) - m[2][p]);
                    s[3][p] += ex2_approx(fmaf(xv, kLog2e, w.w) - m[3][p]);
                }
            }
        }
        // keep -inf as the maximum of an all -inf prefix
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int p = 0; p < C::P; ++p)
                if (cm[q][p] == NEG_INF) m[q][p] = NEG_INF;
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
                    float ly = (m[q][p] == NEG_INF || s[q][p] <= 0.f)
                                   ? NEG_INF
                                   : (m[q][p] + log2f(s[q][p])) * kLn2;
                    int64_t idx = (int64_t)b * N + ((int64_t)to * ny + gy) * nx + gx;
                    err += apply_epilogue<true>(epi, idx, gx, gy, ly);
                }
            }
        }
    }
    if (epi.err_partial != nullptr) {
        float t = block_sum<C::NT>(err, sRed);
        if (threadIdx.x == 0)
        {   // 4 slots per (field, quad, tile): the layout K3's split combine fills one per orientation
            float* o = epi.err_partial + (((int64_t)b * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 4;
            o[0] = t;
            o[1] = 0.f;
            o[2] = 0.f;
            o[3] = 0.f;
        }
    }
}

template <int R>
static cudaError_t launch_lse_r(const se2_kernel_s* k, const float* in, int batch, const Epilogue& epi,
                                cudaStream_t s, int* bpf) {
    using C = LseCfg<R>;
    cudaError_t e = cudaFuncSetAttribute(conv_lse_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::SMEM);
    if (e != cudaSuccess) return e;
    int tiles_x = (k->nx + C::TX - 1) / C::TX;
    int tiles_y = (k->ny + C::TY - 1) / C::TY;
    dim3 grid(tiles_x * tiles_y, (k->nt + 3) / 4, batch);
    if (bpf) *bpf = (int)(grid.x * grid.y) * 4;
    conv_lse_kernel<R><<<grid, C::NT, C::SMEM, s>>>(in, epi.table ? epi.table : k->Lq, k->nx, k->ny, k->nt, tiles_x, epi);
    count_launch();
    return cudaGetLastError();
}

int conv_blocks_per_field_lse(const se2_kernel_s* k) {
    using C = LseCfg<1>;
    int tiles_x = (k->nx + C::TX - 1) / C::TX;
    int tiles_y = (k->ny + C::TY - 1) / C::TY;
    return tiles_x * tiles_y * ((k->nt + 3) / 4) * 4;   // 4 error-partial slots per (tile, quad)
}

cudaError_t launch_conv_lse(const se2_kernel_s* k, const float* in, int batch, const Epilogue& epi,
                            cudaStream_t s, int* bpf) {
    switch (k->R) {
#define SE2_CASE(r) \
    case r: return launch_lse_r<r>(k, in, batch, epi, s, bpf);
        SE2_CASE(0) SE2_CASE(1) SE2_CASE(2) SE2_CASE(3) SE2_CASE(4) SE2_CASE(5) SE2_CASE(6) SE2_CASE(7)
        SE2_CASE(8) SE2_CASE(9) SE2_CASE(10) SE2_CASE(11) SE2_CASE(12) SE2_CASE(13) SE2_CASE(14) SE2_CASE(15)
#undef SE2_CASE
        default: return cudaErrorInvalidValue;
    }
}

int conv_blocks_per_field(const se2_kernel_s* k, bool log_domain, uint32_t flags) {
    if (log_domain) return conv_blocks_per_field_lse(k);
    return conv_tc_active(k, flags) ? conv_blocks_per_field_tc(k) : conv_blocks_per_field_linear(k);
}

}  // namespace se2
