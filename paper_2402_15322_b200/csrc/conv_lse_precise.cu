// K4P: the exact log-domain SE(2) conv with fp64 potentials (the north star's 1e-4 elementwise parity on
// potentials that reach 10^2..10^3 nats; SURVEY ledger L16 / DESIGN.md reading R19):
//
//   ly[b, to, x] = log sum_{ti, dy, dx} exp( L[to, ti, dy, dx] + lv[b, ti, x - (dx, dy)] )
//
// fp32 arithmetic on such magnitudes loses ~1e-5 nats per conv in three places, which the slowly
// contracting modes of the barycenter iteration accumulate past 1e-4 (tools/conv_err_probe.py): the
// rounding of L and of lv (values of hundreds of nats), the sum of the large exponent parts, and the fp32
// accumulation of thousands of terms plus the approximate rescaling between channels.  K4P keeps the
// tiling and the two passes of K4 and removes each loss:
//   * lv (fp64 in HBM) is staged as an exact float pair r_hi + r_lo = lv log2(e); L2 = L log2(e) is an
//     exact float pair table (fp64 formula, split once);
//   * per tap the exponent r_hi + L_hi is formed with TwoSum (exact), the per-output shift m is an
//     INTEGER (floor of the approximate maximum) so the big cancellation t - m is exact, and the small
//     parts (TwoSum error, r_lo, L_lo) are added last: the exponent of every retained term is exact to
//     fp32 rounding of a number of magnitude <~ 30;
//   * each tap row is summed in fp32 (S terms) and the row sums in fp64; rescaling to a new maximum is
//     an exact power of two (ldexp), and ly = (m + log2 S) ln 2 is formed in fp64.
// What remains per conv is ex2.approx's ~2^-22 relative error per term: ~1e-7 nats.  Cost per tap and
// output: 1 MUFU.EX2 + ~11 FP32 ops (K4: 1 + 5).
#include "conv_common.cuh"

namespace se2 {

template <int R>
struct LsePCfg {
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
    static constexpr int RAW = WIN_H * WIN_W;   // the next channel's fp64 window, dense (cp.async target)
    // window hi + lo (converted), the raw fp64 window of the next channel, filter hi + lo + row bounds
    // double-buffered: channel a + 1 loads while channel a computes
    static constexpr size_t SMEM = (size_t)RAW * sizeof(double) + (size_t)(2 * WIN + 2 * (2 * FIL + 4 * S)) * sizeof(float) + 64;
};
// pruning margin (log2 units): a term below 2^-64 of every output it could reach is never evaluated;
// the skipped mass is < S^2 nt 2^-64 < 2^-48 relative
constexpr float kGap = 64.f;

// a staged -inf (zero mass, zero padding) is the finite sentinel -1e30: TwoSum stays NaN-free and its
// terms underflow to exactly 0; a pass-A maximum below -1e29 means "no finite term"
constexpr float kSent = -1e30f;
__device__ __forceinline__ void split2(double x, float& hi, float& lo) {
    if (!(x > -1e300)) {
        hi = kSent;
        lo = 0.f;
        return;
    }
    hi = (float)x;
    lo = (float)(x - (double)hi);
}

template <int R>
__global__ void __launch_bounds__(LsePCfg<R>::NT)
conv_lse_precise_kernel(const double* __restrict__ in, const float* __restrict__ L2hi, const float* __restrict__ L2lo,
                        const float* __restrict__ L2row, int nx, int ny, int nt, int tiles_x, int y_lo, int y_hi,
                        EpiP epi) {
    using C = LsePCfg<R>;
    extern __shared__ __align__(16) float smem[];
    double* sRaw = reinterpret_cast<double*>(smem);                 // [WIN_H * WIN_W] next channel, fp64
    float* sWh = smem + 2 * C::RAW;
    float* sWl = sWh + C::WIN;
    float* sF0 = sWl + C::WIN;   // 2 buffers of [hi FIL][lo FIL][row S x 4]
    constexpr int FBUF = 2 * C::FIL + 4 * C::S;
    __shared__ float sRed[C::NT / 32];

    const int tile = blockIdx.x;
    const int qd = blockIdx.y;
    const int b = blockIdx.z;
    const int x0 = (tile % tiles_x) * C::TX;
    const int y0 = y_lo + (tile / tiles_x) * C::TY;
    const int64_t N = (int64_t)nx * ny * nt;
    const double* vin = in + (int64_t)b * N;
    const int lane = threadIdx.x & 31;
    const int wx = threadIdx.x >> 5;
    const float NEG_INF = -INFINITY;
    const double LOG2E = 1.4426950408889634073599246810019;

    for (int i = threadIdx.x; i < C::WIN_H; i += C::NT)
        for (int c = C::WIN_W; c < C::PITCH; ++c) {
            sWh[i * C::PITCH + c] = kSent;
            sWl[i * C::PITCH + c] = 0.f;
        }

    float m[4][C::P];      // integer shift (log2 units); NEG_INF while no finite term was seen
    double sd[4][C::P];    // sum of 2^(t - m), fp64
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int p = 0; p < C::P; ++p) { m[q][p] = NEG_INF; sd[q][p] = 0.0; }

    // valid outputs of this thread (bit 4 q + p)
    unsigned vmask = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int p = 0; p < C::P; ++p)
            if (4 * qd + q < nt && y0 + lane < y_hi && x0 + wx * C::P + p < nx) vmask |= 1u << (4 * q + p);
    // pruning floor per output orientation of this lane: min over its valid outputs of (shift - kGap);
    // -inf while any of them has no finite term yet
    auto floors = [&](float* lb) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float t = INFINITY;
#pragma unroll
            for (int p = 0; p < C::P; ++p)
                if (vmask & (1u << (4 * q + p))) t = fminf(t, m[q][p]);
            lb[q] = t - kGap;   // NEG_INF stays NEG_INF
        }
    };

    // channels in order of increasing |theta_i - theta_o| around the quad: the dominant ones set the
    // shifts early, so the pruning bounds below bite on the rest
    auto chan = [&](int a) {
        const int off = (a & 1) ? (a + 1) / 2 : -(a / 2);
        return (((4 * qd + 1 + off) % nt) + nt) % nt;
    };
    // asynchronous staging of channel a: the raw fp64 window (zero padding / -inf as -inf) and the
    // channel's filter tables into buffer a & 1; the thread that copied an element converts it
    auto issue = [&](int a) {
        const int ti = chan(a);
        const double* src = vin + (int64_t)ti * nx * ny;
        for (int i = threadIdx.x; i < C::RAW; i += C::NT) {
            const int r = i / C::WIN_W, c = i - r * C::WIN_W;
            const int gy = y0 - R + r, gx = x0 - R + c;
            if (gy >= 0 && gy < ny && gx >= 0 && gx < nx)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(sRaw + i)),
                             "l"(src + (int64_t)gy * nx + gx));
            else
                sRaw[i] = -(double)INFINITY;
        }
        float* fb = sF0 + (a & 1) * FBUF;
        const float* fh = L2hi + ((int64_t)qd * nt + ti) * C::FIL;
        const float* fl = L2lo + ((int64_t)qd * nt + ti) * C::FIL;
        for (int i = threadIdx.x; i < C::FIL / 4; i += C::NT) {
            cp_async16(fb + 4 * i, fh + 4 * i);
            cp_async16(fb + C::FIL + 4 * i, fl + 4 * i);
        }
        const float* rm = L2row + ((int64_t)qd * nt + ti) * C::S * 4;
        for (int i = threadIdx.x; i < C::S; i += C::NT) cp_async16(fb + 2 * C::FIL + 4 * i, rm + 4 * i);
        cp_async_commit();
    };
    issue(0);
    for (int a = 0; a < nt; ++a) {
        cp_async_wait<0>();
        __syncthreads();   // channel a's copies visible; the previous channel's readers of sWh / sWl are done
        for (int i = threadIdx.x; i < C::RAW; i += C::NT) {
            const int r = i / C::WIN_W, c = i - r * C::WIN_W;
            float hi, lo;
            split2(sRaw[i] * LOG2E, hi, lo);
            sWh[r * C::PITCH + c] = hi;
            sWl[r * C::PITCH + c] = lo;
        }
        __syncthreads();   // sRaw free for the next channel, sWh / sWl complete
        if (a + 1 < nt) issue(a + 1);
        const float* sFh = sF0 + (a & 1) * FBUF;
        const float* sFl = sFh + C::FIL;
        const float* sRow = sFh + 2 * C::FIL;   // [S][4] max over each tap row of L2 (pruning bounds)
        const float* wh = sWh + wx * C::P;
        const float* wl = sWl + wx * C::P;
        const float4* fh4 = reinterpret_cast<const float4*>(sFh);
        const float4* fl4 = reinterpret_cast<const float4*>(sFl);
        const float4* rw4 = reinterpret_cast<const float4*>(sRow);

        // channel bound of this warp: max of the window columns it reads + the channel's largest L2 (its
        // centre tap, Ls(0) = 0 >= Ls(d)); a channel below every output's floor is skipped
        float lb[4];
        floors(lb);
        {
            float wm = kSent;
            for (int r = lane; r < C::WIN_H; r += 32)
#pragma unroll
                for (int c = 0; c < C::RL; ++c) wm = fmaxf(wm, wh[r * C::PITCH + c]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));
            const float4 cen = fh4[R * C::S + R];
            const bool any = __any_sync(0xffffffffu, wm + cen.x >= lb[0] || wm + cen.y >= lb[1] ||
                                                         wm + cen.z >= lb[2] || wm + cen.w >= lb[3]);
            if (!any) continue;   // warp-uniform: no term of this channel can reach these outputs
        }

        // pass A: approximate channel maximum (fp32 sums suffice: the shift only has to be near the max)
        float cm[4][C::P];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int p = 0; p < C::P; ++p) cm[q][p] = NEG_INF;
#pragma unroll 1
        for (int dy = 0; dy < C::S; ++dy) {
            const float4* rowp = reinterpret_cast<const float4*>(wh + (lane - dy + 2 * R) * C::PITCH);
            float r[C::RL];
            float rmax = kSent;
#pragma unroll
            for (int j = 0; j < C::RL / 4; ++j) {
                const float4 t = rowp[j];
                r[4 * j + 0] = t.x; r[4 * j + 1] = t.y; r[4 * j + 2] = t.z; r[4 * j + 3] = t.w;
                rmax = fmaxf(fmaxf(rmax, fmaxf(t.x, t.y)), fmaxf(t.z, t.w));
            }
            const float4 rb = rw4[dy];   // max over the row's taps of L2 (per q)
            if (!__any_sync(0xffffffffu, rmax + rb.x >= lb[0] || rmax + rb.y >= lb[1] || rmax + rb.z >= lb[2] ||
                                             rmax + rb.w >= lb[3]))
                continue;   // no tap of this row can raise any shift of the warp
#pragma unroll
            for (int dx = 0; dx < C::S; ++dx) {
                const float4 w = fh4[dy * C::S + dx];
#pragma unroll
                for (int p = 0; p < C::P; ++p) {
                    const float xv = r[p - dx + 2 * R];
                    cm[0][p] = fmaxf(cm[0][p], xv + w.x);
                    cm[1][p] = fmaxf(cm[1][p], xv + w.y);
                    cm[2][p] = fmaxf(cm[2][p], xv + w.z);
                    cm[3][p] = fmaxf(cm[3][p], xv + w.w);
                }
            }
        }
        // new integer shifts; exact power-of-two rescale of the running sums
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int p = 0; p < C::P; ++p) {
                if (!(cm[q][p] > -1e29f)) continue;   // only sentinel terms so far
                const float mn = floorf(cm[q][p]) + 1.f;   // every term t - mn < 1 up to the pass-A rounding
                if (m[q][p] == NEG_INF) {
                    m[q][p] = mn;
                } else if (mn > m[q][p]) {
                    sd[q][p] = ldexp(sd[q][p], (int)(m[q][p] - mn));
                    m[q][p] = mn;
                }
            }
        floors(lb);
        // pass B: sum 2^(t - m) with exact exponents; row sums in fp32, the total in fp64.  A (row,
        // orientation) whose largest term is below 2^-kGap of every output of the warp is skipped.
#pragma unroll 1
        for (int dy = 0; dy < C::S; ++dy) {
            const float4* rowh = reinterpret_cast<const float4*>(wh + (lane - dy + 2 * R) * C::PITCH);
            const float4* rowl = reinterpret_cast<const float4*>(wl + (lane - dy + 2 * R) * C::PITCH);
            float rh[C::RL], rl[C::RL];
            float rmax = kSent;
#pragma unroll
            for (int j = 0; j < C::RL / 4; ++j) {
                const float4 t = rowh[j];
                rh[4 * j + 0] = t.x; rh[4 * j + 1] = t.y; rh[4 * j + 2] = t.z; rh[4 * j + 3] = t.w;
                rmax = fmaxf(fmaxf(rmax, fmaxf(t.x, t.y)), fmaxf(t.z, t.w));
            }
            const float4 rb = rw4[dy];
            const float rbv[4] = {rb.x, rb.y, rb.z, rb.w};
            unsigned live = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) live |= __any_sync(0xffffffffu, rmax + rbv[q] >= lb[q]) ? (1u << q) : 0u;
            if (!live) continue;
#pragma unroll
            for (int j = 0; j < C::RL / 4; ++j) {
                const float4 u = rowl[j];
                rl[4 * j + 0] = u.x; rl[4 * j + 1] = u.y; rl[4 * j + 2] = u.z; rl[4 * j + 3] = u.w;
            }
            const float* frh = reinterpret_cast<const float*>(fh4 + dy * C::S);   // [dx][q]
            const float* frl = reinterpret_cast<const float*>(fl4 + dy * C::S);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (!((live >> q) & 1u)) continue;
                float rs[C::P];
#pragma unroll
                for (int p = 0; p < C::P; ++p) rs[p] = 0.f;
#pragma unroll
                for (int dx = 0; dx < C::S; ++dx) {
                    const float bb = frh[4 * dx + q], blo = frl[4 * dx + q];
#pragma unroll
                    for (int p = 0; p < C::P; ++p) {
                        const float av = rh[p - dx + 2 * R];
                        const float s1 = av + bb;                                   // TwoSum(av, bb)
                        const float bv = s1 - av;
                        const float e1 = (av - (s1 - bv)) + (bb - bv);
                        const float u = (s1 - m[q][p]) + (e1 + (rl[p - dx + 2 * R] + blo));   // s1 - m exact
                        rs[p] += ex2_approx(u);                                     // sentinel -> 0
                    }
                }
#pragma unroll
                for (int p = 0; p < C::P; ++p)
                    if (m[q][p] != NEG_INF) sd[q][p] += (double)rs[p];
            }
        }
    }

    float err = 0.f;
    const int gy = y0 + lane;
    if (gy < y_hi) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int to = 4 * qd + q;
            if (to >= nt) continue;
#pragma unroll
            for (int p = 0; p < C::P; ++p) {
                const int gx = x0 + wx * C::P + p;
                if (gx >= nx) continue;
                const double ly = (m[q][p] == NEG_INF || !(sd[q][p] > 0.0))
                                      ? -(double)INFINITY
                                      : ((double)m[q][p] + log2(sd[q][p])) * 0.69314718055994530941723212145818;
                const int64_t idx = (int64_t)b * N + ((int64_t)to * ny + gy) * nx + gx;
                err += apply_epilogue_precise(epi, idx, ly);
            }
        }
    }
    if (epi.err_partial != nullptr) {
        const float t = block_sum<C::NT>(err, sRed);
        if (threadIdx.x == 0) epi.err_partial[((int64_t)b * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
    }
}

template <int R>
static cudaError_t launch_lsep_r(const se2_kernel_s* k, const double* in, int batch, const EpiP& epi, cudaStream_t s,
                                 int* bpf) {
    using C = LsePCfg<R>;
    cudaError_t e = cudaFuncSetAttribute(conv_lse_precise_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::SMEM);
    if (e != cudaSuccess) return e;
    const int tiles_x = (k->nx + C::TX - 1) / C::TX;
    const int tiles_y = (k->wrows() + C::TY - 1) / C::TY;
    dim3 grid(tiles_x * tiles_y, (k->nt + 3) / 4, batch);
    if (bpf) *bpf = (int)(grid.x * grid.y);
    conv_lse_precise_kernel<R><<<grid, C::NT, C::SMEM, s>>>(in, k->L2hi, k->L2lo, k->L2row, k->nx, k->ny, k->nt,
                                                             tiles_x, k->wlo(), k->whi(), epi);
    count_launch();
    return cudaGetLastError();
}

int conv_blocks_per_field_precise(const se2_kernel_s* k) {
    using C = LsePCfg<1>;
    const int tiles_x = (k->nx + C::TX - 1) / C::TX;
    const int tiles_y = (k->wrows() + C::TY - 1) / C::TY;
    return tiles_x * tiles_y * ((k->nt + 3) / 4);
}

cudaError_t launch_conv_lse_precise(const se2_kernel_s* k, const double* in, int batch, const EpiP& epi,
                                    cudaStream_t s, int* bpf) {
    if (k->L2hi == nullptr) return cudaErrorNotReady;
    switch (k->R) {
#define SE2_CASE(r) \
    case r: return launch_lsep_r<r>(k, in, batch, epi, s, bpf);
        SE2_CASE(0) SE2_CASE(1) SE2_CASE(2) SE2_CASE(3) SE2_CASE(4) SE2_CASE(5) SE2_CASE(6) SE2_CASE(7)
        SE2_CASE(8) SE2_CASE(9) SE2_CASE(10) SE2_CASE(11) SE2_CASE(12) SE2_CASE(13) SE2_CASE(14) SE2_CASE(15)
#undef SE2_CASE
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace se2
