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
//
// Factored (FFMA) path for channels whose staged window lies within kFfmaRangeP nats of the tile's
// minimum (K4P): exp(L + lv) = exp(Lth) exp(Ls + 40) exp(lv - M + 40) exp(M - 80) with M the
// window maximum -- the spatial table Eq = exp(Ls + 40) (fp32, relative rounding only) times
// v~ = exp(lv - M + 40) computed in fp64 from the fp64 potential and rounded once (relative rounding only),
// so no term carries an absolute exponent error however large the potentials are.  Per tap one FFMA; tap
// rows summed in fp32, rows in fp64; the channel's sum S enters the output's (integer shift, fp64 sum) as
// frexp(S) 2^(floor G) 2^frac(G), G = (M - 80 + Lth) log2 e in fp64 (Lth from its fp64 formula).
// Validity (range <= 80 nats): every retained product is a normal float >= e^-42, no sum overflows
// (961 e^80 < 2^127), and the products dropped by underflow are below e^-40 of the output's centre term.
#include <type_traits>

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
constexpr double kFfmaRangeP = 80.0;   // natural log units: FFMA path when max(window) - min(tile) <= this
// compact exact power-of-two scaling / splitting (the libm ldexp / frexp / log2 / exp bodies, inlined per
// output, made the kernel's code overflow the instruction cache)
__device__ __forceinline__ double pow2i(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }
__device__ __forceinline__ double ldexp_fast(double x, int e) {   // exact while the result is normal
    if (e >= -1022 && e <= 1023) return x * pow2i(e);
    int e1 = e / 2, e2 = e - e1;
    e1 = max(-1022, min(1023, e1));
    e2 = max(-1022, min(1023, e2));
    return (x * pow2i(e1)) * pow2i(e2);
}
__device__ __forceinline__ double frexp_pos(double x, int& e) {   // x > 0 normal: x = mant 2^e, mant in [0.5, 1)
    const long long bits = __double_as_longlong(x);
    e = (int)((bits >> 52) & 0x7ff) - 1022;
    return __longlong_as_double((bits & ~(0x7ffLL << 52)) | (1022LL << 52));
}
__device__ __noinline__ double log2_once(double x) { return log2(x); }
__device__ __noinline__ double exp2_once(double x) { return exp2(x); }
// exp(t) for |t| <~ 200 to ~1.5 ulp of fp32: t = th + tl (fp32 pair), exp(th) (expf) times (1 + tl)
__device__ __forceinline__ float exp_pair(double t) {
    if (!(t > -1e300)) return 0.f;   // zero mass / padding (-inf): -inf - -inf would be NaN below
    const float th = (float)t;
    const float tl = (float)(t - (double)th);
    return expf(th) * (1.f + tl);
}

__device__ __forceinline__ void split2(double x, float& hi, float& lo) {
    if (!(x > -1e300)) {
        hi = kSent;
        lo = 0.f;
        return;
    }
    hi = (float)x;
    lo = (float)(x - (double)hi);
}

// channel bounds without staging: per (field, theta, row, 16-column block) the min / max of lv, rounded
// outward to fp32; one thread per segment (16 consecutive doubles of one row)
constexpr int kPSegW = 16;
constexpr int kPMaxNT = 128;                 // channel pruning from these bounds for nt <= 128
constexpr float kGapNat = 44.3614195558365f;  // kGap log2 units in nats
__global__ void lsep_stats_kernel(const double* __restrict__ in, int nx, int ny, int nt, int batch,
                                  float4* __restrict__ st) {
    const int nxb = (nx + kPSegW - 1) / kPSegW;
    const int64_t total = (int64_t)batch * nt * ny * nxb;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int xb = (int)(i % nxb);
        const int64_t row = i / nxb;   // (b, theta, y)
        const double* src = in + row * nx + xb * kPSegW;
        double mn = INFINITY, mx = -INFINITY, mnf = INFINITY;
        const int w = min(kPSegW, nx - xb * kPSegW);
        for (int j = 0; j < w; ++j) {
            const double v = src[j];
            mn = fmin(mn, v);
            mx = fmax(mx, v);
            if (v > -INFINITY) mnf = fmin(mnf, v);
        }
        st[i] = make_float4(__double2float_rd(mn), __double2float_ru(mx), __double2float_rd(mnf), 0.f);
    }
}

template <int R>
__global__ void __launch_bounds__(LsePCfg<R>::NT)
conv_lse_precise_kernel(const double* __restrict__ in, const float* __restrict__ L2hi, const float* __restrict__ L2lo,
                        const float* __restrict__ L2row, const float* __restrict__ Eq, double w3sq_eps, int nx, int ny,
                        int nt, int tiles_x, int y_lo, int y_hi, EpiP epi, int ffma_max_a,
                        unsigned long long* __restrict__ counters, const float4* __restrict__ pst,
                        const float* __restrict__ Lth, const float* __restrict__ LseS, int ngroups,
                        double2* __restrict__ split_out) {
    using C = LsePCfg<R>;
    extern __shared__ __align__(16) float smem[];
    double* sRaw = reinterpret_cast<double*>(smem);                 // [WIN_H * WIN_W] next channel, fp64
    float* sWh = smem + 2 * C::RAW;
    float* sWl = sWh + C::WIN;
    float* sF0 = sWl + C::WIN;   // 2 buffers of [hi FIL][lo FIL][row S x 4]
    constexpr int FBUF = 2 * C::FIL + 4 * C::S;
    __shared__ float sRed[C::NT / 32];
    __shared__ float sCM[kPMaxNT], sCMu[kPMaxNT], sCMn[kPMaxNT], sPM[C::NT], sPMu[C::NT], sPMn[C::NT], sLB[4];
    __shared__ int sAct[kPMaxNT], sNAct;

    const int tile = blockIdx.x;
    // theta_i split (small grids): blockIdx.y = qd * ngroups + grp; the CTA takes every ngroups-th channel of
    // the active list and writes its partial (shift, sum) per output to split_out (combined afterwards)
    const int qd = blockIdx.y / ngroups;
    const int grp = blockIdx.y - qd * ngroups;
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
    auto chan0 = [&](int a) {
        const int off = (a & 1) ? (a + 1) / 2 : -(a / 2);
        return (((4 * qd + 1 + off) % nt) + nt) % nt;
    };
    // channel pruning from the row-segment bounds (nt <= kPMaxNT): a channel ti is skipped when its largest
    // possible total e^{M + Lth + log sum e^Ls} lies more than kGap (log2) below the lower bound
    // LB(to) = max_j (Lth(to, j) + mu_j) of every output of the tile (centre taps), M the max of lv_ti over
    // the window, mu_j the min of lv_j over the tile: skipped mass < nt 2^-64 relative (as the per-warp skip)
    int nact = nt;
    if (nt <= kPMaxNT) {
        const int nxb = (nx + kPSegW - 1) / kPSegW, xb0 = x0 / kPSegW;
        const int parts = C::NT / nt, ti = threadIdx.x % nt, part = threadIdx.x / nt;
        float M = NEG_INF, mu = INFINITY, mnw = INFINITY;   // window max, tile min, window min of the finite lv
        if (part < parts) {
            const float4* sb = pst + (((int64_t)b * nt + ti) * ny) * nxb;
            const int ra = max(0, y0 - R), rb = min(ny - 1, y0 + C::TY - 1 + R);
            for (int y = ra + part; y <= rb; y += parts) {
                const bool own = y >= y0 && y < min(y_hi, y0 + C::TY);
                for (int xb = max(0, xb0 - 1); xb <= min(nxb - 1, xb0 + 1); ++xb) {
                    const float4 v = sb[(int64_t)y * nxb + xb];
                    M = fmaxf(M, v.y);
                    mnw = fminf(mnw, v.z);
                    if (own && xb == xb0) mu = fminf(mu, v.x);
                }
            }
        }
        sPM[threadIdx.x] = M;
        sPMu[threadIdx.x] = mu;
        sPMn[threadIdx.x] = mnw;
        __syncthreads();
        if (threadIdx.x < nt) {
            for (int pp = 1; pp < parts; ++pp) {
                M = fmaxf(M, sPM[pp * nt + threadIdx.x]);
                mu = fminf(mu, sPMu[pp * nt + threadIdx.x]);
                mnw = fminf(mnw, sPMn[pp * nt + threadIdx.x]);
            }
            sCM[threadIdx.x] = M;
            sCMu[threadIdx.x] = mu;
            sCMn[threadIdx.x] = mnw;
        }
        __syncthreads();
        if (wx < 4) {   // warp q: LB(to_q)
            const int to = 4 * qd + wx;
            float lbv = NEG_INF;
            if (to < nt)
                for (int j = lane; j < nt; j += 32) lbv = fmaxf(lbv, Lth[to * nt + j] + sCMu[j]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) lbv = fmaxf(lbv, __shfl_xor_sync(0xffffffffu, lbv, o));
            if (lane == 0) sLB[wx] = lbv;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int n = 0;
            for (int a = 0; a < nt; ++a) {
                const int t = chan0(a);
                const float Mt = sCM[t];
                bool act = false;
                if (Mt > NEG_INF && Mt == Mt)
                    for (int q = 0; q < 4; ++q) {
                        const int to = 4 * qd + q;
                        if (to < nt && !(Mt + Lth[to * nt + t] + LseS[to * nt + t] < sLB[q] - kGapNat)) act = true;
                    }
                if (act) sAct[n++] = t;
            }
            sNAct = n;
        }
        __syncthreads();
        nact = sNAct;
    }
    auto chan = [&](int a) { return nt <= kPMaxNT ? sAct[a] : chan0(a); };
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
        float* fb = sF0 + (((a - grp) / ngroups) & 1) * FBUF;   // this CTA's j-th channel -> buffer j & 1
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
    if (grp < nact) issue(grp);
    for (int a = grp; a < nact; a += ngroups) {
        cp_async_wait<0>();
        __syncthreads();   // channel a's copies visible; the previous channel's readers of sWh / sWl are done
        // path of the channel from the prologue's bounds (no per-element reductions): M >= the window's max,
        // mu <= the tile's min (fp32 rounded outward), so M - mu >= the true range
        double wmax = 0.0, Bd = 0.0;   // Bd: integer base (log2 units) of the exact path's staged values
        bool ffma = false, gridx = false;
        if (nt <= kPMaxNT) {
            const int tic = chan(a);
            const float Mf = sCM[tic], muf = sCMu[tic], mnf = sCMn[tic];
            ffma = a < ffma_max_a && isfinite(Mf) && isfinite(muf) && ((double)Mf - (double)muf <= kFfmaRangeP);
            wmax = (double)Mf;
            if (isfinite(Mf)) {
                Bd = floor((double)Mf * LOG2E) + 1.0;
                // staged values x - B in (-2^14, 0] and the table's |L2| < 2^15 on the 2^-8 grid: every sum of
                // the two (and minus an integer shift) is exact in fp32
                gridx = isfinite(mnf) && ((double)Mf - (double)mnf) * LOG2E < 16384.0;
            }
        }
        const float B = (float)Bd;
        if (ffma) {   // v~ = exp(lv - M + 40) from the fp64 potential, rounded once (zero mass / padding -> 0)
            for (int i = threadIdx.x; i < C::RAW; i += C::NT) {
                const int r = i / C::WIN_W, c = i - r * C::WIN_W;
                sWh[r * C::PITCH + c] = exp_pair(sRaw[i] - wmax + 40.0);
            }
        } else {      // the exact path: lv log2 e - B as a pair, hi on the 2^-8 grid (exact in fp32), lo the rest
            for (int i = threadIdx.x; i < C::RAW; i += C::NT) {
                const int r = i / C::WIN_W, c = i - r * C::WIN_W;
                const double v = sRaw[i];
                float hi = kSent, lo = 0.f;
                if (v > -1e300) {
                    const double x = v * LOG2E - Bd;
                    hi = (float)(rint(x * 256.0) / 256.0);
                    lo = (float)(x - (double)hi);
                }
                sWh[r * C::PITCH + c] = hi;
                sWl[r * C::PITCH + c] = lo;
            }
        }
        __syncthreads();   // sRaw free for the next channel, sWh / sWl complete
        if (a + ngroups < nact) issue(a + ngroups);
        const float* sFh = sF0 + (((a - grp) / ngroups) & 1) * FBUF;
        const float* sFl = sFh + C::FIL;
        const float* sRow = sFh + 2 * C::FIL;   // [S][4] max over each tap row of L2 (pruning bounds)
        const float* wh = sWh + wx * C::P;
        const float* wl = sWl + wx * C::P;
        const float4* fh4 = reinterpret_cast<const float4*>(sFh);
        const float4* fl4 = reinterpret_cast<const float4*>(sFl);
        const float4* rw4 = reinterpret_cast<const float4*>(sRow);

        if (counters != nullptr && threadIdx.x == 0) {
            atomicAdd(&counters[0], ffma ? 1ull : 0ull);
            atomicAdd(&counters[1], 1ull);
        }
        if (ffma) {
            // ---------------- factored path: S = sum_d Eq(d) v~(x - d), one FFMA per tap ----------------
            const int ti = chan(a);
            float lbf[4];
            floors(lbf);
            double Lt[4];
            bool reach = false;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int to = 4 * qd + q;
                int kk = ((to - ti) % nt + nt) % nt;
                if (2 * kk >= nt) kk -= nt;
                const double Th = 6.283185307179586476925286766559 * kk / nt;
                Lt[q] = -w3sq_eps * Th * Th;   // Lth(to, ti), the fp64 formula of tabulate_theta_kernel
                // largest possible term of the channel: exp(M + Lth) (Ls <= 0)
                if (to < nt && (float)((wmax + Lt[q]) * LOG2E) >= lbf[q]) reach = true;
            }
            if (!__any_sync(0xffffffffu, reach)) continue;   // warp-uniform
            const float4* eq4 = reinterpret_cast<const float4*>(Eq + ((int64_t)qd * nt + ti) * C::FIL);
            double accd[4][C::P];
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int p = 0; p < C::P; ++p) accd[q][p] = 0.0;
#pragma unroll 1
            for (int dy = 0; dy < C::S; ++dy) {
                const float4* rowp = reinterpret_cast<const float4*>(wh + (lane - dy + 2 * R) * C::PITCH);
                float r[C::RL];
#pragma unroll
                for (int j = 0; j < C::RL / 4; ++j) {
                    const float4 t = rowp[j];
                    r[4 * j + 0] = t.x; r[4 * j + 1] = t.y; r[4 * j + 2] = t.z; r[4 * j + 3] = t.w;
                }
                float rs[4][C::P];
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int p = 0; p < C::P; ++p) rs[q][p] = 0.f;
                {   // rolled tap loop, 4-wide sliding window of the staged row
                    const float* rowF = wh + (lane - dy + 2 * R) * C::PITCH;
                    float x0v = rowF[2 * R], x1v = rowF[2 * R + 1], x2v = rowF[2 * R + 2], x3v = rowF[2 * R + 3];
#pragma unroll 4
                    for (int dx = 0; dx < C::S; ++dx) {
                        const float4 w = __ldg(eq4 + dy * C::S + dx);
                        const float xs[4] = {x0v, x1v, x2v, x3v};
#pragma unroll
                        for (int p = 0; p < C::P; ++p) {
                            rs[0][p] = fmaf(w.x, xs[p], rs[0][p]);
                            rs[1][p] = fmaf(w.y, xs[p], rs[1][p]);
                            rs[2][p] = fmaf(w.z, xs[p], rs[2][p]);
                            rs[3][p] = fmaf(w.w, xs[p], rs[3][p]);
                        }
                        x3v = x2v; x2v = x1v; x1v = x0v;
                        const int nc = 2 * R - dx - 1;
                        x0v = nc >= 0 ? rowF[nc] : 0.f;
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int p = 0; p < C::P; ++p) accd[q][p] += (double)rs[q][p];
            }
            // fold: the channel's term is accd 2^G, G = (M - 80 + Lth) log2 e; into (m, sd) exactly up to one
            // fp64 rounding: frexp(accd) = mant 2^ex, c = mant 2^frac(G) in [0.5, 2), value = c 2^(ex + floor G)
            // 2^frac(G) per orientation: lane q evaluates it once, every lane reads it by shuffle
            double Fl = 1.0;
            {
                const int ql = lane & 3;
                const double Gl = (wmax - 80.0 + (ql == 0 ? Lt[0] : ql == 1 ? Lt[1] : ql == 2 ? Lt[2] : Lt[3])) * LOG2E;
                Fl = exp2_once(Gl - floor(Gl));
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double G = (wmax - 80.0 + Lt[q]) * LOG2E;
                const double Gi = floor(G);
                const double F = __shfl_sync(0xffffffffu, Fl, q);
#pragma unroll
                for (int p = 0; p < C::P; ++p) {
                    const double sa = accd[q][p];
                    if (!((vmask >> (4 * q + p)) & 1u) || !(sa > 0.0)) continue;
                    int ex;
                    const double mant = frexp_pos(sa, ex);
                    const double cv = mant * F;
                    const int e = ex + (int)Gi;
                    const float ef = (float)(e + 1);            // value < 2^(e + 1)
                    if (m[q][p] == NEG_INF) {
                        m[q][p] = ef;
                        sd[q][p] = ldexp_fast(cv, -1);
                    } else {
                        if (ef > m[q][p]) {
                            sd[q][p] = ldexp_fast(sd[q][p], (int)(m[q][p] - ef));
                            m[q][p] = ef;
                        }
                        sd[q][p] += ldexp_fast(cv, e - (int)m[q][p]);
                    }
                }
            }
            continue;
        }

        // channel bound of this warp: max of the window columns it reads + the channel's largest L2 (its
        // centre tap, Ls(0) = 0 >= Ls(d)); a channel below every output's floor is skipped
        float lb[4];
        floors(lb);
#pragma unroll
        for (int q = 0; q < 4; ++q) lb[q] -= B;   // staged values are relative to B
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
            {   // rolled tap loop, 4-wide sliding window of the staged row (instruction-cache footprint)
                const float* rowA = wh + (lane - dy + 2 * R) * C::PITCH;
                float x0v = rowA[2 * R], x1v = rowA[2 * R + 1], x2v = rowA[2 * R + 2], x3v = rowA[2 * R + 3];
#pragma unroll 4
                for (int dx = 0; dx < C::S; ++dx) {
                    const float4 w = fh4[dy * C::S + dx];
                    const float xs[4] = {x0v, x1v, x2v, x3v};
#pragma unroll
                    for (int p = 0; p < C::P; ++p) {
                        cm[0][p] = fmaxf(cm[0][p], xs[p] + w.x);
                        cm[1][p] = fmaxf(cm[1][p], xs[p] + w.y);
                        cm[2][p] = fmaxf(cm[2][p], xs[p] + w.z);
                        cm[3][p] = fmaxf(cm[3][p], xs[p] + w.w);
                    }
                    x3v = x2v; x2v = x1v; x1v = x0v;
                    const int nc = 2 * R - dx - 1;
                    x0v = nc >= 0 ? rowA[nc] : kSent;
                }
            }
        }
        // new integer shifts; exact power-of-two rescale of the running sums
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int p = 0; p < C::P; ++p) {
                if (!(cm[q][p] > -1e29f)) continue;   // only sentinel terms so far
                const float mn = (float)(floor((double)cm[q][p] + Bd) + 1.0);   // every term t - mn < 1 (absolute)
                if (m[q][p] == NEG_INF) {
                    m[q][p] = mn;
                } else if (mn > m[q][p]) {
                    sd[q][p] = ldexp_fast(sd[q][p], (int)(m[q][p] - mn));
                    m[q][p] = mn;
                }
            }
        floors(lb);
#pragma unroll
        for (int q = 0; q < 4; ++q) lb[q] -= B;
        // pass B: sum 2^(t - m) with exact exponents; row sums in fp32, the total in fp64.  A (row,
        // orientation) whose largest term is below 2^-kGap of every output of the warp is skipped.
#pragma unroll 1
        for (int dy = 0; dy < C::S; ++dy) {
            const float4* rowh = reinterpret_cast<const float4*>(wh + (lane - dy + 2 * R) * C::PITCH);
            const float4* rowl = reinterpret_cast<const float4*>(wl + (lane - dy + 2 * R) * C::PITCH);
            float rh[C::RL];
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
            // per orientation a ROLLED loop over the taps of the row with a 4-wide sliding window of the staged
            // pair (the unrolled S x 4 x P body overflowed the instruction cache: ncu no_instruction 7 / issue)
            const float* rowH = wh + (lane - dy + 2 * R) * C::PITCH;
            const float* rowL = wl + (lane - dy + 2 * R) * C::PITCH;
            const float* frh = reinterpret_cast<const float*>(fh4 + dy * C::S);   // [dx][q]
            const float* frl = reinterpret_cast<const float*>(fl4 + dy * C::S);
            // one orientation's row: exponent (hi + bb) - m + (lo + blo) relative to the base B.  gridx: hi and bb on
            // the 2^-8 grid within 2^15 -> hi + bb and (hi + bb) - m are exact in fp32 (4 FADD + 1 EX2 per term);
            // otherwise TwoSum(hi, bb) (10 FADD)
            auto row_q = [&](auto fast, int q, float mq0, float mq1, float mq2, float mq3, float& rs0, float& rs1,
                             float& rs2, float& rs3) {
                float h0 = rowH[2 * R], h1 = rowH[2 * R + 1], h2 = rowH[2 * R + 2], h3 = rowH[2 * R + 3];
                float l0 = rowL[2 * R], l1 = rowL[2 * R + 1], l2 = rowL[2 * R + 2], l3 = rowL[2 * R + 3];
                auto term = [](float av, float al, float bb, float blo, float mm) {
                    if constexpr (decltype(fast)::value) {
                        return ex2_approx(((av + bb) - mm) + (al + blo));
                    } else {
                        const float s1 = av + bb;                               // TwoSum(av, bb)
                        const float bv = s1 - av;
                        const float e1 = (av - (s1 - bv)) + (bb - bv);
                        return ex2_approx((s1 - mm) + (e1 + (al + blo)));       // s1 - m exact; sentinel -> 0
                    }
                };
#pragma unroll 4
                for (int dx = 0; dx < C::S; ++dx) {
                    const float bb = frh[4 * dx + q], blo = frl[4 * dx + q];
                    rs0 += term(h0, l0, bb, blo, mq0);
                    rs1 += term(h1, l1, bb, blo, mq1);
                    rs2 += term(h2, l2, bb, blo, mq2);
                    rs3 += term(h3, l3, bb, blo, mq3);
                    // window of tap dx + 1: staged columns 2R - dx - 1 .. 2R - dx + 2 (p = 0..3)
                    h3 = h2; h2 = h1; h1 = h0;
                    l3 = l2; l2 = l1; l1 = l0;
                    const int nc = 2 * R - dx - 1;
                    h0 = nc >= 0 ? rowH[nc] : kSent;
                    l0 = nc >= 0 ? rowL[nc] : 0.f;
                }
            };
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (!((live >> q) & 1u)) continue;
                // shifts relative to B (integers: exact); NEG_INF stays (sentinel terms underflow to 0)
                const float m0 = m[q][0] - B, m1 = m[q][1] - B, m2 = m[q][2] - B, m3 = m[q][3] - B;
                float rs0 = 0.f, rs1 = 0.f, rs2 = 0.f, rs3 = 0.f;
                if (gridx)
                    row_q(std::integral_constant<bool, true>(), q, m0, m1, m2, m3, rs0, rs1, rs2, rs3);
                else
                    row_q(std::integral_constant<bool, false>(), q, m0, m1, m2, m3, rs0, rs1, rs2, rs3);
                const float rsv[4] = {rs0, rs1, rs2, rs3};
#pragma unroll
                for (int p = 0; p < C::P; ++p)
                    if (m[q][p] != NEG_INF) sd[q][p] += (double)rsv[p];
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
                                      : ((double)m[q][p] + log2_once(sd[q][p])) * 0.69314718055994530941723212145818;
                const int64_t idx = (int64_t)b * N + ((int64_t)to * ny + gy) * nx + gx;
                if (ngroups > 1)
                    split_out[(int64_t)grp * gridDim.z * N + idx] = make_double2((double)m[q][p], sd[q][p]);
                else
                    err += apply_epilogue_precise(epi, idx, ly);
            }
        }
    }
    if (ngroups == 1 && epi.err_partial != nullptr) {
        const float t = block_sum<C::NT>(err, sRed);
        if (threadIdx.x == 0) epi.err_partial[((int64_t)b * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
    }
}

// theta_i split: combine the groups' (shift m, fp64 sum) per output exactly (2^(m_g - M) scalings), then the
// fp64 epilogue; one CTA per (tile, quad, field) with the main kernel's output mapping and error-partial slot
template <int R>
__global__ void __launch_bounds__(LsePCfg<R>::NT)
lsep_split_combine_kernel(const double2* __restrict__ part, int ngroups, int nx, int ny, int nt, int tiles_x, int y_lo,
                          int y_hi, EpiP epi) {
    using C = LsePCfg<R>;
    __shared__ float sRed[C::NT / 32];
    const int tile = blockIdx.x, qd = blockIdx.y, b = blockIdx.z;
    const int x0 = (tile % tiles_x) * C::TX, y0 = y_lo + (tile / tiles_x) * C::TY;
    const int64_t N = (int64_t)nx * ny * nt, GN = (int64_t)gridDim.z * N;
    const int lane = threadIdx.x & 31, wx = threadIdx.x >> 5;
    float err = 0.f;
    const int gy = y0 + lane;
    if (gy < y_hi) {
        for (int q = 0; q < 4; ++q) {
            const int to = 4 * qd + q;
            if (to >= nt) continue;
            for (int p = 0; p < C::P; ++p) {
                const int gx = x0 + wx * C::P + p;
                if (gx >= nx) continue;
                const int64_t idx = (int64_t)b * N + ((int64_t)to * ny + gy) * nx + gx;
                double M = -(double)INFINITY;
                for (int g = 0; g < ngroups; ++g) {
                    const double2 v = part[g * GN + idx];
                    if (v.y > 0.0) M = fmax(M, v.x);
                }
                double sum = 0.0;
                if (M > -(double)INFINITY)
                    for (int g = 0; g < ngroups; ++g) {
                        const double2 v = part[g * GN + idx];
                        if (v.y > 0.0) sum += ldexp_fast(v.y, (int)(v.x - M));
                    }
                const double ly = (M == -(double)INFINITY || !(sum > 0.0))
                                      ? -(double)INFINITY
                                      : (M + log2_once(sum)) * 0.69314718055994530941723212145818;
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
    const int nquad = (k->nt + 3) / 4;
    if (bpf) *bpf = tiles_x * tiles_y * nquad;
    {
        const int64_t segs = (int64_t)batch * k->nt * k->ny * ((k->nx + kPSegW - 1) / kPSegW);
        lsep_stats_kernel<<<(int)std::min<int64_t>((segs + 255) / 256, 148 * 16), 256, 0, s>>>(in, k->nx, k->ny, k->nt,
                                                                                             batch, k->pstats);
        count_launch();
    }
    // theta_i split over `groups` CTAs per (tile, quad) when the grid is small: the waves model of K3
    // (waves(g) / g; <= 8 groups, the scratch, ~16 CTAs per SM)
    static int slots = 0;
    if (slots == 0) {
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, conv_lse_precise_kernel<R>, C::NT, C::SMEM) !=
                cudaSuccess ||
            per_sm < 1)
            per_sm = 1;
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        slots = per_sm * nsm;
        cudaGetLastError();
    }
    const int base_ctas = tiles_x * tiles_y * nquad * batch;
    int gmax = k->nt < 8 ? k->nt : 8;
    const int gcap = (16 * 148 + base_ctas - 1) / base_ctas;
    if (gmax > gcap) gmax = gcap;
    const size_t per_group = (size_t)batch * k->N();
    if (k->psplit == nullptr || (size_t)gmax * per_group > k->psplit_n) gmax = (int)(k->psplit_n / std::max<size_t>(per_group, 1));
    if (gmax < 1) gmax = 1;
    double best = 1e30;
    for (int g = 1; g <= gmax; ++g) best = fmin(best, (double)(((int64_t)base_ctas * g + slots - 1) / slots) / g);
    int groups = 1;
    for (int g = 1; g <= gmax; ++g)   // the largest g within 5% of the best (c2: g 3 / 5 / 6 / 8 measured 1.62k / 1.69k / - / 1.55k it/s)
        if ((double)(((int64_t)base_ctas * g + slots - 1) / slots) / g <= 1.05 * best) groups = g;
    const char* fg = getenv("SE2_K4P_GROUPS");   // tuning / tests (read per launch)
    const int force_groups = fg ? atoi(fg) : 0;
    if (force_groups > 0) groups = force_groups < gmax ? force_groups : gmax;
    dim3 grid(tiles_x * tiles_y, nquad * groups, batch);
    // channels (in theta-distance order) that may take the factored path; SE2_K4P_EXACT: none (diagnostics)
    const int ffma_max_a = getenv("SE2_K4P_EXACT") ? 0 : (getenv("SE2_K4P_FFMA_A") ? atoi(getenv("SE2_K4P_FFMA_A")) : 1 << 20);
    conv_lse_precise_kernel<R><<<grid, C::NT, C::SMEM, s>>>(
        in, k->L2hi, k->L2lo, k->L2row, k->Eq, k->w3 * k->w3 / k->eps, k->nx, k->ny, k->nt, tiles_x, k->wlo(), k->whi(),
        epi, ffma_max_a, reinterpret_cast<unsigned long long*>(k->lse_counters + 12), k->pstats, k->Lth, k->LseS, groups,
        reinterpret_cast<double2*>(k->psplit));
    count_launch();
    if (groups > 1) {
        dim3 g2(tiles_x * tiles_y, nquad, batch);
        lsep_split_combine_kernel<R><<<g2, C::NT, 0, s>>>(reinterpret_cast<const double2*>(k->psplit), groups, k->nx, k->ny,
                                                          k->nt, tiles_x, k->wlo(), k->whi(), epi);
        count_launch();
    }
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
