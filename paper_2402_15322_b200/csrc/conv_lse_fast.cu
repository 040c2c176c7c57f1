// K3: SE(2) group convolution in the log domain -- theta-factored, shifted FFMA log-sum-exp with a
// gradient-tilted variant, an exact per-tap fallback and exact-bound channel pruning (reading R7;
// DESIGN.md "K3").
//
//   ly[to, x] = log sum_ti sum_d exp( Lth(to,ti) + Ls(to,ti,d) + lv[ti, x - d] )
//
// A stats pass fits, per (field, theta, 32 x 16 tile), the plane psi(h) = a + g.(h - c) (least
// squares, c = tile centre) and records min/max of lv and of the residual r = lv - psi.  Per CTA (a
// tile T, an output-orientation quad, one field) and per input orientation ti:
//   * prune   if  M + Lth + log sum_d e^{Ls} < LB - 30 for every to of the quad, where M bounds lv on
//             the window (T + halo) and LB(to) = max_j (Lth(to,j) + min_T lv_j) <= ly(to, x) on T
//             (centre taps); the skipped mass is < e^-30 of the output per channel;
//   * FFMA    if  M - min_T lv <= 100: v~ = exp(lv - m), m = min_T lv + 62, S = sum_d exp(Ls + 40) v~;
//   * tilted  if the residual range over the window R_hi - R_lo <= 100 (bounded from the 3 x 3 tile
//     FFMA    neighbourhood's planes and residuals): with T(d) = Ls(d) - g.d and c1 = max_d T(d),
//             v~ = exp(r - m), m = R_lo + 62, S = sum_d exp(T(d) - c1 + 40) v~, and the channel's
//             contribution is S exp(psi(x) + c1 - 40 + m + Lth) -- since lv(x-d) = psi(x) - g.d + r(x-d)
//             the steep part of the potential moves into the (per CTA and channel) tilted kernel;
//   * exact   otherwise: the two-pass per-tap log-sum-exp of K4 for this channel.
// In every FFMA variant each term within e^-25 of the channel's largest term is a normal fp32
// product, the sum cannot overflow and underflowed terms total < 961 e^-25 relative.
// The channel results are folded into each output's running (max, sum) in log2 units relative to a
// per-CTA reference, which keeps the fp32 magnitudes small.
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
    static constexpr int NSEG = kRowSegs;        // tap-row segments with their own bound (exact path)
    static constexpr int SEGW = (S + NSEG - 1) / NSEG;
    static constexpr int RMX = S * NSEG * 4;     // per tap-row segment: max over its dx of the L2 table (4 q)
    static constexpr int MAXNT = 128;
    // window x2, L2 filter x2, exp filter x2 (FFMA candidates decided on the staged window), row max x2
    static constexpr size_t SMEM = (size_t)(2 * WIN + 4 * FIL + 2 * RMX) * sizeof(float) + 64;
};
constexpr int kLseTileY = 32, kLseTileX = 16;
constexpr int kStat = 8;   // per tile: a, gx, gy, rmin, rmax, vmin, vmax, valid-plane flag

// Per (field, theta, tile): min/max of lv, least-squares plane psi = a + gx (x - cx) + gy (y - cy)
// about the tile centre (pixel units), and min/max of the residual lv - psi.  One 128-thread block per
// tile (4 values per thread; block reductions through shared memory).
constexpr int kStatT = 128;
__device__ __forceinline__ void stat_reduce3(float& a, float& b, float& c, bool is_min_max, float* sh) {
    // is_min_max: (a, b) = (min, max), c unused; else (a, b, c) summed.  Result in every thread.
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ta = __shfl_xor_sync(0xffffffffu, a, o), tb = __shfl_xor_sync(0xffffffffu, b, o);
        const float tc = __shfl_xor_sync(0xffffffffu, c, o);
        if (is_min_max) { a = fminf(a, ta); b = fmaxf(b, tb); } else { a += ta; b += tb; c += tc; }
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) { sh[w] = a; sh[4 + w] = b; sh[8 + w] = c; }
    __syncthreads();
    a = sh[0]; b = sh[4]; c = sh[8];
#pragma unroll
    for (int i = 1; i < kStatT / 32; ++i) {
        if (is_min_max) { a = fminf(a, sh[i]); b = fmaxf(b, sh[4 + i]); } else { a += sh[i]; b += sh[4 + i]; c += sh[8 + i]; }
    }
}

__global__ void __launch_bounds__(kStatT)
lse_stats_kernel(const float* __restrict__ in, int nx, int ny, int nt, int tiles_x, int tiles_y,
                 float* __restrict__ st) {
    __shared__ float sh[12];
    const int ntile = tiles_x * tiles_y;
    const int th = blockIdx.x / ntile, t = blockIdx.x % ntile;
    const int b = blockIdx.y;
    const int x0 = (t % tiles_x) * kLseTileX, y0 = (t / tiles_x) * kLseTileY;
    const int w = min(kLseTileX, nx - x0), h = min(kLseTileY, ny - y0);
    const float cx = x0 + 0.5f * (w - 1), cy = y0 + 0.5f * (h - 1);
    const float* src = in + ((int64_t)b * nt + th) * nx * ny;
    constexpr int PER = kLseTileY * kLseTileX / kStatT;
    float v[PER];
    float mn = INFINITY, mx = -INFINITY, dummy = 0.f;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int i = threadIdx.x + kStatT * k;
        const int yy = i / kLseTileX, xx = i % kLseTileX;
        v[k] = 0.f;
        if (yy < h && xx < w) {
            v[k] = src[(int64_t)(y0 + yy) * nx + x0 + xx];
            mn = fminf(mn, v[k]);
            mx = fmaxf(mx, v[k]);
        }
    }
    stat_reduce3(mn, mx, dummy, true, sh);
    const bool finite = (mn != -INFINITY) && (mx != INFINITY) && (mn == mn);
    float a = 0.f, gx = 0.f, gy = 0.f, rmn = mn, rmx = mx;
    if (finite) {   // uniform over the block
        // the valid cells form a w x h rectangle: the centred design is orthogonal
        float s0 = 0.f, sx = 0.f, sy = 0.f;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int i = threadIdx.x + kStatT * k;
            const int yy = i / kLseTileX, xx = i % kLseTileX;
            if (yy < h && xx < w) {
                const float d = v[k] - mn;      // shift for conditioning
                s0 += d;
                sx += d * ((float)(x0 + xx) - cx);
                sy += d * ((float)(y0 + yy) - cy);
            }
        }
        stat_reduce3(s0, sx, sy, false, sh);
        const float sxx = (float)h * (float)w * ((float)w * w - 1.f) / 12.f;
        const float syy = (float)w * (float)h * ((float)h * h - 1.f) / 12.f;
        a = mn + s0 / (float)(w * h);
        gx = sxx > 0.f ? sx / sxx : 0.f;
        gy = syy > 0.f ? sy / syy : 0.f;
        rmn = INFINITY;
        rmx = -INFINITY;
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int i = threadIdx.x + kStatT * k;
            const int yy = i / kLseTileX, xx = i % kLseTileX;
            if (yy < h && xx < w) {
                const float r = (v[k] - a) - (gx * ((float)(x0 + xx) - cx) + gy * ((float)(y0 + yy) - cy));
                rmn = fminf(rmn, r);
                rmx = fmaxf(rmx, r);
            }
        }
        stat_reduce3(rmn, rmx, dummy, true, sh);
    }
    if (threadIdx.x == 0) {
        float* o = st + (((int64_t)b * nt + th) * ntile + t) * kStat;
        o[0] = a; o[1] = gx; o[2] = gy; o[3] = rmn; o[4] = rmx; o[5] = mn; o[6] = mx;
        o[7] = finite ? 1.f : 0.f;
    }
}

// extreme values of (psi_j - psi_0) over the pixel rectangle [xa, xb] x [ya, yb] (an affine function)
__device__ __forceinline__ void plane_diff_range(float da, float dgx, float dgy, float cxj, float cyj, float cx0,
                                                 float cy0, float gx0, float gy0, float xa, float xb, float ya,
                                                 float yb, float& lo, float& hi) {
    // psi_j(p) - psi_0(p) = da + gxj (x - cxj) + gyj (y - cyj) - gx0 (x - cx0) - gy0 (y - cy0)
    //                     = const + dgx x + dgy y
    const float c = da - (dgx + gx0) * cxj - (dgy + gy0) * cyj + gx0 * cx0 + gy0 * cy0;
    const float v1 = c + dgx * xa + dgy * ya, v2 = c + dgx * xb + dgy * ya;
    const float v3 = c + dgx * xa + dgy * yb, v4 = c + dgx * xb + dgy * yb;
    lo = fminf(fminf(v1, v2), fminf(v3, v4));
    hi = fmaxf(fmaxf(v1, v2), fmaxf(v3, v4));
}

template <int R>
__global__ void __launch_bounds__(LseFCfg<R>::NT, 4)
conv_lse_fast_kernel(const float* __restrict__ in, const float* __restrict__ Eq, const float* __restrict__ Lq,
                     const float* __restrict__ LqRow,
                     const float* __restrict__ Lth, const float* __restrict__ LseS, const float* __restrict__ st,
                     int nx, int ny, int nt, int tiles_x, int tiles_y, int force_exact, Epilogue epi,
                     int* __restrict__ counters, int ngroups, float* __restrict__ split_out) {
    using C = LseFCfg<R>;
    extern __shared__ __align__(16) float smem[];
    float* sWin = smem;
    float* sFil = smem + 2 * C::WIN;
    float* sFilE = sFil + 2 * C::FIL;   // Eq copy of a candidate channel (path 3 / 5)
    float* sRmx = sFilE + 2 * C::FIL;
    float* sRed = sRmx + 2 * C::RMX;
    __shared__ float sMu[C::MAXNT], sM[C::MAXNT], sLB[4];
    __shared__ float sA[C::MAXNT], sGx[C::MAXNT], sGy[C::MAXNT], sShift[C::MAXNT];
    __shared__ float sCoef[C::MAXNT][4];
    __shared__ float sPart[C::NT / 32][4], sPartD[C::NT / 32][4], sWmax[C::NT / 32];
    __shared__ float sRhi[C::MAXNT];
    __shared__ int sList[C::MAXNT];
    __shared__ int sNAct, sNFast, sNTilt;
    __shared__ float sRef;

    const int tile = blockIdx.x;
    // theta_i split (small grids): blockIdx.y = qd * ngroups + group; the CTA handles the input
    // orientations ti with ti % ngroups == group and writes its partial log-sum to split_out
    const int qd = blockIdx.y / ngroups;
    const int grp = blockIdx.y - qd * ngroups;
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
    const float cx0 = x0 + 0.5f * (min(C::TX, nx - x0) - 1), cy0 = y0 + 0.5f * (min(C::TY, ny - y0) - 1);

    // ---- per-channel bounds from the tile statistics: 4 threads per channel share its 9 neighbour
    // tiles (independent loads in flight), then combine over the 4 lanes ----------------------------
    for (int base = 0; base < nt; base += C::NT / 4) {
        const int i = base + (threadIdx.x >> 2), part = threadIdx.x & 3;
        const bool valid = i < nt;
        float M = NEG_INF, rlo = INFINITY, rhi = -INFINITY, mu = 0.f, a0 = 0.f, gx0 = 0.f, gy0 = 0.f;
        int tok = 0;
        if (valid) {
            const float* s0 = st + (((int64_t)b * nt + i) * ntile + tile) * kStat;
            mu = s0[5];
            a0 = s0[0];
            gx0 = s0[1];
            gy0 = s0[2];
            tok = s0[7] > 0.5f ? 1 : 0;   // tilted bounds of the residual r = lv - psi_0 over the window
            for (int n = part; n < 9; n += 4) {
                const int yy = ty + n / 3 - 1, xx = tx + n % 3 - 1;
                if (yy < 0 || yy >= tiles_y || xx < 0 || xx >= tiles_x) continue;
                const float* sj = st + (((int64_t)b * nt + i) * ntile + yy * tiles_x + xx) * kStat;
                M = fmaxf(M, sj[6]);
                if (!tok) continue;
                if (!(sj[7] > 0.5f)) { tok = 0; continue; }
                const int xa = xx * C::TX, ya = yy * C::TY;
                const int xb = min(xa + C::TX, nx) - 1, yb = min(ya + C::TY, ny) - 1;
                const float cxj = xa + 0.5f * (xb - xa), cyj = ya + 0.5f * (yb - ya);
                float lo, hi;
                plane_diff_range(sj[0] - a0, sj[1] - gx0, sj[2] - gy0, cxj, cyj, cx0, cy0, gx0, gy0, (float)xa,
                                 (float)xb, (float)ya, (float)yb, lo, hi);
                rlo = fminf(rlo, sj[3] + lo);
                rhi = fmaxf(rhi, sj[4] + hi);
            }
        }
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
            M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
            rlo = fminf(rlo, __shfl_xor_sync(0xffffffffu, rlo, o));
            rhi = fmaxf(rhi, __shfl_xor_sync(0xffffffffu, rhi, o));
            tok = min(tok, __shfl_xor_sync(0xffffffffu, tok, o));
        }
        if (valid && part == 0) {
            sMu[i] = mu;
            sM[i] = M;
            sA[i] = a0;
            sGx[i] = gx0;
            sGy[i] = gy0;
            sShift[i] = tok ? ((rhi - rlo <= kFastRange) ? rlo : NAN) : NAN;   // R_lo when a tilt may be valid
            sRhi[i] = rhi;
        }
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
    // status per channel: 0 skip, 1 FFMA, 2 exact, 3 tilt candidate, 5 FFMA candidate.  The bound M
    // is the max over the 3 x 3 tile neighbourhood; candidates (3, 5) are decided on the exact max of
    // the staged window (M - mu <= kFastRange with the window's own max), a tilt candidate then tries
    // the tilted kernel, a plain candidate falls back to the exact path.
    for (int i = threadIdx.x; i < nt; i += C::NT) {
        const float M = sM[i], mu = sMu[i];
        int stt = 0;
        if (M != NEG_INF) {
            bool active = false;
            for (int q = 0; q < 4; ++q) {
                const int to = 4 * qd + q;
                if (to >= nt) continue;
                const float ub = M + Lth[to * nt + i] + LseS[to * nt + i];
                if (!(ub < sLB[q] - kPruneGap)) active = true;
            }
            if (active) {
                if ((force_exact & 3) == 1) stt = 2;
                else if (mu != NEG_INF && (M - mu) <= kFastRange) stt = 1;
                else if ((force_exact & 3) != 2 && sShift[i] == sShift[i]) stt = 3;   // not NaN: tilt valid
                else if (mu != NEG_INF) stt = 5;
                else stt = 2;
            }
        }
        sList[i] = stt;
        if (stt == 1 || stt == 3 || stt == 5)
            for (int q = 0; q < 4; ++q) {
                const int to = 4 * qd + q;
                const float lt = (to < nt) ? Lth[to * nt + i] : 0.f;
                // (m - kEsShift + Lth - ref) log2(e), m = mu + kShiftAbove; (mu - ref) first: both large
                sCoef[i][q] = (((mu - ref) + (kShiftAbove - kEsShift)) + lt) * kLog2e;
            }
    }
    __syncthreads();
    {   // compact the active list (entry = channel | (path << 16)); active channels are dealt
        // round-robin over the split groups by their rank among the actives (ballot prefix counts)
        __shared__ int sWc[C::NT / 32], sWf[C::NT / 32], sWt[C::NT / 32];
        const int i = threadIdx.x;
        const int stt = (i < nt) ? sList[i] : 0;
        const bool act = stt != 0;
        const unsigned bal = __ballot_sync(0xffffffffu, act);
        if (lane == 0) sWc[wx] = __popc(bal);
        __syncthreads();
        int off = 0;
        for (int w2 = 0; w2 < wx; ++w2) off += sWc[w2];
        const int rank = off + __popc(bal & ((1u << lane) - 1u));
        const bool mine = act && (rank % ngroups) == grp;
        const unsigned bm = __ballot_sync(0xffffffffu, mine);
        const unsigned bf = __ballot_sync(0xffffffffu, mine && (stt == 1 || stt == 3));
        const unsigned bt = __ballot_sync(0xffffffffu, mine && stt == 3);
        __syncthreads();   // every sList[i] / sWc read before they are overwritten
        if (mine) sList[rank / ngroups] = i | (stt << 16);
        if (lane == 0) {
            sWc[wx] = __popc(bm);
            sWf[wx] = __popc(bf);
            sWt[wx] = __popc(bt);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int n = 0, nf = 0, ntl = 0;
            for (int w2 = 0; w2 < C::NT / 32; ++w2) {
                n += sWc[w2];
                nf += sWf[w2];
                ntl += sWt[w2];
            }
            sNAct = n;
            sNFast = nf;
            sNTilt = ntl;
        }
    }
    __syncthreads();
    const int nact = sNAct;
    if (counters != nullptr && threadIdx.x == 0) {
        atomicAdd(&counters[0], nact);
        atomicAdd(&counters[1], sNFast);
        atomicAdd(&counters[2], grp == 0 ? nt : 0);   // visited pairs: once per (tile, quad)
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
        if (path == 3 || path == 5) {
            const float* esrc = Eq + ((int64_t)qd * nt + ti) * C::FIL;
            float* de = sFilE + buf * C::FIL;
            for (int i = threadIdx.x; i < C::FIL / 4; i += C::NT) cp_async16(de + 4 * i, esrc + 4 * i);
        }
        const float* rsrc = LqRow + ((int64_t)qd * nt + ti) * C::RMX;
        float* dr = sRmx + buf * C::RMX;
        for (int i = threadIdx.x; i < C::RMX / 4; i += C::NT) cp_async16(dr + 4 * i, rsrc + 4 * i);
        cp_async_commit();
    };

    float Macc[4][C::P], Sacc[4][C::P];
    unsigned vmask = 0;   // outputs of this thread inside the grid (bit 4q + p)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int p = 0; p < C::P; ++p)
            if (4 * qd + q < nt && y0 + lane < ny && x0 + wx * C::P + p < nx) vmask |= 1u << (4 * q + p);
    unsigned rows_live = 0, rows_seen = 0;
    // hinted shifts: verified here (whole-CTA redo) when unsplit; in a theta_i split the partial sums
    // cannot be judged alone, so the combine kernel verifies the total and recomputes bad outputs
    const bool have_hint = (epi.hint_in != nullptr);
    for (int attempt = have_hint ? 0 : 1; attempt < 2; ++attempt) {
    const bool use_hint = (attempt == 0);
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int p = 0; p < C::P; ++p) {
            Macc[q][p] = LOW;
            Sacc[q][p] = 0.f;
            if (use_hint) {
                // shift = previous output + 20 nats, relative to ref, log2 units
                const int to = 4 * qd + q, gy = y0 + lane, gx = x0 + wx * C::P + p;
                if (to < nt && gy < ny && gx < nx) {
                    const float h = epi.hint_in[(int64_t)b * N + ((int64_t)to * ny + gy) * nx + gx] +
                                    ((force_exact & 4) ? kDebugHintBias : 0.f);   // diagnostics: wrong hints
                    if (h > -1e30f && h < 1e30f) Macc[q][p] = ((h - ref) + kHintAbove) * kLog2e;
                }
            }
        }

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
        float* dw = sWin + buf * C::WIN;
        float* df = sFil + buf * C::FIL;
        // transform the elements this thread staged (its own cp.async copies are complete)
        int epath = path;   // effective path of this channel (a candidate may end FFMA, tilted or exact)
        if (path == 3 || path == 5) {
            // exact max of the staged window: the elements this thread staged, then the block
            float wm = NEG_INF;
            for (int i = threadIdx.x; i < C::WIN_H * C::WIN_W; i += C::NT) {
                const int r = i / C::WIN_W, c = i - r * C::WIN_W;
                wm = fmaxf(wm, dw[r * C::PITCH + c]);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));
            if (lane == 0) sWmax[wx] = wm;
            __syncthreads();
            wm = sWmax[0];
#pragma unroll
            for (int w2 = 1; w2 < C::NT / 32; ++w2) wm = fmaxf(wm, sWmax[w2]);
            if (wm - sMu[ti] <= kFastRange) {
                epath = 1;
                df = sFilE + buf * C::FIL;
                if (path == 5 && counters != nullptr && threadIdx.x == 0) atomicAdd(&counters[1], 1);
            } else if (path == 5) {
                epath = 2;
            }
        }
        if (epath == 3) {
            // tilted candidate: T2(d) = (Ls(d) - g.d) log2 e from the staged L table.  c1 = max_d T2 over
            // the box; c1D = max over the taps valid for every output of the tile (a sub-box, clipped by
            // the zero padding).  The shift m = R_lo + 62 - dc, dc = max_q (c1 - c1D) (natural), is valid
            // when R_hi - R_lo + dc <= 100 (K3); otherwise the channel takes the exact path.
            const float gx = sGx[ti], gy = sGy[ti];
            const int xt1 = min(x0 + C::TX, nx) - 1, yt1 = min(y0 + C::TY, ny) - 1;
            const int dxlo = max(-R, xt1 - (nx - 1)), dxhi = min(R, x0);
            const int dylo = max(-R, yt1 - (ny - 1)), dyhi = min(R, y0);
            float lt2[4], pmax[4], pmaxD[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int to = 4 * qd + q;
                lt2[q] = (to < nt ? Lth[to * nt + ti] : 0.f) * kLog2e;
                pmax[q] = -INFINITY;
                pmaxD[q] = -INFINITY;
            }
            // the filter block was copied in 16-byte chunks (one tap's four q values) by thread
            // (chunk % NT): read the same chunks (own cp.async writes are visible)
            const float4* df4 = reinterpret_cast<const float4*>(df);
            for (int i = threadIdx.x; i < C::FIL / 4; i += C::NT) {
                const int dyi = i / C::S, dxi = i - dyi * C::S;
                const float gd = (gx * (float)(dxi - R) + gy * (float)(dyi - R)) * kLog2e;
                const float4 v = df4[i];
                const float t0 = (v.x - lt2[0]) - gd, t1 = (v.y - lt2[1]) - gd;
                const float t2 = (v.z - lt2[2]) - gd, t3 = (v.w - lt2[3]) - gd;
                pmax[0] = fmaxf(pmax[0], t0); pmax[1] = fmaxf(pmax[1], t1);
                pmax[2] = fmaxf(pmax[2], t2); pmax[3] = fmaxf(pmax[3], t3);
                if (dxi - R >= dxlo && dxi - R <= dxhi && dyi - R >= dylo && dyi - R <= dyhi) {
                    pmaxD[0] = fmaxf(pmaxD[0], t0); pmaxD[1] = fmaxf(pmaxD[1], t1);
                    pmaxD[2] = fmaxf(pmaxD[2], t2); pmaxD[3] = fmaxf(pmaxD[3], t3);
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                float v = pmax[q], u = pmaxD[q];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
                    u = fmaxf(u, __shfl_xor_sync(0xffffffffu, u, o));
                }
                if (lane == 0) { sPart[wx][q] = v; sPartD[wx][q] = u; }
            }
            __syncthreads();
            float c1[4], dc = 0.f;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                c1[q] = sPart[0][q];
                float cD = sPartD[0][q];
#pragma unroll
                for (int w2 = 1; w2 < C::NT / 32; ++w2) {
                    c1[q] = fmaxf(c1[q], sPart[w2][q]);
                    cD = fmaxf(cD, sPartD[w2][q]);
                }
                dc = fmaxf(dc, (c1[q] - cD) * kLn2);        // -inf cD (empty sub-box) -> +inf
            }
            const float rlo = sShift[ti], rhi = sRhi[ti];
            if ((rhi - rlo) + dc <= kFastRange) {
                const float a0 = sA[ti];
                const float m = rlo + kShiftAbove - dc;
                for (int i = threadIdx.x; i < C::WIN_H * C::WIN_W; i += C::NT) {
                    int r = i / C::WIN_W, c = i - r * C::WIN_W;
                    const float hx = (float)(x0 - R + c) - cx0, hy = (float)(y0 - R + r) - cy0;
                    float v = dw[r * C::PITCH + c];
                    dw[r * C::PITCH + c] = ex2_approx(((v - a0) - (gx * hx + gy * hy) - m) * kLog2e);
                }
                const float sh = kEsShift * kLog2e;
                float4* dfw = reinterpret_cast<float4*>(df);
                for (int i = threadIdx.x; i < C::FIL / 4; i += C::NT) {
                    const int dyi = i / C::S, dxi = i - dyi * C::S;
                    const float gd = (gx * (float)(dxi - R) + gy * (float)(dyi - R)) * kLog2e;
                    float4 v = dfw[i];
                    v.x = ex2_approx(((v.x - lt2[0]) - gd) - c1[0] + sh);
                    v.y = ex2_approx(((v.y - lt2[1]) - gd) - c1[1] + sh);
                    v.z = ex2_approx(((v.z - lt2[2]) - gd) - c1[2] + sh);
                    v.w = ex2_approx(((v.w - lt2[3]) - gd) - c1[3] + sh);
                    dfw[i] = v;
                }
                if (threadIdx.x < 4) {
                    const int q = threadIdx.x, to = 4 * qd + q;
                    const float lt = (to < nt) ? Lth[to * nt + ti] : 0.f;
                    const float c1q = (q == 0) ? c1[0] : (q == 1) ? c1[1] : (q == 2) ? c1[2] : c1[3];
                    // contribution = S exp(psi(x) + c1 - 40 + m + Lth): relative to ref, natural -> log2
                    sCoef[ti][q] = (((a0 - ref) + (m - kEsShift) + lt) * kLog2e) + c1q;
                }
                if (counters != nullptr && threadIdx.x == 0) atomicAdd(&counters[3], 1);
            } else {
                epath = 2;
                if (counters != nullptr && threadIdx.x == 0) atomicAdd(&counters[1], -1);  // not an FFMA pair
            }
        }
        if (epath == 1 || epath == 2) {
            const float shift = (epath == 1) ? (sMu[ti] + kShiftAbove) : ref;   // FFMA: m = mu + 62
            for (int i = threadIdx.x; i < C::WIN_H * C::WIN_W; i += C::NT) {
                int r = i / C::WIN_W, c = i - r * C::WIN_W;
                float v = dw[r * C::PITCH + c];
                float u = (v - shift) * kLog2e;
                dw[r * C::PITCH + c] = (epath == 1) ? ex2_approx(u) : u;
            }
        }
        __syncthreads();
        const float* win = dw + wx * C::P;
        const float4* fil = reinterpret_cast<const float4*>(df);
        float acc[4][C::P];
        if (epath != 2) {
            // ---------------- FFMA paths: S = sum_d Ktilde(d) * v~(x - d)
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
            // per-output tilt psi(x) - a (log2 units); zero on the untilted path
            const float gx2 = (epath == 3) ? sGx[ti] * kLog2e : 0.f, gy2 = (epath == 3) ? sGy[ti] * kLog2e : 0.f;
            const float ty2 = gy2 * ((float)(y0 + lane) - cy0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float cf = sCoef[ti][q] + ty2;
#pragma unroll
                for (int p = 0; p < C::P; ++p) {
                    const float tilt = gx2 * ((float)(x0 + wx * C::P + p) - cx0);
                    const float t = lg2_norm(acc[q][p]) + (cf + tilt);     // lg2(0) = -inf: no contribution
                    const float mx = fmaxf(Macc[q][p], t);
                    Sacc[q][p] = Sacc[q][p] * ex2_approx(Macc[q][p] - mx) + ex2_approx(t - mx);
                    Macc[q][p] = mx;
                }
            }
        } else {
            // ---------------- exact path: two passes over the taps of this channel (pass A, the
            // per-output maximum, is skipped when the output shift comes from a verified hint).
            // Row pruning: the row dy of taps is skipped by the whole warp when, for every output of
            // every lane, its largest possible term  max_dx L2(dy, .) + max(row segment of lv)  is below
            // thr = (lower bound of the output) - gap, in pass B: the running max (<= ly) - kRowGap, or
            // with a hint the verified floor h - kHintDrop - kRowGap; the skipped terms then total
            // < S^2 nt e^-25 of the output.  (Pruning pass A as well costs 87 registers; pass A only
            // runs without a hint.)
            const float4* rmx = reinterpret_cast<const float4*>(sRmx + buf * C::RMX);
            float thr[4];
            auto set_thr = [&](float drop2) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    float t = INFINITY;
#pragma unroll
                    for (int p = 0; p < C::P; ++p)
                        if (vmask & (1u << (4 * q + p))) t = fminf(t, Macc[q][p]);
                    thr[q] = t - drop2;
                }
            };
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int p = 0; p < C::P; ++p) acc[q][p] = Macc[q][p];
#pragma unroll 1
            for (int dy = 0; dy < (use_hint ? 0 : C::S); ++dy) {
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
            if (!use_hint) {
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int p = 0; p < C::P; ++p) {
                        const float mn = acc[q][p];      // >= Macc (LOW sentinel when nothing finite yet)
                        Sacc[q][p] *= ex2_approx(Macc[q][p] - mn);
                        Macc[q][p] = mn;
                    }
            }
            set_thr((use_hint ? (kHintAbove + kHintDrop + kRowGap) : kRowGap) * kLog2e);
#pragma unroll 1
            for (int dy = 0; dy < C::S; ++dy) {
                const float4* rowp = reinterpret_cast<const float4*>(win + (lane - dy + 2 * R) * C::PITCH);
                float r[C::RL];
#pragma unroll
                for (int j = 0; j < C::RL / 4; ++j) {
                    float4 t = rowp[j];
                    r[4 * j + 0] = t.x; r[4 * j + 1] = t.y; r[4 * j + 2] = t.z; r[4 * j + 3] = t.w;
                }
                // per segment k (taps dx in [k SEGW, (k+1) SEGW)) and output orientation q: bound = max_dx
                // L2_q + max of the r entries those taps read (indices 2R - dx + p); warp vote per (k, q),
                // so a live segment only spends exps on the orientations that can reach their outputs
                unsigned segq = 0;   // bit 4 k + q
#pragma unroll
                for (int k = 0; k < C::NSEG; ++k) {
                    const int dxlo = k * C::SEGW;
                    const int dxhi = (dxlo + C::SEGW - 1 < C::S - 1) ? dxlo + C::SEGW - 1 : C::S - 1;
                    float sm = -INFINITY;
                    if (dxlo <= dxhi) {
#pragma unroll
                        for (int j = 2 * R - dxhi; j <= 2 * R - dxlo + C::P - 1; ++j) sm = fmaxf(sm, r[j]);
                    }
                    const float4 m4 = rmx[dy * C::NSEG + k];
                    const unsigned l = (__any_sync(0xffffffffu, sm + m4.x >= thr[0]) ? 1u : 0u) |
                                       (__any_sync(0xffffffffu, sm + m4.y >= thr[1]) ? 2u : 0u) |
                                       (__any_sync(0xffffffffu, sm + m4.z >= thr[2]) ? 4u : 0u) |
                                       (__any_sync(0xffffffffu, sm + m4.w >= thr[3]) ? 8u : 0u);
                    segq |= l << (4 * k);
                    rows_seen += 4;
                    rows_live += __popc(l);
                }
                if (!segq) continue;
                const float* frow = reinterpret_cast<const float*>(fil + dy * C::S);   // [dx][q]
#pragma unroll
                for (int k = 0; k < C::NSEG; ++k) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        if (!((segq >> (4 * k + q)) & 1u)) continue;
#pragma unroll
                        for (int dx = k * C::SEGW; dx < (k + 1) * C::SEGW && dx < C::S; ++dx) {
                            const float w = frow[4 * dx + q];
#pragma unroll
                            for (int p = 0; p < C::P; ++p)
                                Sacc[q][p] += ex2_approx((r[p - dx + 2 * R] + w) - Macc[q][p]);
                        }
                    }
                }
            }
        }
        __syncthreads();
    }
    if (!use_hint || ngroups > 1) break;
    // verify the hinted shifts: every stored output must have a finite, non-overflowing sum and lie at
    // least at h - kHintDrop (sum >= e^-(kHintAbove + kHintDrop) relative to the shift h + kHintAbove: the
    // floor the row pruning assumed); otherwise the CTA redoes two-pass
    bool bad = false;
    const float hint_floor = exp2f(-(kHintAbove + kHintDrop) * kLog2e);
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int p = 0; p < C::P; ++p) {
            const int to = 4 * qd + q, gyy = y0 + lane, gxx = x0 + wx * C::P + p;
            if (to < nt && gyy < ny && gxx < nx) {
                const float sv = Sacc[q][p];
                if (!(sv >= hint_floor && sv <= 1.2676506e30f)) bad = true;   // [e^-(above+drop), 2^100]
            }
        }
    if (!__syncthreads_or(bad)) break;
    if (counters != nullptr && threadIdx.x == 0) atomicAdd(&counters[4], 1);   // hint redo
    }

    if (counters != nullptr && lane == 0 && rows_seen > 0) {
        unsigned long long* rc = reinterpret_cast<unsigned long long*>(counters + 8);
        atomicAdd(&rc[0], (unsigned long long)rows_live);
        atomicAdd(&rc[1], (unsigned long long)rows_seen);
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
                    if (ngroups > 1)
                        split_out[(int64_t)grp * gridDim.z * N + idx] = ly;   // partial: combined later
                    else
                        err += apply_epilogue<true>(epi, idx, gx, gy, ly);
                }
            }
        }
    }
    if (ngroups == 1 && epi.err_partial != nullptr) {
        float t = block_sum<C::NT>(err, sRed);
        if (threadIdx.x == 0) {   // error partials: 4 slots per (field, quad, tile), the split combine fills one per q
            float* o = epi.err_partial + (((int64_t)b * gridDim.y + qd) * gridDim.x + tile) * 4;
            o[0] = t;
            o[1] = 0.f;
            o[2] = 0.f;
            o[3] = 0.f;
        }
    }
}

// exact log-sum-exp of one output over every input orientation and tap (two passes, the definition),
// computed by the whole warp (taps dealt over the lanes, warp max / sum): the combine kernel's fallback
// when a hinted shift failed (rare; correct always).  Every lane must call it with the same output.
__device__ __noinline__ float exact_lse_point_warp(const float* __restrict__ vin, const float* __restrict__ Lq, int nx,
                                                   int ny, int nt, int R, int to, int y, int x, int lane) {
    const int S = 2 * R + 1, qd = to >> 2, q = to & 3;
    const int total = nt * S * S;
    float m = -INFINITY;
    for (int t = lane; t < total; t += 32) {
        const int ti = t / (S * S), d = t - ti * S * S, dy = d / S - R, dx = d % S - R;
        const int hy = y - dy, hx = x - dx;
        if (hy < 0 || hy >= ny || hx < 0 || hx >= nx) continue;
        m = fmaxf(m, vin[((int64_t)ti * ny + hy) * nx + hx] * kLog2e +
                         Lq[((((int64_t)qd * nt + ti) * S * S) + d) * 4 + q]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (m == -INFINITY) return -INFINITY;
    float sacc = 0.f;
    for (int t = lane; t < total; t += 32) {
        const int ti = t / (S * S), d = t - ti * S * S, dy = d / S - R, dx = d % S - R;
        const int hy = y - dy, hx = x - dx;
        if (hy < 0 || hy >= ny || hx < 0 || hx >= nx) continue;
        sacc += ex2_approx(vin[((int64_t)ti * ny + hy) * nx + hx] * kLog2e +
                           Lq[((((int64_t)qd * nt + ti) * S * S) + d) * 4 + q] - m);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
    return (m + log2f(sacc)) * kLn2;
}

// Combine the theta_i-group partials of a split launch: ly = LSE_g ly_g, then the fused epilogue.
// One CTA per (tile, quad, field) as in the main kernel (so the error partials keep the unsplit
// layout), but kCombT threads, each with a few outputs (x fastest: coalesced partial reads).
constexpr int kCombT = 256;
template <int R>
__global__ void __launch_bounds__(kCombT)
lse_split_combine_kernel(const float* __restrict__ part, int ngroups, int nx, int ny, int nt, int tiles_x,
                         Epilogue epi, const float* __restrict__ in, const float* __restrict__ Lq,
                         int* __restrict__ counters, float hint_bias) {
    // one CTA per (tile, output orientation, field): 4x the CTAs of the main kernel's (tile, quad) grid
    using C = LseFCfg<R>;
    __shared__ float sRed[kCombT / 32];
    const int tile = blockIdx.x, to = blockIdx.y, b = blockIdx.z;
    const int qd = to >> 2, q = to & 3;
    const int x0 = (tile % tiles_x) * C::TX, y0 = (tile / tiles_x) * C::TY;
    const int64_t N = (int64_t)nx * ny * nt;
    const int64_t GN = (int64_t)gridDim.z * N;
    const int lane = threadIdx.x & 31;
    constexpr int NOUT = C::TY * C::TX;   // outputs of the (tile, orientation) block
    float err = 0.f;
    for (int o = threadIdx.x; o < NOUT; o += kCombT) {   // same trip count for every lane
        const int gy = y0 + o / C::TX, gx = x0 + o % C::TX;
        const bool ok = to < nt && gy < ny && gx < nx;
        const int64_t idx = ok ? (int64_t)b * N + ((int64_t)to * ny + gy) * nx + gx : 0;
        float ly = -INFINITY;
        bool bad = false;
        if (ok) {
            float m = -INFINITY;
            for (int g = 0; g < ngroups; ++g) m = fmaxf(m, part[g * GN + idx]);
            ly = m;
            if (m != -INFINITY) {
                float s = 0.f;
                for (int g = 0; g < ngroups; ++g) s += expf(part[g * GN + idx] - m);
                ly = m + logf(s);
            }
            if (epi.hint_in != nullptr) {
                // the partials used shift = hint + kHintAbove and rows pruned against the floor
                // h - kHintDrop: valid iff no overflow (finite) and the total reached that floor
                const float h = epi.hint_in[idx] + hint_bias;
                bad = !(ly < 1e30f && ly >= h - kHintDrop);
            }
        }
        unsigned mask = __ballot_sync(0xffffffffu, bad);
        while (mask) {   // warp-cooperative exact recomputation of each failed output
            const int src = __ffs(mask) - 1;
            mask &= mask - 1;
            const int yy = __shfl_sync(0xffffffffu, gy, src);
            const int xx = __shfl_sync(0xffffffffu, gx, src);
            const float v = exact_lse_point_warp(in + (int64_t)b * N, Lq, nx, ny, nt, R, to, yy, xx, lane);
            if (lane == src) {
                ly = v;
                if (counters != nullptr) atomicAdd(&counters[4], 1);
            }
        }
        if (ok) err += apply_epilogue<true>(epi, idx, gx, gy, ly);
    }
    if (epi.err_partial != nullptr) {
        float t = block_sum<kCombT>(err, sRed);
        if (threadIdx.x == 0) {
            const int ntile = gridDim.x, nquad = (gridDim.y + 3) / 4;
            epi.err_partial[(((int64_t)b * nquad + qd) * ntile + tile) * 4 + q] = t;
        }
    }
}

template <int R>
static cudaError_t launch_lsef_r(const se2_kernel_s* k, const float* in, int batch, const Epilogue& epi,
                                 cudaStream_t s, int* bpf, float* stats, int force_exact, int* counters,
                                 float* split_scratch, size_t split_floats) {
    using C = LseFCfg<R>;
    const int tiles_x = (k->nx + C::TX - 1) / C::TX;
    const int tiles_y = (k->ny + C::TY - 1) / C::TY;
    const int ntile = tiles_x * tiles_y;
    {
        dim3 g(k->nt * ntile, batch);
        lse_stats_kernel<<<g, kStatT, 0, s>>>(in, k->nx, k->ny, k->nt, tiles_x, tiles_y, stats);
        count_launch();
    }
    cudaError_t e = cudaFuncSetAttribute(conv_lse_fast_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::SMEM);
    if (e != cudaSuccess) return e;
    const int nquad = (k->nt + 3) / 4;
    // split the input orientations over `groups` CTAs per (tile, quad), then combine.  The per-channel
    // loop of one CTA is latency-bound and only a few CTAs fit per SM, so the grid is sized in waves:
    // waves(g) / g = ceil(base g / slots) / g models the time of the busiest SM (per-CTA work ~ 1/g); up to
    // 8 groups / the scratch / ~16 CTAs per SM.  Measured sweep (tools/sweep_groups.sh): c1 best at 5
    // (6.6k it/s vs 6.3k at 8), c2 at 7-8 (4.68k vs 4.40k at 3), c3 at 3-4 (341-345 vs 299 unsplit).
    const int base_ctas = ntile * nquad * batch;
    static int slots = 0;
    if (slots == 0) {
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, conv_lse_fast_kernel<R>, C::NT, C::SMEM) != cudaSuccess ||
            per_sm < 1)
            per_sm = 1;
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        slots = per_sm * nsm;
        cudaGetLastError();
    }
    int gmax = k->nt < 8 ? k->nt : 8;
    const int gcap = (16 * 148 + base_ctas - 1) / base_ctas;   // no more than ~16 CTAs per SM in total
    if (gmax > gcap) gmax = gcap;
    if ((size_t)gmax * batch * k->N() > split_floats) gmax = (int)(split_floats / ((size_t)batch * k->N()));
    if (gmax < 1 || (force_exact & 8)) gmax = 1;   // 8: diagnostics, no split
    double best = 1e30;
    for (int g = 1; g <= gmax; ++g)
        best = fmin(best, (double)(((int64_t)base_ctas * g + slots - 1) / slots) / g);
    int groups = 1;   // the largest g within 13% of the best (small CTAs also balance uneven channel work)
    for (int g = 1; g <= gmax; ++g)
        if ((double)(((int64_t)base_ctas * g + slots - 1) / slots) / g <= 1.13 * best) groups = g;
    static const int force_groups = getenv("SE2_K3_GROUPS") ? atoi(getenv("SE2_K3_GROUPS")) : 0;   // tuning
    if (force_groups > 0) groups = force_groups < gmax ? force_groups : gmax;
    if (bpf) *bpf = ntile * nquad * 4;
    dim3 grid(ntile, nquad * groups, batch);
    conv_lse_fast_kernel<R><<<grid, C::NT, C::SMEM, s>>>(in, k->Eq, k->Lq, k->LqRow, k->Lth, k->LseS, stats, k->nx, k->ny,
                                                          k->nt, tiles_x, tiles_y, force_exact, epi, counters,
                                                          groups, split_scratch);
    count_launch();
    if (groups > 1) {
        dim3 g2(ntile, nquad * 4, batch);   // one CTA per (tile, output orientation); slots of padding
        lse_split_combine_kernel<R><<<g2, kCombT, 0, s>>>(split_scratch, groups, k->nx, k->ny, k->nt, tiles_x, epi, in,
                                                         k->Lq, counters, (force_exact & 4) ? kDebugHintBias : 0.f);
        count_launch();
    }
    return cudaGetLastError();
}

size_t lse_fast_stats_floats(const se2_kernel_s* k, int batch) {
    const int tiles_x = (k->nx + kLseTileX - 1) / kLseTileX;
    const int tiles_y = (k->ny + kLseTileY - 1) / kLseTileY;
    return (size_t)batch * k->nt * tiles_x * tiles_y * kStat;
}

int conv_blocks_per_field_lse_fast(const se2_kernel_s* k) {
    const int tiles_x = (k->nx + kLseTileX - 1) / kLseTileX;
    const int tiles_y = (k->ny + kLseTileY - 1) / kLseTileY;
    return tiles_x * tiles_y * ((k->nt + 3) / 4) * 4;   // 4 error-partial slots per (tile, quad)
}

cudaError_t launch_conv_lse_fast(const se2_kernel_s* k, const float* in, int batch, const Epilogue& epi,
                                 cudaStream_t s, int* bpf, float* stats, int force_exact, int* counters,
                                 float* split_scratch, size_t split_floats) {
    if (k->nt > LseFCfg<1>::MAXNT) return cudaErrorInvalidValue;
    switch (k->R) {
#define SE2_CASE(r) \
    case r: return launch_lsef_r<r>(k, in, batch, epi, s, bpf, stats, force_exact, counters, split_scratch, split_floats);
        SE2_CASE(0) SE2_CASE(1) SE2_CASE(2) SE2_CASE(3) SE2_CASE(4) SE2_CASE(5) SE2_CASE(6) SE2_CASE(7)
        SE2_CASE(8) SE2_CASE(9) SE2_CASE(10) SE2_CASE(11) SE2_CASE(12) SE2_CASE(13) SE2_CASE(14) SE2_CASE(15)
#undef SE2_CASE
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace se2
