// K10: SE(2) group convolution, linear domain, on the 5th-generation tensor cores (tcgen05), with
// fp32 accuracy recovered by a 3-pass BF16 split (the same operator as K2).
//
//   y[b, to, y, x] = sum_ti sum_{dyi, dxi < S} Wl[to, ti, dyi, dxi] * v[b, ti, y + R - dyi, x + R - dxi]
//
// Formulation: one CTA owns 8 output rows y0..y0+7 x one block of 16 output
// orientations x all nx pixels of those rows.  For every input row yi and every filter column dxi one
// tcgen05 MMA chain computes
//
//   D[(r, to)][x] += sum_{ti in window} A[(r, to)][ti] * B[x][ti],
//   A[(r, to)][ti] = Wl[to, ti, y0 + r + R - yi, dxi]    (rows with dyi outside the box: 0)
//   B[x][ti]       = v[ti, yi, x + R - dxi]               (pixels shifted by a descriptor offset)
//
// with M = 128 = 8 rows x 16 orientations, N = the row's pixels (<= 256), K = the theta window of the
// orientation block (32 orientations covering the fp32 band, or all of them when nt <= 32).  Both
// operands are K-major SWIZZLE_NONE ("interleave") shared-memory tiles:
//   * B is a padded input row stored [ti chunk][x'][8 ti] (16 B per pixel), so a pixel shift dxi is
//     a +16 B start-address change of the descriptor -- no im2col;
//   * A is stored [dxi][chunk][j = dyi + 7][16 to][8 ti], so the 8 output rows r of one input row yi
//     (dyi = y0 + r + R - yi, consecutive) form one contiguous 2 KB tile per chunk.
// fp32 accuracy: x = hi + lo with hi = bf16(x), lo = bf16(x - hi) for both operands; the chain adds
// hi.hi + hi.lo + lo.hi (per-term error <= 3 * 2^-18 relative; simulated on c4m in DESIGN.md).
//
// Roles (320 threads): warp 0 lane 0 is the TMA producer (an NA-stage weight ring, one 5-D tensor copy
// per stage, and a 2-stage ring of split input rows, 8 bulk copies per row); warp 1 lane 0 issues the
// MMAs and commits each stage back; warps 2-9 add every input row's TMEM sums into registers (round to
// nearest; the tensor core's own accumulation truncates) and read the correction accumulator.
//
// Geometry (chosen per kernel for its max_batch):
//   * rows mode: one CTA per (rows <= 8 output rows, orientation block, field); the epilogue runs in the
//     kernel through a shared-memory transpose (coalesced along x);
//   * balanced mode: 8-row tiles; the tiles' input-row chains are concatenated and split into equal runs
//     over <= 148 CTAs (<= 3 pieces per tile); every piece writes its sums to an L2-resident partial
//     buffer and tc_pieces_epilogue_kernel adds the pieces in order and applies the fused epilogue.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "conv_common.cuh"

namespace se2 {

namespace {

constexpr int kTcRows = 8;     // rows of the MMA M tile (8 rows x 16 orientations = 128)
constexpr int kTcBlk = 16;     // output orientations per CTA
constexpr int kTcPadX = 16;    // zero pixels left of x = 0 in the split input rows (>= R)
constexpr int kTcNA = 6;       // weight-ring stages
// stages of a row whose correction MMAs are issued before waiting for the previous row's flush (the
// rest interleave main and corrections per K-step, which keeps consecutive MMAs on different TMEM
// accumulators: 0.579 -> 0.524 ms at c4; 1 early stage measured best, 0.511 ms, against 0/2/4/6)
constexpr int kTcEarly = 1;
// input rows per main-accumulator chain (flushed to registers after each): 2 halves the flush bubbles;
// truncation bound 2 x S x K/16 = 124 steps of 2^-23 at R 15, inside R18
constexpr int kTcFlushRows = 2;
constexpr int kTcThreads = 320;   // warp 0: TMA producer, warp 1: MMA issuer, warps 2-9: accumulators / epilogue
constexpr int kTcFlushWarps = 8;

struct TcGeom {
    int npad;    // MMA N: nx rounded up to 16
    int nxp;     // padded row length (pixels) of the split input: npad + 2 * kTcPadX
    int nch;     // theta chunks of 8
    int nwin;    // chunks in the theta window of one orientation block (2 or 4)
    int nj;      // dyi + 7 range: S + 14
    int nblk;    // orientation blocks
    size_t a_stage, b_stage, smem;
    int tmem_cols;
};

__host__ __device__ inline int tc_chunk0(int blk, int nch, int nwin) {
    return (nwin == nch) ? 0 : ((2 * blk - 1 + nch) % nch);
}

TcGeom tc_geom(const se2_kernel_s* k) {
    TcGeom g;
    g.npad = (k->nx + 15) / 16 * 16;
    g.nxp = g.npad + 2 * kTcPadX;
    g.nch = k->nt / 8;
    g.nwin = g.nch <= 4 ? g.nch : 4;
    g.nj = k->S + 14;
    g.nblk = k->nt / kTcBlk;
    g.a_stage = (size_t)2 * g.nwin * kTcRows * kTcBlk * 16;          // hi + lo, 2 KB per chunk
    g.b_stage = (size_t)2 * g.nwin * g.nxp * 16;                     // hi + lo rows
    size_t pipe = 2 * g.b_stage + kTcNA * g.a_stage;
    size_t epi = (size_t)128 * (g.npad + 1) * sizeof(float);         // TMEM -> smem transpose
    g.smem = std::max(pipe, epi) + 1024;                              // + barriers / scratch
    // per accumulator: the npad columns, and every x32 tcgen05.ld of the column-half flush
    // (columns h * npad/2 + c .. + 31 with c < npad/2) must stay inside the allocation
    g.tmem_cols = 32;
    while (g.tmem_cols < std::max(g.npad, g.npad / 2 + 32)) g.tmem_cols *= 2;
    g.tmem_cols *= 2;   // main (hi.hi) + correction (hi.lo + lo.hi) accumulators
    return g;
}

// programmatic dependent launch: block until the preceding kernel in the stream has completed and its
// writes are visible (a no-op for a normally launched kernel)
__device__ __forceinline__ void tc_grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;   // descriptor version (sm_100); base offset 0; layout SWIZZLE_NONE
    return d;
}

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// bounded wait: a pipeline bug traps (a launch error) instead of hanging the device
__device__ __forceinline__ void tc_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    long long spins = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (++spins > (1ll << 31)) __trap();
    }
}

struct TcArgs {
    const __nv_bfloat16* xk;   // split input rows: [hl][batch][ny][nch][nxp][8]
    const __nv_bfloat16* wk;   // split weights:    [hl][nblk][S][nwin][nj][16][8]
    size_t xk_hl, wk_hl;       // elements between the hi and lo halves
    int nx, ny, nt, R, S;
    int npad, nxp, nch, nwin, nj;
    uint32_t a_stage, b_stage;
    int tmem_cols;
    int rows_out;              // output rows a CTA owns (<= kTcRows; the M tile's remaining rows are discarded)
    int y_lo, y_hi;            // output window (kernel's win_lo / win_hi): rows outside are input-only halos
    // balanced mode (PIECES): 8-row tiles, CTA c takes chain units [c q, (c + 1) q) of the concatenated
    // (tile, input row) list; every piece's sums go to `part` [tile][piece < 3][128][npad]
    int batch, nblk, ngroups, ug, q;
    float* part;
};

// chain length (input rows) of 8-row group g, and the units before it within one (field, block)
__device__ __forceinline__ int tc_group_len(const TcArgs& a, int g) {
    const int y0 = a.y_lo + g * kTcRows;
    return min(a.ny - 1, min(a.y_hi - 1, y0 + kTcRows - 1) + a.R) - max(0, y0 - a.R) + 1;
}
__device__ __forceinline__ int tc_group_prefix(const TcArgs& a, int g) {
    int s = 0;
    for (int i = 0; i < g; ++i) s += tc_group_len(a, i);
    return s;
}

struct TcPiece {
    int b, blk, y0, ylo;   // field, orientation block, first output row, first input row of the tile's chain
    int r0, r1;            // this piece: chain rows [r0, r1) (input rows ylo + r0 ...)
    int tile, p;           // tile index (field, block, group) and the piece's index within the tile
};

// piece k of this CTA; false when the CTA has fewer pieces
template <bool PIECES>
__device__ __forceinline__ bool tc_piece(const TcArgs& a, int k, TcPiece& pc) {
    if (!PIECES) {
        if (k > 0) return false;
        pc.y0 = a.y_lo + blockIdx.x * a.rows_out;
        pc.blk = blockIdx.y;
        pc.b = blockIdx.z;
        pc.ylo = max(0, pc.y0 - a.R);
        pc.r0 = 0;
        pc.r1 = min(a.ny - 1, min(a.y_hi - 1, pc.y0 + a.rows_out - 1) + a.R) - pc.ylo + 1;
        pc.tile = 0;
        pc.p = 0;
        return true;
    }
    const int U = a.batch * a.nblk * a.ug;
    const int c = blockIdx.x;
    const int uend = min(U, (c + 1) * a.q);
    int u = c * a.q;
    for (int kk = 0; u < uend; ++kk) {
        const int grp = u / a.ug, rem = u - grp * a.ug;
        int g = 0, pre = 0;
        while (pre + tc_group_len(a, g) <= rem) { pre += tc_group_len(a, g); ++g; }
        const int st = grp * a.ug + pre, len = tc_group_len(a, g);
        const int r1 = min(len, uend - st);
        if (kk == k) {
            pc.b = grp / a.nblk;
            pc.blk = grp - pc.b * a.nblk;
            pc.y0 = a.y_lo + g * kTcRows;
            pc.ylo = max(0, pc.y0 - a.R);
            pc.r0 = u - st;
            pc.r1 = r1;
            pc.tile = grp * a.ngroups + g;
            pc.p = c - st / a.q;
            return true;
        }
        u = st + r1;
    }
    return false;
}

// input split: v[b][ti][y][x] (fp32) -> hi/lo bf16 rows [b][y][chunk][x' = x + kTcPadX][8]
__global__ void tc_split_input_kernel(const float* __restrict__ v, __nv_bfloat16* __restrict__ xk, size_t xk_hl,
                                      int nx, int ny, int nt, int nxp, int batch) {
    tc_grid_dep_wait();   // reads the previous kernel's output (launched with PDL)
    const int nch = nt / 8;
    const int64_t total = (int64_t)batch * ny * nch * nxp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int xp = (int)(i % nxp);
        int64_t t = i / nxp;
        const int c = (int)(t % nch);
        t /= nch;
        const int y = (int)(t % ny);
        const int b = (int)(t / ny);
        const int x = xp - kTcPadX;
        __align__(16) __nv_bfloat16 hi[8], lo[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            float f = 0.f;
            if (x >= 0 && x < nx) f = v[(((int64_t)b * nt + c * 8 + e) * ny + y) * nx + x];
            const __nv_bfloat16 h = __float2bfloat16_rn(f);
            hi[e] = h;
            lo[e] = __float2bfloat16_rn(f - __bfloat162float(h));
        }
        reinterpret_cast<uint4*>(xk)[i] = *reinterpret_cast<const uint4*>(hi);
        reinterpret_cast<uint4*>(xk + xk_hl)[i] = *reinterpret_cast<const uint4*>(lo);
    }
}

// weight split: Wl[to][ti][S][SP] (fp32) -> hi/lo [blk][dxi][c][j][to_l][8]
__global__ void tc_split_weights_kernel(const float* __restrict__ Wl, __nv_bfloat16* __restrict__ wk, size_t wk_hl,
                                        int nt, int S, int nch, int nwin, int nj, int nblk) {
    const int SP = (S + 3) / 4 * 4;
    const int64_t total = (int64_t)nblk * S * nwin * nj * kTcBlk;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int tol = (int)(i % kTcBlk);
        int64_t t = i / kTcBlk;
        const int j = (int)(t % nj);
        t /= nj;
        const int c = (int)(t % nwin);
        t /= nwin;
        const int dxi = (int)(t % S);
        const int blk = (int)(t / S);
        const int to = blk * kTcBlk + tol;
        const int chunk = (tc_chunk0(blk, nch, nwin) + c) % nch;
        const int dyi = j - 7;
        __align__(16) __nv_bfloat16 hi[8], lo[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int ti = chunk * 8 + e;
            float w = 0.f;
            if (dyi >= 0 && dyi < S) w = Wl[(((int64_t)to * nt + ti) * S + dyi) * SP + dxi];
            const __nv_bfloat16 h = __float2bfloat16_rn(w);
            hi[e] = h;
            lo[e] = __float2bfloat16_rn(w - __bfloat162float(h));
        }
        reinterpret_cast<uint4*>(wk)[i] = *reinterpret_cast<const uint4*>(hi);
        reinterpret_cast<uint4*>(wk + wk_hl)[i] = *reinterpret_cast<const uint4*>(lo);
    }
}

template <bool PIECES>
__global__ void __launch_bounds__(kTcThreads, 1)
conv_tc_kernel(TcArgs a, Epilogue epi, const __grid_constant__ CUtensorMap wmap) {
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* sB = smem;                                   // [2][hl][nwin][nxp][16 B]
    unsigned char* sA = smem + 2 * (size_t)a.b_stage;           // [NA][hl][nwin][8 j][16 to][16 B]
    __shared__ __align__(8) uint64_t fullB[2], emptyB[2], fullA[kTcNA], emptyA[kTcNA], rowdone[2], flushed, cflushed;
    __shared__ uint32_t tmem_base;
    __shared__ float sRed[kTcThreads / 32];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(a.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < 2; ++i) { mbar_init(&fullB[i], 1); mbar_init(&emptyB[i], 1); }
        for (int i = 0; i < kTcNA; ++i) { mbar_init(&fullA[i], 1); mbar_init(&emptyA[i], 1); }
        mbar_init(&rowdone[0], 1);
        mbar_init(&rowdone[1], 1);
        mbar_init(&flushed, kTcFlushWarps);
        mbar_init(&cflushed, kTcFlushWarps);
        mbar_fence_init();
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;

    const size_t row_elems = (size_t)a.nch * a.nxp * 8;               // one (b, y) row of the split input
    const uint32_t chunk_bytes_b = (uint32_t)a.nxp * 16;
    if (warp == 0) {
      if (lane == 0) {
        // ---------------- producer ----------------
        // global input-row counter gr (all pieces of this CTA): B ring stage gr & 1, weight stage (gr S + dxi)
        auto load_b = [&](int gr, const TcPiece& pc, int yi) {
            const int st = gr & 1;
            if (gr >= 2) tc_wait(&emptyB[st], (uint32_t)(((gr >> 1) - 1) & 1));
            mbar_expect_tx(&fullB[st], a.b_stage);
            const int chunk0 = tc_chunk0(pc.blk, a.nch, a.nwin);
            for (int hl = 0; hl < 2; ++hl) {
                const __nv_bfloat16* row = a.xk + hl * a.xk_hl + ((size_t)pc.b * a.ny + yi) * row_elems;
                for (int c = 0; c < a.nwin; ++c) {
                    const int ch = (chunk0 + c) % a.nch;
                    bulk_load(sB + st * (size_t)a.b_stage + (size_t)(hl * a.nwin + c) * chunk_bytes_b,
                              row + (size_t)ch * a.nxp * 8, chunk_bytes_b, &fullB[st]);
                }
            }
        };
        const int b_after = min(kTcNA - 1, a.S - 1);
        const uint32_t sA_u = smem_u32(sA), fullA_u = smem_u32(&fullA[0]);
        const CUtensorMap* wm = &wmap;
        TcPiece pc, pn;
        int gr = 0;
        // PDL: the weight stages do not depend on the preceding kernels, the input rows do (the split
        // kernel): B(0) is loaded after the first weight stages, behind the grid-dependency wait
        bool b0 = false;
        for (int k = 0; tc_piece<PIECES>(a, k, pc); ++k) {
            for (int rr = pc.r0; rr < pc.r1; ++rr, ++gr) {
                const int yi = pc.ylo + rr;
                const int j0 = pc.y0 + a.R - yi + 7;
                for (int dxi = 0; dxi < a.S; ++dxi) {
                    const int t = gr * a.S + dxi;
                    const int st = t % kTcNA;
                    if (t >= kTcNA) tc_wait(&emptyA[st], (uint32_t)(((t / kTcNA) - 1) & 1));
                    mbar_expect_tx(&fullA[st], a.a_stage);
                    // one TMA box per stage: [hl 2][chunk nwin][j 8][16 to x 8 ti]
                    tma_load_5d(sA_u + (uint32_t)st * a.a_stage, wm, fullA_u + 8u * (uint32_t)st, 0, j0, 0,
                                pc.blk * a.S + dxi, 0);
                    if (!b0 && dxi == b_after) {
                        tc_grid_dep_wait();
                        TcPiece p0;
                        tc_piece<PIECES>(a, 0, p0);
                        load_b(0, p0, p0.ylo + p0.r0);
                        b0 = true;
                    }
                    if (dxi == b_after) {   // the next input row (this piece's, or the next piece's first)
                        if (rr + 1 < pc.r1) load_b(gr + 1, pc, yi + 1);
                        else if (tc_piece<PIECES>(a, k + 1, pn)) load_b(gr + 1, pn, pn.ylo + pn.r0);
                    }
                }
            }
        }
      }
      __syncwarp();
    } else if (warp == 1) {
      if (lane == 0) {
        // ---------------- MMA issuer ----------------
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(a.npad >> 3) << 17) |
                               ((uint32_t)(128 >> 4) << 24);
        const uint64_t dA0 = tc_desc(smem_u32(sA), 2048, 128);
        const uint64_t dB0 = tc_desc(smem_u32(sB), chunk_bytes_b, 128);
        const int ksteps = a.nwin / 2;
        const uint32_t tcor = tmem + (uint32_t)(a.tmem_cols / 2);   // correction accumulator (hi.lo + lo.hi)
        uint32_t acc_c = 0;
        auto issue_corr = [&](int t, int stb, int dxi) {
            const int st = t % kTcNA;
            tc_wait(&fullA[st], (uint32_t)((t / kTcNA) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t offA = (uint32_t)(st * a.a_stage);
            const uint32_t offB = (uint32_t)(stb * a.b_stage + (kTcPadX + a.R - dxi) * 16);
            for (int ks = 0; ks < ksteps; ++ks) {
                const uint32_t ah = offA + (uint32_t)(2 * ks) * 2048, al = ah + (uint32_t)a.nwin * 2048;
                const uint32_t bh = offB + (uint32_t)(2 * ks) * chunk_bytes_b, bl = bh + (uint32_t)a.nwin * chunk_bytes_b;
                tc_mma(tcor, dA0 + (ah >> 4), dB0 + (bl >> 4), idesc, acc_c);
                acc_c = 1;
                tc_mma(tcor, dA0 + (al >> 4), dB0 + (bh >> 4), idesc, 1);
            }
        };
        auto issue_main = [&](int t, int stb, int dxi, bool restart) {
            const int st = t % kTcNA;
            const uint32_t offA = (uint32_t)(st * a.a_stage);
            const uint32_t offB = (uint32_t)(stb * a.b_stage + (kTcPadX + a.R - dxi) * 16);
            for (int ks = 0; ks < ksteps; ++ks) {
                const uint32_t ah = offA + (uint32_t)(2 * ks) * 2048;
                const uint32_t bh = offB + (uint32_t)(2 * ks) * chunk_bytes_b;
                tc_mma(tmem, dA0 + (ah >> 4), dB0 + (bh >> 4), idesc, (!restart || dxi > 0 || ks > 0) ? 1u : 0u);
            }
            tc_commit(&emptyA[st]);
        };
        // steady state: per K-step main (hi.hi), then the two corrections sharing its A / B operand
        auto issue_both = [&](int t, int stb, int dxi, bool restart) {
            const int st = t % kTcNA;
            tc_wait(&fullA[st], (uint32_t)((t / kTcNA) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t offA = (uint32_t)(st * a.a_stage);
            const uint32_t offB = (uint32_t)(stb * a.b_stage + (kTcPadX + a.R - dxi) * 16);
            for (int ks = 0; ks < ksteps; ++ks) {
                const uint32_t ah = offA + (uint32_t)(2 * ks) * 2048, al = ah + (uint32_t)a.nwin * 2048;
                const uint32_t bh = offB + (uint32_t)(2 * ks) * chunk_bytes_b, bl = bh + (uint32_t)a.nwin * chunk_bytes_b;
                tc_mma(tcor, dA0 + (ah >> 4), dB0 + (bl >> 4), idesc, acc_c);              // A_hi shared with
                acc_c = 1;
                tc_mma(tmem, dA0 + (ah >> 4), dB0 + (bh >> 4), idesc, (!restart || dxi > 0 || ks > 0) ? 1u : 0u);   // <- B_hi
                tc_mma(tcor, dA0 + (al >> 4), dB0 + (bh >> 4), idesc, 1);                   // shared with
            }
            tc_commit(&emptyA[st]);
        };
        TcPiece pc;
        int gr = 0, gs = 0;   // input rows and main-accumulator chains issued so far
        for (int k = 0; tc_piece<PIECES>(a, k, pc); ++k) {
            if (k > 0) {   // the correction accumulator restarts per piece: the previous piece's was read
                tc_wait(&cflushed, (uint32_t)((k - 1) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;");
                acc_c = 0;
            }
            for (int rr = pc.r0; rr < pc.r1; ++rr, ++gr) {
                const int stb = gr & 1;
                tc_wait(&fullB[stb], (uint32_t)((gr >> 1) & 1));
                // The main accumulator restarts every kTcFlushRows input rows of a piece and the
                // accumulator warps must first have read the previous chain's sums: the correction MMAs
                // of the row's first P stages are issued before that wait so the tensor pipe stays busy.
                const bool restart = (rr - pc.r0) % kTcFlushRows == 0;
                const int P = (restart && gs > 0) ? min(kTcEarly, a.S) : 0;
                for (int dxi = 0; dxi < P; ++dxi) issue_corr(gr * a.S + dxi, stb, dxi);
                if (restart && gs > 0) {
                    tc_wait(&flushed, (uint32_t)((gs - 1) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;");
                }
                for (int dxi = 0; dxi < P; ++dxi) issue_main(gr * a.S + dxi, stb, dxi, restart);
                for (int dxi = P; dxi < a.S; ++dxi) issue_both(gr * a.S + dxi, stb, dxi, restart);
                tc_commit(&emptyB[stb]);
                tc_commit(&rowdone[gr & 1]);   // 2-deep ring: the issuer runs at most one chain (<= 2 rows) ahead
                if ((rr - pc.r0) % kTcFlushRows == kTcFlushRows - 1 || rr == pc.r1 - 1) ++gs;   // chain end
            }
        }
      }
      __syncwarp();
    }
    // ---------------- accumulation of the per-row partial sums (fp32, round to nearest) ----------------
    // The tensor core's fp32 accumulation truncates; restarting the main accumulator every input row
    // bounds that to one row's chain (S x K/16 steps) and the row sums are added here in registers.
    float* T = reinterpret_cast<float*>(smem);   // [128][npad + 1] after the pipeline has drained
    const int pitch = a.npad + 1;
    float err = 0.f;
    const int half = a.npad / 2;
    TcPiece pc;
    if (warp >= 2) {
        tc_grid_dep_wait();   // partial / output writes after the preceding kernels (PDL launch)
        const int q = warp & 3, h = (warp - 2) >> 2;        // TMEM lane quarter (warp % 4) and column half
        const int m = 32 * q + lane;
        const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(h * half);
        int gr = 0;
        for (int k = 0; tc_piece<PIECES>(a, k, pc); ++k) {
            float sum[128];
#pragma unroll
            for (int j = 0; j < 128; ++j) sum[j] = 0.f;
            for (int rr = pc.r0; rr < pc.r1; ++rr, ++gr) {
                tc_wait(&rowdone[gr & 1], (uint32_t)((gr >> 1) & 1));
                if (!((rr - pc.r0) % kTcFlushRows == kTcFlushRows - 1 || rr == pc.r1 - 1)) continue;   // mid-chain
                __syncwarp();
                asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
                for (int c = 0; c < 128; c += 32) {
                    if (c < half) {
                        uint32_t v[32];
                        asm volatile(
                            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                              "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                              "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                              "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                            : "r"(tl + (uint32_t)c));
                        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
                        for (int j = 0; j < 32; ++j) sum[c + j] += __uint_as_float(v[j]);
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&flushed)) : "memory");
            }
            // the correction accumulator (complete with the piece's last row commit)
            const uint32_t tc2 = tl + (uint32_t)(a.tmem_cols / 2);
            float* prow = PIECES ? a.part + ((size_t)pc.tile * 3 + pc.p) * 128 * a.npad + (size_t)m * a.npad + h * half
                                 : nullptr;
#pragma unroll
            for (int c = 0; c < 128; c += 32) {
                if (c < half) {
                    uint32_t v[32];
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                        : "r"(tc2 + (uint32_t)c));
                    asm volatile("tcgen05.wait::ld.sync.aligned;");
                    if (PIECES) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4)
                            if (c + j < half)
                                *reinterpret_cast<float4*>(prow + c + j) =
                                    make_float4(sum[c + j] + __uint_as_float(v[j]), sum[c + j + 1] + __uint_as_float(v[j + 1]),
                                                sum[c + j + 2] + __uint_as_float(v[j + 2]),
                                                sum[c + j + 3] + __uint_as_float(v[j + 3]));
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (c + j < half) T[m * pitch + h * half + c + j] = sum[c + j] + __uint_as_float(v[j]);
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&cflushed)) : "memory");
        }
    }
    if (!PIECES) {
        __syncthreads();   // T complete (every warp reaches this; the role warps have finished their loops)
        tc_piece<false>(a, 0, pc);
        if (warp >= 2) {
            const int64_t N = (int64_t)a.nx * a.ny * a.nt;
            const int f = warp - 2;
            for (int mm = 0; mm < 128 / kTcFlushWarps; ++mm) {
                const int m = (128 / kTcFlushWarps) * f + mm;
                const int r = m / kTcBlk, tol = m % kTcBlk;
                const int y = pc.y0 + r, to = pc.blk * kTcBlk + tol;
                if (y >= a.y_hi || r >= a.rows_out) continue;
                const int64_t rowbase = (int64_t)pc.b * N + ((int64_t)to * a.ny + y) * a.nx;
                for (int x = lane; x < a.nx; x += 32) err += apply_epilogue<false>(epi, rowbase + x, x, y, T[m * pitch + x]);
            }
        }
        if (epi.err_partial != nullptr) {
            const float t = block_sum<kTcThreads>(err, sRed);
            if (tid == 0)
                epi.err_partial[(int64_t)pc.b * (gridDim.x * gridDim.y) + blockIdx.y * gridDim.x + blockIdx.x] = t;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols));
}

// balanced mode: sum each output's piece partials (1-3, in piece order) and apply the fused epilogue;
// one block per (8-row group, orientation, field) -- one tile row block -- threads along x (coalesced)
__global__ void __launch_bounds__(256) tc_pieces_epilogue_kernel(TcArgs a, Epilogue epi) {
    __shared__ float sRed[32];
    __shared__ int sNp;
    tc_grid_dep_wait();   // the partials of the MMA kernel (PDL launch)
    const int g = blockIdx.x, to = blockIdx.y, b = blockIdx.z;
    const int blk = to / kTcBlk, grp = b * a.nblk + blk;
    if (threadIdx.x < 32) {   // warp 0: the group's unit offset as a strided sum + shuffle reduction
        int pre = 0;
        for (int i = threadIdx.x; i < g; i += 32) pre += tc_group_len(a, i);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
        if (threadIdx.x == 0) {
            const int st = grp * a.ug + pre, len = tc_group_len(a, g);
            sNp = (st + len - 1) / a.q - st / a.q + 1;
        }
    }
    __syncthreads();
    const int np = sNp;
    const float* tile = a.part + ((size_t)(grp * a.ngroups + g) * 3) * 128 * a.npad;
    const int64_t N = (int64_t)a.nx * a.ny * a.nt;
    // 256 threads: 4 consecutive x per thread (float4 partial loads; npad % 16 == 0), rows r and r + 4
    const int x0 = (threadIdx.x & 63) * 4, r0 = threadIdx.x >> 6;
    float4 v[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int r = r0 + 4 * k;
        if (x0 >= a.npad) break;   // narrow rows: no load past the row (npad % 16 == 0, so x0 + 3 < npad)
        const float4* src = reinterpret_cast<const float4*>(tile + (size_t)(r * kTcBlk + (to % kTcBlk)) * a.npad + x0);
        v[k] = src[0];
        for (int p = 1; p < np; ++p) {
            const float4 w = src[(size_t)p * 32 * a.npad];   // 128 * npad floats = 32 * npad float4
            v[k].x += w.x; v[k].y += w.y; v[k].z += w.z; v[k].w += w.w;
        }
    }
    float err = 0.f;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int r = r0 + 4 * k, y = a.y_lo + g * kTcRows + r;
        if (y >= a.y_hi || x0 >= a.nx) continue;
        const int64_t rowbase = (int64_t)b * N + ((int64_t)to * a.ny + y) * a.nx;
        const float vv[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (x0 + j < a.nx) err += apply_epilogue<false>(epi, rowbase + x0 + j, x0 + j, y, vv[j]);
    }
    if (epi.err_partial != nullptr) {
        const float t = block_sum<256>(err, sRed);
        if (threadIdx.x == 0) epi.err_partial[(int64_t)b * (gridDim.x * gridDim.y) + (int64_t)to * gridDim.x + g] = t;
    }
}

}  // namespace

bool conv_tc_eligible(const se2_kernel_s* k) {
    if (getenv("SE2_NO_TC") != nullptr) return false;
    if (k->nt % 16 != 0 || k->nx > 256 || k->R > kTcPadX) return false;
    if (k->nt / 8 > 4 && k->band > 8) return false;   // the 32-orientation window must cover the band
    return true;
}

// output rows per CTA: fewer than the M tile's 8 when that fills the SMs in the same number of waves
// (c4: 7 rows -> 37 x 4 = 148 CTAs, one wave, each chain 37 instead of 38 input rows).  Chosen for the
// kernel's max_batch so that every launch (and the error-partial layout) uses one geometry.
static int tc_rows_out(const se2_kernel_s* k) {
    int best = kTcRows;
    double best_cost = 1e300;
    for (int rows = kTcRows; rows >= 4; --rows) {
        const double ctas = (double)((k->wrows() + rows - 1) / rows) * (k->nt / kTcBlk) * k->max_batch;
        const double cost = std::ceil(ctas / 148.0) * std::min(k->ny, rows + 2 * k->R);
        if (cost < best_cost - 1e-9) { best_cost = cost; best = rows; }
    }
    return best;
}

// balanced mode geometry (host mirror of tc_group_len / tc_group_prefix)
static int tc_group_len_h(const se2_kernel_s* k, int g) {
    const int y0 = k->wlo() + g * kTcRows;
    return std::min(k->ny - 1, std::min(k->whi() - 1, y0 + kTcRows - 1) + k->R) - std::max(0, y0 - k->R) + 1;
}
static int tc_ngroups(const se2_kernel_s* k) { return (k->wrows() + kTcRows - 1) / kTcRows; }
static void tc_units(const se2_kernel_s* k, int batch, int* ug, int* lmax, long long* U) {
    const int ngroups = tc_ngroups(k);
    *ug = 0;
    *lmax = 0;
    for (int g = 0; g < ngroups; ++g) {
        *ug += tc_group_len_h(k, g);
        *lmax = std::max(*lmax, tc_group_len_h(k, g));
    }
    *U = (long long)batch * (k->nt / kTcBlk) * (*ug);
}
// units per CTA in the balanced mode: ceil(U / 148), at least half the longest chain (<= 3 pieces per tile)
static int tc_units_per_cta(const se2_kernel_s* k, int batch) {
    int ug, lmax;
    long long U;
    tc_units(k, batch, &ug, &lmax, &U);
    return (int)std::max<long long>((U + 147) / 148, (lmax + 1) / 2);
}

int conv_blocks_per_field_tc(const se2_kernel_s* k) {
    if (k->tc_part != nullptr) return tc_ngroups(k) * k->nt;   // balanced: epilogue blocks
    const int rows = tc_rows_out(k);
    return (k->wrows() + rows - 1) / rows * (k->nt / kTcBlk);
}

// 5-D tensor map over split weights w: one TMA box per pipeline stage ([hl][chunk][8 j][16 to x 8 ti])
static cudaError_t tc_weight_map(const se2_kernel_s* k, void* w, void** map_out) {
    const TcGeom g = tc_geom(k);
    const size_t wk_hl = (size_t)g.nblk * k->S * g.nwin * g.nj * kTcBlk * 8;
    CUtensorMap* m = new CUtensorMap;
    const uint64_t dims[5] = {(uint64_t)kTcBlk * 8, (uint64_t)g.nj, (uint64_t)g.nwin, (uint64_t)g.nblk * k->S, 2};
    const uint64_t strides[4] = {(uint64_t)kTcBlk * 8 * 2, (uint64_t)g.nj * kTcBlk * 8 * 2,
                                 (uint64_t)g.nwin * g.nj * kTcBlk * 8 * 2, (uint64_t)wk_hl * 2};
    const uint32_t box[5] = {(uint32_t)kTcBlk * 8, (uint32_t)kTcRows, (uint32_t)g.nwin, 1, 2};
    if (!make_tmap_5d(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, w, dims, strides, box)) {
        delete m;
        return cudaErrorInvalidValue;
    }
    *map_out = m;
    return cudaSuccess;
}

// K10 weights of the transport-cost table rho^2 exp(-rho^2/eps) (se2_transport_cost, NEXT #2): same
// layout as the Gibbs weights, built on the first cost evaluation after k->Wcl is tabulated
cudaError_t conv_tc_prepare_cost(se2_kernel_s* k, cudaStream_t s) {
    if (k->tc_w == nullptr || k->tc_wc != nullptr || k->Wcl == nullptr) return cudaSuccess;
    const TcGeom g = tc_geom(k);
    cudaError_t e = cudaMalloc(&k->tc_wc, 2 * k->tc_w_hl * sizeof(__nv_bfloat16));
    if (e != cudaSuccess) return e;
    e = tc_weight_map(k, k->tc_wc, &k->tc_wcmap);
    if (e != cudaSuccess) return e;
    tc_split_weights_kernel<<<592, 256, 0, s>>>(k->Wcl, reinterpret_cast<__nv_bfloat16*>(k->tc_wc), k->tc_w_hl, k->nt,
                                                k->S, g.nch, g.nwin, g.nj, g.nblk);
    count_launch();
    return cudaGetLastError();
}

// default-engine and geometry decisions for the kernel's output window (at build, and again when
// se2_kernel_set_window changes the window): tc_fast (K10 vs K2 cost model) and the balanced mode's
// partial buffer (allocated when that mode is chosen)
cudaError_t conv_tc_decide(se2_kernel_s* k) {
    if (k->tc_w == nullptr) return cudaSuccess;
    const TcGeom g = tc_geom(k);
    cudaError_t e = cudaSuccess;
    {
        // cost model at batch 1 (measured on B200, K10): K10 = waves x one CTA's MMA chain
        // ((8 + 2R) rows x S taps x K/16 steps x 3 passes x N/2 cycles) at ~70% of the tensor floor,
        // K2 = 2 nnz N flop at ~60 TFLOP/s (0.82 of the FFMA peak)
        const int rows = tc_rows_out(k);
        const double ctas = (double)((k->wrows() + rows - 1) / rows) * g.nblk;
        const double waves = std::ceil(ctas / 148.0);
        const double row_cyc = (double)k->S * (g.nwin / 2) * 3 * (g.npad / 2);   // one input row's MMA chain
        double t10 = waves * std::min(k->ny, rows + 2 * k->R) * row_cyc / 0.7 / 1.9e9 + 8e-6;
        // the balanced mode (chosen below when it is cheaper): q input rows per SM + its epilogue pass
        t10 = std::min(t10, tc_units_per_cta(k, 1) * row_cyc / 0.7 / 1.9e9 + 20e-6);
        const double t2 = 2.0 * (double)k->nnz_taps * k->nx * k->wrows() * k->nt / 60e12 + 4e-6;
        k->tc_fast = getenv("SE2_TC_DEFAULT") ? (atoi(getenv("SE2_TC_DEFAULT")) != 0) : (t10 < t2);
    }
    {
        // balanced mode (8-row tiles split into equal runs of input rows over 148 CTAs + an epilogue
        // kernel) when its per-SM chain beats the row-count mode's; decided for max_batch
        int ug, lmax;
        long long U;
        tc_units(k, k->max_batch, &ug, &lmax, &U);
        const int q = tc_units_per_cta(k, k->max_batch);
        const int rows = tc_rows_out(k);
        const double ctas = (double)((k->wrows() + rows - 1) / rows) * g.nblk * k->max_batch;
        const double rows_cost = std::ceil(ctas / 148.0) * std::min(k->ny, rows + 2 * k->R);
        const bool want = getenv("SE2_TC_PIECES") ? (atoi(getenv("SE2_TC_PIECES")) != 0) : (q < 0.95 * rows_cost);
        if (want && k->tc_part == nullptr) {
            // sized for the whole grid: any later output window has at most as many 8-row tiles
            const size_t tiles = (size_t)k->max_batch * g.nblk * ((k->ny + kTcRows - 1) / kTcRows);
            e = cudaMalloc(&k->tc_part, tiles * 3 * 128 * g.npad * sizeof(float));
            if (e != cudaSuccess) return e;
        } else if (!want && k->tc_part != nullptr) {
            cudaFree(k->tc_part);
            k->tc_part = nullptr;
        }
    }
    return e;
}

cudaError_t conv_tc_prepare(se2_kernel_s* k) {
    if (!conv_tc_eligible(k)) return cudaSuccess;
    const TcGeom g = tc_geom(k);
    const size_t wk_hl = (size_t)g.nblk * k->S * g.nwin * g.nj * kTcBlk * 8;
    const size_t xk_hl = (size_t)k->max_batch * k->ny * g.nch * g.nxp * 8;
    cudaError_t e = cudaMalloc(&k->tc_w, 2 * wk_hl * sizeof(__nv_bfloat16));
    if (e == cudaSuccess) e = cudaMalloc(&k->tc_x, 2 * xk_hl * sizeof(__nv_bfloat16));
    if (e != cudaSuccess) return e;
    k->tc_w_hl = wk_hl;
    k->tc_x_hl = xk_hl;
    e = conv_tc_decide(k);
    if (e != cudaSuccess) return e;
    e = tc_weight_map(k, k->tc_w, &k->tc_wmap);
    if (e != cudaSuccess) return e;
    tc_split_weights_kernel<<<592, 256>>>(k->Wl, reinterpret_cast<__nv_bfloat16*>(k->tc_w), wk_hl, k->nt, k->S, g.nch,
                                          g.nwin, g.nj, g.nblk);
    count_launch();
    // the attribute is per function: set the maximum once (each launch passes its own size)
    int optin = 0;
    cudaFuncAttributes fa;
    e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, k->device);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, conv_tc_kernel<false>);
    if (e != cudaSuccess) return e;
    const int dyn_max = optin - (int)fa.sharedSizeBytes;
    if ((int)g.smem > dyn_max) return cudaErrorInvalidValue;
    e = cudaFuncSetAttribute(conv_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, conv_tc_kernel<true>);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(conv_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 optin - (int)fa.sharedSizeBytes);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

void conv_tc_release(se2_kernel_s* k) {
    delete reinterpret_cast<CUtensorMap*>(k->tc_wmap);
    delete reinterpret_cast<CUtensorMap*>(k->tc_wcmap);
    if (k->tc_wc) cudaFree(k->tc_wc);
    if (k->tc_part) cudaFree(k->tc_part);
    k->tc_wmap = k->tc_wcmap = k->tc_wc = nullptr;
    k->tc_part = nullptr;
}

cudaError_t launch_conv_tc(const se2_kernel_s* k, const float* in, int batch, const Epilogue& epi, cudaStream_t s,
                           int* bpf) {
    const TcGeom g = tc_geom(k);
    __nv_bfloat16* xk = reinterpret_cast<__nv_bfloat16*>(k->tc_x);
    // the three K10 kernels are launched with programmatic stream serialization (PDL): each may start
    // while its predecessor drains and waits (griddepcontrol.wait) before consuming its results
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    auto cfg_of = [&](dim3 grid, dim3 block, size_t smem) {
        cudaLaunchConfig_t c = {};
        c.gridDim = grid;
        c.blockDim = block;
        c.dynamicSmemBytes = smem;
        c.stream = s;
        c.attrs = pdl;
        c.numAttrs = 1;
        return c;
    };
    {
        // one (field, row, chunk, pixel) item per thread: all 8 plane loads of every item in flight
        const long long items = (long long)batch * k->ny * (k->nt / 8) * g.nxp;
        cudaLaunchConfig_t c = cfg_of(dim3((unsigned)std::min<long long>((items + 255) / 256, 1 << 20)), dim3(256), 0);
        cudaError_t e = cudaLaunchKernelEx(&c, tc_split_input_kernel, in, xk, k->tc_x_hl, k->nx, k->ny, k->nt, g.nxp, batch);
        if (e != cudaSuccess) return e;
    }
    count_launch();
    TcArgs a;
    a.xk = xk;
    const bool cost = epi.table != nullptr;   // the transport-cost table (launch only when tc_wc exists)
    a.wk = reinterpret_cast<const __nv_bfloat16*>(cost ? k->tc_wc : k->tc_w);
    a.xk_hl = k->tc_x_hl;
    a.wk_hl = k->tc_w_hl;
    a.nx = k->nx; a.ny = k->ny; a.nt = k->nt; a.R = k->R; a.S = k->S;
    a.npad = g.npad; a.nxp = g.nxp; a.nch = g.nch; a.nwin = g.nwin; a.nj = g.nj;
    a.a_stage = (uint32_t)g.a_stage;
    a.b_stage = (uint32_t)g.b_stage;
    a.tmem_cols = g.tmem_cols;
    a.y_lo = k->wlo();
    a.y_hi = k->whi();
    const CUtensorMap* wm = reinterpret_cast<const CUtensorMap*>(cost ? k->tc_wcmap : k->tc_wmap);
    if (k->tc_part != nullptr) {
        // balanced mode: 8-row tiles, equal runs of chain units per CTA, partials + epilogue kernel
        long long U;
        int lmax;
        tc_units(k, batch, &a.ug, &lmax, &U);
        a.rows_out = kTcRows;
        a.batch = batch;
        a.nblk = g.nblk;
        a.ngroups = tc_ngroups(k);
        a.q = tc_units_per_cta(k, batch);
        a.part = reinterpret_cast<float*>(k->tc_part);
        const int ncta = (int)((U + a.q - 1) / a.q);
        {
            cudaLaunchConfig_t c = cfg_of(dim3(ncta), dim3(kTcThreads), g.smem);
            cudaError_t e = cudaLaunchKernelEx(&c, conv_tc_kernel<true>, a, epi, *wm);
            if (e != cudaSuccess) return e;
        }
        count_launch();
        {
            cudaLaunchConfig_t c = cfg_of(dim3(a.ngroups, k->nt, batch), dim3(256), 0);
            cudaError_t e = cudaLaunchKernelEx(&c, tc_pieces_epilogue_kernel, a, epi);
            if (e != cudaSuccess) return e;
        }
        count_launch();
        if (bpf) *bpf = a.ngroups * k->nt;
        return cudaGetLastError();
    }
    a.rows_out = tc_rows_out(k);
    a.part = nullptr;
    dim3 grid((k->wrows() + a.rows_out - 1) / a.rows_out, g.nblk, batch);
    if (bpf) *bpf = (int)(grid.x * grid.y);
    {
        cudaLaunchConfig_t c = cfg_of(grid, dim3(kTcThreads), g.smem);
        cudaError_t e = cudaLaunchKernelEx(&c, conv_tc_kernel<false>, a, epi, *wm);
        if (e != cudaSuccess) return e;
    }
    count_launch();
    return cudaGetLastError();
}

}  // namespace se2
