// K10: SE(2) group convolution, linear domain, on the 5th-generation tensor cores (tcgen05), with
// fp32 accuracy recovered by a 3-pass BF16 split (the same operator as K2).
//
//   y[b, to, y, x] = sum_ti sum_{dyi, dxi < S} Wl[to, ti, dyi, dxi] * v[b, ti, y + R - dyi, x + R - dxi]
//
// Formulation: one CTA owns a tile of kr output rows y0.. x one block of kb output
// orientations x all nx pixels of those rows.  For every input row yi and every filter column dxi one
// tcgen05 MMA chain computes
//
//   D[(r, to)][x] += sum_{ti in window} A[(r, to)][ti] * B[x][ti],
//   A[(r, to)][ti] = Wl[to, ti, y0 + r + R - yi, dxi]    (rows with dyi outside the box: 0)
//   B[x][ti]       = v[ti, yi, x + R - dxi]               (pixels shifted by a descriptor offset)
//
// with M = 128 = kr rows x kb orientations, N = the row's pixels (<= 256), K = the theta window.  Two
// geometries:
//   * classic (nt = 16): kr = 8, kb = 16, K = all orientations;
//   * narrow (nt >= 32): kr = 16, kb = 8 orientations to = 8 blk + 4 .. 8 blk + 11, and per tile EITHER
//     the narrow window ti in [8 blk, 8 blk + 16) (K = 16: every |to - ti| <= 4 kept) when the tile's
//     bound proves the taps outside it negligible --
//        wout[blk] * max_{window rows} |v| <= 2^-30 * min_{tile rows, block chunks} v,   v >= 0 on the window
//     (every output is >= its centre tap W = 1 times v[to, y, x] and the dropped taps sum to <= wout
//     times the window maximum: relative error <= 2^-30) -- OR the wide window [8 blk - 8, 8 blk + 24)
//     (K = 32, exact for bands <= 12).  Input-row statistics come from the split kernel.
// Both operands are K-major SWIZZLE_NONE ("interleave") shared-memory tiles:
//   * B is a padded input row stored [ti chunk][x'][8 ti] (16 B per pixel), so a pixel shift dxi is
//     a +16 B start-address change of the descriptor -- no im2col;
//   * A is stored [dxi][chunk][j = dyi + kr - 1][kb to][8 ti], so the kr output rows r of one input row yi
//     (dyi = y0 + r + R - yi, consecutive) form one contiguous 2 KB tile per chunk.
// fp32 accuracy: x = hi + lo with hi = bf16(x), lo = bf16(x - hi) for both operands; the chain adds
// hi.hi + hi.lo + lo.hi (per-term error <= 3 * 2^-18 relative; simulated on c4m in DESIGN.md).
//
// Roles (320 threads): warp 0 lane 0 is the TMA producer (an NA-stage weight ring, one 5-D tensor copy
// per stage, and a 2-stage ring of split input rows, one bulk copy per chunk); warp 1 lane 0 issues the
// MMAs and commits each stage back; warps 2-9 add every input row's TMEM sums into registers (round to
// nearest; the tensor core's own accumulation truncates) and read the correction accumulator; warp 2
// first decides the window of each of the CTA's tiles.
//
// Geometry (chosen per kernel for its max_batch):
//   * rows mode: one CTA per (rows <= kr output rows, orientation block, field); the epilogue runs in the
//     kernel through a shared-memory transpose (coalesced along x);
//   * balanced mode: kr-row tiles; the tiles' input-row chains are concatenated and split into equal runs
//     over <= 148 CTAs (<= 3 pieces per tile on whole grids, up to 12 on thin row slabs); every piece writes its sums to an L2-resident partial
//     buffer and tc_pieces_epilogue_kernel adds the pieces in order and applies the fused epilogue.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "conv_common.cuh"

namespace se2 {

namespace {

constexpr int kTcPadX = 16;    // zero pixels left of x = 0 in the split input rows (>= R)
constexpr int kTcNAMax = 8;    // weight-ring stages (allocated); TcGeom::na of them are used
// The first stage of a chain issues its correction MMAs before waiting for the previous chain's flush
// (the rest interleave main and corrections per K-step, which keeps consecutive MMAs on different TMEM
// accumulators: 0.579 -> 0.524 ms at c4; 1 early stage measured best, 0.511 ms, against 0/2/4/6)
// input rows per main-accumulator chain (flushed to registers after each): 8 / (chunks of the window),
// i.e. 2 rows at K = 32 and 4 rows at K = 16 -- the truncation bound stays rows x S x K/16 <= 124 steps
// of 2^-23 at R 15 (inside R18) and the flush bubbles are halved against flushing every row
constexpr int kTcMaxFlushRows = 16;  // depth of the row-done ring (>= the longest chain: one barrier per row of a chain)
// a weight stage is 32 KB: two filter columns of the 4-chunk window or four of a 2-chunk window (the
// single issuing thread's per-stage work -- barrier wait, descriptors, commit -- is amortised over 12 MMAs)
constexpr uint32_t kTcAStage = 2u * 8u * 2048u;
// filter columns per stage (nwa is 2 or 4: no integer division on the single-thread issue path)
__host__ __device__ constexpr int tc_cols(int nwa) { return nwa == 2 ? 4 : 2; }
// input rows per main-accumulator chain: 8 / nwl
__host__ __device__ constexpr int tc_chain_rows(int nwl, int chain16) { return nwl == 2 ? chain16 : 2; }
constexpr int kTcThreads = 320;   // warp 0: TMA producer, warp 1: MMA issuer, warps 2-9: accumulators / epilogue
constexpr int kTcFlushWarps = 8;
constexpr int kTcMaxPieces = 4;   // pieces per CTA in the balanced mode (<= 3 by construction)
constexpr float kTcNarrowEta = 9.313225746154785e-10f;   // 2^-30: relative bound of the narrow window's dropped taps

struct TcGeom {
    bool nar;    // narrow geometry (16 rows x 8 orientations, per-tile 16- or 32-wide window)
    int kr, kb;  // rows and orientations of the M tile (kr x kb = 128)
    int npad;    // MMA N: nx rounded up to 16
    int nxp;     // padded row length (pixels) of the split input: npad + 2 * kTcPadX
    int nch;     // theta chunks of 8
    int nwin;    // chunks of the stored theta window of one orientation block (classic: 2 or 4; narrow: 4)
    int nj;      // dyi + kr - 1 range: S + 2 (kr - 1)
    int nblk;    // orientation blocks
    size_t a_stage, b_stage, smem;
    int tmem_cols;
    int na;      // weight-ring stages
};

__host__ __device__ inline int tc_chunk0(int blk, int nch, int nwin) {
    return (nwin == nch) ? 0 : ((2 * blk - 1 + nch) % nch);
}
// first chunk of the stored window of block blk: classic as above; narrow: the wide window's first
// chunk blk - 1 (the narrow window is chunks 1, 2 of it)
__host__ __device__ inline int tc_win0(bool nar, int blk, int nch, int nwin) {
    return nar ? (blk - 1 + nch) % nch : tc_chunk0(blk, nch, nwin);
}
// output orientation of M-tile orientation tol of block blk
__host__ __device__ inline int tc_to(bool nar, int blk, int tol, int nt) {
    return nar ? (8 * blk + 4 + tol) % nt : 16 * blk + tol;
}

// narrow geometry where it applies (>= 4 theta chunks, so the 32-wide window has distinct chunks, and
// a band the wide window covers); SE2_TC_NAR=0 keeps the classic geometry (A/B measurements)
bool tc_use_narrow(const se2_kernel_s* k) {
    if (k->nt / 8 < 4 || k->band > 12) return false;
    const char* e = getenv("SE2_TC_NAR");
    return e == nullptr || atoi(e) != 0;
}

TcGeom tc_geom(const se2_kernel_s* k) {
    TcGeom g;
    g.nar = k->tc_nar;   // decided once in conv_tc_prepare
    g.kr = g.nar ? 16 : 8;
    g.kb = 128 / g.kr;
    g.npad = (k->nx + 15) / 16 * 16;
    g.nxp = g.npad + 2 * kTcPadX;
    g.nch = k->nt / 8;
    g.nwin = g.nar ? 4 : (g.nch <= 4 ? g.nch : 4);
    g.nj = k->S + 2 * (g.kr - 1);
    g.nblk = k->nt / g.kb;
    g.a_stage = kTcAStage;   // hi + lo x (2 columns x 4 chunks | 4 columns x 2 chunks), 2 KB per chunk (kr j x kb to x 16 B)
    g.b_stage = (size_t)2 * g.nwin * g.nxp * 16;                     // hi + lo rows
    g.na = getenv("SE2_TC_NA") ? std::max(2, std::min(kTcNAMax, atoi(getenv("SE2_TC_NA")))) : 4;
    size_t pipe = 2 * g.b_stage + g.na * g.a_stage;
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
// ... and its counterpart (SE2_TC_PDL_EARLY=1, an experiment): at the top of each K10 kernel, so that once every
// block of this grid has started the next kernel's blocks may take the SM resources that free up and run to
// their griddepcontrol.wait.  Measured no gain (c4 conv 0.338 vs 0.335 ms): off by default.
__device__ __forceinline__ void tc_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// One lane of a converged warp, chosen with elect.sync: ptxas then knows a single thread runs the role's
// code and emits bare UTCHMMA / UTMALDG / UTCBAR instructions; under `lane == 0` it wraps every one of
// them in its own ELECT / branch loop (6 SASS per MMA on the issue path).
__device__ __forceinline__ bool tc_elect_one() {
    uint32_t e;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
    return e != 0;
}

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
// one filter column of the steady-state chain, as ONE asm block (the compiler wraps every tcgen05 asm
// statement of a single active lane in an elect loop; one block per column amortises it): per K-step the
// correction hi.lo into tc, the main hi.hi into tm, the correction lo.hi into tc.  ah / bh are the hi
// descriptors, alo / blo the hi -> lo descriptor offsets, accm / accc the enable-input flags of the first
// main / correction MMA.
__device__ __forceinline__ void tc_mma_col(uint32_t tc, uint32_t tm, uint64_t ah, uint64_t bh, uint64_t alo,
                                           uint64_t blo, uint32_t idesc, uint32_t accc, uint32_t accm) {
    asm volatile(
        "{\n\t.reg .pred pc, pm, pt;\n\t.reg .b64 al, bl;\n\t"
        "setp.ne.b32 pc, %7, 0;\n\tsetp.ne.b32 pm, %8, 0;\n\tsetp.eq.b32 pt, 0, 0;\n\t"
        "add.s64 bl, %3, %6;\n\tadd.s64 al, %2, %5;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %2, bl, %4, pc;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %3, %4, pm;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], al, %3, %4, pt;\n\t}"
        ::"r"(tc), "r"(tm), "l"(ah), "l"(bh), "r"(idesc), "l"(alo), "l"(blo), "r"(accc), "r"(accm));
}
// two consecutive filter columns (a 2-column stage of a K = 16 window): the second column's operands are
// ah + ae (next column's weights) and bh - 1 (the input row shifted by one pixel = 16 B)
__device__ __forceinline__ void tc_mma_col2(uint32_t tc, uint32_t tm, uint64_t ah, uint64_t bh, uint64_t ae,
                                            uint64_t alo, uint64_t blo, uint32_t idesc, uint32_t accc, uint32_t accm,
                                            uint64_t bstep) {
    asm volatile(
        "{\n\t.reg .pred pc, pm, pt;\n\t.reg .b64 al, bl, a2, b2, al2, bl2;\n\t"
        "setp.ne.b32 pc, %8, 0;\n\tsetp.ne.b32 pm, %9, 0;\n\tsetp.eq.b32 pt, 0, 0;\n\t"
        "add.s64 bl, %3, %7;\n\tadd.s64 al, %2, %6;\n\t"
        "add.s64 a2, %2, %5;\n\tsub.s64 b2, %3, %10;\n\t"
        "add.s64 bl2, b2, %7;\n\tadd.s64 al2, a2, %6;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %2, bl, %4, pc;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %3, %4, pm;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], al, %3, %4, pt;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a2, bl2, %4, pt;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], a2, b2, %4, pt;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], al2, b2, %4, pt;\n\t}"
        ::"r"(tc), "r"(tm), "l"(ah), "l"(bh), "r"(idesc), "l"(ae), "l"(alo), "l"(blo), "r"(accc), "r"(accm), "l"(bstep));
}
__device__ __forceinline__ void tc_commit_u32(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// bounded wait: a pipeline bug traps (a launch error) instead of hanging the device
__device__ __forceinline__ void tc_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    uint32_t spins = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (++spins == (1u << 31)) __trap();
    }
}

struct TcArgs {
    const __nv_bfloat16* xk;   // split input rows: [hl][batch][ny][nch][nxp][8]
    const __nv_bfloat16* wk;   // split weights:    [hl][nblk][S][nwin][nj][kb][8]
    size_t xk_hl, wk_hl;       // elements between the hi and lo halves
    int nx, ny, nt, R, S;
    int npad, nxp, nch, nwin, nj;
    int nar, kr, kb;           // geometry (TcGeom)
    int na;                    // weight-ring stages
    int chain16;               // input rows per main-accumulator chain at K = 16 (power of 2, <= kTcMaxFlushRows)
    uint32_t a_stage, b_stage;
    int pdl_early;             // griddepcontrol.launch_dependents at the top of the kernels (SE2_TC_PDL_EARLY=1; off by default)
    int epi_split;             // pieces epilogue: blocks per (row group, orientation)
    int epi_vec;               // pieces epilogue: 4 outputs per thread with 16-byte loads / stores (tc_epilogue4)
    int diag;                  // timing diagnostics (wrong results): bit 0 = no pixel shift of the B descriptor, bit 1 = MMAs of half the N, bit 2 = no weight loads after the first ring fill
    uint32_t a_tx;             // bytes one weight-stage TMA box delivers (kTcAStage; halved by a timing diagnostic)
    int tmem_cols;
    int rows_out;              // output rows a CTA owns (<= kr; the M tile's remaining rows are discarded)
    int y_lo, y_hi;            // output window (kernel's win_lo / win_hi): rows outside are input-only halos
    // balanced mode (PIECES): kr-row tiles, CTA c takes chain units [c q, (c + 1) q) of the concatenated
    // (tile, input row) list; every piece's sums go to `part` [tile][piece < pt][128][npad]
    int batch, nblk, ngroups, ug, q;
    int pt;                    // piece slots per tile in `part`: ceil(longest chain / q) + 1 (3 on the whole c4 grid)
    float* part;
    // narrow geometry: per (field, input row, chunk) (min v, max |v|) of this launch's input, the weight
    // mass outside each block's narrow window, and the tile counters (instrumentation)
    const float2* stats;
    const float* wout;
    unsigned long long* cnt;
};

// chain length (input rows) of kr-row group g, and the units before it within one (field, block)
__device__ __forceinline__ int tc_group_len(const TcArgs& a, int g) {
    const int y0 = a.y_lo + g * a.kr;
    return min(a.ny - 1, min(a.y_hi - 1, y0 + a.kr - 1) + a.R) - max(0, y0 - a.R) + 1;
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
            pc.y0 = a.y_lo + g * a.kr;
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

// narrow geometry: may tile (field b, block blk, output rows from y0) use the 16-wide window?  Warp-
// collective (every lane returns the decision).  Dropped taps of output (to, y, x): ti outside the
// window, sum <= wout[blk] * max_window |v|; the output is >= its centre tap (W = 1) times v[to, y, x]
// when v >= 0 on the whole window.  Inputs with NaN / Inf / negative entries take the wide window.
__device__ bool tc_tile_narrow(const TcArgs& a, int b, int blk, int y0, int rows) {
    const int lane = threadIdx.x & 31;
    const float wo = a.wout[blk];
    const int ylo = max(0, y0 - a.R), yhi = min(a.ny - 1, y0 + rows - 1 + a.R);
    const int ohi = min(min(a.ny, a.y_hi), y0 + rows) - 1;
    const int c0 = blk, c1 = (blk + 1) % a.nch;
    const float2* st = a.stats + (size_t)b * a.ny * a.nch;
    float wmin = INFINITY, wmax = 0.f, tmin = INFINITY;
    bool finite = true;
#pragma unroll 4
    for (int i = lane; i < (yhi - ylo + 1) * a.nch; i += 32) {
        const int y = ylo + i / a.nch, c = i % a.nch;
        const float2 v = __ldg(st + (size_t)y * a.nch + c);
        finite = finite && isfinite(v.x) && isfinite(v.y);
        wmin = fminf(wmin, v.x);
        wmax = fmaxf(wmax, v.y);
        if (y >= y0 && y <= ohi && (c == c0 || c == c1)) tmin = fminf(tmin, v.x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        wmin = fminf(wmin, __shfl_xor_sync(0xffffffffu, wmin, o));
        wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
        tmin = fminf(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
    }
    finite = __all_sync(0xffffffffu, finite);
    if (wo == 0.f) return true;   // nothing outside the narrow window (band <= 4)
    return finite && wmin >= 0.f && tmin > 0.f && wo * wmax <= kTcNarrowEta * tmin;
}

// input split: v[b][ti][y][x] (fp32) -> hi/lo bf16 rows [b][y][chunk][x' = x + kTcPadX][8]; one block per
// (field, row, chunk), one padded pixel per thread (all 8 plane loads in flight); optionally the row's
// (min v, max |v|) over the 8 planes and the nx real pixels (stats[b][y][chunk])
__global__ void tc_split_input_kernel(const float* __restrict__ v, __nv_bfloat16* __restrict__ xk, size_t xk_hl,
                                      int nx, int ny, int nt, int nxp, float2* __restrict__ stats, int pdl_early) {
    __shared__ float sMin[32], sMax[32];
    if (pdl_early) tc_launch_dependents();
    tc_grid_dep_wait();   // reads the previous kernel's output (launched with PDL)
    const int nch = nt / 8;
    const int64_t row = blockIdx.x;   // (b, y, c)
    const int c = (int)(row % nch);
    const int64_t by = row / nch;
    const int y = (int)(by % ny);
    const int b = (int)(by / ny);
    float mn = INFINITY, mx = 0.f;
    for (int xp = threadIdx.x; xp < nxp; xp += blockDim.x) {
        const int x = xp - kTcPadX;
        __align__(16) __nv_bfloat16 hi[8], lo[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            float f = 0.f;
            if (x >= 0 && x < nx) {
                f = v[(((int64_t)b * nt + c * 8 + e) * ny + y) * nx + x];
                mn = fminf(mn, f);
                mx = fmaxf(mx, fabsf(f));
                if (f != f) mn = -INFINITY;   // NaN: never the narrow window
            }
            const __nv_bfloat16 h = __float2bfloat16_rn(f);
            hi[e] = h;
            lo[e] = __float2bfloat16_rn(f - __bfloat162float(h));
        }
        const int64_t i = row * nxp + xp;
        reinterpret_cast<uint4*>(xk)[i] = *reinterpret_cast<const uint4*>(hi);
        reinterpret_cast<uint4*>(xk + xk_hl)[i] = *reinterpret_cast<const uint4*>(lo);
    }
    if (stats == nullptr) return;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) { sMin[w] = mn; sMax[w] = mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < nw; ++i) { mn = fminf(mn, sMin[i]); mx = fmaxf(mx, sMax[i]); }
        stats[row] = make_float2(mn, mx);
    }
}

// weight split: Wl[to][ti][S][SP] (fp32) -> hi/lo [blk][dxi][c][j][to_l < kb][8]
__global__ void tc_split_weights_kernel(const float* __restrict__ Wl, __nv_bfloat16* __restrict__ wk, size_t wk_hl,
                                        int nt, int S, int nch, int nwin, int nj, int nblk, int nar) {
    const int SP = (S + 3) / 4 * 4;
    const int kb = nar ? 8 : 16, jofs = 128 / kb - 1;
    const int64_t total = (int64_t)nblk * S * nwin * nj * kb;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int tol = (int)(i % kb);
        int64_t t = i / kb;
        const int j = (int)(t % nj);
        t /= nj;
        const int c = (int)(t % nwin);
        t /= nwin;
        const int dxi = (int)(t % S);
        const int blk = (int)(t / S);
        const int to = tc_to(nar != 0, blk, tol, nt);
        const int chunk = (tc_win0(nar != 0, blk, nch, nwin) + c) % nch;
        const int dyi = j - jofs;
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

// narrow geometry: wout[blk] = max over the block's orientations of the weight mass outside its narrow
// window (chunks blk, blk + 1), summed in fp64 and rounded up.  One block per orientation block.
__global__ void tc_wout_kernel(const float* __restrict__ Wl, float* __restrict__ wout, int nt, int S) {
    __shared__ double sSum[8];
    const int blk = blockIdx.x, nch = nt / 8, SP = (S + 3) / 4 * 4;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;   // 8 warps: one output orientation each
    const int to = tc_to(true, blk, warp, nt);
    double acc = 0.0;
    for (int ti = 0; ti < nt; ++ti) {
        const int c = ti / 8;
        if (c == blk || c == (blk + 1) % nch) continue;
        const float* w = Wl + ((int64_t)to * nt + ti) * S * SP;
        for (int i = lane; i < S * SP; i += 32) acc += (double)w[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) sSum[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int i = 0; i < 8; ++i) m = fmax(m, sSum[i]);
        wout[blk] = m == 0.0 ? 0.f : __double2float_ru(m * (1.0 + 1e-6));
    }
}

template <bool PIECES>
__global__ void __launch_bounds__(kTcThreads, 1)
conv_tc_kernel(TcArgs a, Epilogue epi, const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap wmapn) {
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* sB = smem;                                   // [2][hl][nwl][nxp][16 B]
    unsigned char* sA = smem + 2 * (size_t)a.b_stage;           // [NA][hl][nwl][kr j][kb to][16 B]
    __shared__ __align__(8) uint64_t fullB[2], emptyB[2], fullA[kTcNAMax], emptyA[kTcNAMax], rowdone[kTcMaxFlushRows],
        flushed, cflushed,
        flagbar;
    __shared__ uint32_t tmem_base;
    __shared__ float sRed[kTcThreads / 32];
    __shared__ int sNwl[kTcMaxPieces];   // theta chunks of each piece's window (narrow: 2 or 4; classic: nwin)

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (a.pdl_early) tc_launch_dependents();
    const long long t_entry = (a.diag & 8) ? clock64() : 0;   // SE2_TC_DIAG_PROF

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(a.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < 2; ++i) { mbar_init(&fullB[i], 1); mbar_init(&emptyB[i], 1); }
        for (int i = 0; i < a.na; ++i) { mbar_init(&fullA[i], 1); mbar_init(&emptyA[i], 1); }
        for (int i = 0; i < kTcMaxFlushRows; ++i) mbar_init(&rowdone[i], 1);
        mbar_init(&flushed, kTcFlushWarps);
        mbar_init(&cflushed, kTcFlushWarps);
        mbar_init(&flagbar, 1);
        mbar_fence_init();
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;

    const size_t row_elems = (size_t)a.nch * a.nxp * 8;               // one (b, y) row of the split input
    const uint32_t chunk_bytes_b = (uint32_t)a.nxp * 16;
    if (warp == 0) {
      if (tc_elect_one()) {
        // ---------------- producer ----------------
        // global input-row counter gr (all pieces of this CTA): B ring stage gr & 1, weight stage (gr S + dxi)
        auto load_b = [&](int gr, const TcPiece& pc, int nwl, int yi) {
            const int st = gr & 1;
            if (gr >= 2) tc_wait(&emptyB[st], (uint32_t)(((gr >> 1) - 1) & 1));
            mbar_expect_tx(&fullB[st], 2u * (uint32_t)nwl * chunk_bytes_b);
            const int chunk0 = tc_win0(a.nar != 0, pc.blk, a.nch, a.nwin) + ((a.nar && nwl == 2) ? 1 : 0);
            for (int hl = 0; hl < 2; ++hl) {
                const __nv_bfloat16* row = a.xk + hl * a.xk_hl + ((size_t)pc.b * a.ny + yi) * row_elems;
                for (int c = 0; c < nwl; ++c) {
                    const int ch = (chunk0 + c) % a.nch;
                    bulk_load(sB + st * (size_t)a.b_stage + (size_t)(hl * nwl + c) * chunk_bytes_b,
                              row + (size_t)ch * a.nxp * 8, chunk_bytes_b, &fullB[st]);
                }
            }
        };
        const uint32_t sA_u = smem_u32(sA), fullA_u = smem_u32(&fullA[0]);
        // weight stage t of piece pc (input row yi, filter columns dxi .. dxi + 8 / nwl - 1): one TMA box
        // [hl 2][column 8 / nwl][chunk nwl][j kr][kb to x 8 ti] (32 KB)
        int pst = 0, prnd = 0;   // ring slot and round of the next weight stage (t = prnd * na + pst)
        auto load_a = [&](int t, const TcPiece& pc, int yi, int dxi, int nwl) {
            const int st = pst;
            if (prnd > 0) tc_wait(&emptyA[st], (uint32_t)((prnd - 1) & 1));
            if (++pst == a.na) { pst = 0; ++prnd; }
            if ((a.diag & 4) && t >= a.na) {   // timing diagnostic: no weight traffic after the first ring fill
                mbar_expect_tx(&fullA[st], 0);
                return;
            }
            mbar_expect_tx(&fullA[st], a.a_tx);
            const int j0 = pc.y0 + a.R - yi + a.kr - 1;
            const bool n2 = a.nar && nwl == 2;   // the narrow window of the narrow geometry (second map)
            tma_load_5d(sA_u + (uint32_t)st * a.a_stage, n2 ? (const void*)&wmapn : (const void*)&wmap,
                        fullA_u + 8u * (uint32_t)st, 0, j0, n2 ? 1 : 0, pc.blk * a.S + dxi, 0);
        };
        const int b_after = min((a.na - 1) * tc_cols(a.nwin), a.S - 1);   // filter column that triggers the next row
        TcPiece pc, pn;
        // PDL: the first weight stages do not depend on the preceding kernels (loaded with the full stored
        // window, one filter column each: the tile's window is decided from the split kernel's
        // statistics); the input rows do
        int t = 0, dpre = 0;   // stages issued, filter columns prefetched
        if (tc_piece<PIECES>(a, 0, pc))
            while (dpre < b_after) {
                load_a(t++, pc, pc.ylo + pc.r0, dpre, a.nwin);
                dpre += tc_cols(a.nwin);
            }
        tc_wait(&flagbar, 0);   // warp 2 has passed the grid-dependency wait and decided every piece's window
        tc_grid_dep_wait();
        int gr = 0;
        for (int k = 0; tc_piece<PIECES>(a, k, pc); ++k) {
            const int nwl = sNwl[k];
            const int nd = tc_cols(nwl);   // filter columns per stage
            if (k == 0) load_b(0, pc, nwl, pc.ylo + pc.r0);
            for (int rr = pc.r0; rr < pc.r1; ++rr, ++gr) {
                const int yi = pc.ylo + rr;
                const int d0 = gr == 0 ? dpre : 0;
                bool nextb = false;   // the next input row's B stage has been requested
                for (int dxi = d0; dxi < a.S; dxi += nd) {
                    load_a(t++, pc, yi, dxi, nwl);
                    // the next input row (this piece's, or the next piece's first) after the stage holding
                    // filter column b_after (or the row's first stage when the prefetch passed it)
                    if (!nextb && b_after < dxi + nd) {
                        nextb = true;
                        if (rr + 1 < pc.r1) load_b(gr + 1, pc, nwl, yi + 1);
                        else if (tc_piece<PIECES>(a, k + 1, pn)) load_b(gr + 1, pn, sNwl[k + 1], pn.ylo + pn.r0);
                    }
                }
                if (!nextb) {   // the prefetch covered the whole first row
                    if (rr + 1 < pc.r1) load_b(gr + 1, pc, nwl, yi + 1);
                    else if (tc_piece<PIECES>(a, k + 1, pn)) load_b(gr + 1, pn, sNwl[k + 1], pn.ylo + pn.r0);
                }
            }
        }
      }
      __syncwarp();
    } else if (warp == 1) {
      if (tc_elect_one()) {
        // ---------------- MMA issuer ----------------
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(((a.diag & 2) ? a.npad / 2 : a.npad) >> 3) << 17) |
                               ((uint32_t)(128 >> 4) << 24);
        const uint64_t dA0 = tc_desc(smem_u32(sA), 2048, 128);
        const uint64_t dB0 = tc_desc(smem_u32(sB), chunk_bytes_b, 128);
        const uint32_t tcor = tmem + (uint32_t)(a.tmem_cols / 2);   // correction accumulator (hi.lo + lo.hi)
        uint32_t acc_c = 0;
        int nwl = a.nwin;   // the current piece's window (chunks): K = 8 nwl, nwl / 2 K-steps
        // operand offsets of K-step ks of weight stage st against input-row stage stb, filter column dxi
        // Per stage the descriptors are formed once (the 14-bit start-address fields never carry: shared
        // addresses < 256 KB) and stepped per filter column / K-step: the single issuing thread must stay
        // well ahead of the 128-cycle MMAs.  Stage layout [hl][column e < 4 / nwa][chunk nwa][2 KB].
        const uint64_t aLo = kTcAStage / 2 / 16, aK = 2 * 2048 / 16, bK = 2 * chunk_bytes_b / 16;
        int ist = 0, irnd = 0;   // ring slot and round of the next weight stage to consume
        const uint64_t bstep = (a.diag & 1) ? 0 : 1;   // descriptor step of one pixel (16 B)

        // corrections (hi.lo + lo.hi) of one filter column
        auto issue_corr = [&](uint64_t dAh, uint64_t dBh, uint64_t bLo, int ksteps) {
            for (int ks = 0; ks < ksteps; ++ks) {
                const uint64_t ah = dAh + ks * aK, bh = dBh + ks * bK;
                tc_mma(tcor, ah, bh + bLo, idesc, acc_c);
                acc_c = 1;
                tc_mma(tcor, ah + aLo, bh, idesc, 1);
            }
        };
        auto issue_main = [&](uint64_t dAh, uint64_t dBh, int ksteps, uint32_t acc0) {
            for (int ks = 0; ks < ksteps; ++ks) tc_mma(tmem, dAh + ks * aK, dBh + ks * bK, idesc, ks ? 1u : acc0);
        };
        // steady state: per K-step main (hi.hi), then the two corrections sharing its A / B operand
        auto issue_both = [&](uint64_t dAh, uint64_t dBh, uint64_t bLo, int ksteps, uint32_t acc0) {
            for (int ks = 0; ks < ksteps; ++ks) {
                tc_mma_col(tcor, tmem, dAh + ks * aK, dBh + ks * bK, aLo, bLo, idesc, acc_c, ks ? 1u : acc0);
                acc_c = 1;
            }
        };
        const uint32_t emptyA_u = smem_u32(&emptyA[0]);
        // stages the producer prefetched before the windows were known (the stored window, tc_cols(nwin)
        // filter columns each; mirrors the producer's prefetch loop)
        const int b_after = min((a.na - 1) * tc_cols(a.nwin), a.S - 1);
        const int npre = (b_after + tc_cols(a.nwin) - 1) / tc_cols(a.nwin);
        tc_wait(&flagbar, 0);
        // SE2_TC_DIAG_PROF: cycles the issuer spends in total and waiting on its barriers (cnt[2..6])
        const bool prof = (a.diag & 8) != 0 && a.cnt != nullptr;
        long long pt0 = prof ? clock64() : 0, pwA = 0, pwB = 0, pwF = 0, ptmp = 0;
        TcPiece pc;
        int gr = 0, gs = 0, t = 0;   // input rows, main-accumulator chains and weight stages issued so far
        for (int k = 0; tc_piece<PIECES>(a, k, pc); ++k) {
            nwl = sNwl[k];
            const int fr = tc_chain_rows(nwl, a.chain16);   // input rows per main-accumulator chain (power of 2)
            if (k > 0) {   // the correction accumulator restarts per piece: the previous piece's was read
                if (prof) ptmp = clock64();
                tc_wait(&cflushed, (uint32_t)((k - 1) & 1));
                if (prof) pwF += clock64() - ptmp;
                asm volatile("tcgen05.fence::after_thread_sync;");
                acc_c = 0;
            }
            for (int rr = pc.r0; rr < pc.r1; ++rr, ++gr) {
                const int stb = gr & 1;
                if (prof) ptmp = clock64();
                tc_wait(&fullB[stb], (uint32_t)((gr >> 1) & 1));
                if (prof) pwB += clock64() - ptmp;
                // The main accumulator restarts every fr input rows of a piece and the accumulator warps
                // must first have read the previous chain's sums: the correction MMAs of the row's first
                // stage are issued before that wait so the tensor pipe stays busy.
                const bool restart = ((rr - pc.r0) & (fr - 1)) == 0;
                // chain restart: the corrections of the row's first stage are issued before the wait for
                // the accumulator warps' flush, its main MMAs after it (0-4 such stages measured alike at c4)
                bool early = restart && gs > 0;
                const int ksteps = nwl / 2;
                const uint64_t bLo = (uint64_t)nwl * chunk_bytes_b / 16;
                for (int dxi = 0; dxi < a.S; ++t) {
                    const int st = ist;
                    if (prof) ptmp = clock64();
                    tc_wait(&fullA[st], (uint32_t)(irnd & 1));
                    if (prof) pwA += clock64() - ptmp;
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    if (++ist == a.na) { ist = 0; ++irnd; }
                    const int nwa = t < npre ? a.nwin : nwl;                    // chunks loaded into the stage
                    const int nv = min(tc_cols(nwa), a.S - dxi);               // its filter columns
                    // a narrow tile on a stage prefetched with the wide window reads the middle chunks
                    const uint64_t dAh = dA0 + (uint64_t)((st * a.a_stage + (nwa > nwl ? 2048u : 0u)) >> 4);
                    const uint64_t dBh = dB0 + (uint64_t)((stb * a.b_stage + (bstep ? kTcPadX + a.R - dxi : kTcPadX) * 16) >> 4);
                    const uint64_t aE = (uint64_t)nwa * 2048 / 16;             // next filter column's weights
                    const uint32_t first = (!restart || dxi > 0) ? 1u : 0u;     // enable-input of the chain's first main MMA
                    if (early) {
                        for (int e = 0; e < nv; ++e) issue_corr(dAh + e * aE, dBh - e * bstep, bLo, ksteps);
                        if (prof) ptmp = clock64();
                        tc_wait(&flushed, (uint32_t)((gs - 1) & 1));
                        if (prof) pwF += clock64() - ptmp;
                        asm volatile("tcgen05.fence::after_thread_sync;");
                        for (int e = 0; e < nv; ++e) issue_main(dAh + e * aE, dBh - e * bstep, ksteps, (dxi + e) ? 1u : 0u);
                        early = false;
                    } else if (ksteps == 1) {   // K = 16 windows: two filter columns per asm block
                        int e = 0;
                        for (; e + 1 < nv; e += 2) {
                            tc_mma_col2(tcor, tmem, dAh + e * aE, dBh - e * bstep, aE, aLo, bLo, idesc, acc_c, e ? 1u : first, bstep);
                            acc_c = 1;
                        }
                        if (e < nv) issue_both(dAh + e * aE, dBh - e * bstep, bLo, 1, e ? 1u : first);
                    } else {
                        for (int e = 0; e < nv; ++e) issue_both(dAh + e * aE, dBh - e * bstep, bLo, ksteps, e ? 1u : first);
                    }
                    tc_commit_u32(emptyA_u + 8u * (uint32_t)st);
                    dxi += nv;
                }
                tc_commit(&emptyB[stb]);
                // row-done ring, one barrier per row of a chain: the issuer runs at most one chain ahead
                tc_commit(&rowdone[gr % kTcMaxFlushRows]);
                if (((rr - pc.r0) & (fr - 1)) == fr - 1 || rr == pc.r1 - 1) ++gs;   // chain end
            }
        }
        if (prof) {
            atomicAdd(&a.cnt[2], (unsigned long long)(clock64() - pt0));
            atomicAdd(&a.cnt[3], (unsigned long long)pwA);
            atomicAdd(&a.cnt[4], (unsigned long long)pwB);
            atomicAdd(&a.cnt[5], (unsigned long long)pwF);
            atomicAdd(&a.cnt[6], 1ull);
            atomicAdd(&a.cnt[7], (unsigned long long)(pt0 - t_entry));   // kernel entry -> the issuer's loop
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
        tc_grid_dep_wait();   // statistics, partial / output writes after the preceding kernels (PDL launch)
        {
            // the window of every piece (narrow geometry: decided per tile from the split kernel's row
            // statistics; every piece of a tile takes the same decision): warp 2 + k decides piece k, then
            // warp 2 releases producer and issuer
            if (tc_piece<PIECES>(a, warp - 2, pc)) {
                int nwl = a.nwin;
                if (a.nar) {
                    const int rows = PIECES ? a.kr : a.rows_out;
                    nwl = tc_tile_narrow(a, pc.b, pc.blk, pc.y0, rows) ? 2 : 4;
                    if (lane == 0 && a.cnt != nullptr && pc.r0 == 0) {
                        atomicAdd(&a.cnt[0], 1ull);
                        if (nwl == 4) atomicAdd(&a.cnt[1], 1ull);
                    }
                }
                if (lane == 0) sNwl[warp - 2] = nwl;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kTcFlushWarps * 32) : "memory");   // warps 2-9
            if (warp == 2 && lane == 0)
                asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&flagbar)) : "memory");
        }
        tc_wait(&flagbar, 0);   // every piece's window (sNwl), hence its chain length
        const int q = warp & 3, h = (warp - 2) >> 2;        // TMEM lane quarter (warp % 4) and column half
        const int m = 32 * q + lane;
        const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(h * half);
        int gr = 0;
        for (int k = 0; tc_piece<PIECES>(a, k, pc); ++k) {
            float sum[128];
#pragma unroll
            for (int j = 0; j < 128; ++j) sum[j] = 0.f;
            const int fr = tc_chain_rows(sNwl[k], a.chain16);   // rows per main-accumulator chain (after flagbar: see below)
            for (int rr = pc.r0; rr < pc.r1; ++rr, ++gr) {
                tc_wait(&rowdone[gr % kTcMaxFlushRows], (uint32_t)((gr / kTcMaxFlushRows) & 1));
                if (!(((rr - pc.r0) & (fr - 1)) == fr - 1 || rr == pc.r1 - 1)) continue;   // mid-chain
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
            float* prow = PIECES ? a.part + ((size_t)pc.tile * a.pt + pc.p) * 128 * a.npad + (size_t)m * a.npad + h * half
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
        if ((a.diag & 8) && a.cnt != nullptr && warp == 2 && lane == 0)   // kernel entry -> the last piece's sums stored
            atomicAdd(&a.cnt[8], (unsigned long long)(clock64() - t_entry));
    }
    if (!PIECES) {
        __syncthreads();   // T complete (every warp reaches this; the role warps have finished their loops)
        tc_piece<false>(a, 0, pc);
        if (warp >= 2) {
            const int64_t N = (int64_t)a.nx * a.ny * a.nt;
            const int f = warp - 2;
            for (int mm = 0; mm < 128 / kTcFlushWarps; ++mm) {
                const int m = (128 / kTcFlushWarps) * f + mm;
                const int r = m / a.kb, tol = m % a.kb;
                const int y = pc.y0 + r, to = tc_to(a.nar != 0, pc.blk, tol, a.nt);
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

// apply_epilogue<false> (conv_common.cuh) for 4 consecutive outputs of one row with 16-byte loads / stores: the
// same expressions per output and the same order of the error sum, for the ops of the linear solvers (store,
// divide, multiply, entropic and porous prox), boundary rows to the peer halos / send buffers included.  The scalar form cost ~69 instructions per output and
// made the pieces epilogue issue-bound (ncu: issue active 62%, L2 32%).
__device__ __forceinline__ void tc_epilogue4(const Epilogue& e, int64_t idx, int ix, int iy, const float (&y)[4],
                                             float& err) {
    if (e.err_a != nullptr) {
        const float4 ao = *reinterpret_cast<const float4*>(e.err_a + idx);
        const float4 mu = *reinterpret_cast<const float4*>(e.err_mu + idx);
        err += fabsf(ao.x * y[0] - mu.x);
        err += fabsf(ao.y * y[1] - mu.y);
        err += fabsf(ao.z * y[2] - mu.z);
        err += fabsf(ao.w * y[3] - mu.w);
    }
    float o[4];
    if (e.op == EPI_STORE) {
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = y[j];
    } else if (e.op == EPI_PROX && e.prox_kind == 2) {   // porous medium: safeguarded Newton per output
        float s[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (y[j] < kDivFloor && e.guard != nullptr) atomicAdd(&e.guard[0], 1u);
            const float lz = logf(fmaxf(y[j], kDivFloor));
            bool conv;
            const float u = porous_prox_u(lz, e.prox_lnc, e.prox_m1, &conv);
            if (!conv && e.guard != nullptr) atomicAdd(&e.guard[1], 1u);
            o[j] = expf(u - lz);
            s[j] = expf(u);
        }
        if (e.out2 != nullptr) *reinterpret_cast<float4*>(e.out2 + idx) = make_float4(s[0], s[1], s[2], s[3]);
    } else if (e.op == EPI_PROX) {
        const float dyp = ((float)iy + 0.5f - e.cy) * e.hy;
        float s[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float dxp = ((float)(ix + j) + 0.5f - e.cx) * e.hx;
            const float V = dxp * dxp + dyp * dyp;
            if (y[j] < kDivFloor && e.guard != nullptr) atomicAdd(&e.guard[0], 1u);
            const float z = fmaxf(y[j], kDivFloor);
            o[j] = exp2f(-e.prox_p * log2f(z) - e.prox_q * V * kLog2e);
            s[j] = o[j] * z;
        }
        if (e.out2 != nullptr) *reinterpret_cast<float4*>(e.out2 + idx) = make_float4(s[0], s[1], s[2], s[3]);
    } else {
        const float4 t4 = *reinterpret_cast<const float4*>(e.target + idx);
        const float t[4] = {t4.x, t4.y, t4.z, t4.w};
        if (e.op == EPI_DIVIDE) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (y[j] < kDivFloor && e.guard != nullptr) atomicAdd(&e.guard[0], 1u);
                o[j] = t[j] / fmaxf(y[j], kDivFloor);
            }
        } else {   // EPI_MULTIPLY
#pragma unroll
            for (int j = 0; j < 4; ++j) o[j] = t[j] * y[j];
        }
    }
    const float4 o4 = make_float4(o[0], o[1], o[2], o[3]);
    *reinterpret_cast<float4*>(e.out + idx) = o4;
    if (e.slab_hi > 0) {   // boundary rows into the neighbours' halo rows / the send buffers (as apply_epilogue)
        const int64_t plane = idx / ((int64_t)e.ny_self * e.nx_self);
        if (e.halo_up != nullptr && iy < e.slab_lo + e.slab_halo)
            *reinterpret_cast<float4*>(e.halo_up + (plane * e.ny_up + iy + e.up_shift) * e.nx_self + ix) = o4;
        if (e.halo_dn != nullptr && iy >= e.slab_hi - e.slab_halo)
            *reinterpret_cast<float4*>(e.halo_dn + (plane * e.ny_dn + iy - e.dn_shift) * e.nx_self + ix) = o4;
    }
}

// balanced mode: sum each output's piece partials (1-3, in piece order) and apply the fused epilogue;
// one block per (kr-row group, orientation, field) -- one tile row block -- threads along x (coalesced)
__global__ void __launch_bounds__(256, 4) tc_pieces_epilogue_kernel(TcArgs a, Epilogue epi) {
    __shared__ float sRed[32];
    if (a.pdl_early) tc_launch_dependents();
    tc_grid_dep_wait();   // the partials of the MMA kernel (PDL launch)
    const int g = blockIdx.x / a.epi_split, kpart = blockIdx.x % a.epi_split, to = blockIdx.y, b = blockIdx.z;
    // the M-tile orientation of `to`: classic blocks of 16 from 0; narrow blocks of 8 from 4
    const int u = a.nar ? (to - 4 + a.nt) % a.nt : to;
    const int blk = u / a.kb, tol = u % a.kb, grp = b * a.nblk + blk;
    // the group's unit offset (every thread: a few integer ops per group, no block barrier) and its pieces
    int pre = 0;
    for (int i = 0; i < g; ++i) pre += tc_group_len(a, i);
    const int st = grp * a.ug + pre, len = tc_group_len(a, g);
    const int np = (st + len - 1) / a.q - st / a.q + 1;
    const float* tile = a.part + ((size_t)(grp * a.ngroups + g) * a.pt) * 128 * a.npad;
    const int64_t N = (int64_t)a.nx * a.ny * a.nt;
    // 256 threads: 4 consecutive x per thread (float4 partial loads; npad % 16 == 0), rows r0 + 4 k.
    // Every partial load of the thread is issued before the first use (up to 4 rows x 3 pieces in flight).
    const int x0 = (threadIdx.x & 63) * 4, r0 = threadIdx.x >> 6;
    constexpr int kMaxR = 4;   // rows per thread: kr / 4 <= 4
    float4 v[kMaxR];
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
        const int r = r0 + 4 * k;
        v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r >= a.kr || x0 >= a.npad || (a.epi_split > 1 && k != kpart)) continue;
        const float4* src = reinterpret_cast<const float4*>(tile + (size_t)(r * a.kb + tol) * a.npad + x0);
        const float4 w0 = src[0];
        const float4 w1 = np > 1 ? src[(size_t)32 * a.npad] : make_float4(0.f, 0.f, 0.f, 0.f);   // 128 npad floats
        const float4 w2 = np > 2 ? src[(size_t)64 * a.npad] : make_float4(0.f, 0.f, 0.f, 0.f);   // = 32 npad float4
        v[k].x = (w0.x + w1.x) + w2.x;   // pieces added in order (as before: ((p0 + p1) + p2))
        v[k].y = (w0.y + w1.y) + w2.y;
        v[k].z = (w0.z + w1.z) + w2.z;
        v[k].w = (w0.w + w1.w) + w2.w;
        for (int p = 3; p < np; ++p) {   // thin output windows (row slabs): short runs, up to kTcTilePieces per tile
            const float4 w = src[(size_t)p * 32 * a.npad];
            v[k].x += w.x; v[k].y += w.y; v[k].z += w.z; v[k].w += w.w;
        }
    }
    float err = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxR; ++k) {
        const int r = r0 + 4 * k;
        const int y = a.y_lo + g * a.kr + r;
        if (r >= a.kr || y >= a.y_hi || x0 >= a.nx || (a.epi_split > 1 && k != kpart)) continue;
        const int64_t rowbase = (int64_t)b * N + ((int64_t)to * a.ny + y) * a.nx;
        const float vv[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
        if (a.epi_vec) {   // nx % 4 == 0, 16-byte aligned fields and halo buffers, a vector op (uniform per launch)
            // (a slab epilogue on a kernel without an output window: rows outside the slab are a neighbour's)
            if (epi.slab_hi > 0 && (y < epi.slab_lo || y >= epi.slab_hi)) continue;
            tc_epilogue4(epi, rowbase + x0, x0, y, vv, err);
            continue;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (x0 + j < a.nx) err += apply_epilogue<false>(epi, rowbase + x0 + j, x0 + j, y, vv[j]);
    }
    if (epi.err_partial != nullptr) {
        const float t = block_sum<256>(err, sRed);
        if (threadIdx.x == 0) epi.err_partial[(int64_t)b * (gridDim.x * gridDim.y) + (int64_t)to * gridDim.x + blockIdx.x] = t;
    }
}

}  // namespace

bool conv_tc_eligible(const se2_kernel_s* k) {
    if (getenv("SE2_NO_TC") != nullptr) return false;
    if (k->nt % 16 != 0 || k->nx > 256 || k->R > kTcPadX) return false;
    // the stored window must cover the band: classic 32-wide window (nt > 32) +-8, narrow wide window +-12
    if (k->nt / 8 > 4 && k->band > (tc_use_narrow(k) ? 12 : 8)) return false;
    return true;
}

// output rows per CTA: fewer than the M tile's kr when that fills the SMs in the same number of waves.
// Chosen for the kernel's max_batch so that every launch (and the error-partial layout) uses one geometry.
static int tc_rows_out(const se2_kernel_s* k) {
    const TcGeom g = tc_geom(k);
    int best = g.kr;
    double best_cost = 1e300;
    for (int rows = g.kr; rows >= g.kr / 2; --rows) {
        const double ctas = (double)((k->wrows() + rows - 1) / rows) * g.nblk * k->max_batch;
        const double cost = std::ceil(ctas / 148.0) * std::min(k->ny, rows + 2 * k->R);
        if (cost < best_cost - 1e-9) { best_cost = cost; best = rows; }
    }
    return best;
}

// balanced mode geometry (host mirror of tc_group_len)
static int tc_group_len_h(const se2_kernel_s* k, int kr, int g) {
    const int y0 = k->wlo() + g * kr;
    return std::min(k->ny - 1, std::min(k->whi() - 1, y0 + kr - 1) + k->R) - std::max(0, y0 - k->R) + 1;
}
static int tc_ngroups(const se2_kernel_s* k) {
    const int kr = tc_geom(k).kr;
    return (k->wrows() + kr - 1) / kr;
}
static void tc_units(const se2_kernel_s* k, int batch, int* ug, int* lmax, long long* U) {
    const TcGeom gm = tc_geom(k);
    const int ngroups = tc_ngroups(k);
    *ug = 0;
    *lmax = 0;
    for (int g = 0; g < ngroups; ++g) {
        *ug += tc_group_len_h(k, gm.kr, g);
        *lmax = std::max(*lmax, tc_group_len_h(k, gm.kr, g));
    }
    *U = (long long)batch * gm.nblk * (*ug);
}
// units per CTA in the balanced mode: ceil(U / 148), and long enough that a tile has at most kTcTilePieces
// pieces.  On the whole c4 grid that is 39 of a 46-row chain (<= 3 pieces per tile); on a thin output window
// (one of 8 row slabs: 16 tiles) the runs go down to 5 rows so that all 148 SMs still take part.
constexpr int kTcTilePieces = 12;
static int tc_units_per_cta(const se2_kernel_s* k, int batch) {
    int ug, lmax;
    long long U;
    tc_units(k, batch, &ug, &lmax, &U);
    return (int)std::max<long long>((U + 147) / 148, (lmax + kTcTilePieces - 2) / (kTcTilePieces - 1));
}
// piece slots per tile of a launch: a chain of lmax rows cut into runs of q touches at most this many CTAs
static int tc_tile_pieces(const se2_kernel_s* k, int batch) {
    int ug, lmax;
    long long U;
    tc_units(k, batch, &ug, &lmax, &U);
    const int q = tc_units_per_cta(k, batch);
    return std::max(3, (lmax + q - 1) / q + 1);
}

// pieces epilogue: blocks per (kr-row group, orientation) -- 4 (one of the thread rows r0 + 4 k each) when the
// grid would otherwise leave most SMs without a block (thin output windows: 128 blocks on one of 8 c4 slabs)
static int tc_epi_split(const se2_kernel_s* k) { return tc_ngroups(k) * k->nt < 2 * 148 ? 4 : 1; }

int conv_blocks_per_field_tc(const se2_kernel_s* k) {
    if (k->tc_part != nullptr) return tc_ngroups(k) * tc_epi_split(k) * k->nt;   // balanced: epilogue blocks
    const int rows = tc_rows_out(k);
    return (k->wrows() + rows - 1) / rows * tc_geom(k).nblk;
}

// 5-D tensor map over split weights w: one TMA box per pipeline stage ([hl][chunk nbox][kr j][kb to x 8 ti])
static cudaError_t tc_weight_map(const se2_kernel_s* k, void* w, int nbox, void** map_out) {
    const TcGeom g = tc_geom(k);
    const size_t wk_hl = (size_t)g.nblk * k->S * g.nwin * g.nj * g.kb * 8;
    CUtensorMap* m = new CUtensorMap;
    const uint64_t dims[5] = {(uint64_t)g.kb * 8, (uint64_t)g.nj, (uint64_t)g.nwin, (uint64_t)g.nblk * k->S, 2};
    const uint64_t strides[4] = {(uint64_t)g.kb * 8 * 2, (uint64_t)g.nj * g.kb * 8 * 2,
                                 (uint64_t)g.nwin * g.nj * g.kb * 8 * 2, (uint64_t)wk_hl * 2};
    // 8 / nbox filter columns per box (past the block's last column the box reads the next block's first
    // columns or zero fill, never used)
    // SE2_TC_DIAG_HALFW (timing diagnostic, wrong results): half the weight rows per stage -- does the weight
    // stream (L2 -> shared memory, 2.7 KB per MMA) cost MMA time?
    static const bool halfw = getenv("SE2_TC_DIAG_HALFW") != nullptr;
    const uint32_t box[5] = {(uint32_t)g.kb * 8, (uint32_t)(halfw ? g.kr / 2 : g.kr), (uint32_t)nbox, (uint32_t)tc_cols(nbox), 2};
    if (!make_tmap_5d(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, w, dims, strides, box)) {
        delete m;
        return cudaErrorInvalidValue;
    }
    *map_out = m;
    return cudaSuccess;
}

// split weights + tensor maps (+ the narrow window's outside mass) of one weight table
static cudaError_t tc_build_weights(se2_kernel_s* k, const float* W, void* wk, void** map, void** mapn, float** wout,
                                    cudaStream_t s) {
    const TcGeom g = tc_geom(k);
    cudaError_t e = tc_weight_map(k, wk, g.nwin, map);
    if (e == cudaSuccess && g.nar) e = tc_weight_map(k, wk, 2, mapn);
    if (e != cudaSuccess) return e;
    tc_split_weights_kernel<<<592, 256, 0, s>>>(W, reinterpret_cast<__nv_bfloat16*>(wk), k->tc_w_hl, k->nt, k->S, g.nch,
                                                g.nwin, g.nj, g.nblk, g.nar ? 1 : 0);
    count_launch();
    if (g.nar) {
        e = cudaMalloc(wout, g.nblk * sizeof(float));
        if (e != cudaSuccess) return e;
        tc_wout_kernel<<<g.nblk, 256, 0, s>>>(W, *wout, k->nt, k->S);
        count_launch();
    }
    return cudaGetLastError();
}

// K10 weights of the transport-cost table rho^2 exp(-rho^2/eps) (se2_transport_cost, NEXT #2): same
// layout as the Gibbs weights, built on the first cost evaluation after k->Wcl is tabulated
cudaError_t conv_tc_prepare_cost(se2_kernel_s* k, cudaStream_t s) {
    if (k->tc_w == nullptr || k->tc_wc != nullptr || k->Wcl == nullptr) return cudaSuccess;
    cudaError_t e = cudaMalloc(&k->tc_wc, 2 * k->tc_w_hl * sizeof(__nv_bfloat16));
    if (e != cudaSuccess) return e;
    return tc_build_weights(k, k->Wcl, k->tc_wc, &k->tc_wcmap, &k->tc_wcmapn, &k->tc_woutc, s);
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
        // ((kr + 2R) rows x S taps x K/16 steps x 3 passes x N/2 cycles) at ~70% of the tensor floor,
        // K2 = 2 nnz N flop at ~60 TFLOP/s (0.82 of the FFMA peak).  Narrow geometry: K = 16 assumed.
        const int rows = tc_rows_out(k);
        const double ctas = (double)((k->wrows() + rows - 1) / rows) * g.nblk;
        const double waves = std::ceil(ctas / 148.0);
        const double row_cyc = (double)k->S * ((g.nar ? 2 : g.nwin) / 2) * 3 * (g.npad / 2);   // one input row's chain
        double t10 = waves * std::min(k->ny, rows + 2 * k->R) * row_cyc / 0.7 / 1.9e9 + 8e-6;
        // the balanced mode (chosen below when it is cheaper): q input rows per SM + its epilogue pass
        t10 = std::min(t10, tc_units_per_cta(k, 1) * row_cyc / 0.7 / 1.9e9 + 20e-6);
        const double t2 = 2.0 * (double)k->nnz_taps * k->nx * k->wrows() * k->nt / 60e12 + 4e-6;
        k->tc_fast = getenv("SE2_TC_DEFAULT") ? (atoi(getenv("SE2_TC_DEFAULT")) != 0) : (t10 < t2);
    }
    {
        // balanced mode (kr-row tiles split into equal runs of input rows over 148 CTAs + an epilogue
        // kernel) when its per-SM chain beats the row-count mode's; decided for max_batch
        int ug, lmax;
        long long U;
        tc_units(k, k->max_batch, &ug, &lmax, &U);
        const int q = tc_units_per_cta(k, k->max_batch);
        const int rows = tc_rows_out(k);
        const double ctas = (double)((k->wrows() + rows - 1) / rows) * g.nblk * k->max_batch;
        const double rows_cost = std::ceil(ctas / 148.0) * std::min(k->ny, rows + 2 * k->R);
        const bool want = getenv("SE2_TC_PIECES") ? (atoi(getenv("SE2_TC_PIECES")) != 0) : (q < 0.95 * rows_cost);
        if (want) {
            // tiles x piece slots of the current output window, for every batch size a launch may use
            size_t need = 0;
            for (int b = 1; b <= k->max_batch; ++b)
                need = std::max(need, (size_t)b * g.nblk * tc_ngroups(k) * tc_tile_pieces(k, b));
            need *= (size_t)128 * g.npad * sizeof(float);
            if (k->tc_part == nullptr || need > k->tc_part_bytes) {
                if (k->tc_part != nullptr) cudaFree(k->tc_part);
                k->tc_part = nullptr;
                e = cudaMalloc(&k->tc_part, need);
                if (e != cudaSuccess) return e;
                k->tc_part_bytes = need;
            }
        } else if (k->tc_part != nullptr) {
            cudaFree(k->tc_part);
            k->tc_part = nullptr;
            k->tc_part_bytes = 0;
        }
    }
    return e;
}

cudaError_t conv_tc_prepare(se2_kernel_s* k) {
    if (!conv_tc_eligible(k)) return cudaSuccess;
    k->tc_nar = tc_use_narrow(k);
    const TcGeom g = tc_geom(k);
    const size_t wk_hl = (size_t)g.nblk * k->S * g.nwin * g.nj * g.kb * 8;
    const size_t xk_hl = (size_t)k->max_batch * k->ny * g.nch * g.nxp * 8;
    cudaError_t e = cudaMalloc(&k->tc_w, 2 * wk_hl * sizeof(__nv_bfloat16));
    if (e == cudaSuccess) e = cudaMalloc(&k->tc_x, 2 * xk_hl * sizeof(__nv_bfloat16));
    if (e == cudaSuccess) e = cudaMalloc(&k->tc_stats, (size_t)k->max_batch * k->ny * g.nch * sizeof(float2));
    if (e == cudaSuccess) e = cudaMalloc(&k->tc_cnt, 10 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(k->tc_cnt, 0, 10 * sizeof(unsigned long long));
    if (e != cudaSuccess) return e;
    k->tc_w_hl = wk_hl;
    k->tc_x_hl = xk_hl;
    e = conv_tc_decide(k);
    if (e != cudaSuccess) return e;
    e = tc_build_weights(k, k->Wl, k->tc_w, &k->tc_wmap, &k->tc_wmapn, &k->tc_wout, 0);
    if (e != cudaSuccess) return e;
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
    delete reinterpret_cast<CUtensorMap*>(k->tc_wmapn);
    delete reinterpret_cast<CUtensorMap*>(k->tc_wcmapn);
    if (k->tc_wc) cudaFree(k->tc_wc);
    if (k->tc_part) cudaFree(k->tc_part);
    if (k->tc_wout) cudaFree(k->tc_wout);
    if (k->tc_woutc) cudaFree(k->tc_woutc);
    if (k->tc_stats) cudaFree(k->tc_stats);
    if (k->tc_cnt) cudaFree(k->tc_cnt);
    k->tc_wmap = k->tc_wcmap = k->tc_wc = k->tc_wmapn = k->tc_wcmapn = nullptr;
    k->tc_part = nullptr;
    k->tc_wout = k->tc_woutc = nullptr;
    k->tc_stats = nullptr;
    k->tc_cnt = nullptr;
}

cudaError_t conv_tc_tile_counts(const se2_kernel_s* k, int64_t* tiles, int64_t* wide, bool reset) {
    unsigned long long h[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (k->tc_cnt != nullptr) {
        cudaError_t e = cudaMemcpy(h, k->tc_cnt, sizeof(h), cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && reset) e = cudaMemset(k->tc_cnt, 0, sizeof(h));
        if (e != cudaSuccess) return e;
    }
    if (getenv("SE2_TC_DIAG_PROF") && h[6] > 0)   // issuer cycle profile (timing diagnostic), mean per CTA
        fprintf(stderr, "K10 issuer per CTA: %.0f cycles in its loop; waiting on weights %.0f, input rows %.0f, flushes %.0f (%llu CTAs)\n",
                (double)h[2] / h[6], (double)h[3] / h[6], (double)h[4] / h[6], (double)h[5] / h[6], h[6]);
    if (getenv("SE2_TC_DIAG_PROF") && h[6] > 0)
        fprintf(stderr, "K10 per CTA: %.0f cycles from kernel entry to the issuer's loop, %.0f to the last piece's sums stored\n",
                (double)h[7] / h[6], (double)h[8] / h[6]);
    *tiles = (int64_t)h[0];
    *wide = (int64_t)h[1];
    return cudaSuccess;
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
    float2* stats = g.nar ? reinterpret_cast<float2*>(k->tc_stats) : nullptr;
    // (measured: 0.338 vs 0.335 ms per c4 conv with the early trigger, so it is off by default)
    static const int pdl_early = getenv("SE2_TC_PDL_EARLY") ? 1 : 0;
    static const bool skip_split = getenv("SE2_TC_DIAG_SKIP_SPLIT") != nullptr;   // timing diagnostics only
    if (!skip_split) {
        // one block per (field, row, chunk), one padded pixel per thread: all 8 plane loads in flight
        const long long rows = (long long)batch * k->ny * g.nch;
        // (a 4-pixels-per-thread form with 16-byte plane loads measured no faster, 11.9 vs 11.2 us: each of its
        // store instructions half-fills 32 sectors; this form's stores are fully coalesced)
        const int threads = std::min(1024, (g.nxp + 31) / 32 * 32);
        cudaLaunchConfig_t c = cfg_of(dim3((unsigned)rows), dim3(threads), 0);
        cudaError_t e = cudaLaunchKernelEx(&c, tc_split_input_kernel, in, xk, k->tc_x_hl, k->nx, k->ny, k->nt, g.nxp, stats, pdl_early);
        if (e != cudaSuccess) return e;
        count_launch();
    }
    TcArgs a;
    a.xk = xk;
    const bool cost = epi.table != nullptr;   // the transport-cost table (launch only when tc_wc exists)
    a.wk = reinterpret_cast<const __nv_bfloat16*>(cost ? k->tc_wc : k->tc_w);
    a.xk_hl = k->tc_x_hl;
    a.wk_hl = k->tc_w_hl;
    a.nx = k->nx; a.ny = k->ny; a.nt = k->nt; a.R = k->R; a.S = k->S;
    a.npad = g.npad; a.nxp = g.nxp; a.nch = g.nch; a.nwin = g.nwin; a.nj = g.nj;
    a.nar = g.nar ? 1 : 0;
    a.na = g.na;
    a.chain16 = 4;   // 4 x S x 1 K-step <= 124 truncation steps at R 15 (R18); SE2_TC_CHAIN16: measurements only
    if (getenv("SE2_TC_CHAIN16")) {
        const int c = atoi(getenv("SE2_TC_CHAIN16"));
        if (c == 1 || c == 2 || c == 4 || c == 8 || c == 16) a.chain16 = c;
    }
    a.kr = g.kr;
    a.kb = g.kb;
    a.a_stage = (uint32_t)g.a_stage;
    a.b_stage = (uint32_t)g.b_stage;
    a.epi_vec = 0;
    a.pdl_early = pdl_early;
    a.epi_split = tc_epi_split(k);
    a.diag = (getenv("SE2_TC_DIAG_NOSHIFT") ? 1 : 0) | (getenv("SE2_TC_DIAG_HALFN") ? 2 : 0) |
             (getenv("SE2_TC_DIAG_NOWLOAD") ? 4 : 0) | (getenv("SE2_TC_DIAG_PROF") ? 8 : 0);
    a.a_tx = getenv("SE2_TC_DIAG_HALFW") ? kTcAStage / 2 : kTcAStage;
    a.tmem_cols = g.tmem_cols;
    a.y_lo = k->wlo();
    a.y_hi = k->whi();
    a.stats = stats;
    a.wout = cost ? k->tc_woutc : k->tc_wout;
    a.cnt = k->tc_cnt;
    a.nblk = g.nblk;
    const CUtensorMap* wm = reinterpret_cast<const CUtensorMap*>(cost ? k->tc_wcmap : k->tc_wmap);
    const CUtensorMap* wmn = g.nar ? reinterpret_cast<const CUtensorMap*>(cost ? k->tc_wcmapn : k->tc_wmapn) : wm;
    if (k->tc_part != nullptr) {
        // balanced mode: kr-row tiles, equal runs of chain units per CTA, partials + epilogue kernel
        long long U;
        int lmax;
        tc_units(k, batch, &a.ug, &lmax, &U);
        a.rows_out = g.kr;
        a.batch = batch;
        a.ngroups = tc_ngroups(k);
        a.q = tc_units_per_cta(k, batch);
        a.pt = tc_tile_pieces(k, batch);
        a.part = reinterpret_cast<float*>(k->tc_part);
        const int ncta = (int)((U + a.q - 1) / a.q);
        {
            cudaLaunchConfig_t c = cfg_of(dim3(ncta), dim3(kTcThreads), g.smem);
            cudaError_t e = cudaLaunchKernelEx(&c, conv_tc_kernel<true>, a, epi, *wm, *wmn);
            if (e != cudaSuccess) return e;
        }
        count_launch();
        static const bool scalar_epi = getenv("SE2_TC_EPI1") != nullptr;   // A/B measurements
        auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
        const bool vec_op = epi.op == EPI_STORE || epi.op == EPI_DIVIDE || epi.op == EPI_MULTIPLY || epi.op == EPI_PROX;
        a.epi_vec = (!scalar_epi && vec_op && k->nx % 4 == 0 && al16(epi.halo_up) && al16(epi.halo_dn) &&
                     al16(epi.out) && al16(epi.out2) && al16(epi.target) && al16(epi.err_a) && al16(epi.err_mu))
                        ? 1 : 0;
        static const bool skip_epi = getenv("SE2_TC_DIAG_SKIP_EPI") != nullptr;   // timing diagnostics only
        if (!skip_epi) {
            cudaLaunchConfig_t c = cfg_of(dim3(a.ngroups * a.epi_split, k->nt, batch), dim3(256), 0);
            cudaError_t e = cudaLaunchKernelEx(&c, tc_pieces_epilogue_kernel, a, epi);
            if (e != cudaSuccess) return e;
            count_launch();
        }
        if (bpf) *bpf = a.ngroups * a.epi_split * k->nt;
        return cudaGetLastError();
    }
    a.rows_out = tc_rows_out(k);
    a.batch = batch;
    a.ngroups = 0;
    a.ug = 0;
    a.q = 0;
    a.pt = 0;
    a.part = nullptr;
    dim3 grid((k->wrows() + a.rows_out - 1) / a.rows_out, g.nblk, batch);
    if (bpf) *bpf = (int)(grid.x * grid.y);
    {
        cudaLaunchConfig_t c = cfg_of(grid, dim3(kTcThreads), g.smem);
        cudaError_t e = cudaLaunchKernelEx(&c, conv_tc_kernel<false>, a, epi, *wm, *wmn);
        if (e != cudaSuccess) return e;
    }
    count_launch();
    return cudaGetLastError();
}

}  // namespace se2
