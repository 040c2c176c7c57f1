// Internal declarations of the se2ot CUDA library (sm_100a).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "se2ot.h"

namespace se2 {

// thread-local last error message (se2_last_error)
void set_error(const std::string& msg);
// process-wide count of kernel launches issued by this library (se2_launch_count)
void count_launch(int64_t n = 1);

#define SE2_CUDA_TRY(expr)                                                                   \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess) {                                                             \
            ::se2::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));            \
            return SE2_ECUDA;                                                                \
        }                                                                                    \
    } while (0)

#define SE2_CHECK_ARG(cond, msg)                                                             \
    do {                                                                                     \
        if (!(cond)) {                                                                       \
            ::se2::set_error(msg);                                                           \
            return SE2_EINVAL;                                                               \
        }                                                                                    \
    } while (0)

constexpr int kMaxRadius = 15;
constexpr float kDivFloor = 1e-30f;   // division guard (reading R9)
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
// factored log-domain engine (conv_lse_fast.cu): spatial table stored as exp(Ls + kEsShift); a
// channel is handled by the FFMA path when its window range (max over the window - min over the
// tile, natural log units) is at most kFastRange (validity derivation in DESIGN.md, K3)
constexpr float kEsShift = 40.f;
constexpr float kFastRange = 100.f;
constexpr float kShiftAbove = 62.f;   // per-channel shift m = tile min + kShiftAbove
constexpr float kPruneGap = 30.f;     // channels whose upper bound is < lower bound - kPruneGap are skipped
// exact path row pruning (K3): a row of taps is skipped for a warp when its largest possible term is
// more than kRowGap nats below a lower bound of every output of the warp; with a hint h (previous
// output) the shift is h + kHintAbove and the result is accepted only if ly >= h - kHintDrop
constexpr float kRowGap = 25.f;
constexpr int kRowSegs = 3;   // each tap row is pruned in 3 segments of ceil(S/3) taps
constexpr float kHintAbove = 20.f;
constexpr float kHintDrop = 10.f;
constexpr float kDebugHintBias = 60.f;   // SE2_DEBUG_BAD_HINTS: hints read 60 nats too high (tests the redo paths)

// Epilogue ops of the fused conv (see se2_conv_update in se2ot.h)
enum EpiOp : int {
    EPI_STORE = 0,
    EPI_DIVIDE = 1,     // out = target / max(y, floor)   | log: target - ly
    EPI_MULTIPLY = 2,   // out = target * y               | log: target + ly
    EPI_PROX = 3,       // out = max(y,floor)^-p exp(-q V) | log: -p ly - q V
    EPI_ERRONLY = 4,    // no store; only the marginal-error partial
    EPI_DOT = 5,        // no store; partial += a * y (log: exp(alpha + ly)) -- transport cost
};

// Everything an epilogue needs; plain-old-data passed by value to the kernels.
struct Epilogue {
    int op = EPI_STORE;
    const float* table = nullptr;    // table override (cost tables); null = the kernel's Gibbs tables
    // log domain (K3): the previous iteration's output of the same operator, used as the per-output
    // shift of the exact path (skips its max pass; verified, with a two-pass redo); ly is written to
    // hint_out (may alias hint_in: same thread, same index)
    const float* hint_in = nullptr;
    float* hint_out = nullptr;
    const float* target = nullptr;   // [batch][N]
    float* out = nullptr;            // [batch][N]
    float* out2 = nullptr;           // EPI_PROX only: s = prox(z) = b * z (or its log-domain form exp(beta + lz))
    // marginal-error fusion: err += |a_old * y - mu| with a_old = err_a (read before out is written)
    const float* err_a = nullptr;    // [batch][N] (linear a, or alpha in log domain); null = no error
    const float* err_mu = nullptr;   // [batch][N] linear mu
    float* err_partial = nullptr;    // [batch][blocks_per_field]
    // prox (entropy + potential): p = tau/(eps+tau) exponent, q = tau/(eps+tau) potential factor
    int prox_kind = 1;               // 1 entropy + potential, 2 porous medium
    float prox_p = 0.f, prox_q = 0.f;
    float prox_lnc = 0.f, prox_m1 = 0.f; // porous: ln c, c = tau m / (eps (m-1)) cell^{1-m}; m1 = m - 1
    // guard counters (device, k->guard): [0] linear-domain denominators clamped at kDivFloor (R9, SPEC
    // S:219 "counted and reported"), [1] porous prox sites whose safeguarded Newton did not converge
    unsigned int* guard = nullptr;
    float cx = 0.f, cy = 0.f, hx = 0.f, hy = 0.f;
    // slab decomposition with peer-memory halos (se2_conv_update_slab): own rows [slab_lo, slab_hi) of a
    // plane of ny_self x nx_self; slab_hi == 0: off
    int slab_lo = 0, slab_hi = 0, slab_halo = 0, ny_self = 0, nx_self = 0;
    float* halo_up = nullptr;
    int up_shift = 0, ny_up = 0;
    float* halo_dn = nullptr;
    int dn_shift = 0, ny_dn = 0;
};

// Epilogue of the fp64 log-domain engine (K4P, conv_lse_precise.cu): the same ops in fp64
struct EpiP {
    int op = EPI_STORE;
    const double* target = nullptr;  // [batch][N] log targets
    double* out = nullptr;
    const double* err_a = nullptr;   // marginal error |exp(a_old + ly) - mu| (a_old read before out is written)
    const float* err_mu = nullptr;
    float* err_partial = nullptr;    // [batch][blocks_per_field]
};

struct Timing {
    bool on = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;  // pool
    size_t used = 0;
    int64_t all_launches = 0;
};

}  // namespace se2

struct se2_kernel_s {
    int device = 0;
    int nx = 0, ny = 0, nt = 0, R = 0, S = 0;
    double eps = 0, w1 = 0, w2 = 0, w3 = 0;
    double hx = 0, hy = 0;  // cell sizes ([0,1]^2 units)
    int max_batch = 1;
    int band = 0;           // fp32-nonzero theta half band (bins)
    int64_t nnz_taps = 0;   // per output
    int64_t nnz_normal_taps = 0;   // per output: taps whose fp32 value is a normal number (the algorithmic work)
    // device tables, theta-quad interleaved: [nt/4][nt][S][S][4]  (to = 4*qd + q)
    float* Eq = nullptr;    // exp(Ls + kEsShift) fp32, quad-interleaved (factored LSE engine)
    float* Lth = nullptr;   // [nt][nt] theta part of L (natural log)
    float* LseS = nullptr;  // [nt][nt] log sum_taps exp(Ls)
    float* Lq = nullptr;    // -rho^2/eps * log2(e) fp32
    float* LqRow = nullptr; // [nt/4][nt][S][kRowSegs][4] max of Lq over each tap-row segment (exact path)
    float* Wl = nullptr;    // exp(-rho^2/eps) fp32, layout [to][ti][S][SP], SP = S rounded up to 4 (zero pad)
    float* Wcl = nullptr;   // cost tables (built on first se2_transport_cost): rho^2 exp(-rho^2/eps), Wl layout
    float* Lcq = nullptr;   //   and log2(rho^2) + L2, Lq layout
    size_t table_bytes = 0;
    void* extra = nullptr;        // grow-only workspaces (api.cu)
    float* lstats = nullptr;      // [max_batch][nt][tiles][8] per-tile plane fit + ranges of log fields (K3)
    int* lse_counters = nullptr;  // K3 path counters: active, FFMA (incl. tilted), visited, tilted pairs,
                                  // hint redos; [8..11] = two uint64: exact-path rows live / visited
    float* split = nullptr;       // K3 theta_i-split partials (small grids): [groups][max_batch][N]
    size_t split_floats = 0;
    // K10 (conv_tc.cu): BF16 hi/lo split weights [2][nblk][S][nwin][S+14][16][8] and input rows
    // [2][max_batch][ny][nt/8][nx_pad + 32][8]; null when K10 does not apply to this grid
    void* tc_w = nullptr;
    void* tc_x = nullptr;
    size_t tc_w_hl = 0, tc_x_hl = 0;
    void* tc_wmap = nullptr;      // CUtensorMap (5-D) over tc_w: one TMA per weight stage
    void* tc_wc = nullptr;        // the same for the transport-cost table Wcl (built with it)
    void* tc_part = nullptr;      // balanced mode: per-piece partial sums [tiles][pieces per tile][128][npad] (null: off)
    size_t tc_part_bytes = 0;
    void* tc_wcmap = nullptr;
    bool tc_fast = false;         // cost model: K10 beats K2 on this grid (default engine)
    // K10 narrow geometry (nt >= 32): 16 rows x 8 orientations per M tile, a 16-orientation K window per
    // tile when a per-tile bound proves the rest of the band negligible, else the 32-wide window
    bool tc_nar = false;
    void* tc_wmapn = nullptr;     // CUtensorMap boxes of the narrow window (Gibbs / cost weights)
    void* tc_wcmapn = nullptr;
    float* tc_wout = nullptr;     // [nblk] max over the block's orientations of the weight mass outside the narrow window
    float* tc_woutc = nullptr;    //   the same for the cost table
    void* tc_stats = nullptr;     // float2 [max_batch][ny][nt/8]: (min v, max |v|) per input row and theta chunk
    unsigned long long* tc_cnt = nullptr;   // [2] tiles, tiles on the wide window (instrumentation)
    unsigned int* guard = nullptr;  // [4] guard counters (Epilogue::guard), zeroed per solve
    float* L2hi = nullptr;          // K4P: L log2(e) as an exact float pair, Lq layout (built on first use)
    float* L2lo = nullptr;
    float* L2row = nullptr;         // K4P pruning bounds: [nt/4][nt][S][4] max over each tap row of L2hi
    float4* pstats = nullptr;       // K4P channel bounds: per (field, theta, row, 16-column block) (min lv, max lv,
                                    //   min over the finite lv, -)
    void* psplit = nullptr;         // K4P theta_i split partials: double2 (shift, sum) [groups][max_batch][N]
    size_t psplit_n = 0;            //   capacity in double2
    // output window (slab decomposition, se2_kernel_set_window): every conv computes and stores only the
    // output rows [win_lo, win_hi) of each plane; rows outside are input-only halo rows.  Default: all.
    int win_lo = 0, win_hi = 0;
    int wlo() const { return win_lo; }
    int whi() const { return win_hi > 0 ? win_hi : ny; }
    int wrows() const { return whi() - wlo(); }
    se2::Timing timing;
    int64_t N() const { return (int64_t)nx * ny * nt; }
};

namespace se2 {

// conv launchers (conv_linear.cu / conv_lse.cu).  in: [batch][N]; epilogue describes the output.
// returns the number of CTAs per field (for error partial reduction).
cudaError_t launch_conv_linear(const se2_kernel_s* k, const float* in, int batch, const Epilogue& epi,
                               cudaStream_t s, int* blocks_per_field);
cudaError_t launch_conv_lse(const se2_kernel_s* k, const float* in, int batch, const Epilogue& epi,
                            cudaStream_t s, int* blocks_per_field);
int conv_blocks_per_field(const se2_kernel_s* k, bool log_domain, uint32_t flags = 0);
// K10 (conv_tc.cu): tensor-core linear conv; used for the Gibbs-kernel linear conv when prepared
bool conv_tc_eligible(const se2_kernel_s* k);
cudaError_t conv_tc_prepare(se2_kernel_s* k);
cudaError_t conv_tc_decide(se2_kernel_s* k);   // re-run K10's engine / geometry choice (window changes)
void conv_tc_release(se2_kernel_s* k);
cudaError_t conv_tc_prepare_cost(se2_kernel_s* k, cudaStream_t s);
// K10 narrow geometry: tiles launched / tiles that took the wide (32-orientation) window (instrumentation)
cudaError_t conv_tc_tile_counts(const se2_kernel_s* k, int64_t* tiles, int64_t* wide, bool reset);
int conv_blocks_per_field_tc(const se2_kernel_s* k);
cudaError_t launch_conv_tc(const se2_kernel_s* k, const float* in, int batch, const Epilogue& epi, cudaStream_t s,
                           int* bpf);
// K10 when prepared and either forced (SE2_LIN_TC) or predicted faster than K2 (tc_fast, cost model in
// conv_tc.cu); SE2_LIN_FFMA forces K2
inline bool conv_tc_active(const se2_kernel_s* k, uint32_t flags) {
    return k->tc_w != nullptr && (flags & SE2_LIN_FFMA) == 0 && (k->tc_fast || (flags & SE2_LIN_TC) != 0);
}
// a linear conv with this epilogue runs on K10: the Gibbs table, or the cost table once its K10
// weights exist
inline bool conv_tc_route(const se2_kernel_s* k, uint32_t flags, const Epilogue& epi) {
    if (!conv_tc_active(k, flags)) return false;
    return epi.table == nullptr || (epi.table == k->Wcl && k->tc_wc != nullptr);
}
int conv_blocks_per_field_linear(const se2_kernel_s* k);
int conv_blocks_per_field_lse(const se2_kernel_s* k);
// K9 (sinkhorn_small.cu): whole log-domain Sinkhorn of a small grid in one cluster launch
int k9_cluster_size(const se2_kernel_s* k);   // 0: not applicable
cudaError_t launch_sinkhorn_small(const se2_kernel_s* k, const float* mu, const float* nu, float* a, float* b,
                                  int batch, int iters, bool warm, float* err_partial, double* trace, int C,
                                  cudaStream_t s);
cudaError_t launch_conv_lse_fast(const se2_kernel_s* k, const float* in, int batch, const Epilogue& epi,
                                 cudaStream_t s, int* bpf, float* stats, int force_exact, int* counters,
                                 float* split_scratch, size_t split_floats);
size_t lse_fast_stats_floats(const se2_kernel_s* k, int batch);

// K4P (conv_lse_precise.cu): exact log-domain conv, fp64 potentials
cudaError_t launch_conv_lse_precise(const se2_kernel_s* k, const double* in, int batch, const EpiP& epi,
                                    cudaStream_t s, int* bpf);
int conv_blocks_per_field_precise(const se2_kernel_s* k);
cudaError_t tabulate_precise(se2_kernel_s* k, cudaStream_t s);   // L2hi / L2lo on first use

// tabulation (tabulate.cu)
cudaError_t tabulate(se2_kernel_s* k, cudaStream_t s);
cudaError_t tabulate_cost(se2_kernel_s* k, cudaStream_t s);

// elementwise / reductions (elementwise.cu)
cudaError_t launch_fill(float* x, int64_t n, float v, cudaStream_t s);
cudaError_t launch_log(const float* x, float* y, int64_t n, cudaStream_t s);
cudaError_t launch_reduce_partials(const float* partial, int batch, int nblocks, double* out,
                                   cudaStream_t s);
cudaError_t launch_bary_logmean(int n, int nsolve, int64_t N, const float* ld, const float* lam_dev,
                                float* lbar, cudaStream_t s);
cudaError_t launch_bary_reduce_update(int nranks, const float* const* parts, int n_local, int64_t N, float* lv,
                                      const float* ld, float* lbar, cudaStream_t s);
cudaError_t launch_bary_logmean_update(int n, int nsolve, int64_t N, const float* ld, const float* lam_dev, float* lbar,
                                       float* lv, float* lv_lo, cudaStream_t s);
cudaError_t launch_bary_update_log(int n, int nsolve, int64_t N, float* lv, float* lv_lo, const float* ld,
                                   const float* lbar, cudaStream_t s);
cudaError_t launch_bary_update_lin(int n, int nsolve, int64_t N, float* v, const float* d,
                                   const float* lam_dev, float* bary, unsigned int* guard, cudaStream_t s);
cudaError_t launch_sum(const float* x, int64_t n, double* out_dev, double* scratch, cudaStream_t s);
cudaError_t launch_scale(float* x, int64_t n, const double* sum_dev, cudaStream_t s);
cudaError_t launch_sum_rows(const float* x, int planes, int ny, int nx, int row0, int rows, double* out_dev,
                            double* scratch, cudaStream_t s);
cudaError_t launch_scale_rows(float* x, int planes, int ny, int nx, int row0, int rows, double f, cudaStream_t s);
cudaError_t launch_count_nonfinite(const float* x, int64_t n, int* count_dev, cudaStream_t s);
// fp64 state of the precise barycenter
cudaError_t launch_log_f64(const float* x, double* y, int64_t n, cudaStream_t s);
cudaError_t launch_fill_f64(double* x, int64_t n, double v, cudaStream_t s);
cudaError_t launch_bary_logmean_update_f64(int n, int nsolve, int64_t N, const double* ld, const double* lam_dev,
                                           double* lbar, double* lv, cudaStream_t s);
cudaError_t launch_count_nonfinite_f64(const double* x, int64_t n, int* count_dev, cudaStream_t s);
cudaError_t launch_bary_logmean_f64(int n, int nsolve, int64_t N, const double* ld, const double* lam_dev,
                                    double* lbar, cudaStream_t s);
cudaError_t launch_bary_update_f64(int n, int nsolve, int64_t N, const double* ld, const double* lbar, double* lv,
                                   cudaStream_t s);

}  // namespace se2
