/*
 * se2ot.h -- C ABI of the B200-native entropic optimal transport hot path on SE(2)
 *            (arXiv 2402.15322, "Optimal Transport on the Lie Group of Roto-translations").
 *
 * Citations: P:n = line n of the paper text, with the equation label.
 *
 * The library implements ONE thing: the Sinkhorn / convolutional Wasserstein-barycenter
 * scaling loop, whose cost is the application of the Gibbs kernel
 *     K(g) = exp(-rho_b(g)^2 / eps)
 * as a left-invariant SE(2) group convolution
 *     (K v)(g) = sum_h K(h^{-1} g) v(h),   and K^T = K
 * with rho_b the half-angle distance approximation (eq. eq:rhob).
 *
 * Conventions (all entry points):
 *  - Lattice: nx x ny x ntheta on [0,1]^2 x [0,2pi); cell centres x_i = (i+1/2)/nx,
 *    y_j = (j+1/2)/ny, theta_k = 2 pi k/ntheta (readings R1, R2).
 *  - Kernel support: spatial box |ix_g-ix_h| <= radius, |iy_g-iy_h| <= radius, all theta
 *    offsets; zero padding outside the window (R3).
 *  - Field arrays: fp32, contiguous, layout [batch][ntheta][ny][nx] (x fastest), DEVICE
 *    pointers on the kernel's device unless stated otherwise.  The caller owns every array.
 *  - Log-domain state (SE2_LOG_DOMAIN) holds natural logs of the scalings (alpha = log a ...).
 *  - Every call is stream-ordered on `stream` (a cudaStream_t; NULL = legacy default stream).
 *    Calls that return host scalars / traces synchronise that stream before returning.
 *  - No exceptions cross the ABI; errors are returned as se2_status, with a thread-local
 *    message from se2_last_error().  Warnings are >= 100 and leave outputs valid.
 *  - A kernel object may be used by one stream at a time (it owns scratch buffers).
 */
#ifndef SE2OT_H
#define SE2OT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SE2OT_ABI_VERSION 1

#if defined(__GNUC__)
#define SE2_API __attribute__((visibility("default")))
#else
#define SE2_API
#endif

typedef struct CUstream_st* se2_stream; /* == cudaStream_t */

typedef enum {
    SE2_OK = 0,
    SE2_EINVAL = 1,       /* bad argument (null pointer, size, eps <= 0, lambdas off simplex ...) */
    SE2_ENOMEM = 2,       /* device allocation failed                                            */
    SE2_ECUDA = 3,        /* CUDA runtime error (message has the CUDA error string)              */
    SE2_ENCCL = 4,        /* NCCL error / NCCL unavailable (multi-GPU calls)                     */
    SE2_ENONFINITE = 5,   /* NaN/Inf produced by the iteration (SPEC NonFiniteIterate)           */
    SE2_EUNSUPPORTED = 6, /* configuration the kernels do not implement (e.g. radius > 15)       */
    SE2_WKERNEL_TOO_WIDE = 100, /* warning: support box exceeds the grid (call succeeded)        */
    SE2_WGUARD_HIT = 101,       /* warning: the solve clamped linear-domain denominators at 1e-30
                                   (R9; "counted and reported"); se2_guard_stats has the count */
    SE2_WPROX_NOCONV = 102      /* warning: porous-medium prox sites whose safeguarded Newton iteration
                                   missed its tolerance in 64 steps (count in se2_guard_stats)     */
} se2_status;

/* Flags */
#define SE2_LOG_DOMAIN 0x1u   /* state/fields are natural logs; conv is log-sum-exp (R7)      */
#define SE2_WARM_START 0x2u   /* sinkhorn: use the b (beta) array as b^(0) instead of 1;
                                 barycenter: use v_state as the initial v_i (resume)              */
#define SE2_TRACE_ERR 0x4u    /* compute the marginal error every iteration (fused)           */
#define SE2_LSE_EXACT 0x8u    /* log domain: force the exact per-tap log-sum-exp engine (K4; also used for ntheta > 128) */
#define SE2_LSE_NOTILT 0x10u  /* diagnostics: K3 without its gradient-tilted FFMA path           */
#define SE2_LSE_K3EXACT 0x20u /* diagnostics: K3 with every active channel on its exact path     */
#define SE2_NO_GRAPH 0x40u    /* solvers: launch directly instead of replaying a CUDA graph       */
#define SE2_NO_PERSISTENT 0x80u /* se2_sinkhorn: never use the one-launch cluster solver (K9)     */
#define SE2_DEBUG_BAD_HINTS 0x100u /* diagnostics: K3 reads its exact-path hints 60 nats too high, so
                                      every hinted output must take the verified fallback (redo) */
#define SE2_DEBUG_NO_SPLIT 0x200u  /* diagnostics: K3 without the theta_i split (one CTA per tile-quad) */
#define SE2_LIN_FFMA 0x400u        /* linear domain: force the fp32 FFMA conv (K2)                     */
#define SE2_LIN_TC 0x800u          /* linear domain: force the tensor-core conv (K10, 3-pass BF16 split)
                                      on every grid it covers (default: only where its cost model
                                      predicts it beats K2; see se2_kernel_stats.tensor_cores)        */

typedef struct {
    int32_t nx, ny, ntheta;
    double hx, hy;  /* cell sizes in [0,1]^2 units; 0 -> 1/nx, 1/ny.  A slab of a larger grid keeps the
                       global cell size (R1) while ny counts its own rows (+ halos).            */
} se2_grid;

typedef struct {
    double w1, w2, w3; /* left-invariant metric diag(w1^2, w2^2, w3^2) in the frame A1,A2,A3 */
} se2_metric;

typedef struct se2_kernel_s* se2_kernel; /* opaque: device tables + scratch */

typedef struct {
    int64_t box_taps;     /* ntheta * (2r+1)^2: taps per output in the support box                 */
    int64_t nnz_taps;     /* taps per output whose fp32 value is nonzero (the linear path's work)  */
    int32_t theta_band;   /* k: fp32-nonzero theta offsets are |theta_o - theta_i| <= k bins       */
    int32_t radius;
    double zeta;          /* spatial anisotropy max(w1,w2)/min(w1,w2)                      */
    size_t table_bytes;   /* device bytes held by the tables                                       */
    int32_t tensor_cores; /* 1: linear convs with the Gibbs kernel run on the tensor-core engine (K10,
                             3-pass BF16 split) by default; 0: on the fp32 FFMA engine (K2) unless
                             SE2_LIN_TC (2: K10 available on request only)                          */
    int64_t nnz_normal_taps; /* taps per output whose fp32 value is a NORMAL number: the algorithmic work
                             count of the roofline (subnormal taps < 2^-126 are below every retained
                             term's resolution)                                          */
} se2_kernel_stats;

/* ------------------------------------------------------------------------------------------
 * se2_kernel_build -- tabulate the Gibbs kernel once (App. A "K_eps <- exp(-rho_b^2/eps)").
 *   Tables W[to][ti][dy][dx] = exp(-rho_b((0,0,theta_i)^{-1} (dx/nx, dy/ny, theta_o))^2/eps) (fp32,
 *   computed in fp64 and rounded) and its log L = -rho_b^2/eps, on device `device`.
 *   radius: spatial half-width r (support (2r+1)^2), 0 <= r <= 15.
 *   max_batch: largest batch any later call will use (scratch is sized for it; >= 1).
 *   Errors: SE2_EINVAL (null out, eps <= 0, w <= 0, sizes <= 0), SE2_EUNSUPPORTED (r > 15),
 *   SE2_ENOMEM, SE2_ECUDA.  Warning SE2_WKERNEL_TOO_WIDE if 2r+1 > min(nx, ny).
 * ---------------------------------------------------------------------------------------- */
SE2_API se2_status se2_kernel_build(const se2_grid* grid, const se2_metric* metric, double eps, int32_t radius,
                            int32_t max_batch, int32_t device, se2_kernel* out);
SE2_API se2_status se2_kernel_stats_get(se2_kernel k, se2_kernel_stats* out);
SE2_API void se2_kernel_destroy(se2_kernel k); /* idempotent on NULL */

/* Output window of a slab kernel (multi-GPU slab decomposition, B:north_star "split into spatial
 * slabs"): after this call every conv of `k` computes and stores only the output rows
 * [row_lo, row_hi) of each plane (marginal errors / sums likewise); the other rows of the kernel's grid
 * are input-only halo rows holding the neighbours' boundary rows (or zero padding at the global
 * edges).  The tensor-core and FFMA linear engines launch only the window's tiles; the log-domain
 * engines mask their stores.  (0, ny) restores the whole grid.  Errors: SE2_EINVAL. */
SE2_API se2_status se2_kernel_set_window(se2_kernel k, int32_t row_lo, int32_t row_hi);

/* ------------------------------------------------------------------------------------------
 * se2_conv -- y = K v (the same operator serves K^T), batch fields at once.
 *   Linear: out = K in.  SE2_LOG_DOMAIN: out = log(K exp(in)) (exact log-sum-exp).
 *   in, out: device [batch][N]; in != out.  batch <= max_batch.
 * ---------------------------------------------------------------------------------------- */
SE2_API se2_status se2_conv(se2_kernel k, const float* in, float* out, int32_t batch, uint32_t flags,
                    se2_stream stream);

/* Prox of the second marginal term F2 (eq. equ:scaling_iterations). */
typedef enum {
    SE2_PROX_MARGINAL = 0,          /* F2 = indicator{= nu}: prox = nu -> Sinkhorn        */
    SE2_PROX_ENTROPY_POTENTIAL = 1, /* F2 = tau * (sum s(log s - 1) + sum V s): JKO step; */
                                    /* b = z^{-tau/(eps+tau)} exp(-tau V/(eps+tau)) (reading R10)     */
    SE2_PROX_POROUS = 2             /* F2 = tau/(m-1) int rho^m dH, the porous-medium energy of the    */
                                    /* paper's gradient flow, rho = s/cell the density on   */
                                    /* cells of Haar measure dx dy dtheta: s = prox(z) solves per site   */
                                    /* (tau m/(eps(m-1))) (s/cell)^{m-1} + log(s/z) = 0 (Newton in log s)*/
} se2_prox_kind;

typedef struct {
    int32_t kind;        /* se2_prox_kind                                                           */
    double tau;          /* JKO time step                                                           */
    double cx, cy;       /* potential centre in cell units of this (slab) grid                      */
    double hx, hy;       /* cell sizes: V(i,j) = ((i + 1/2 - cx) hx)^2 + ((j + 1/2 - cy) hy)^2      */
    double m;            /* porous-medium exponent m > 1 (SE2_PROX_POROUS only)                      */
} se2_prox;

typedef struct {
    int32_t iters;       /* scaling iterations (fixed count, no early stop; reading R5)             */
    uint32_t flags;      /* SE2_LOG_DOMAIN | SE2_WARM_START | SE2_TRACE_ERR                          */
} se2_opts;

/* ------------------------------------------------------------------------------------------
 * se2_sinkhorn -- scaling iterations:  a = mu / K b ;  b = prox(K^T a) / K^T a,
 *   starting from b^(0) = 1 (or the given b with SE2_WARM_START).  With prox = NULL or
 *   SE2_PROX_MARGINAL this is Sinkhorn (nu required); with
 *   SE2_PROX_ENTROPY_POTENTIAL it is the inner solve of one entropic JKO step (nu ignored).
 *   batch independent problems are solved at once (mu, nu, a, b: [batch][N]).
 *   a, b: outputs (scalings, or alpha = log a, beta = log b under SE2_LOG_DOMAIN).
 *   err_trace_host: nullable host array [iters][batch]; with SE2_TRACE_ERR it receives
 *   e_l = sum |a * K b - mu| after the l-th b-update (R8).  Divisions are guarded at 1e-30 (R9).
 *   Errors: SE2_EINVAL, SE2_ECUDA, SE2_ENONFINITE (checked at the end of the solve).
 * ---------------------------------------------------------------------------------------- */
SE2_API se2_status se2_sinkhorn(se2_kernel k, const float* mu, const float* nu, float* a, float* b, int32_t batch,
                        const se2_prox* prox, const se2_opts* opts, double* err_trace_host,
                        se2_stream stream);

/* ------------------------------------------------------------------------------------------
 * se2_jko_step -- one entropic JKO step = se2_sinkhorn with the entropy+potential or
 *   porous-medium prox, then mu_next = b * K^T a normalised to mass 1 (R10).  mass_host (nullable) receives
 *   sum(b * K^T a) before normalisation.  mu_k, mu_next: [N] device (may not alias).
 * ---------------------------------------------------------------------------------------- */
SE2_API se2_status se2_jko_step(se2_kernel k, const float* mu_k, float* mu_next, float* a, float* b,
                        const se2_prox* prox, const se2_opts* opts, double* mass_host,
                        double* err_trace_host, se2_stream stream);

/* ------------------------------------------------------------------------------------------
 * se2_barycenter -- App. A, iterated Bregman projections:
 *     v_i, w_i <- 1
 *     for j: mu <- 1; for i: w_i <- mu_i / K v_i ; d_i <- v_i K w_i ; mu <- mu d_i^lambda_i
 *            for i: v_i <- v_i mu / d_i
 *   nsolve independent barycenter problems over the SAME n inputs with different weights
 *   (c1: the 5 interpolation weights t -> (t, 1-t)) run batched (nsolve*n fields per conv).
 *   mus: device [n][N] input measures.  lambdas: HOST [nsolve][n], each row on the simplex
 *   within 1e-9 (SE2_EINVAL otherwise); lambda_i = 0 terms are skipped (R6).
 *   bary: device [nsolve][N] output mu (log mu under SE2_LOG_DOMAIN), as returned by App. A.
 *   v_state, w_state: nullable device [nsolve][n][N] outputs (v_i, w_i or their logs).  With
 *   SE2_WARM_START, v_state (required) is also the INPUT: the iteration resumes from those v_i instead of
 *   v_i = 1 (w_i is recomputed from them first): a solve split into calls of j1 and j2 iterations
 *   continues the same iterates as one call of j1 + j2 (up to fp32 rounding: the log-domain running
 *   sum's compensation term restarts at 0).
 *   err_trace_host: nullable host [iters][nsolve]; with SE2_TRACE_ERR receives
 *   sum_i lambda_i sum|w_i K v_i - mu_i| after each v-update (R8).
 * ---------------------------------------------------------------------------------------- */
SE2_API se2_status se2_barycenter(se2_kernel k, int32_t n, int32_t nsolve, const float* mus, const double* lambdas,
                          float* bary, float* v_state, float* w_state, const se2_opts* opts,
                          double* err_trace_host, se2_stream stream);

/* ------------------------------------------------------------------------------------------
 * se2_barycenter_precise -- App. A in the log domain with the potentials held in fp64 and every
 *   conv on K4P (channels within 80 nats on a factored FFMA path whose terms carry only relative rounding;
 *   the rest per tap with exponents exact in fp32 (grid-aligned float pairs, integer shifts); fp64
 *   accumulation; ~1e-7 nats per conv): the engine of the north star's elementwise 1e-4
 *   parity on potentials of 10^2..10^3 nats (reading R19, SURVEY ledger L16).  Same arguments as
 *   se2_barycenter with fp64 outputs: lbary [nsolve][N] = log mu, lv_state / lw_state (nullable)
 *   [nsolve][n][N] = log v_i / log w_i (with SE2_WARM_START lv_state is also the initial log v_i).
 *   SE2_LOG_DOMAIN is implied.  The L2 pair table is built on the first call.
 * se2_conv_precise -- out = log(K exp(in)) on K4P, fp64 fields [batch][N].
 * ---------------------------------------------------------------------------------------- */
SE2_API se2_status se2_barycenter_precise(se2_kernel k, int32_t n, int32_t nsolve, const float* mus,
                                          const double* lambdas, double* lbary, double* lv_state, double* lw_state,
                                          const se2_opts* opts, double* err_trace_host, se2_stream stream);
SE2_API se2_status se2_conv_precise(se2_kernel k, const double* in, double* out, int32_t batch, se2_stream stream);

/* ------------------------------------------------------------------------------------------
 * se2_marginal_error -- err_host[i] = sum_x |a_i(x) (K b_i)(x) - mu_i(x)|  (R8) for
 *   i < batch.  Under SE2_LOG_DOMAIN a, b are logs.  Deterministic two-stage reduction.
 * ---------------------------------------------------------------------------------------- */
SE2_API se2_status se2_marginal_error(se2_kernel k, const float* a, const float* b, const float* mu, int32_t batch,
                              uint32_t flags, double* err_host, se2_stream stream);

/* ------------------------------------------------------------------------------------------
 * se2_transport_cost -- cost_host[i] = <pi_i, c> = sum_{x,y} a_i(x) K(x,y) rho_b(x,y)^2 b_i(y) for the plan
 *   pi = a K b of a scaling solution (R11; the transport term of the entropic W_2^2, P:186-195,
 *   SURVEY NEXT #2) without materialising pi: one conv of b with the cost table K rho^2.  Under
 *   SE2_LOG_DOMAIN a, b are logs.  Cost tables are built on the first call.
 * ---------------------------------------------------------------------------------------- */
SE2_API se2_status se2_transport_cost(se2_kernel k, const float* a, const float* b, int32_t batch, uint32_t flags,
                                      double* cost_host, se2_stream stream);

/* ------------------------------------------------------------------------------------------
 * Step-level entry points (used by the multi-GPU driver, which owns the loop and the collectives).
 * se2_conv_update: out = target (op) K in, fused in the conv epilogue:
 *   op = SE2_EPI_DIVIDE:   out = target / max(K in, 1e-30)     | log: out = target - LSE(in)
 *   op = SE2_EPI_MULTIPLY: out = target * (K in)               | log: out = target + LSE(in)
 *   op = SE2_EPI_PROX:     out = prox(K in)/K in  (JKO proxes, `prox` required; target unused)
 * target: device [batch][N] (log targets under SE2_LOG_DOMAIN).
 * ---------------------------------------------------------------------------------------- */
#define SE2_EPI_DIVIDE 1
#define SE2_EPI_MULTIPLY 2
#define SE2_EPI_PROX 3
SE2_API se2_status se2_conv_update(se2_kernel k, const float* in, const float* target, float* out, int32_t batch,
                           int32_t op, const se2_prox* prox, uint32_t flags, se2_stream stream);

/* Barycenter log-mean pieces (App. A, mu <- prod d_i^lambda_i, v_i <- v_i mu / d_i), in logs:
 *   se2_bary_logmean: lbar[N] = sum_{i<n, lambda_i != 0} lambdas[i] * ld[i][N]   (lambdas HOST)
 *   se2_bary_update:  lv[i] += lbar - ld[i] for i < n.   Log-domain arrays. */
SE2_API se2_status se2_bary_logmean(int32_t n, int64_t N, const float* ld, const double* lambdas, float* lbar,
                            se2_stream stream);
SE2_API se2_status se2_bary_update(int32_t n, int64_t N, float* lv, const float* ld, const float* lbar,
                           se2_stream stream);

/* Slab decomposition with peer-memory halos (a rank's grid rows [r0, r1) plus R halo rows each side):
 * the conv's epilogue stores the output rows [own_lo, own_hi) of this slab only, and ALSO stores
 * rows [own_lo, own_lo + halo) into the upper neighbour's array `up` at row (row + up_shift) and rows
 * [own_hi - halo, own_hi) into the lower neighbour's array `dn` at row (row - dn_shift) (plane strides
 * ny_up / ny_dn rows of nx); up / dn may be null (global edges).  Rows outside [own_lo, own_hi) are
 * not stored and do not enter the marginal error.  The caller orders the peers' writes with a
 * cross-rank barrier before the next conv reads its halos. */
typedef struct {
    int32_t own_lo, own_hi, halo;
    float* up;
    int32_t up_shift, ny_up;
    float* dn;
    int32_t dn_shift, ny_dn;
} se2_slab;
SE2_API se2_status se2_conv_update_slab(se2_kernel k, const float* in, const float* target, float* out, int32_t batch,
                                        int32_t op, const se2_prox* prox, uint32_t flags, const se2_slab* slab,
                                        se2_stream stream);

/* Fused cross-rank log-mean reduction + v-update of the sharded barycenter (App. A with the inputs
 * spread over ranks; the allreduce and the update in ONE kernel reading the peers' buffers directly):
 *   lbar[x] = sum_{r < nranks} partials[r][x]      (rank order -> bit-identical on every rank)
 *   lv[i][x] += lbar[x] - ld[i][x]                 for the n_local inputs of this rank (may be 0)
 * partials_dev: DEVICE array of nranks device pointers to [N] fp32 buffers -- normally the peers'
 * buffers mapped into this process (symmetric memory / CUDA IPC over NVLink); every buffer must be
 * complete before the call (the caller's cross-rank barrier).  lbar: [N] out (may alias nothing). */
SE2_API se2_status se2_bary_reduce_update(int32_t nranks, const float* const* partials_dev, int32_t n_local,
                                          int64_t N, float* lv, const float* ld, float* lbar, se2_stream stream);

/* Rows [row0, row0 + rows) of every plane of a [planes][ny][nx] device array (slab decomposition):
 * deterministic fp64 sum to the host, and in-place scaling by `factor`. */
SE2_API se2_status se2_sum_rows(const float* x, int32_t planes, int32_t ny, int32_t nx, int32_t row0, int32_t rows,
                                double* out_host, se2_stream stream);
SE2_API se2_status se2_scale_rows(float* x, int32_t planes, int32_t ny, int32_t nx, int32_t row0, int32_t rows,
                                  double factor, se2_stream stream);

/* Sum of a device array (deterministic), result in double on the host. */
SE2_API se2_status se2_sum(const float* x, int64_t n, double* out_host, se2_stream stream);

/* Log-domain engine (K3) path counters since the last reset: (tile-quad, theta_i) pairs that were
 * active after pruning, handled by an FFMA path (plain or gradient-tilted), visited in total, handled
 * by the tilted FFMA path, and CTAs whose hinted exact-path shift failed verification (redone). */
SE2_API se2_status se2_lse_path_stats(se2_kernel k, int64_t* active_pairs, int64_t* ffma_pairs,
                                      int64_t* visited_pairs, int64_t* tilted_pairs, int64_t* hint_redos,
                                      int32_t reset);

/* K3 exact-path row pruning counters since the last reset (synchronises the device): tap-row
 * segments (warp, input orientation, dy, one of 3 dx segments) evaluated / visited.  A segment is
 * skipped when its largest possible term lies more than 25 nats below a lower bound of every output
 * of the warp (K3). */
SE2_API se2_status se2_lse_row_stats(se2_kernel k, int64_t* rows_live, int64_t* rows_visited, int32_t reset);

/* Tensor-core linear conv (K10), narrow geometry (nt >= 32; K10): tiles computed since the
 * last reset, and those among them that took the 32-orientation window because the tile's bound
 * (taps outside the 16-orientation window <= 2^-30 of every output) did not hold.  Synchronises the
 * device.  Both counts are 0 for kernels without K10 or with the classic geometry. */
SE2_API se2_status se2_tc_tile_stats(se2_kernel k, int64_t* tiles, int64_t* wide_tiles, int32_t reset);

/* fp64-potential log-domain engine (K4P, se2_barycenter_precise): (CTA, input orientation) channels that
 * took the factored FFMA path / all channels visited, and CTAs whose hinted shifts failed verification and
 * were redone two-pass, since the last reset (synchronises the device). */
SE2_API se2_status se2_precise_path_stats(se2_kernel k, int64_t* ffma_channels, int64_t* channels, int64_t* hint_redos,
                                          int32_t reset);

/* Instrumentation: when enabled, every conv launch is bracketed by CUDA events on its stream;
 * se2_timing_get returns the number of conv launches and their summed device time (ms)
 * since the last reset (synchronises the events). */
SE2_API se2_status se2_timing_enable(se2_kernel k, int32_t on);
SE2_API se2_status se2_timing_get(se2_kernel k, int64_t* n_launches, double* conv_ms, int64_t* all_launches);

/* Guard counters of the kernel object since its last solve started (se2_sinkhorn / se2_jko_step /
 * se2_barycenter reset them; step-level calls such as se2_conv_update accumulate): linear-domain
 * denominators clamped at 1e-30 (R9) and porous prox sites without convergence.  reset != 0
 * zeroes them after reading.  Synchronises the device. */
SE2_API se2_status se2_guard_stats(se2_kernel k, int64_t* div_clamps, int64_t* prox_noconv, int32_t reset);

/* Number of kernel launches this library has issued in this process (all entry points). */
SE2_API int64_t se2_launch_count(void);

/* ------------------------------------------------------------------------------------------
 * Lifting and projection: images and orientation fields <-> measures on the
 * SE(2) grid.  A lifting context (se2_cake) owns the cake-wavelet bank and the reduction scratch of
 * these calls; all arrays are device fp32, images [batch][ny][nx], SE(2) fields
 * [batch][ntheta][ny][nx] (theta_k = 2 pi k / ntheta), contiguous, caller-owned.  Calls returning
 * host scalars synchronise the stream.
 *
 * se2_cake_build -- cake wavelets (App. B; reading R15): in the Fourier domain on the
 *   size x size DFT lattice omega = 2 pi k / size,
 *     psi^_j(omega) = B_deg( wrap(arg omega - theta_j - pi/2) / (2 pi / ntheta) ) W(|omega|),
 *     W(rho) = 1 for rho <= c pi, exp(-(rho - c pi)^2 / (2 ((1 - c) pi / 2)^2)) beyond,  psi^_j(0) = 1/ntheta,
 *   B_deg the centred cardinal B-spline, c = radial_cut; the table is Re psi_j(d) =
 *   size^-2 sum_omega psi^_j(omega) cos(omega . d), d in [-R, R]^2 (size = 2R + 1 odd), computed on the
 *   device in fp64.  Requires ntheta >= spline_degree + 1, 0 <= spline_degree <= 7, 0 < radial_cut < 1.
 * se2_lift_image -- orientation score (eq. `eq:lift`): U[b][j][y][x] = sum_d Re psi_j(d)
 *   f[b][y + dy][x + dx], zero padding outside the image.
 * se2_split_signed -- (eq. `eq:tildeW-v1`): Upos = max(U, 0) / m+, Uneg = max(-U, 0) / m-
 *   per field of n elements; masses_host[b][0..1] = (m+, m-) in fp64; a part with zero mass is all zeros.
 *   floor_rel > 0 adds floor_rel * max(part) to every site of a nonempty part before normalising (the
 *   configs' "1e-6 floor" input recipe; keeps the log-domain App. A iteration off empty windows, R17).
 * se2_project -- (eq. `eq:proj`): img[b][y][x] = sum_j U[b][j][y][x].
 * se2_project_signed -- (eq. `eq:final`): img = max(m+ P(Upos) - m- P(Uneg), 0) / sum, the
 *   "dominant positive response" normalised to mass 1; masses from se2_split_signed (host [batch][2]);
 *   mass_host[b] = the sum before normalisation (0 -> img all zeros).
 * se2_lift_field -- orientation-field lift (eq. `equ:lifting_vector_field`): U[b][k][y][x] =
 *   mag / m if k is the bin of angle (d_S1(angle, theta_k) < pi/ntheta, the lower bin at exactly pi/ntheta,
 *   reading R16; decided in fp64 as k = ceil(wrap_[0,2pi)(angle) ntheta / 2pi - 1/2) mod ntheta), else 0;
 *   m = sum mag (mass_host[b]).  mag must be >= 0.
 * se2_reconstruct_field -- (eq. `equ:reconstruction_vector_field`): mag = sum_k U, angle =
 *   theta of the first maximum over k; sites with mag < threshold or mag == 0 get (0, 0).
 * ---------------------------------------------------------------------------------------- */
typedef struct se2_cake_s* se2_cake; /* opaque lifting context */
SE2_API se2_status se2_cake_build(int32_t ntheta, int32_t size, int32_t spline_degree, double radial_cut,
                                  int32_t device, se2_cake* out);
SE2_API se2_status se2_cake_get(se2_cake c, float* table_host /* ntheta*size*size, nullable */, int32_t* ntheta,
                                int32_t* size);
SE2_API void se2_cake_destroy(se2_cake c);
SE2_API se2_status se2_lift_image(se2_cake c, const float* f, float* U, int32_t nx, int32_t ny, int32_t batch,
                                  se2_stream stream);
SE2_API se2_status se2_split_signed(se2_cake c, const float* U, float* Upos, float* Uneg, int64_t n, int32_t batch,
                                    double floor_rel, double* masses_host, se2_stream stream);
SE2_API se2_status se2_project(se2_cake c, const float* U, float* img, int32_t nx, int32_t ny, int32_t batch,
                               se2_stream stream);
SE2_API se2_status se2_project_signed(se2_cake c, const float* Upos, const float* Uneg, const double* masses_host,
                                      float* img, int32_t nx, int32_t ny, int32_t batch, double* mass_host,
                                      se2_stream stream);
/* se2_interp_masses -- Step 4 of the image interpolation: the +/- masses of b_t linearly
 *   interpolated between the two images', m_t = (1 - t) m(f0) + t m(f1), for each t (host arrays:
 *   masses [2][2] from se2_split_signed of the two images, ts [nts], out [nts][2]).  t in [0, 1]. */
SE2_API se2_status se2_interp_masses(const double* masses_host, const double* ts_host, int32_t nts, double* out_host);
SE2_API se2_status se2_lift_field(se2_cake c, const float* angle, const float* mag, float* U, int32_t nx, int32_t ny,
                                  int32_t batch, double* mass_host, se2_stream stream);
SE2_API se2_status se2_reconstruct_field(se2_cake c, const float* U, float* angle, float* mag, int32_t nx, int32_t ny,
                                         int32_t batch, float threshold, se2_stream stream);
/* y[i] = exp(x[i]) (expf), e.g. a log-domain barycenter -> the measure the projection takes. */
SE2_API se2_status se2_exp(const float* x, float* y, int64_t n, se2_stream stream);
/* y[i] = log(x[i]) (logf; log 0 = -inf), e.g. measures -> log-domain targets. */
SE2_API se2_status se2_log(const float* x, float* y, int64_t n, se2_stream stream);

/* ------------------------------------------------------------------------------------------
 * Multi-GPU (B:north_star: "independent barycenter inputs ... go per GPU, with an NCCL allreduce over
 * NVLink for the barycenter log-mean, and a single large grid is split into spatial slabs with NVLink
 * halo exchange").  One rank per GPU (one process each); every rank calls every function below
 * collectively, in the same order.
 *
 * se2_comm_unique_id -- 128-byte NCCL unique id (rank 0 creates it, the caller broadcasts it, e.g. with
 *   torch.distributed).  NCCL is resolved at run time (dlopen libnccl.so.2; the build torch loaded is
 *   reused).  Errors: SE2_ENCCL (no NCCL).
 * se2_comm_init -- communicator of nranks ranks on `device` (ncclCommInitRank; nranks = 1 needs no id
 *   and no NCCL -- given an id it still builds a one-rank NCCL communicator and the solvers run their
 *   collectives on it: the NCCL transport on one GPU).  se2_comm_init_loopback -- nranks communicators in ONE process on one device (out
 *   [nranks]), each to be driven by its own host thread: the exchanges are device copies / reductions
 *   ordered by CUDA events and host rendezvous (no kernel waits on another rank's kernel) -- the test
 *   transport of the multi-rank logic on one GPU.
 * se2_comm_split -- sub-communicator of the ranks with the same color, ordered by key (ncclCommSplit);
 *   c3 on 8 GPUs: color = slab index -> the 4 input ranks of a slab (log-mean allreduce), color = input
 *   -> the 2 slab ranks of an input (halo exchange).
 * se2_comm_allreduce -- in-place sum of count floats (f64 = 0) or doubles over the ranks.
 * ---------------------------------------------------------------------------------------- */
typedef struct se2_comm_s* se2_comm;
#define SE2_COMM_ID_BYTES 128
SE2_API se2_status se2_comm_unique_id(uint8_t* id_out /* SE2_COMM_ID_BYTES */);
SE2_API se2_status se2_comm_init(const uint8_t* id, int32_t nranks, int32_t rank, int32_t device, se2_comm* out);
SE2_API se2_status se2_comm_init_loopback(int32_t nranks, int32_t device, se2_comm* out /* [nranks] */);
SE2_API se2_status se2_comm_split(se2_comm parent, int32_t color, int32_t key, se2_comm* out);
SE2_API se2_status se2_comm_info(se2_comm c, int32_t* nranks, int32_t* rank);
SE2_API se2_status se2_comm_allreduce(se2_comm c, void* buf, int64_t count, int32_t f64, se2_stream stream);
SE2_API void se2_comm_destroy(se2_comm c); /* idempotent on NULL */

/* Decomposition of one rank.  The kernel is built on the LOCAL grid: the rank's owned rows plus halo_top
 * rows above and halo_bot rows below (halo = R toward a neighbour slab, 0 at a global edge; cell sizes of
 * the global grid, R1), and its output window is set to the owned rows.  Fields are local arrays
 * [..][ntheta][halo_top + rows + halo_bot][nx]. */
typedef struct {
    se2_comm reduce;     /* ranks whose inputs form the same barycenters (allreduce of the log-mean); NULL: none */
    se2_comm slabs;      /* the row slabs of the same fields, rank order = row order; NULL: the whole grid */
    int32_t halo_top, halo_bot;
} se2_dist;

/* se2_jko_step_dist -- se2_jko_step on a row slab: per inner iteration two convs over the owned rows,
 *   each followed by the exchange of R boundary rows with the neighbour slabs (packed by the conv
 *   epilogue); mass and error trace summed over the slabs (the same values on every rank).  mu_next's
 *   halo rows are zero.  One rank (dist with NULL communicators) is se2_jko_step exactly. */
SE2_API se2_status se2_jko_step_dist(se2_kernel k, const se2_dist* dist, const float* mu_k, float* mu_next, float* a,
                                     float* b, const se2_prox* prox, const se2_opts* opts, double* mass_host,
                                     double* err_trace_host, se2_stream stream);
/* se2_barycenter_dist -- App. A (log domain) with this rank's n inputs (mus [n][N_local], lambdas HOST
 *   [nsolve][n]: this rank's share of weights that sum to 1 over all `reduce` ranks); per iteration one
 *   allreduce of the partial sum_i lambda_i log d_i over `reduce` and, with slabs, halo exchanges of w_i and
 *   v_i.  bary: [nsolve][N_local] log mu on every rank.  Trace: sum over all inputs and slabs. */
SE2_API se2_status se2_barycenter_dist(se2_kernel k, const se2_dist* dist, int32_t n, int32_t nsolve, const float* mus,
                                       const double* lambdas, float* bary, float* v_state, float* w_state,
                                       const se2_opts* opts, double* err_trace_host, se2_stream stream);

/* se2_barycenter_precise_dist -- se2_barycenter_precise (fp64 potentials, K4P) with this rank's n inputs
 *   (mus [n][N] float, lambdas HOST [nsolve][n]: this rank's share of weights that sum to 1 over all `reduce`
 *   ranks); per iteration one fp64 allreduce of the partial sum_i lambda_i log d_i over `reduce` and, with
 *   `slabs`, exchanges of the fp64 w_i / v_i boundary rows (R rows toward each neighbour; the kernel is built on
 *   the local grid as for se2_barycenter_dist).  lbary [nsolve][N_local] (fp64 log barycenter; its owned rows
 *   on every rank of the slab), lv_state / lw_state [nsolve][n][N_local] fp64 (nullable).  Trace: the
 *   lambda-weighted error summed over all ranks' inputs and slabs. */
SE2_API se2_status se2_barycenter_precise_dist(se2_kernel k, const se2_dist* dist, int32_t n, int32_t nsolve,
                                               const float* mus, const double* lambdas, double* lbary, double* lv_state,
                                               double* lw_state, const se2_opts* opts, double* err_trace_host,
                                               se2_stream stream);

SE2_API const char* se2_last_error(void);
SE2_API int32_t se2_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SE2OT_H */
