// Elementwise updates and deterministic reductions of the scaling loop (HBM-bound, tiny next to
// the convolutions): barycenter geometric mean (App. A), JKO finish (R10), sums.
#include <math.h>

#include "conv_common.cuh"

namespace se2 {

static inline int grid_for(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    if (b > 148 * 16) b = 148 * 16;
    if (b < 1) b = 1;
    return (int)b;
}

__global__ void fill_kernel(float* x, int64_t n, float v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = v;
}
cudaError_t launch_fill(float* x, int64_t n, float v, cudaStream_t s) {
    fill_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, n, v);
    count_launch();
    return cudaGetLastError();
}

__global__ void log_kernel(const float* x, float* y, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = logf(x[i]);
}
cudaError_t launch_log(const float* x, float* y, int64_t n, cudaStream_t s) {
    log_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, y, n);
    count_launch();
    return cudaGetLastError();
}

// out[b] = sum_{i < nblocks} partial[b][i], fixed order (one block per b) -> deterministic.
__global__ void reduce_partials_kernel(const float* partial, int nblocks, double* out) {
    __shared__ double red[256];
    const int b = blockIdx.x;
    double t = 0.0;
    for (int i = threadIdx.x; i < nblocks; i += blockDim.x) t += (double)partial[(int64_t)b * nblocks + i];
    red[threadIdx.x] = t;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[b] = red[0];
}
cudaError_t launch_reduce_partials(const float* partial, int batch, int nblocks, double* out, cudaStream_t s) {
    reduce_partials_kernel<<<batch, 256, 0, s>>>(partial, nblocks, out);
    count_launch();
    return cudaGetLastError();
}

// lbar[sv][x] = sum_i lam[sv][i] * ld[sv][i][x]  (lambda_i = 0 skipped: d^0 = 1, reading R6)
__global__ void bary_logmean_kernel(int n, int nsolve, int64_t N, const float* ld, const float* lam,
                                    float* lbar) {
    const int64_t total = (int64_t)nsolve * N;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int sv = (int)(t / N);
        const int64_t x = t - (int64_t)sv * N;
        float acc = 0.f;
        for (int i = 0; i < n; ++i) {
            float l = lam[sv * n + i];
            if (l != 0.f) acc += l * ld[((int64_t)sv * n + i) * N + x];
        }
        lbar[t] = acc;
    }
}
cudaError_t launch_bary_logmean(int n, int nsolve, int64_t N, const float* ld, const float* lam_dev, float* lbar,
                                cudaStream_t s) {
    bary_logmean_kernel<<<grid_for((int64_t)nsolve * N, 256), 256, 0, s>>>(n, nsolve, N, ld, lam_dev, lbar);
    count_launch();
    return cudaGetLastError();
}

// lv[sv][i] += lbar[sv] - ld[sv][i]   (App. A: v_i <- v_i mu / d_i, in logs).  log v_i is a running
// sum over the iterations; with lv_lo != null it is carried as an unevaluated fp32 pair (hi, lo)
// (two-sum compensation), so the rounding of a 100-1000 nat potential to fp32 does not accumulate
// into a drift of the gauge; lv (hi) is what the convolutions read.
__global__ void bary_update_log_kernel(int n, int nsolve, int64_t N, float* lv, float* lv_lo, const float* ld,
                                       const float* lbar) {
    const int64_t total = (int64_t)nsolve * n * N;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = t / N;          // field index sv*n + i
        const int64_t x = t - f * N;
        const int sv = (int)(f / n);
        const float dlt = lbar[(int64_t)sv * N + x] - ld[t];
        if (lv_lo == nullptr) {
            lv[t] = lv[t] + dlt;
        } else {
            const float hi = lv[t];
            const float y = dlt + lv_lo[t];
            const float s = hi + y;                        // two-sum (Knuth): s + e == hi + y exactly
            const float bb = s - hi;
            const float e = (hi - (s - bb)) + (y - bb);
            lv[t] = s;
            lv_lo[t] = (s == s && fabsf(s) != INFINITY) ? e : 0.f;
        }
    }
}
// fused single-GPU barycenter step (App. A): per (solve, site) lbar = sum_i lambda_i ld_i (lambda_i = 0
// skipped, R6), then lv_i += lbar - ld_i with the compensated two-sum -- one pass over ld instead of two
__global__ void bary_logmean_update_kernel(int n, int nsolve, int64_t N, const float* __restrict__ ld,
                                           const float* __restrict__ lam, float* __restrict__ lbar,
                                           float* __restrict__ lv, float* __restrict__ lv_lo) {
    const int64_t total = (int64_t)nsolve * N;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int sv = (int)(t / N);
        const int64_t x = t - (int64_t)sv * N;
        float acc = 0.f;
        for (int i = 0; i < n; ++i) {
            const float l = lam[sv * n + i];
            if (l != 0.f) acc += l * ld[((int64_t)sv * n + i) * N + x];
        }
        lbar[t] = acc;
        for (int i = 0; i < n; ++i) {
            const int64_t j = ((int64_t)sv * n + i) * N + x;
            const float dlt = acc - ld[j];
            const float hi = lv[j];
            const float y = dlt + lv_lo[j];
            const float s2 = hi + y;                       // two-sum (Knuth): s2 + e == hi + y exactly
            const float bb = s2 - hi;
            const float e = (hi - (s2 - bb)) + (y - bb);
            lv[j] = s2;
            lv_lo[j] = (s2 == s2 && fabsf(s2) != INFINITY) ? e : 0.f;
        }
    }
}
cudaError_t launch_bary_logmean_update(int n, int nsolve, int64_t N, const float* ld, const float* lam_dev, float* lbar,
                                       float* lv, float* lv_lo, cudaStream_t s) {
    bary_logmean_update_kernel<<<grid_for((int64_t)nsolve * N, 256), 256, 0, s>>>(n, nsolve, N, ld, lam_dev, lbar, lv,
                                                                                   lv_lo);
    count_launch();
    return cudaGetLastError();
}

// sharded barycenter: lbar = sum over ranks of the partial log-means (peer buffers, rank order), then
// lv_i += lbar - ld_i for the local inputs -- the allreduce fused with the update
__global__ void bary_reduce_update_kernel(int nranks, const float* const* __restrict__ parts, int n_local, int64_t N,
                                          float* __restrict__ lv, const float* __restrict__ ld,
                                          float* __restrict__ lbar) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < N; x += (int64_t)gridDim.x * blockDim.x) {
        float acc = 0.f;
        for (int r = 0; r < nranks; ++r) acc += parts[r][x];
        if (lbar != nullptr) lbar[x] = acc;
        for (int i = 0; i < n_local; ++i) lv[(int64_t)i * N + x] += acc - ld[(int64_t)i * N + x];
    }
}
cudaError_t launch_bary_reduce_update(int nranks, const float* const* parts, int n_local, int64_t N, float* lv,
                                      const float* ld, float* lbar, cudaStream_t s) {
    bary_reduce_update_kernel<<<grid_for(N, 256), 256, 0, s>>>(nranks, parts, n_local, N, lv, ld, lbar);
    count_launch();
    return cudaGetLastError();
}

// ---- fp64 state of the precise barycenter (K4P) ----
__global__ void log_f64_kernel(const float* x, double* y, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float v = x[i];
        y[i] = v > 0.f ? log((double)v) : -(double)INFINITY;
    }
}
cudaError_t launch_log_f64(const float* x, double* y, int64_t n, cudaStream_t s) {
    log_f64_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, y, n);
    count_launch();
    return cudaGetLastError();
}
__global__ void fill_f64_kernel(double* x, int64_t n, double v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) x[i] = v;
}
cudaError_t launch_fill_f64(double* x, int64_t n, double v, cudaStream_t s) {
    fill_f64_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, n, v);
    count_launch();
    return cudaGetLastError();
}
// lbar = sum_i lambda_i ld_i (lambda_i = 0 skipped, R6); lv_i += lbar - ld_i  -- in fp64
__global__ void bary_logmean_update_f64_kernel(int n, int nsolve, int64_t N, const double* __restrict__ ld,
                                               const double* __restrict__ lam, double* __restrict__ lbar,
                                               double* __restrict__ lv) {
    const int64_t total = (int64_t)nsolve * N;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int sv = (int)(t / N);
        const int64_t x = t - (int64_t)sv * N;
        double acc = 0.0;
        for (int i = 0; i < n; ++i) {
            const double l = lam[sv * n + i];
            if (l != 0.0) acc += l * ld[((int64_t)sv * n + i) * N + x];
        }
        lbar[t] = acc;
        for (int i = 0; i < n; ++i) {
            const int64_t j = ((int64_t)sv * n + i) * N + x;
            lv[j] += acc - ld[j];
        }
    }
}
cudaError_t launch_bary_logmean_update_f64(int n, int nsolve, int64_t N, const double* ld, const double* lam_dev,
                                           double* lbar, double* lv, cudaStream_t s) {
    bary_logmean_update_f64_kernel<<<grid_for((int64_t)nsolve * N, 256), 256, 0, s>>>(n, nsolve, N, ld, lam_dev, lbar, lv);
    count_launch();
    return cudaGetLastError();
}
// the distributed fp64 barycenter: this rank's partial sum_i lambda_i ld_i (all-reduced over the input ranks
// by the caller), then lv_i += lbar - ld_i
__global__ void bary_logmean_f64_kernel(int n, int nsolve, int64_t N, const double* __restrict__ ld,
                                        const double* __restrict__ lam, double* __restrict__ lbar) {
    const int64_t total = (int64_t)nsolve * N;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int sv = (int)(t / N);
        const int64_t x = t - (int64_t)sv * N;
        double acc = 0.0;
        for (int i = 0; i < n; ++i) {
            const double l = lam[sv * n + i];
            if (l != 0.0) acc += l * ld[((int64_t)sv * n + i) * N + x];
        }
        lbar[t] = acc;
    }
}
cudaError_t launch_bary_logmean_f64(int n, int nsolve, int64_t N, const double* ld, const double* lam_dev,
                                    double* lbar, cudaStream_t s) {
    bary_logmean_f64_kernel<<<grid_for((int64_t)nsolve * N, 256), 256, 0, s>>>(n, nsolve, N, ld, lam_dev, lbar);
    count_launch();
    return cudaGetLastError();
}
__global__ void bary_update_f64_kernel(int n, int nsolve, int64_t N, const double* __restrict__ ld,
                                       const double* __restrict__ lbar, double* __restrict__ lv) {
    const int64_t total = (int64_t)nsolve * n * N;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < total; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = j / N, x = j - f * N;
        lv[j] += lbar[(f / n) * N + x] - ld[j];
    }
}
cudaError_t launch_bary_update_f64(int n, int nsolve, int64_t N, const double* ld, const double* lbar, double* lv,
                                   cudaStream_t s) {
    bary_update_f64_kernel<<<grid_for((int64_t)nsolve * n * N, 256), 256, 0, s>>>(n, nsolve, N, ld, lbar, lv);
    count_launch();
    return cudaGetLastError();
}
__global__ void count_nonfinite_f64_kernel(const double* x, int64_t n, int* count) {
    int c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        c += (isnan(x[i]) || (isinf(x[i]) && x[i] > 0.0)) ? 1 : 0;   // -inf is a valid log(0)
    if (c) atomicAdd(count, c);
}
cudaError_t launch_count_nonfinite_f64(const double* x, int64_t n, int* count_dev, cudaStream_t s) {
    count_nonfinite_f64_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, n, count_dev);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_bary_update_log(int n, int nsolve, int64_t N, float* lv, float* lv_lo, const float* ld,
                                   const float* lbar, cudaStream_t s) {
    bary_update_log_kernel<<<grid_for((int64_t)nsolve * n * N, 256), 256, 0, s>>>(n, nsolve, N, lv, lv_lo, ld, lbar);
    count_launch();
    return cudaGetLastError();
}

// Linear domain: mu = prod_i d_i^lambda_i ; v_i <- v_i * mu / max(d_i, floor); bary = mu.
__global__ void bary_update_lin_kernel(int n, int nsolve, int64_t N, float* v, const float* d, const float* lam,
                                       float* bary, unsigned int* guard) {
    const int64_t total = (int64_t)nsolve * N;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int sv = (int)(t / N);
        const int64_t x = t - (int64_t)sv * N;
        float mu = 1.f;
        for (int i = 0; i < n; ++i) {
            float l = lam[sv * n + i];
            if (l != 0.f) mu *= powf(d[((int64_t)sv * n + i) * N + x], l);
        }
        for (int i = 0; i < n; ++i) {
            int64_t o = ((int64_t)sv * n + i) * N + x;
            if (d[o] < kDivFloor && guard != nullptr) atomicAdd(&guard[0], 1u);   // counted clamp (R9)
            v[o] = v[o] * mu / fmaxf(d[o], kDivFloor);
        }
        bary[t] = mu;
    }
}
cudaError_t launch_bary_update_lin(int n, int nsolve, int64_t N, float* v, const float* d, const float* lam_dev,
                                   float* bary, unsigned int* guard, cudaStream_t s) {
    bary_update_lin_kernel<<<grid_for((int64_t)nsolve * N, 256), 256, 0, s>>>(n, nsolve, N, v, d, lam_dev, bary, guard);
    count_launch();
    return cudaGetLastError();
}

// Deterministic sum: fixed grid of 296 blocks -> fp64 partials -> one block.
constexpr int kSumBlocks = 296;
__global__ void sum_stage1(const float* x, int64_t n, double* part) {
    __shared__ double red[256];
    double t = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        t += (double)x[i];
    red[threadIdx.x] = t;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
__global__ void sum_stage2(const double* part, int nb, double* out) {
    __shared__ double red[256];
    double t = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) t += part[i];
    red[threadIdx.x] = t;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = red[0];
}
cudaError_t launch_sum(const float* x, int64_t n, double* out_dev, double* scratch, cudaStream_t s) {
    sum_stage1<<<kSumBlocks, 256, 0, s>>>(x, n, scratch);
    count_launch();
    sum_stage2<<<1, 256, 0, s>>>(scratch, kSumBlocks, out_dev);
    count_launch();
    return cudaGetLastError();
}

// rows [row0, row0 + rows) of each of the `planes` planes of a [planes][ny][nx] array
__global__ void sum_rows_stage1(const float* x, int planes, int ny, int nx, int row0, int rows, double* part) {
    __shared__ double red[256];
    const int64_t n = (int64_t)planes * rows * nx;
    double t = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = i / ((int64_t)rows * nx);
        const int64_t rem = i - p * rows * nx;
        const int r = (int)(rem / nx), c = (int)(rem - (int64_t)r * nx);
        t += (double)x[(p * ny + row0 + r) * nx + c];
    }
    red[threadIdx.x] = t;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
cudaError_t launch_sum_rows(const float* x, int planes, int ny, int nx, int row0, int rows, double* out_dev,
                            double* scratch, cudaStream_t s) {
    sum_rows_stage1<<<kSumBlocks, 256, 0, s>>>(x, planes, ny, nx, row0, rows, scratch);
    count_launch();
    sum_stage2<<<1, 256, 0, s>>>(scratch, kSumBlocks, out_dev);
    count_launch();
    return cudaGetLastError();
}
__global__ void scale_rows_kernel(float* x, int planes, int ny, int nx, int row0, int rows, double f) {
    const int64_t n = (int64_t)planes * rows * nx;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = i / ((int64_t)rows * nx);
        const int64_t rem = i - p * rows * nx;
        const int r = (int)(rem / nx), c = (int)(rem - (int64_t)r * nx);
        float* e = x + (p * ny + row0 + r) * nx + c;
        *e = (float)((double)*e * f);
    }
}
cudaError_t launch_scale_rows(float* x, int planes, int ny, int nx, int row0, int rows, double f, cudaStream_t s) {
    scale_rows_kernel<<<grid_for((int64_t)planes * rows * nx, 256), 256, 0, s>>>(x, planes, ny, nx, row0, rows, f);
    count_launch();
    return cudaGetLastError();
}

__global__ void scale_kernel(float* x, int64_t n, const double* sum) {
    const double inv = 1.0 / sum[0];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = (float)((double)x[i] * inv);
}
cudaError_t launch_scale(float* x, int64_t n, const double* sum_dev, cudaStream_t s) {
    scale_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, n, sum_dev);
    count_launch();
    return cudaGetLastError();
}

__global__ void count_nonfinite_kernel(const float* x, int64_t n, int* count) {
    int c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        c += (isnan(x[i]) || (isinf(x[i]) && x[i] > 0.f)) ? 1 : 0;   // -inf is a valid log(0)
    if (c) atomicAdd(count, c);
}
cudaError_t launch_count_nonfinite(const float* x, int64_t n, int* count_dev, cudaStream_t s) {
    count_nonfinite_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, n, count_dev);
    count_launch();
    return cudaGetLastError();
}

}  // namespace se2
