// Lifting and projection (include/se2ot.h "Lifting and projection"):
//   cake-wavelet tabulation (fp64, on the device), orientation score (direct correlation), +/- split
//   with deterministic mass reductions, theta projection, signed recombination, orientation-field
//   lift and argmax reconstruction.  Every step runs here; the host only validates and orders launches.
// Citations: P:n = PAPER.md line n (eq. labels in DESIGN.md).  Readings R15 (cake wavelets), R16 (bin
// boundary) in DESIGN.md.
#include <math.h>

#include <string>

#include "se2_internal.cuh"

using namespace se2;

struct se2_cake_s {
    int device = 0;
    int nt = 0, L = 0, R = 0, degree = 0;
    double cut = 0;
    float* table = nullptr;     // [nt][L][L]  Re psi_j(dy, dx)
    double* scratch = nullptr;  // reduction partials / masses (grow-only)
    size_t scratch_n = 0;
};

namespace {

constexpr double kTwoPi = 6.283185307179586476925286766559;
constexpr double kPi = 3.1415926535897932384626433832795;

struct Guard {
    int prev = -1;
    explicit Guard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~Guard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// centred cardinal B-spline of degree k by the truncated-power sum
//   B_k(x) = 1/k! sum_{i=0}^{k+1} (-1)^i C(k+1, i) (x + (k+1)/2 - i)_+^k
__device__ double bspline_tp(double x, int k) {
    if (k == 0) return (x >= -0.5 && x < 0.5) ? 1.0 : 0.0;
    const double h = 0.5 * (k + 1);
    if (x <= -h || x >= h) return 0.0;
    double acc = 0.0, binom = 1.0, fact = 1.0;
    for (int i = 2; i <= k; ++i) fact *= i;
    for (int i = 0; i <= k + 1; ++i) {
        const double t = x + h - i;
        if (t > 0.0) {
            double p = 1.0;
            for (int e = 0; e < k; ++e) p *= t;
            acc += ((i & 1) ? -binom : binom) * p;
        }
        binom = binom * (double)(k + 1 - i) / (double)(i + 1);
    }
    const double v = acc / fact;
    return v > 0.0 ? v : 0.0;
}

// Re psi_j(dy, dx) = L^-2 sum_{k2, k1} psi^_j(omega) cos(omega_x dx + omega_y dy), one thread per entry
__global__ void cake_tabulate_kernel(int nt, int L, int degree, double cut, float* __restrict__ table) {
    const int total = nt * L * L;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    const int j = idx / (L * L), rem = idx - j * L * L;
    const int R = (L - 1) / 2;
    const int dy = rem / L - R, dx = rem % L - R;
    const double s = kTwoPi / nt;
    const double thj = kTwoPi * j / nt;
    const double r0 = cut * kPi, sig = (1.0 - cut) * kPi * 0.5;
    double acc = 0.0;
    for (int k2 = -R; k2 <= R; ++k2) {
        const double wy = kTwoPi * k2 / L;
        for (int k1 = -R; k1 <= R; ++k1) {
            const double wx = kTwoPi * k1 / L;
            double hat;
            if (k1 == 0 && k2 == 0) {
                hat = 1.0 / nt;                                        // DC split uniformly
            } else {
                const double rho = sqrt(wx * wx + wy * wy);
                const double W = rho <= r0 ? 1.0 : exp(-(rho - r0) * (rho - r0) / (2.0 * sig * sig));
                double a = atan2(wy, wx) - thj - 0.5 * kPi;           // wedge of theta_j at theta_j + pi/2
                a = a - kTwoPi * floor((a + kPi) / kTwoPi);           // wrap into [-pi, pi)
                hat = bspline_tp(a / s, degree) * W;
            }
            acc += hat * cos(wx * dx + wy * dy);
        }
    }
    table[idx] = (float)(acc / ((double)L * L));
}

// U[b][j][y][x] = sum_{dy,dx} T[j][dy][dx] f[b][y+dy][x+dx]; 16 x 16 outputs per CTA, the f tile (with
// an R halo, zero outside the image) and one orientation's filter in shared memory.  Generic kernel for
// banks wider than 31 x 31 (the register-blocked one below covers R <= 15)
constexpr int kLT = 16;
__global__ void lift_image_kernel(const float* __restrict__ f, const float* __restrict__ T, float* __restrict__ U,
                                  int nx, int ny, int nt, int L) {
    extern __shared__ float sm[];
    const int R = (L - 1) / 2;
    const int TW = kLT + 2 * R;
    float* tile = sm;                 // [TW][TW]
    float* fil = sm + TW * TW;        // [L][L]
    const int b = blockIdx.z;
    const int x0 = blockIdx.x * kLT, y0 = blockIdx.y * kLT;
    const float* fb = f + (int64_t)b * nx * ny;
    for (int i = threadIdx.x; i < TW * TW; i += blockDim.x) {
        const int r = i / TW, c = i - r * TW;
        const int gy = y0 - R + r, gx = x0 - R + c;
        tile[i] = (gy >= 0 && gy < ny && gx >= 0 && gx < nx) ? fb[(int64_t)gy * nx + gx] : 0.f;
    }
    const int tx = threadIdx.x % kLT, ty = threadIdx.x / kLT;
    const int gx = x0 + tx, gy = y0 + ty;
    for (int j = 0; j < nt; ++j) {
        __syncthreads();   // tile ready / previous filter consumed
        for (int i = threadIdx.x; i < L * L; i += blockDim.x) fil[i] = T[(int64_t)j * L * L + i];
        __syncthreads();
        float acc = 0.f;
        for (int a = 0; a < L; ++a) {
            const float* trow = tile + (ty + a) * TW + tx;
            const float* frow = fil + a * L;
            for (int c = 0; c < L; ++c) acc = fmaf(frow[c], trow[c], acc);
        }
        if (gx < nx && gy < ny) U[(((int64_t)b * nt + j) * ny + gy) * nx + gx] = acc;
    }
}

// Register-blocked orientation scores (the K3 FFMA geometry): one CTA = a 16 x 32 output tile x one
// quad of orientations; lanes are rows, each warp 4 columns; per filter row the thread loads its input
// row segment (LDS.128) and issues 16 FFMA per tap against one LDS.128 broadcast of the 4 orientations'
// filter values (the bank re-laid out quad-interleaved in shared memory).
template <int R>
struct LiftCfg {
    static constexpr int L = 2 * R + 1, P = 4, WX = 4, NT = 32 * WX, TY = 32, TX = P * WX;
    static constexpr int RL = ((P + 2 * R) + 3) / 4 * 4;
    static constexpr int NEED = (WX - 1) * P + RL;
    static constexpr int P0 = (NEED + 3) / 4 * 4;
    static constexpr int PITCH = ((P0 / 4) % 2 == 1) ? P0 : P0 + 4;   // pitch/4 odd: conflict-free rows
    static constexpr int WIN_H = TY + 2 * R;
    static constexpr size_t SMEM = (size_t)(WIN_H * PITCH + 4 * L * L) * sizeof(float);
};

template <int R>
__global__ void __launch_bounds__(LiftCfg<R>::NT)
lift_image_rb_kernel(const float* __restrict__ f, const float* __restrict__ T, float* __restrict__ U, int nx, int ny,
                     int nt, int tiles_x) {
    using C = LiftCfg<R>;
    extern __shared__ __align__(16) float sm[];
    float* win = sm;                                                     // [WIN_H][PITCH]
    float4* fil = reinterpret_cast<float4*>(sm + C::WIN_H * C::PITCH);   // [L*L] quad-interleaved
    const int tile = blockIdx.x, qd = blockIdx.y, b = blockIdx.z;
    const int x0 = (tile % tiles_x) * C::TX, y0 = (tile / tiles_x) * C::TY;
    const float* fb = f + (int64_t)b * nx * ny;
    for (int i = threadIdx.x; i < C::WIN_H * C::PITCH; i += C::NT) {
        const int r = i / C::PITCH, c = i - r * C::PITCH;
        const int gy = y0 - R + r, gx = x0 - R + c;
        win[i] = (gy >= 0 && gy < ny && gx >= 0 && gx < nx) ? fb[(int64_t)gy * nx + gx] : 0.f;
    }
    for (int i = threadIdx.x; i < C::L * C::L; i += C::NT) {
        float v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int to = 4 * qd + q;
            v[q] = to < nt ? T[(int64_t)to * C::L * C::L + i] : 0.f;
        }
        fil[i] = make_float4(v[0], v[1], v[2], v[3]);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wx = threadIdx.x >> 5;
    float acc[4][C::P];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int p = 0; p < C::P; ++p) acc[q][p] = 0.f;
#pragma unroll 1
    for (int dy = 0; dy < C::L; ++dy) {
        const float4* rowp = reinterpret_cast<const float4*>(win + (lane + dy) * C::PITCH + wx * C::P);
        float r[C::RL];
#pragma unroll
        for (int j = 0; j < C::RL / 4; ++j) {
            const float4 t = rowp[j];
            r[4 * j] = t.x; r[4 * j + 1] = t.y; r[4 * j + 2] = t.z; r[4 * j + 3] = t.w;
        }
        const float4* frow = fil + dy * C::L;
#pragma unroll
        for (int dx = 0; dx < C::L; ++dx) {
            const float4 w = frow[dx];
#pragma unroll
            for (int p = 0; p < C::P; ++p) {
                const float xv = r[p + dx];
                acc[0][p] = fmaf(w.x, xv, acc[0][p]);
                acc[1][p] = fmaf(w.y, xv, acc[1][p]);
                acc[2][p] = fmaf(w.z, xv, acc[2][p]);
                acc[3][p] = fmaf(w.w, xv, acc[3][p]);
            }
        }
    }
    const int gy = y0 + lane;
    if (gy >= ny) return;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int to = 4 * qd + q;
        if (to >= nt) continue;
        float* row = U + (((int64_t)b * nt + to) * ny + gy) * nx;
#pragma unroll
        for (int p = 0; p < C::P; ++p) {
            const int gx = x0 + wx * C::P + p;
            if (gx < nx) row[gx] = acc[q][p];
        }
    }
}

template <int R>
static cudaError_t launch_lift_rb(const se2_cake_s* c, const float* f, float* U, int nx, int ny, int batch,
                                  cudaStream_t s) {
    using C = LiftCfg<R>;
    cudaError_t e = cudaFuncSetAttribute(lift_image_rb_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::SMEM);
    if (e != cudaSuccess) return e;
    const int tiles_x = (nx + C::TX - 1) / C::TX, tiles_y = (ny + C::TY - 1) / C::TY;
    dim3 grid(tiles_x * tiles_y, (c->nt + 3) / 4, batch);
    lift_image_rb_kernel<R><<<grid, C::NT, C::SMEM, s>>>(f, c->table, U, nx, ny, c->nt, tiles_x);
    return cudaGetLastError();
}

static cudaError_t launch_lift_image(const se2_cake_s* c, const float* f, float* U, int nx, int ny, int batch,
                                     cudaStream_t s) {
    switch (c->R) {
#define SE2_LCASE(r) \
    case r: return launch_lift_rb<r>(c, f, U, nx, ny, batch, s);
        SE2_LCASE(0) SE2_LCASE(1) SE2_LCASE(2) SE2_LCASE(3) SE2_LCASE(4) SE2_LCASE(5) SE2_LCASE(6) SE2_LCASE(7)
        SE2_LCASE(8) SE2_LCASE(9) SE2_LCASE(10) SE2_LCASE(11) SE2_LCASE(12) SE2_LCASE(13) SE2_LCASE(14) SE2_LCASE(15)
#undef SE2_LCASE
        default: return cudaErrorNotSupported;   // wider banks: the generic kernel
    }
}

// per-block partials of one field: fp64 sums and maxima of max(U,0), max(-U,0): part[b][blk][4]
constexpr int kRedT = 256;
__global__ void signed_partials_kernel(const float* __restrict__ U, int64_t n, double* __restrict__ part) {
    __shared__ double sp[kRedT], sn[kRedT];
    __shared__ float xp[kRedT], xn[kRedT];
    const int b = blockIdx.y;
    const float* u = U + (int64_t)b * n;
    double p = 0.0, q = 0.0;
    float mp = 0.f, mq = 0.f;
    for (int64_t i = blockIdx.x * (int64_t)kRedT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kRedT) {
        const float v = u[i];
        if (v > 0.f) { p += v; mp = fmaxf(mp, v); } else { q -= v; mq = fmaxf(mq, -v); }
    }
    sp[threadIdx.x] = p;
    sn[threadIdx.x] = q;
    xp[threadIdx.x] = mp;
    xn[threadIdx.x] = mq;
    __syncthreads();
    for (int o = kRedT / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            sp[threadIdx.x] += sp[threadIdx.x + o];
            sn[threadIdx.x] += sn[threadIdx.x + o];
            xp[threadIdx.x] = fmaxf(xp[threadIdx.x], xp[threadIdx.x + o]);
            xn[threadIdx.x] = fmaxf(xn[threadIdx.x], xn[threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double* o = part + ((int64_t)b * gridDim.x + blockIdx.x) * 4;
        o[0] = sp[0];
        o[1] = sn[0];
        o[2] = xp[0];
        o[3] = xn[0];
    }
}

// m[b] = (sum+, sum-, max+, max-) from the block partials (fixed order)
__global__ void signed_reduce_kernel(const double* __restrict__ part, int nblk, double* __restrict__ m) {
    __shared__ double red[4][kRedT];
    const int b = blockIdx.x;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int i = threadIdx.x; i < nblk; i += kRedT) {
        const double* q = part + ((int64_t)b * nblk + i) * 4;
        a0 += q[0];
        a1 += q[1];
        a2 = fmax(a2, q[2]);
        a3 = fmax(a3, q[3]);
    }
    red[0][threadIdx.x] = a0;
    red[1][threadIdx.x] = a1;
    red[2][threadIdx.x] = a2;
    red[3][threadIdx.x] = a3;
    __syncthreads();
    for (int o = kRedT / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            red[0][threadIdx.x] += red[0][threadIdx.x + o];
            red[1][threadIdx.x] += red[1][threadIdx.x + o];
            red[2][threadIdx.x] = fmax(red[2][threadIdx.x], red[2][threadIdx.x + o]);
            red[3][threadIdx.x] = fmax(red[3][threadIdx.x], red[3][threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x < 4) m[4 * b + threadIdx.x] = red[threadIdx.x][0];
}

// out[b][c] = sum_blk part[b][blk][c] in a fixed order (one block per field, c < nc)
__global__ void reduce_fixed_kernel(const double* __restrict__ part, int nblk, int nc, double* __restrict__ out) {
    __shared__ double red[kRedT];
    const int b = blockIdx.x;
    for (int c = 0; c < nc; ++c) {
        double t = 0.0;
        for (int i = threadIdx.x; i < nblk; i += kRedT) t += part[((int64_t)b * nblk + i) * nc + c];
        red[threadIdx.x] = t;
        __syncthreads();
        for (int o = kRedT / 2; o > 0; o >>= 1) {
            if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
            __syncthreads();
        }
        if (threadIdx.x == 0) out[b * nc + c] = red[0];
        __syncthreads();
    }
}

// U+- = (max(+-U, 0) + floor max+-) / (m+- + floor max+- n); an empty part (m = 0) stays zero
__global__ void split_normalise_kernel(const float* __restrict__ U, float* __restrict__ Up, float* __restrict__ Un,
                                       int64_t n, const double* __restrict__ m, double floor_rel) {
    const int b = blockIdx.y;
    const double mp = m[4 * b], mn = m[4 * b + 1];
    const double fp = floor_rel * m[4 * b + 2], fn = floor_rel * m[4 * b + 3];
    const double tp = mp + fp * (double)n, tn = mn + fn * (double)n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float v = U[(int64_t)b * n + i];
        const double pv = v > 0.f ? (double)v : 0.0, nv = v < 0.f ? -(double)v : 0.0;
        Up[(int64_t)b * n + i] = mp > 0.0 ? (float)((pv + fp) / tp) : 0.f;
        Un[(int64_t)b * n + i] = mn > 0.0 ? (float)((nv + fn) / tn) : 0.f;
    }
}

__global__ void project_kernel(const float* __restrict__ U, float* __restrict__ img, int64_t plane, int nt) {
    const int b = blockIdx.y;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < plane; i += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int j = 0; j < nt; ++j) acc += U[((int64_t)b * nt + j) * plane + i];
        img[(int64_t)b * plane + i] = (float)acc;
    }
}

// img = max(m+ P(Up) - m- P(Un), 0) (unnormalised) and per-block partial sums part[b][blk]
__global__ void project_signed_kernel(const float* __restrict__ Up, const float* __restrict__ Un,
                                      const double* __restrict__ m, float* __restrict__ img, double* __restrict__ part,
                                      int64_t plane, int nt) {
    __shared__ double red[kRedT];
    const int b = blockIdx.y;
    const double mp = m[2 * b], mn = m[2 * b + 1];
    double t = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)kRedT + threadIdx.x; i < plane; i += (int64_t)gridDim.x * kRedT) {
        double pp = 0.0, pn = 0.0;
        for (int j = 0; j < nt; ++j) {
            pp += Up[((int64_t)b * nt + j) * plane + i];
            pn += Un[((int64_t)b * nt + j) * plane + i];
        }
        double v = mp * pp - mn * pn;
        v = v > 0.0 ? v : 0.0;
        img[(int64_t)b * plane + i] = (float)v;
        t += v;
    }
    red[threadIdx.x] = t;
    __syncthreads();
    for (int o = kRedT / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[(int64_t)b * gridDim.x + blockIdx.x] = red[0];
}

// img /= sum (recomputing the unnormalised value in fp64 from the inputs keeps one rounding)
__global__ void project_signed_normalise_kernel(const float* __restrict__ Up, const float* __restrict__ Un,
                                                const double* __restrict__ m, const double* __restrict__ tot,
                                                float* __restrict__ img, int64_t plane, int nt) {
    const int b = blockIdx.y;
    const double mp = m[2 * b], mn = m[2 * b + 1], s = tot[b];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < plane; i += (int64_t)gridDim.x * blockDim.x) {
        double pp = 0.0, pn = 0.0;
        for (int j = 0; j < nt; ++j) {
            pp += Up[((int64_t)b * nt + j) * plane + i];
            pn += Un[((int64_t)b * nt + j) * plane + i];
        }
        double v = mp * pp - mn * pn;
        v = v > 0.0 ? v : 0.0;
        img[(int64_t)b * plane + i] = s > 0.0 ? (float)(v / s) : 0.f;
    }
}

// per-block fp64 partial sums of mag: part[b][blk]
__global__ void sum_partials_kernel(const float* __restrict__ x, int64_t n, double* __restrict__ part) {
    __shared__ double red[kRedT];
    const int b = blockIdx.y;
    double t = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)kRedT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kRedT)
        t += x[(int64_t)b * n + i];
    red[threadIdx.x] = t;
    __syncthreads();
    for (int o = kRedT / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[(int64_t)b * gridDim.x + blockIdx.x] = red[0];
}

// bin of an orientation angle in fp64 (R16): a in [0, 2pi), k = ceil(a N / 2pi - 1/2) mod N
__device__ __forceinline__ int angle_bin(float angle, int nt) {
    double a = fmod((double)angle, kTwoPi);
    if (a != 0.0 && a < 0.0) a += kTwoPi;
    const double t = a * (double)nt / kTwoPi;
    int k = (int)ceil(t - 0.5);
    k %= nt;
    if (k < 0) k += nt;
    return k;
}

__global__ void lift_field_kernel(const float* __restrict__ ang, const float* __restrict__ mag,
                                  const double* __restrict__ tot, float* __restrict__ U, int64_t plane, int nt) {
    const int b = blockIdx.y;
    const double s = tot[b];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < plane; i += (int64_t)gridDim.x * blockDim.x) {
        const int k = angle_bin(ang[(int64_t)b * plane + i], nt);
        const float v = s > 0.0 ? (float)((double)mag[(int64_t)b * plane + i] / s) : 0.f;
        for (int j = 0; j < nt; ++j) U[((int64_t)b * nt + j) * plane + i] = (j == k) ? v : 0.f;
    }
}

__global__ void reconstruct_field_kernel(const float* __restrict__ U, float* __restrict__ ang, float* __restrict__ mag,
                                         int64_t plane, int nt, float thr) {
    const int b = blockIdx.y;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < plane; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        float best = -INFINITY;
        int kb = 0;
        for (int j = 0; j < nt; ++j) {
            const float v = U[((int64_t)b * nt + j) * plane + i];
            s += v;
            if (v > best) { best = v; kb = j; }      // strict: the first maximum
        }
        const bool keep = (s >= (double)thr) && (s > 0.0);
        ang[(int64_t)b * plane + i] = keep ? (float)(kTwoPi * kb / nt) : 0.f;
        mag[(int64_t)b * plane + i] = keep ? (float)s : 0.f;
    }
}

__global__ void exp_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = expf(x[i]);
}

inline int blocks_for(int64_t n, int t) {
    int64_t g = (n + t - 1) / t;
    if (g > 148 * 8) g = 148 * 8;
    return (int)(g < 1 ? 1 : g);
}

se2_status check_cake(se2_cake c) {
    if (c == nullptr || c->table == nullptr) {
        set_error("invalid se2_cake handle");
        return SE2_EINVAL;
    }
    return SE2_OK;
}

se2_status ensure_scratch(se2_cake c, size_t n) {
    if (c->scratch_n >= n) return SE2_OK;
    if (c->scratch) cudaFree(c->scratch);
    c->scratch = nullptr;
    c->scratch_n = 0;
    if (cudaMalloc(&c->scratch, n * sizeof(double)) != cudaSuccess) {
        set_error("lifting scratch allocation failed");
        return SE2_ENOMEM;
    }
    c->scratch_n = n;
    return SE2_OK;
}

se2_status launch_ok(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string(what) + ": " + cudaGetErrorString(e));
        return SE2_ECUDA;
    }
    return SE2_OK;
}

}  // namespace

extern "C" {

SE2_API se2_status se2_cake_build(int32_t ntheta, int32_t size, int32_t spline_degree, double radial_cut,
                                  int32_t device, se2_cake* out) {
    SE2_CHECK_ARG(out != nullptr, "out must be non-null");
    *out = nullptr;
    SE2_CHECK_ARG(size >= 1 && size % 2 == 1 && size <= 63, "size must be odd, 1..63");
    SE2_CHECK_ARG(spline_degree >= 0 && spline_degree <= 7, "spline_degree must be in [0, 7]");
    SE2_CHECK_ARG(ntheta >= spline_degree + 1 && ntheta <= 1024, "ntheta must be >= spline_degree + 1 (and <= 1024)");
    SE2_CHECK_ARG(radial_cut > 0.0 && radial_cut < 1.0, "radial_cut must be in (0, 1)");
    Guard g(device);
    se2_cake c = new se2_cake_s();
    c->device = device;
    c->nt = ntheta;
    c->L = size;
    c->R = (size - 1) / 2;
    c->degree = spline_degree;
    c->cut = radial_cut;
    const int total = ntheta * size * size;
    if (cudaMalloc(&c->table, sizeof(float) * total) != cudaSuccess) {
        delete c;
        set_error("cake table allocation failed");
        return SE2_ENOMEM;
    }
    cake_tabulate_kernel<<<(total + 127) / 128, 128>>>(ntheta, size, spline_degree, radial_cut, c->table);
    count_launch();
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        cudaFree(c->table);
        delete c;
        set_error(std::string("cake tabulation: ") + cudaGetErrorString(e));
        return SE2_ECUDA;
    }
    *out = c;
    return SE2_OK;
}

SE2_API se2_status se2_cake_get(se2_cake c, float* table_host, int32_t* ntheta, int32_t* size) {
    if (check_cake(c) != SE2_OK) return SE2_EINVAL;
    Guard g(c->device);
    if (ntheta) *ntheta = c->nt;
    if (size) *size = c->L;
    if (table_host)
        SE2_CUDA_TRY(cudaMemcpy(table_host, c->table, sizeof(float) * c->nt * c->L * c->L, cudaMemcpyDeviceToHost));
    return SE2_OK;
}

SE2_API void se2_cake_destroy(se2_cake c) {
    if (!c) return;
    Guard g(c->device);
    if (c->table) cudaFree(c->table);
    if (c->scratch) cudaFree(c->scratch);
    delete c;
}

SE2_API se2_status se2_lift_image(se2_cake c, const float* f, float* U, int32_t nx, int32_t ny, int32_t batch,
                                  se2_stream stream) {
    if (check_cake(c) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(f && U && nx >= 1 && ny >= 1 && batch >= 1, "bad arguments");
    Guard g(c->device);
    if (c->R <= 15) {   // register-blocked kernel (FFMA-bound)
        const cudaError_t e = launch_lift_image(c, f, U, nx, ny, batch, (cudaStream_t)stream);
        count_launch();
        if (e != cudaSuccess) {
            set_error(std::string("lift_image: ") + cudaGetErrorString(e));
            return SE2_ECUDA;
        }
        return SE2_OK;
    }
    const int TW = kLT + 2 * c->R;
    const size_t smem = sizeof(float) * ((size_t)TW * TW + (size_t)c->L * c->L);
    SE2_CUDA_TRY(cudaFuncSetAttribute(lift_image_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid((nx + kLT - 1) / kLT, (ny + kLT - 1) / kLT, batch);
    lift_image_kernel<<<grid, kLT * kLT, smem, (cudaStream_t)stream>>>(f, c->table, U, nx, ny, c->nt, c->L);
    count_launch();
    return launch_ok("lift_image");
}

SE2_API se2_status se2_split_signed(se2_cake c, const float* U, float* Upos, float* Uneg, int64_t n, int32_t batch,
                                    double floor_rel, double* masses_host, se2_stream stream) {
    if (check_cake(c) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(U && Upos && Uneg && n >= 1 && batch >= 1, "bad arguments");
    SE2_CHECK_ARG(floor_rel >= 0.0, "floor_rel must be >= 0");
    Guard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int nblk = blocks_for(n, kRedT) > 256 ? 256 : blocks_for(n, kRedT);
    se2_status st = ensure_scratch(c, (size_t)batch * nblk * 4 + 4 * (size_t)batch);
    if (st != SE2_OK) return st;
    double* part = c->scratch;
    double* m = part + (size_t)batch * nblk * 4;
    signed_partials_kernel<<<dim3(nblk, batch), kRedT, 0, s>>>(U, n, part);
    signed_reduce_kernel<<<batch, kRedT, 0, s>>>(part, nblk, m);
    split_normalise_kernel<<<dim3(blocks_for(n, 256), batch), 256, 0, s>>>(U, Upos, Uneg, n, m, floor_rel);
    count_launch(3);
    st = launch_ok("split_signed");
    if (st != SE2_OK) return st;
    if (masses_host) {
        double h[4 * 64];
        for (int b0 = 0; b0 < batch; b0 += 64) {
            const int nb = batch - b0 < 64 ? batch - b0 : 64;
            SE2_CUDA_TRY(cudaMemcpyAsync(h, m + 4 * b0, sizeof(double) * 4 * nb, cudaMemcpyDeviceToHost, s));
            SE2_CUDA_TRY(cudaStreamSynchronize(s));
            for (int b = 0; b < nb; ++b) {
                masses_host[2 * (b0 + b)] = h[4 * b];
                masses_host[2 * (b0 + b) + 1] = h[4 * b + 1];
            }
        }
    }
    return SE2_OK;
}

SE2_API se2_status se2_project(se2_cake c, const float* U, float* img, int32_t nx, int32_t ny, int32_t batch,
                               se2_stream stream) {
    if (check_cake(c) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(U && img && nx >= 1 && ny >= 1 && batch >= 1, "bad arguments");
    Guard g(c->device);
    const int64_t plane = (int64_t)nx * ny;
    project_kernel<<<dim3(blocks_for(plane, 256), batch), 256, 0, (cudaStream_t)stream>>>(U, img, plane, c->nt);
    count_launch();
    return launch_ok("project");
}

SE2_API se2_status se2_interp_masses(const double* masses_host, const double* ts_host, int32_t nts, double* out_host) {
    SE2_CHECK_ARG(masses_host != nullptr && ts_host != nullptr && out_host != nullptr && nts >= 0, "bad arguments");
    for (int i = 0; i < nts; ++i) {
        const double t = ts_host[i];
        SE2_CHECK_ARG(t >= 0.0 && t <= 1.0, "t must lie in [0, 1]");
        for (int s = 0; s < 2; ++s) out_host[2 * i + s] = (1.0 - t) * masses_host[s] + t * masses_host[2 + s];
    }
    return SE2_OK;
}

se2_status se2_project_signed(se2_cake c, const float* Upos, const float* Uneg, const double* masses_host,
                                      float* img, int32_t nx, int32_t ny, int32_t batch, double* mass_host,
                                      se2_stream stream) {
    if (check_cake(c) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(Upos && Uneg && masses_host && img && nx >= 1 && ny >= 1 && batch >= 1, "bad arguments");
    for (int b = 0; b < batch; ++b)
        SE2_CHECK_ARG(masses_host[2 * b] >= 0.0 && masses_host[2 * b + 1] >= 0.0, "masses must be >= 0");
    Guard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t plane = (int64_t)nx * ny;
    const int nblk = blocks_for(plane, kRedT) > 256 ? 256 : blocks_for(plane, kRedT);
    se2_status st = ensure_scratch(c, (size_t)batch * nblk + 3 * (size_t)batch);
    if (st != SE2_OK) return st;
    double* part = c->scratch;
    double* m = part + (size_t)batch * nblk;
    double* tot = m + 2 * (size_t)batch;
    SE2_CUDA_TRY(cudaMemcpyAsync(m, masses_host, sizeof(double) * 2 * batch, cudaMemcpyHostToDevice, s));
    project_signed_kernel<<<dim3(nblk, batch), kRedT, 0, s>>>(Upos, Uneg, m, img, part, plane, c->nt);
    reduce_fixed_kernel<<<batch, kRedT, 0, s>>>(part, nblk, 1, tot);
    project_signed_normalise_kernel<<<dim3(blocks_for(plane, 256), batch), 256, 0, s>>>(Upos, Uneg, m, tot, img, plane,
                                                                                       c->nt);
    count_launch(3);
    st = launch_ok("project_signed");
    if (st != SE2_OK) return st;
    if (mass_host) SE2_CUDA_TRY(cudaMemcpyAsync(mass_host, tot, sizeof(double) * batch, cudaMemcpyDeviceToHost, s));
    SE2_CUDA_TRY(cudaStreamSynchronize(s));   // masses_host staging buffer is the caller's
    return SE2_OK;
}

SE2_API se2_status se2_lift_field(se2_cake c, const float* angle, const float* mag, float* U, int32_t nx, int32_t ny,
                                  int32_t batch, double* mass_host, se2_stream stream) {
    if (check_cake(c) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(angle && mag && U && nx >= 1 && ny >= 1 && batch >= 1, "bad arguments");
    Guard g(c->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t plane = (int64_t)nx * ny;
    const int nblk = blocks_for(plane, kRedT) > 256 ? 256 : blocks_for(plane, kRedT);
    se2_status st = ensure_scratch(c, (size_t)batch * nblk + (size_t)batch);
    if (st != SE2_OK) return st;
    double* part = c->scratch;
    double* tot = part + (size_t)batch * nblk;
    sum_partials_kernel<<<dim3(nblk, batch), kRedT, 0, s>>>(mag, plane, part);
    reduce_fixed_kernel<<<batch, kRedT, 0, s>>>(part, nblk, 1, tot);
    lift_field_kernel<<<dim3(blocks_for(plane, 256), batch), 256, 0, s>>>(angle, mag, tot, U, plane, c->nt);
    count_launch(3);
    st = launch_ok("lift_field");
    if (st != SE2_OK) return st;
    if (mass_host) {
        SE2_CUDA_TRY(cudaMemcpyAsync(mass_host, tot, sizeof(double) * batch, cudaMemcpyDeviceToHost, s));
        SE2_CUDA_TRY(cudaStreamSynchronize(s));
    }
    return SE2_OK;
}

SE2_API se2_status se2_reconstruct_field(se2_cake c, const float* U, float* angle, float* mag, int32_t nx, int32_t ny,
                                         int32_t batch, float threshold, se2_stream stream) {
    if (check_cake(c) != SE2_OK) return SE2_EINVAL;
    SE2_CHECK_ARG(U && angle && mag && nx >= 1 && ny >= 1 && batch >= 1, "bad arguments");
    Guard g(c->device);
    const int64_t plane = (int64_t)nx * ny;
    reconstruct_field_kernel<<<dim3(blocks_for(plane, 256), batch), 256, 0, (cudaStream_t)stream>>>(U, angle, mag, plane,
                                                                                                   c->nt, threshold);
    count_launch();
    return launch_ok("reconstruct_field");
}

__global__ void log_elem_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = logf(x[i]);
}

SE2_API se2_status se2_log(const float* x, float* y, int64_t n, se2_stream stream) {
    SE2_CHECK_ARG(x && y && n >= 1, "bad arguments");
    log_elem_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(x, y, n);
    count_launch();
    return launch_ok("log");
}

SE2_API se2_status se2_exp(const float* x, float* y, int64_t n, se2_stream stream) {
    SE2_CHECK_ARG(x && y && n >= 1, "bad arguments");
    exp_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(x, y, n);
    count_launch();
    return launch_ok("exp");
}

}  // extern "C"
