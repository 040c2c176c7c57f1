// K1: Gibbs-kernel tabulation (App. A "K_eps <- exp(-rho_b^2/eps)").
//
// For output orientation theta_o = 2 pi to/nt, input orientation theta_i = 2 pi ti/nt and spatial
// offset (dx, dy) cells (dx = ix_g - ix_h), the relative element is
//     h^{-1} g = ( R_{-theta_i} (dx/nx, dy/ny),  wrap(theta_o - theta_i) ),   wrap into [-pi, pi)
// and the half-angle coordinates and rho_b give
//     W = exp(-rho_b^2/eps),   L2 = -rho_b^2/eps * log2(e).
// rho_b^2 splits into a theta part and a spatial part (the spatial part vanishes at dx = dy = 0):
//     L = Lth(to, ti) + Ls(to, ti, dx, dy),  Lth = -w3^2 Theta^2/eps,  Ls = -(w1^2 b1^2 + w2^2 b2^2)/eps
// which the log-domain engine uses (factored per input orientation).  Computed in fp64, stored fp32:
//   Wl [to][ti][S][SP]           W (linear engine, rows padded to SP = 4*ceil(S/4) with zeros)
//   Lq [nt/4][nt][S][S][4]       L2 = L log2(e) (exact LSE engine; theta-quad interleaved so one
//                                16-byte shared-memory broadcast feeds four output orientations)
//   Eq [nt/4][nt][S][S][4]       exp(Ls + kEsShift) (factored LSE engine)
//   Lth[to][ti], LseS[to][ti]    Lth and log sum_{dx,dy} exp(Ls) (natural logs)
//   LqRow [nt/4][nt][S][G][4]    max of Lq over each of the G = kRowSegs segments of a tap row (the
//                                exact path's bounds; an empty segment is -inf)
#include <math.h>

#include <algorithm>

#include "se2_internal.cuh"

namespace se2 {

__global__ void tabulate_kernel(double hx, double hy, int nt, int R, double eps, double w1, double w2,
                                double w3, float* __restrict__ Eq, float* __restrict__ Lq,
                                float* __restrict__ Wl, int* __restrict__ nnz_pair) {
    const int S = 2 * R + 1;
    const int64_t total = (int64_t)nt * nt * S * S;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        int dxi = (int)(idx % S);
        int dyi = (int)((idx / S) % S);
        int ti = (int)((idx / ((int64_t)S * S)) % nt);
        int to = (int)(idx / ((int64_t)S * S * nt));
        const double two_pi = 6.283185307179586476925286766559;
        double ddx = (double)(dxi - R) * hx;
        double ddy = (double)(dyi - R) * hy;
        double thi = two_pi * ti / nt;
        // R_{-theta_i} applied to the spatial offset
        double ci = cos(thi), si = sin(thi);
        double X = ci * ddx + si * ddy;
        double Y = -si * ddx + ci * ddy;
        // wrap(theta_o - theta_i) into [-pi, pi): integer bin offset k in [-nt/2, nt/2)
        int k = ((to - ti) % nt + nt) % nt;
        if (2 * k >= nt) k -= nt;
        double Th = two_pi * k / nt;
        double ch = cos(0.5 * Th), sh = sin(0.5 * Th);
        double b1 = X * ch + Y * sh;
        double b2 = -X * sh + Y * ch;
        double b3 = Th;
        double rho2s = w1 * w1 * b1 * b1 + w2 * w2 * b2 * b2;
        double rho2 = rho2s + w3 * w3 * b3 * b3;
        double e = -rho2 / eps;
        float wv = (float)exp(e);
        int qd = to >> 2, q = to & 3;
        int64_t o = ((((int64_t)qd * nt + ti) * S + dyi) * S + dxi) * 4 + q;
        Eq[o] = (float)exp(-rho2s / eps + (double)kEsShift);
        Lq[o] = (float)(e * 1.4426950408889634073599246810019);
        const int SP = (S + 3) / 4 * 4;
        Wl[(((int64_t)to * nt + ti) * S + dyi) * SP + dxi] = wv;
        if (wv != 0.0f) atomicAdd(&nnz_pair[to * nt + ti], 1);
        if (wv >= 1.17549435e-38f) atomicAdd(&nnz_pair[nt * nt + to * nt + ti], 1);   // fp32 normals
    }
}

// K4P table: L2 = -rho_b^2/eps log2(e) as a float pair hi + lo (hi on the 2^-8 grid, lo the remainder), Lq layout
__global__ void tabulate_l2pair_kernel(double hx, double hy, int nt, int R, double eps, double w1, double w2,
                                       double w3, float* __restrict__ L2hi, float* __restrict__ L2lo) {
    const int S = 2 * R + 1;
    const int64_t total = (int64_t)nt * nt * S * S;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int dxi = (int)(idx % S);
        const int dyi = (int)((idx / S) % S);
        const int ti = (int)((idx / ((int64_t)S * S)) % nt);
        const int to = (int)(idx / ((int64_t)S * S * nt));
        const double two_pi = 6.283185307179586476925286766559;
        const double ddx = (double)(dxi - R) * hx, ddy = (double)(dyi - R) * hy;
        const double thi = two_pi * ti / nt;
        const double ci = cos(thi), si = sin(thi);
        const double X = ci * ddx + si * ddy, Y = -si * ddx + ci * ddy;   // R_{-theta_i} (dx, dy)
        int k = ((to - ti) % nt + nt) % nt;
        if (2 * k >= nt) k -= nt;
        const double Th = two_pi * k / nt;                                  // wrap(theta_o - theta_i)
        const double ch = cos(0.5 * Th), sh = sin(0.5 * Th);
        const double b1 = X * ch + Y * sh, b2 = -X * sh + Y * ch;            // half-angle coordinates
        const double rho2 = w1 * w1 * b1 * b1 + w2 * w2 * b2 * b2 + w3 * w3 * Th * Th;
        const double l2 = -rho2 / eps * 1.4426950408889634073599246810019;
        const int64_t o = ((((int64_t)(to >> 2) * nt + ti) * S + dyi) * S + dxi) * 4 + (to & 3);
        // hi on the 2^-8 grid (exact in fp32 for |l2| < 2^15): K4P adds it to grid-aligned staged potentials
        // without rounding; lo = the (tiny) remainder
        const float hi = fabs(l2) < 32768.0 ? (float)(rint(l2 * 256.0) / 256.0) : (float)l2;
        L2hi[o] = hi;
        L2lo[o] = (float)(l2 - (double)hi);
    }
}

// K4P row bounds: L2row[qd][ti][dy][q] = max over dx of L2hi[qd][ti][dy][dx][q]
__global__ void tabulate_l2row_kernel(int nt, int S, const float* __restrict__ L2hi, float* __restrict__ L2row) {
    const int64_t total = (int64_t)((nt + 3) / 4) * nt * S * 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int q = (int)(i & 3);
        const int64_t row = i >> 2;   // (qd, ti, dy)
        float m = -INFINITY;
        for (int dx = 0; dx < S; ++dx) m = fmaxf(m, L2hi[(row * S + dx) * 4 + q]);
        L2row[i] = m;
    }
}

cudaError_t tabulate_precise(se2_kernel_s* k, cudaStream_t s) {
    if (k->L2hi != nullptr) return cudaSuccess;
    const size_t n = (size_t)((k->nt + 3) / 4) * k->nt * k->S * k->S * 4;
    cudaError_t e = cudaMalloc(&k->L2hi, n * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&k->L2lo, n * sizeof(float));
    if (e == cudaSuccess) e = cudaMemsetAsync(k->L2hi, 0, n * sizeof(float), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(k->L2lo, 0, n * sizeof(float), s);
    if (e != cudaSuccess) return e;
    const int64_t total = (int64_t)k->nt * k->nt * k->S * k->S;
    tabulate_l2pair_kernel<<<(int)std::min<int64_t>((total + 255) / 256, 148 * 32), 256, 0, s>>>(
        k->hx, k->hy, k->nt, k->R, k->eps, k->w1, k->w2, k->w3, k->L2hi, k->L2lo);
    count_launch();
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return e;
    const size_t nr = (size_t)((k->nt + 3) / 4) * k->nt * k->S * 4;
    e = cudaMalloc(&k->L2row, nr * sizeof(float));
    if (e != cudaSuccess) return e;
    tabulate_l2row_kernel<<<(int)std::min<size_t>((nr + 255) / 256, 148 * 32), 256, 0, s>>>(k->nt, k->S, k->L2hi, k->L2row);
    count_launch();
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    k->table_bytes += 2 * n * sizeof(float) + nr * sizeof(float);
    if (e == cudaSuccess)
        e = cudaMalloc(&k->pstats, (size_t)k->max_batch * k->nt * k->ny * ((k->nx + 15) / 16) * sizeof(float4));
    if (e == cudaSuccess) {   // split partials: up to 8 groups, at most 64 MB
        size_t n2 = (size_t)8 * k->max_batch * k->N();
        n2 = std::min<size_t>(n2, ((size_t)64 << 20) / sizeof(double2));
        if (n2 >= (size_t)2 * k->max_batch * k->N()) {
            e = cudaMalloc(&k->psplit, n2 * sizeof(double2));
            k->psplit_n = n2;
        }
    }
    return e;
}

// Lth[to][ti] = -w3^2 Theta^2/eps ; LseS[to][ti] = log sum_{dx,dy} exp(Ls(to,ti,dx,dy))  (fp64 sums)
__global__ void tabulate_theta_kernel(double hx, double hy, int nt, int R, double eps, double w1, double w2,
                                      double w3, float* __restrict__ Lth, float* __restrict__ LseS) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nt * nt) return;
    const int to = p / nt, ti = p % nt;
    const double two_pi = 6.283185307179586476925286766559;
    int k = ((to - ti) % nt + nt) % nt;
    if (2 * k >= nt) k -= nt;
    const double Th = two_pi * k / nt;
    const double thi = two_pi * ti / nt;
    const double ci = cos(thi), si = sin(thi), ch = cos(0.5 * Th), sh = sin(0.5 * Th);
    double acc = 0.0;
    for (int dyi = -R; dyi <= R; ++dyi)
        for (int dxi = -R; dxi <= R; ++dxi) {
            double ddx = (double)dxi * hx, ddy = (double)dyi * hy;
            double X = ci * ddx + si * ddy, Y = -si * ddx + ci * ddy;
            double b1 = X * ch + Y * sh, b2 = -X * sh + Y * ch;
            acc += exp(-(w1 * w1 * b1 * b1 + w2 * w2 * b2 * b2) / eps);
        }
    Lth[p] = (float)(-w3 * w3 * Th * Th / eps);
    LseS[p] = (float)log(acc);
}

// cost-weighted tables for the transport cost <pi, rho^2>: Wc = rho^2 exp(-rho^2/eps)
// (linear layout) and Lc2 = (log(rho^2) - rho^2/eps) log2(e) (quad layout; -inf where rho = 0)
__global__ void tabulate_cost_kernel(double hx, double hy, int nt, int R, double eps, double w1, double w2, double w3,
                                     float* __restrict__ Wcl, float* __restrict__ Lcq) {
    const int S = 2 * R + 1;
    const int SP = (S + 3) / 4 * 4;
    const int64_t total = (int64_t)nt * nt * S * S;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        int dxi = (int)(idx % S);
        int dyi = (int)((idx / S) % S);
        int ti = (int)((idx / ((int64_t)S * S)) % nt);
        int to = (int)(idx / ((int64_t)S * S * nt));
        const double two_pi = 6.283185307179586476925286766559;
        double ddx = (double)(dxi - R) * hx, ddy = (double)(dyi - R) * hy;
        double thi = two_pi * ti / nt;
        double ci = cos(thi), si = sin(thi);
        double X = ci * ddx + si * ddy, Y = -si * ddx + ci * ddy;
        int kk = ((to - ti) % nt + nt) % nt;
        if (2 * kk >= nt) kk -= nt;
        double Th = two_pi * kk / nt;
        double ch = cos(0.5 * Th), sh = sin(0.5 * Th);
        double b1 = X * ch + Y * sh, b2 = -X * sh + Y * ch;
        double rho2 = w1 * w1 * b1 * b1 + w2 * w2 * b2 * b2 + w3 * w3 * Th * Th;
        Wcl[(((int64_t)to * nt + ti) * S + dyi) * SP + dxi] = (float)(rho2 * exp(-rho2 / eps));
        int qd = to >> 2, q = to & 3;
        int64_t o = ((((int64_t)qd * nt + ti) * S + dyi) * S + dxi) * 4 + q;
        Lcq[o] = rho2 > 0.0 ? (float)((log(rho2) - rho2 / eps) * 1.4426950408889634073599246810019) : -INFINITY;
    }
}

// LqRow[qd][ti][dy][g][q] = max over dx in segment g of Lq[qd][ti][dy][dx][q] (after tabulate_kernel)
__global__ void tabulate_rowmax_kernel(int nquads, int nt, int S, const float* __restrict__ Lq,
                                       float* __restrict__ LqRow) {
    const int G = kRowSegs, W = (S + G - 1) / G;
    const int64_t total = (int64_t)nquads * nt * S * G * 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int q = (int)(i & 3);
        const int g = (int)((i >> 2) % G);
        const int64_t row = (i >> 2) / G;   // (qd, ti, dy)
        float m = -INFINITY;
        for (int dx = g * W; dx < (g + 1) * W && dx < S; ++dx) m = fmaxf(m, Lq[(row * S + dx) * 4 + q]);
        LqRow[i] = m;
    }
}

cudaError_t tabulate_cost(se2_kernel_s* k, cudaStream_t s) {
    const int64_t total = (int64_t)k->nt * k->nt * k->S * k->S;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 148 * 32) blocks = 148 * 32;
    tabulate_cost_kernel<<<blocks, 256, 0, s>>>(k->hx, k->hy, k->nt, k->R, k->eps, k->w1, k->w2, k->w3, k->Wcl,
                                                 k->Lcq);
    count_launch();
    return cudaGetLastError();
}

cudaError_t tabulate(se2_kernel_s* k, cudaStream_t s) {
    const int nt = k->nt, S = k->S;
    const int64_t total = (int64_t)nt * nt * S * S;
    int* nnz_dev = nullptr;
    cudaError_t e = cudaMalloc(&nnz_dev, 2 * sizeof(int) * nt * nt);   // nonzero, normal
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(nnz_dev, 0, 2 * sizeof(int) * nt * nt, s);
    // padding entries of a partial last quad (nt % 4 != 0) stay zero / -inf-like
    int threads = 256;
    int blocks = (int)((total + threads - 1) / threads);
    if (blocks > 148 * 32) blocks = 148 * 32;
    tabulate_kernel<<<blocks, threads, 0, s>>>(k->hx, k->hy, nt, k->R, k->eps, k->w1, k->w2, k->w3,
                                               k->Eq, k->Lq, k->Wl, nnz_dev);
    tabulate_theta_kernel<<<(nt * nt + 127) / 128, 128, 0, s>>>(k->hx, k->hy, nt, k->R, k->eps, k->w1, k->w2,
                                                                  k->w3, k->Lth, k->LseS);
    {
        const int nquads = (nt + 3) / 4;
        const int64_t rows = (int64_t)nquads * nt * S * kRowSegs * 4;
        tabulate_rowmax_kernel<<<(int)((rows + 255) / 256), 256, 0, s>>>(nquads, nt, S, k->Lq, k->LqRow);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) { cudaFree(nnz_dev); return e; }
    std::vector<int> nnz(2 * nt * nt);
    e = cudaMemcpyAsync(nnz.data(), nnz_dev, 2 * sizeof(int) * nt * nt, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(nnz_dev);
    if (e != cudaSuccess) return e;
    int band = 0;
    int64_t nnz_total = 0, nnz_normal = 0;
    for (int i = 0; i < nt * nt; ++i) nnz_normal += nnz[nt * nt + i];
    for (int to = 0; to < nt; ++to)
        for (int ti = 0; ti < nt; ++ti) {
            if (nnz[to * nt + ti] == 0) continue;
            int kk = ((to - ti) % nt + nt) % nt;
            if (2 * kk >= nt) kk -= nt;
            if (kk < 0) kk = -kk;
            if (kk > band) band = kk;
            nnz_total += nnz[to * nt + ti];
        }
    k->band = band;
    k->nnz_taps = nnz_total / nt;
    k->nnz_normal_taps = nnz_normal / nt;
    return cudaSuccess;
}

}  // namespace se2
