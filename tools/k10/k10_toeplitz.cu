// K10 probe 2 (round-2 groundwork, not on the product path): the Toeplitz-in-x formulation.
// For one input orientation ti and one filter row: D[px][ti + j] += sum_k X_ti[px + k] W_ti[j][k]
// (k < 32 = the 31 dx taps + 1 zero, j < 16 = the 11 theta offsets + 5 zero), with A read from an
// 8x-expanded row Xe[p] = X[p .. p+7] (16 B per pixel) so that a K-major SWIZZLE_NONE descriptor with
// LBO = SBO = 128 B walks the Toeplitz matrix; the MMA for ti accumulates into TMEM columns ti..ti+15,
// so the theta band lands on the output orientations without any data movement.
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cmath>

constexpr int M = 128, N = 16, KD = 32, NTI = 64, PXE = M + KD;   // expanded pixels per row
constexpr int XS = PXE * 16;                                       // bytes per ti of the expanded row
constexpr int WS = N * KD * 2;                                     // bytes per ti of W (hi only)
constexpr int NCOL = 128;                                          // TMEM columns (>= NTI + N)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__global__ void k10_toeplitz(const __nv_bfloat16* __restrict__ X, const __nv_bfloat16* __restrict__ W, float* __restrict__ D,
                             int reps, long long* cycles, int colmask) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* sX = sm;                 // [ti][p][8]: Xe
    unsigned char* sW = sm + NTI * XS;      // [ti][kchunk 4][n 16][8]
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t mbar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // expand: Xe[ti][p][e] = X[ti][p + e] (X rows are PXE + 8 long)
    __nv_bfloat16* xe = reinterpret_cast<__nv_bfloat16*>(sX);
    for (int i = tid; i < NTI * PXE * 8; i += blockDim.x) {
        const int e = i & 7, p = (i >> 3) % PXE, ti = i / (8 * PXE);
        xe[i] = X[ti * (PXE + 8) + p + e];
    }
    for (int i = tid; i < NTI * WS / 16; i += blockDim.x) reinterpret_cast<uint4*>(sW)[i] = reinterpret_cast<const uint4*>(W)[i];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(NCOL));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    if (tid == 0) {
        // zero the accumulator columns first: one MMA per column block with enable_input_d = 0 would only
        // clear its own 16 columns; instead clear all NCOL columns with tcgen05.st from the epilogue warps
    }
    // clear TMEM (each warp its 32 lanes, all columns)
    {
        const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16);
        for (int c = 0; c < NCOL; c += 8)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr + c), "r"(0u));
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    long long t0 = 0;
    if (tid == 0) {
        t0 = clock64();
        // descriptors are linear in the start address (bits 0-13 = addr >> 4): build once, add offsets
        const uint64_t da0 = desc_kmajor(smem_u32(sX), 128, 128);
        const uint64_t db0 = desc_kmajor(smem_u32(sW), N * 16, 128);
        for (int rep = 0; rep < reps; ++rep) {
#pragma unroll 4
            for (int ti = 0; ti < NTI; ++ti) {
#pragma unroll
                for (int kc = 0; kc < KD / 16; ++kc) {
                    const uint64_t da = da0 + (uint64_t)((ti * XS + kc * 256) >> 4);
                    const uint64_t db = db0 + (uint64_t)((ti * WS + 2 * kc * N * 16) >> 4);
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                                 ::"r"(tmem + (ti & colmask)), "l"(da), "l"(db), "r"(idesc));
                }
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
    }
    {
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                         : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0u));
    }
    if (tid == 0) *cycles = clock64() - t0;
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16);
    const int m = 32 * warp + lane;
    for (int c = 0; c < NTI + N; c += 8) {
        uint32_t v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(taddr + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 8; ++j) D[m * (NTI + N) + c + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(NCOL));
}

int main(int argc, char** argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 1;
    // X[ti][PXE + 8] row values; W[ti][kchunk][n][8] with W_ti[n][k] at [ti][k/8][n][k%8]
    std::vector<__nv_bfloat16> X(NTI * (PXE + 8)), W((size_t)NTI * WS / 2);
    std::vector<float> Xf(X.size()), Wf(W.size());
    srand(2);
    for (size_t i = 0; i < X.size(); ++i) { X[i] = __float2bfloat16((rand() % 17 - 8) / 8.0f); Xf[i] = __bfloat162float(X[i]); }
    for (size_t i = 0; i < W.size(); ++i) { W[i] = __float2bfloat16((rand() % 9 - 4) / 4.0f); Wf[i] = __bfloat162float(W[i]); }
    __nv_bfloat16 *dX, *dW; float* dD; long long* dc;
    cudaMalloc(&dX, X.size() * 2); cudaMalloc(&dW, W.size() * 2); cudaMalloc(&dD, M * (NTI + N) * 4); cudaMalloc(&dc, 8);
    cudaMemcpy(dX, X.data(), X.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dW, W.data(), W.size() * 2, cudaMemcpyHostToDevice);
    const size_t smem = (size_t)NTI * XS + (size_t)NTI * WS;
    cudaFuncSetAttribute(k10_toeplitz, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int colmask = argc > 2 ? atoi(argv[2]) : -1;
    k10_toeplitz<<<1, 128, smem>>>(dX, dW, dD, reps, dc, colmask);
    cudaError_t e = cudaGetLastError(); if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error: %s (smem %zu)\n", cudaGetErrorString(e), smem); return 1; }
    std::vector<float> D(M * (NTI + N)); long long cyc;
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost); cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < M; ++m)
        for (int col = 0; col < NTI + N; ++col) {
            double acc = 0;
            for (int ti = 0; ti < NTI; ++ti) {
                const int n = col - (ti & colmask);
                if (n < 0 || n >= N) continue;
                for (int k = 0; k < KD; ++k) acc += (double)Xf[ti * (PXE + 8) + m + k] * Wf[((size_t)ti * (KD / 8) + k / 8) * N * 8 + n * 8 + k % 8];
            }
            acc *= reps;
            maxerr = fmax(maxerr, fabs(acc - D[m * (NTI + N) + col]));
            maxref = fmax(maxref, fabs(acc));
        }
    const double mmas = (double)reps * NTI * (KD / 16);
    printf("k10 toeplitz: reps %d  max|err| %.3e (max|ref| %.1f)  %.1f cycles per 128x16x16 MMA\n", reps, maxerr, maxref, cyc / mmas);
    return 0;
}
