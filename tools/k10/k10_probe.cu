// K10 probe (round-2 groundwork, not on the product path): does a tcgen05 BF16 MMA with the A operand
// read from a pixel-shifted K-major SWIZZLE_NONE window compute
//     D[m][n] = sum_dx sum_k X[m + dx][k] W_dx[n][k]        (m < 128 pixels, n < 64, k < 64)
// and how many cycles does one 128x64x16 MMA take in that layout?  Standalone: nvcc -arch=sm_100a.
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cmath>

constexpr int M = 128, N = 64, KT = 64, NCH = KT / 8, TAPS = 16, PX = M + TAPS - 1;
constexpr int CS = PX * 16;          // bytes per K chunk of the X window: [chunk][px][8 bf16]
constexpr int WS = N * 16;           // bytes per K chunk of one tap's W: [chunk][n][8 bf16]

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_kmajor(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;            // version (Blackwell)
    return d;                          // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__global__ void k10_probe(const __nv_bfloat16* __restrict__ X, const __nv_bfloat16* __restrict__ W, float* __restrict__ D,
                          int reps, long long* cycles) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* sX = sm;                       // NCH * CS
    unsigned char* sW = sm + NCH * CS;            // TAPS * NCH * WS
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t mbar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // stage operands (plain copies; the layouts are the global ones)
    const int nx = NCH * CS / 16, nw = TAPS * NCH * WS / 16;
    for (int i = tid; i < nx; i += blockDim.x) reinterpret_cast<uint4*>(sX)[i] = reinterpret_cast<const uint4*>(X)[i];
    for (int i = tid; i < nw; i += blockDim.x) reinterpret_cast<uint4*>(sW)[i] = reinterpret_cast<const uint4*>(W)[i];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");   // generic-proxy smem writes -> async proxy (MMA reads)
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    long long t0 = 0, t1 = 0;
    if (tid == 0) {
        t0 = clock64();
        const uint64_t da0 = desc_kmajor(smem_u32(sX), CS, 128);
        const uint64_t db0 = desc_kmajor(smem_u32(sW), WS, 128);
        for (int rep = 0; rep < reps; ++rep) {
#pragma unroll 2
            for (int dx = 0; dx < TAPS; ++dx) {
#pragma unroll
                for (int kc = 0; kc < KT / 16; ++kc) {
                    const uint64_t da = da0 + (uint64_t)(((2 * kc) * CS + dx * 16) >> 4);
                    const uint64_t db = db0 + (uint64_t)(((dx * NCH + 2 * kc) * WS) >> 4);
                    const uint32_t acc = (rep > 0 || dx > 0 || kc > 0) ? 1u : 0u;
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                                 ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
                }
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
    }
    // wait for the MMAs (phase 0)
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                         : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0u));
        }
    }
    if (tid == 0) { t1 = clock64(); *cycles = t1 - t0; }
    asm volatile("tcgen05.fence::after_thread_sync;");
    // TMEM -> registers: warp w reads lanes [32w, 32w + 32), 64 columns
    uint32_t v[64];
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16);
#pragma unroll
    for (int c = 0; c < 64; c += 8) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[c]), "=r"(v[c + 1]), "=r"(v[c + 2]), "=r"(v[c + 3]), "=r"(v[c + 4]), "=r"(v[c + 5]),
                       "=r"(v[c + 6]), "=r"(v[c + 7])
                     : "r"(taddr + c));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int m = 32 * warp + lane;
    for (int n = 0; n < N; ++n) D[m * N + n] = __uint_as_float(v[n]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

int main(int argc, char** argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 1;
    // X[chunk][px][8], W[tap][chunk][n][8]
    std::vector<__nv_bfloat16> X(NCH * PX * 8), W((size_t)TAPS * NCH * N * 8);
    std::vector<float> Xf(X.size()), Wf(W.size());
    srand(1);
    for (size_t i = 0; i < X.size(); ++i) { X[i] = __float2bfloat16((rand() % 17 - 8) / 8.0f); Xf[i] = __bfloat162float(X[i]); }
    for (size_t i = 0; i < W.size(); ++i) { W[i] = __float2bfloat16((rand() % 9 - 4) / 4.0f); Wf[i] = __bfloat162float(W[i]); }
    __nv_bfloat16 *dX, *dW; float* dD; long long* dc;
    cudaMalloc(&dX, X.size() * 2); cudaMalloc(&dW, W.size() * 2); cudaMalloc(&dD, M * N * 4); cudaMalloc(&dc, 8);
    cudaMemcpy(dX, X.data(), X.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dW, W.data(), W.size() * 2, cudaMemcpyHostToDevice);
    const size_t smem = (size_t)NCH * CS + (size_t)TAPS * NCH * WS;
    cudaFuncSetAttribute(k10_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k10_probe<<<1, 128, smem>>>(dX, dW, dD, reps, dc);
    cudaError_t e = cudaGetLastError(); if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error: %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> D(M * N); long long cyc;
    cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost); cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double acc = 0;
            for (int dx = 0; dx < TAPS; ++dx)
                for (int k = 0; k < KT; ++k)
                    acc += (double)Xf[((k / 8) * PX + m + dx) * 8 + k % 8] * Wf[(((size_t)dx * NCH + k / 8) * N + n) * 8 + k % 8];
            acc *= reps;
            maxerr = fmax(maxerr, fabs(acc - D[m * N + n]));
            maxref = fmax(maxref, fabs(acc));
        }
    const double mmas = (double)reps * TAPS * (KT / 16);
    printf("k10 probe: reps %d  max|err| %.3e (max|ref| %.1f)  %.1f cycles per 128x64x16 MMA (issue loop incl.)\n", reps, maxerr,
           maxref, cyc / mmas);
    return 0;
}
