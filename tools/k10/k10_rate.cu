// K10 rate probe (not on the product path): the measured cycles per tcgen05 BF16 MMA of K10's shape and
// operand layout -- M = 128, N = 256, K = 16, both operands K-major SWIZZLE_NONE from shared memory, A a
// 2 KB-per-chunk weight tile (SBO 128, LBO 2048), B a padded input row [chunk][x'][8 ti] (SBO 128, LBO =
// row chunk bytes) read at a pixel-shifted start -- issued by one thread on every SM at once, in K10's
// column-pair order (corr, main, corr, corr, main, corr into two accumulators).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o k10_rate tools/k10/k10_rate.cu && ./k10_rate
// Measured on B200 (gpurun_out/r02bf, r02bp-br; profiles/r02_conv_tc_c4.md):
//   * 128.0 cycles per MMA on 1 SM and on all 148 at once (2.19 PFLOP/s, ~1.81 GHz under that load), with or
//     without the pixel shift, into one or two accumulators; 64.0 at N = 128; a tcgen05.commit every 6 / 12 /
//     24 MMAs costs nothing;
//   * the tensor pipe queues about ONE MMA beyond the running one: an issuer pause of D cycles every 12 MMAs
//     (the `idle` sweep below) costs D - ~70 cycles of pipe time (D = 128 -> 133.6 cycles per MMA, 256 -> 143.4,
//     512 -> 162.9, 1024 -> 208.4).  The issuing thread cannot run ahead, so every gap between two of its
//     UTCHMMAs beyond ~70 cycles is lost -- K10's stage and row boundaries are that loss (its loop keeps the
//     pipe ~90% busy).
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.b32 p, 0, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc));
}

__global__ void __launch_bounds__(128, 1) k10_rate(int n, int nmma, int mode, int shift, int commit_every, int delay, long long* cycles) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t mbar, mbar2;
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t a_bytes = 32768, chunk_b = 288 * 16, b_bytes = 4 * chunk_b;   // A: hi/lo x 4 col x 2 chunk x 2 KB; B: hi/lo x 2 chunks
    for (uint32_t i = tid; i < (a_bytes + b_bytes) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u + i;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(smem_u32(&mbar2)));   // never completes
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tmem_base, tc = tmem_base + 256;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    long long t0 = 0;
    if (tid == 0) {
        const uint64_t dA = desc_kmajor(smem_u32(sm), 2048, 128);
        const uint64_t dB = desc_kmajor(smem_u32(sm + a_bytes), chunk_b, 128) + 16 + 15;   // pixel 31 (pad 16 + R 15)
        const uint64_t aLo = a_bytes / 2 / 16, bLo = 2 * chunk_b / 16, aE = 2 * 2048 / 16;
        t0 = clock64();
        for (int i = 0; i < nmma; i += 6) {
            const int e = (i / 6) & 1;   // the stage's column pair
            const uint64_t a1 = dA + e * 2 * aE, b1 = dB - (shift ? (i / 6) % 30 : 0), a2 = a1 + aE, b2 = b1 - (shift ? 1 : 0);
            if ((mode & 3) == 0) {
                mma(tc, a1, b1 + bLo, idesc); mma(tm, a1, b1, idesc); mma(tc, a1 + aLo, b1, idesc);
                mma(tc, a2, b2 + bLo, idesc); mma(tm, a2, b2, idesc); mma(tc, a2 + aLo, b2, idesc);
            } else if ((mode & 3) == 1) {
                mma(tm, a1, b1 + bLo, idesc); mma(tm, a1, b1, idesc); mma(tm, a1 + aLo, b1, idesc);
                mma(tm, a2, b2 + bLo, idesc); mma(tm, a2, b2, idesc); mma(tm, a2 + aLo, b2, idesc);
            } else {
                mma(tc, a1, b1 + bLo, idesc); mma(tm, a1, b1, idesc); mma(tc, a1 + aLo, b1, idesc);
                mma(tm, a2, b2 + bLo, idesc); mma(tc, a2, b2, idesc); mma(tm, a2 + aLo, b2, idesc);
            }
            // K10 commits every weight stage (12 MMAs) back to the producer: does a commit cost pipe time?
            if (commit_every && ((i / 6 + 1) % commit_every) == 0) {
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar2)));
                // queue-depth probe: the issuer idles `delay` cycles at every stage boundary; the delay the
                // tensor pipe's instruction queue hides shows how far ahead the issuer can be
                if (delay > 0) {
                    const long long t = clock64();
                    while (clock64() - t < delay) {}
                }
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
    }
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n\t}"
                     : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0u));
    if (tid == 0) cycles[blockIdx.x] = clock64() - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main(int argc, char** argv) {
    const int nmma = 6 * 2000;
    long long* dc;
    cudaMalloc(&dc, 148 * 8);
    const size_t smem = 32768 + 4 * 288 * 16 + 1024;
    cudaFuncSetAttribute(k10_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int n : {256})
        for (int mode : {0})
            for (int shift = 1; shift < 2; ++shift)
              for (int commit_every : {2})   // a stage boundary every 12 MMAs
              for (int delay : {0, 64, 128, 192, 256, 384, 512, 768, 1024})
                for (int grid : {1, 148}) {
                    cudaEvent_t e0, e1;
                    cudaEventCreate(&e0); cudaEventCreate(&e1);
                    k10_rate<<<grid, 128, smem>>>(n, nmma, mode, shift, commit_every, delay, dc);   // warm-up
                    cudaEventRecord(e0);
                    k10_rate<<<grid, 128, smem>>>(n, nmma, mode, shift, commit_every, delay, dc);
                    cudaEventRecord(e1);
                    cudaError_t e = cudaDeviceSynchronize();
                    if (e != cudaSuccess) { printf("CUDA error: %s\n", cudaGetErrorString(e)); return 1; }
                    long long c[148];
                    cudaMemcpy(c, dc, grid * 8, cudaMemcpyDeviceToHost);
                    long long mx = 0;
                    for (int i = 0; i < grid; ++i) mx = c[i] > mx ? c[i] : mx;
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    printf("N %3d mode %d shift %d boundary every %d column pairs, idle %4d cycles, grid %3d: %.1f cycles per MMA (max over CTAs), kernel %.3f ms -> %.0f TFLOP/s\n",
                           n, mode, shift, commit_every, delay, grid, (double)mx / nmma, ms, 2.0 * 128 * n * 16 * nmma * grid / (ms * 1e-3) / 1e12);
                }
    return 0;
}
