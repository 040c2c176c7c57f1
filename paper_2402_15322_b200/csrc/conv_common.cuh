// Shared device helpers of the two conv engines (linear FFMA and exact log-sum-exp).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "se2_internal.cuh"

namespace se2 {

bool make_field_tmap(CUtensorMap* map, const float* base, int nx, int ny, int planes, int boxw, int boxh);
bool make_tmap_5d(CUtensorMap* map, CUtensorMapDataType dtype, const void* base, const uint64_t* dims,
                  const uint64_t* strides, const uint32_t* box);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// 4-byte async copy global -> shared with zero fill when !valid (src-size 0)
__device__ __forceinline__ void cp_async4(void* dst, const float* src, bool valid) {
    int sz = valid ? 4 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(sz));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- mbarrier + TMA (cp.async.bulk) helpers -----------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}
// 3-D tensor tile global -> shared (TMA), completion counted on `bar`; out-of-bounds elements are
// filled per the tensor map (zeros here)
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
// 5-D tensor tile global -> shared (TMA), destination / barrier as shared-window addresses
__device__ __forceinline__ void tma_load_5d(uint32_t dst, const void* tmap, uint32_t bar, int c0, int c1, int c2, int c3,
                                            int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
        ::"r"(dst), "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
        : "memory");
}
// contiguous bulk copy global -> shared (bytes % 16 == 0), completion counted on `bar`
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// 2^x for x <= 0 on the FMA pipe (frees the MUFU pipe, which bounds the exact log-sum-exp): x is
// clamped at -125 (2^-125 is far below any retained term), n = rint(x) by the 1.5*2^23 trick,
// 2^f = e^{f ln 2} for |f| <= 1/2 by its degree-6 Taylor polynomial (relative error < 1.3e-7, the
// accuracy of ex2.approx), scaled by adding n to the exponent bits.
__device__ __forceinline__ float ex2_poly(float x) {
    x = fmaxf(x, -125.f);
    const float t = x + 12582912.f;
    const float n = t - 12582912.f;
    const float f = x - n;
    float p = 1.5403530393381608e-4f;          // ln2^6 / 720
    p = fmaf(p, f, 1.3333558146428443e-3f);    // ln2^5 / 120
    p = fmaf(p, f, 9.6181291076284772e-3f);    // ln2^4 / 24
    p = fmaf(p, f, 5.5504108664821580e-2f);    // ln2^3 / 6
    p = fmaf(p, f, 2.4022650695910071e-1f);    // ln2^2 / 2
    p = fmaf(p, f, 6.9314718055994531e-1f);    // ln2
    p = fmaf(p, f, 1.f);
    const int ni = __float_as_int(t) - 0x4B400000;
    return __int_as_float(__float_as_int(p) + (ni << 23));
}

__device__ __forceinline__ float lg2_approx(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// log2 of a positive normal x with ABSOLUTE error ~2^-22: the exponent is taken exactly from the bits
// and lg2.approx only sees the mantissa in [1, 2) (where its error is absolute).  lg2.approx on large
// arguments has a relative error, i.e. ~1e-5 absolute at x ~ 2^100, which biased the log-domain
// convs systematically.  x <= 0 or subnormal -> -inf.
__device__ __forceinline__ float lg2_norm(float x) {
    const int ix = __float_as_int(x);
    const int e = (ix >> 23) - 127;
    const float m = __int_as_float((ix & 0x007fffff) | 0x3f800000);
    return (ix >= 0x00800000) ? ((float)e + lg2_approx(m)) : -INFINITY;
}

// Block-wide deterministic sum of one float per thread; result valid in thread 0.
template <int NT>
__device__ __forceinline__ float block_sum(float v, float* red /* >= NT/32 floats */) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) red[w] = v;
    __syncthreads();
    float t = 0.f;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < NT / 32; ++i) t += red[i];
    }
    return t;
}

// Porous-medium prox: u = log s solves g(u) = c e^{(m-1) u} + u - log z = 0, g convex and
// increasing.  Bracket: g(lz) > 0, and at lo = min(lz - 50, (ln 50 - ln c)/(m-1)) both c e^{(m-1) lo} <= 50 and
// lo - lz <= -50, so g(lo) <= 0.  Newton from lz, falling back to bisection of the bracket whenever a step
// leaves it or fails to halve it (safeguarded Newton); c e^{...} is evaluated as exp(ln c + (m-1) u) with the
// exponent capped at 88 (no overflow far above the root).  Returns u; *conv = false when 64 steps did not converge.
__device__ __forceinline__ float porous_prox_u(float lz, float lnc, float m1, bool* conv) {
    float lo = fminf(lz - 50.f, (3.9120230054f - lnc) / m1), hi = lz;
    float u = lz, dold = hi - lo;
    *conv = false;
    for (int it = 0; it < 64; ++it) {
        const float ex = expf(fminf(lnc + m1 * u, 88.f));
        const float g = ex + u - lz;
        if (g > 0.f) hi = u; else lo = u;
        const float dg = m1 * ex + 1.f;
        float un = u - g / dg;
        if (!(un > lo && un < hi) || fabsf(2.f * g) > fabsf(dold * dg)) un = 0.5f * (lo + hi);
        dold = un - u;
        u = un;
        if (fabsf(dold) <= 1e-7f * (1.f + fabsf(u)) || hi - lo <= 1e-7f * (1.f + fabsf(u))) {
            *conv = true;
            break;
        }
    }
    return u;
}

// Apply the fused epilogue to one conv output.  y_lin: linear-domain value (linear engine),
// or ly (natural log) in the log engine.  Returns the marginal-error contribution.
template <bool LOG>
__device__ __forceinline__ float apply_epilogue(const Epilogue& e, int64_t idx, int ix, int iy, float y) {
    float err = 0.f;
    // the engine's own shift hint for the next iteration: every row it computed, halo rows included
    // (their outputs are not stored, but a stale hint there would only force the verified redo)
    if (LOG && e.hint_out != nullptr && e.slab_hi > 0) e.hint_out[idx] = y;
    if (e.slab_hi > 0 && (iy < e.slab_lo || iy >= e.slab_hi)) return 0.f;   // a neighbour's row: not ours
    if (e.op == EPI_DOT) return LOG ? expf(e.err_a[idx] + y) : e.err_a[idx] * y;
    if (e.err_a != nullptr) {
        float a_old = e.err_a[idx];
        float mu = e.err_mu[idx];
        float row = LOG ? expf(a_old + y) : a_old * y;
        err = fabsf(row - mu);
    }
    if (LOG && e.hint_out != nullptr && e.slab_hi == 0) e.hint_out[idx] = y;
    float o;
    switch (e.op) {
        case EPI_STORE: o = y; break;
        case EPI_DIVIDE:
            if (LOG) {
                const float t = e.target[idx];
                o = (t == -INFINITY) ? -INFINITY : t - y;   // log(0 / y) = -inf, as 0 / max(y, floor) = 0
            } else {
                if (y < kDivFloor && e.guard != nullptr) atomicAdd(&e.guard[0], 1u);
                o = e.target[idx] / fmaxf(y, kDivFloor);
            }
            break;
        case EPI_MULTIPLY: o = LOG ? (e.target[idx] + y) : (e.target[idx] * y); break;
        case EPI_PROX: {
            if (e.prox_kind == 2) {
                // porous medium: safeguarded Newton on u = log s (porous_prox_u); sites not converged
                // in 64 steps are counted
                if (!LOG && y < kDivFloor && e.guard != nullptr) atomicAdd(&e.guard[0], 1u);
                const float lz = LOG ? y : logf(fmaxf(y, kDivFloor));
                bool conv;
                const float u = porous_prox_u(lz, e.prox_lnc, e.prox_m1, &conv);
                if (!conv && e.guard != nullptr) atomicAdd(&e.guard[1], 1u);
                o = LOG ? (u - lz) : expf(u - lz);
                if (e.out2 != nullptr) e.out2[idx] = expf(u);
                break;
            }
            float dxp = ((float)ix + 0.5f - e.cx) * e.hx, dyp = ((float)iy + 0.5f - e.cy) * e.hy;
            float V = dxp * dxp + dyp * dyp;
            if (LOG) {
                o = -e.prox_p * y - e.prox_q * V;
                if (e.out2 != nullptr) e.out2[idx] = expf(o + y);
            } else {
                if (y < kDivFloor && e.guard != nullptr) atomicAdd(&e.guard[0], 1u);
                float z = fmaxf(y, kDivFloor);
                o = exp2f(-e.prox_p * log2f(z) - e.prox_q * V * kLog2e);
                if (e.out2 != nullptr) e.out2[idx] = o * z;
            }
            break;
        }
        default: return err;  // EPI_ERRONLY
    }
    e.out[idx] = o;
    if (e.slab_hi > 0) {   // boundary rows into the neighbours' halo rows (peer memory)
        const int64_t plane = idx / ((int64_t)e.ny_self * e.nx_self);
        if (e.halo_up != nullptr && iy < e.slab_lo + e.slab_halo)
            e.halo_up[(plane * e.ny_up + iy + e.up_shift) * e.nx_self + ix] = o;
        if (e.halo_dn != nullptr && iy >= e.slab_hi - e.slab_halo)
            e.halo_dn[(plane * e.ny_dn + iy - e.dn_shift) * e.nx_self + ix] = o;
    }
    return err;
}

// K4P's epilogue (fp64 potentials): out = target -+ ly, error of the previous iterate |a_old K b - mu|
// out-of-line copy for kernels that apply the epilogue to many outputs per thread at their end (the log
// engines): one body instead of one inlined per output keeps the kernel's code small
template <bool LOG>
__device__ __noinline__ float apply_epilogue_call(const Epilogue& e, int64_t idx, int ix, int iy, float y) {
    return apply_epilogue<LOG>(e, idx, ix, iy, y);
}

static __device__ __noinline__ float apply_epilogue_precise(const EpiP& e, int64_t idx, double ly) {
    float err = 0.f;
    if (e.err_a != nullptr) err = fabsf((float)exp(e.err_a[idx] + ly) - e.err_mu[idx]);
    double o;
    switch (e.op) {
        case EPI_STORE: o = ly; break;
        case EPI_DIVIDE: {
            const double t = e.target[idx];
            o = (t == -(double)INFINITY) ? -(double)INFINITY : t - ly;   // log(0 / y) = -inf
            break;
        }
        case EPI_MULTIPLY: o = e.target[idx] + ly; break;
        default: return err;   // EPI_ERRONLY
    }
    e.out[idx] = o;
    return err;
}

}  // namespace se2
