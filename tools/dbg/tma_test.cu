// standalone TMA sanity test (debug only)
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <vector>
#include "../../paper_2402_15322_b200/csrc/conv_common.cuh"
using namespace se2;
__global__ void k_bulk(const float* src, float* out, int mode, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(128) float sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 4096);
    if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_fence_init(); }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (mode == 0) { mbar_expect_tx(bar, 1024); bulk_load(sm, src, 1024, bar); }
        else if (mode == 1) { mbar_expect_tx(bar, 16 * 8 * 4); tma_load_3d(sm, &tmap, bar, 0, 0, 0); }
        else { mbar_expect_tx(bar, 16 * 8 * 4); tma_load_3d(sm, &tmap, bar, -4, -2, 1); }
    }
    mbar_wait(bar, 0);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = sm[i];
}
int main() {
    std::vector<float> h(64 * 64 * 4);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
    float *d, *o; cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 4096 * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap map;
    bool ok = make_field_tmap(&map, d, 64, 64, 4, 16, 8);
    printf("tmap ok %d\n", ok);
    for (int mode = 0; mode < 3; ++mode) {
        cudaMemset(o, 0, 4096 * 4);
        k_bulk<<<1, 128, 4096 * 4 + 64>>>(d, o, mode, map);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> r(256);
        cudaMemcpy(r.data(), o, 256 * 4, cudaMemcpyDeviceToHost);
        printf("mode %d: %s  out[0..3]=%g %g %g %g out[16]=%g out[20]=%g\n", mode, cudaGetErrorString(e), r[0], r[1], r[2], r[3], r[16], r[36]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
