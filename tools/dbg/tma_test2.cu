#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <vector>
#include "../../paper_2402_15322_b200/csrc/conv_common.cuh"
using namespace se2;
__global__ void kt(const float* fsrc, float* out, int mode, int bw, int bh, int cx, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(128) float sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 8192);
    const CUtensorMap* tp = &tmap;
    if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_fence_init(); }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (mode & 4) fence_proxy_async();
        uint32_t bytes = bw * bh * 4 + ((mode & 2) ? 512 : 0);
        mbar_expect_tx(bar, bytes);
        if (mode & 1) tma_load_3d(sm, tp, bar, cx, -5, 3);
        else tma_load_3d(sm, tp, bar, 0, 0, 0);
        if (mode & 2) bulk_load(sm + 7000, fsrc, 512, bar);
    }
    mbar_wait(bar, 0);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = sm[i];
}
int main() {
    std::vector<float> h(64 * 64 * 8);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
    float *d, *o; cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 4096 * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap map;
    bool ok = make_field_tmap(&map, d, 64, 64, 8, 16, 8);
    int cxs[] = {4, 3, 1, 5, 0, -4, -8, -1, -3, -5};
    for (int cx : cxs) {
        kt<<<1, 64, 8192 * 4 + 64>>>(d, o, 1, 16, 8, cx, map);
        cudaError_t e = cudaDeviceSynchronize();
        printf("cx %d: %s\n", cx, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
