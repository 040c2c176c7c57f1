// Host-side TMA tensor-map creation (driver entry point fetched through the runtime, no -lcuda).
#include <cuda.h>
#include <stdlib.h>
#include <cuda_runtime.h>

#include "conv_common.cuh"

namespace se2 {

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t encode_fn() {
    static PFN_encodeTiled_t fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled_t>(p);
    }
    return fn;
}

// fp32 field [planes][ny][nx] -> tensor map with box {boxw, boxh, 1}; false if TMA cannot describe it
// (row stride not a multiple of 16 B, misaligned base, box too large) -> the caller uses cp.async.
bool make_field_tmap(CUtensorMap* map, const float* base, int nx, int ny, int planes, int boxw, int boxh) {
    static const bool disabled = getenv("SE2_NO_TMA") != nullptr;   // diagnostics: force the cp.async path
    if (disabled) return false;
    PFN_encodeTiled_t fn = encode_fn();
    if (!fn) return false;
    if ((nx * sizeof(float)) % 16 != 0 || (reinterpret_cast<uintptr_t>(base) % 16) != 0) return false;
    if (boxw > 256 || boxh > 256 || (boxw * sizeof(float)) % 16 != 0) return false;
    cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)nx * sizeof(float), (cuuint64_t)nx * ny * sizeof(float)};
    cuuint32_t box[3] = {(cuuint32_t)boxw, (cuuint32_t)boxh, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// generic 5-D tiled map (dims / box innermost first, strides in bytes of dims 1..4), no swizzle, no
// OOB handling needed by the caller; false if the driver rejects it
bool make_tmap_5d(CUtensorMap* map, CUtensorMapDataType dtype, const void* base, const uint64_t* dims,
                  const uint64_t* strides, const uint32_t* box) {
    PFN_encodeTiled_t fn = encode_fn();
    if (!fn) return false;
    cuuint64_t d[5], st[4];
    cuuint32_t b[5], estr[5] = {1, 1, 1, 1, 1};
    for (int i = 0; i < 5; ++i) { d[i] = dims[i]; b[i] = box[i]; }
    for (int i = 0; i < 4; ++i) st[i] = strides[i];
    CUresult r = fn(map, dtype, 5, const_cast<void*>(base), d, st, b, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace se2
