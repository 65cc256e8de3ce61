// TMA tensor-map construction (driver entry point fetched through the runtime, so the
// library does not link libcuda directly).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace wino {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_tiled_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// fp32 3-D map: dims (d0 innermost, d1, d2) with row strides s1, s2 in bytes; box (b0, b1, 1);
// 128-byte swizzle (b0*4 must be 128) — with 32-byte atoms for MN-major tf32 operands
// (UMMA layout SWIZZLE_128B_BASE32B); out-of-bounds elements read as zero.
inline int& last_tmap_error() {
    static thread_local int e = 0;
    return e;
}

inline bool make_map_3d_sw(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                           uint64_t s2, uint32_t b0, uint32_t b1, CUtensorMapSwizzle sw,
                           CUtensorMapDataType dt);

inline bool make_map_3d(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                        uint64_t s2, uint32_t b0, uint32_t b1, bool atom32 = false) {
    return make_map_3d_sw(map, base, d0, d1, d2, s1, s2, b0, b1,
                          atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
}

// same with an explicit swizzle mode (output staging boxes use 64- or 128-byte swizzles) and
// element type (uint8 for the int8 digit tensors of wino_ozaki.cuh)
inline bool make_map_3d_sw(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                           uint64_t s2, uint32_t b0, uint32_t b1, CUtensorMapSwizzle sw,
                           CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32) {
    EncodeTiledFn fn = encode_tiled_fn();
    if (!fn) {
        last_tmap_error() = -1;
        return false;
    }
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {s1, s2};
    cuuint32_t box[3] = {b0, b1, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = fn(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    last_tmap_error() = (int)r;
    return r == CUDA_SUCCESS;
}

// uint8 4-D map (d0 innermost .. d3) over a dense [d3][d2][d1][d0] byte tensor; box (b0, b1, 1, d3):
// one load brings a box of every d3 plane (the exact dW_F digit planes, wino_xdw.cuh)
inline bool make_map_4d_u8(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3,
                           uint32_t b0, uint32_t b1, CUtensorMapSwizzle sw) {
    EncodeTiledFn fn = encode_tiled_fn();
    if (!fn) {
        last_tmap_error() = -1;
        return false;
    }
    cuuint64_t dims[4] = {d0, d1, d2, d3};
    cuuint64_t strides[3] = {d0, d0 * d1, d0 * d1 * d2};
    cuuint32_t box[4] = {b0, b1, 1, (cuuint32_t)d3};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(base), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    last_tmap_error() = (int)r;
    return r == CUDA_SUCCESS;
}

}  // namespace wino
