// maps2d.cuh -- TMA descriptors of the 2D engine (sweep2p.cuh, sweep2v.cuh, tri2t.cuh): 68 x 68
// windows (64 x 64 box + the 2-node halo of PAPER:828-833) of the two iterate buffers and 64 x 64
// tiles of b and of the face arrays, encoded once per grid at sw_decompose.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace sw {

constexpr int T2 = 64;    // box edge
constexpr int WW = 68;    // window edge (box + 2 halo each side)

struct Maps2d {
    CUtensorMap x[2];
    CUtensorMap b;       // 64 x 64 tiles of b (L2 prefetch)
    CUtensorMap f[2];    // 64 x 64 tiles of F_x, F_y (variable coefficients only)
    bool ok = false, fok = false;
};

inline bool sweep2d_supported(const Geo &G) {
    return G.dim == 2 && G.T[0] == T2 && G.T[1] == T2 && G.off[0] == 0 && (G.P0 % 2) == 0;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    }
    return fn;
}

inline bool encode_2d(CUtensorMap *m, const double *base, int64_t pad0, int64_t pad1, int box0, int box1) {
    EncodeTiledFn enc = get_encode();
    if (!enc || !base) return false;
    cuuint64_t dims[2] = {(cuuint64_t)pad0, (cuuint64_t)pad1};
    cuuint64_t strides[1] = {(cuuint64_t)(pad0 * sizeof(double))};
    cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)box1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void *)base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

inline bool make_maps2d(Maps2d &M, const double *x0, const double *x1, const double *b, const double *fx,
                        const double *fy, int64_t pad0, int64_t pad1) {
    M.ok = encode_2d(&M.x[0], x0, pad0, pad1, WW, WW) && encode_2d(&M.x[1], x1, pad0, pad1, WW, WW) &&
           encode_2d(&M.b, b, pad0, pad1, T2, T2);
    M.fok = fx && fy && encode_2d(&M.f[0], fx, pad0, pad1, T2, T2) && encode_2d(&M.f[1], fy, pad0, pad1, T2, T2);
    return M.ok;
}

}  // namespace sw
