// tma.cuh -- Tensor Memory Accelerator staging of Q planes (sm_100a).
//
// One elected producer thread moves a whole R4 box of the next z-plane of Q
// (all five components) from HBM into shared memory with
// cp.async.bulk.tensor; completion is tracked by a transaction-count
// mbarrier per buffer (double-buffered), and an arrival-count mbarrier per
// buffer tells the issuer when every producer has finished reading it.  x and y are periodic by index in
// the HBM layout (kernels_staged.cuh) and TMA tiles do not wrap, so the box
// moves in parts that are each contiguous in HBM after wrapping their origin
// (WsParts); the producers address every element through its part.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>

namespace mpfd_b200 {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "MPFD_MBAR_WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra MPFD_MBAR_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 4-D tile load (x, y, component, plane) into shared memory, completing on bar
__device__ __forceinline__ void tma_load4(void* dst, const CUtensorMap* map, int x, int y, int c, int z,
                                          unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6];" ::"r"(smem_u32(dst)),
        "l"((unsigned long long)map), "r"(x), "r"(y), "r"(c), "r"(z), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"((unsigned long long)map) : "memory");
}

// Staging layout of one R4 box (TX + 8 by TY + 8 points, 5 components):
// three x-parts -- the 4-column low rim, the TX centre columns, the 4-column
// high rim -- each cut into 4-row groups.  One TMA box moves one (part,
// group) with all five components, landing as [5][4][w] (x fastest) at a
// 128-byte aligned offset; parts are [group][5][4][w].  Every box is
// contiguous in HBM after wrapping its origin when nx is a multiple of TX
// and ny, TY are multiples of 4, so periodic tiles need no special case:
// 3 x (TY + 8) / 4 boxes per plane.
struct WsTma {
    CUtensorMap map[2];  // box (4, 4, 5, 1) and (TX, 4, 5, 1)
};

template <int TX, int TY, class QS>
struct WsParts {
    static constexpr int R4Y = TY + 8;
    static constexpr int NG = R4Y / 4;  // 4-row groups
    __host__ __device__ static constexpr int w(int xp) { return xp == 1 ? TX : 4; }
    // one group of one part, padded to 128 bytes (in elements)
    __host__ __device__ static constexpr int gstride(int xp) {
        return (int)((((size_t)5 * 4 * w(xp) * sizeof(QS) + 127) & ~(size_t)127) / sizeof(QS));
    }
    __host__ __device__ static constexpr int offset(int xp) {  // elements
        return xp == 0 ? 0 : (xp == 1 ? NG * gstride(0) : NG * (gstride(0) + gstride(1)));
    }
    static constexpr size_t total = (size_t)NG * (gstride(0) + gstride(1) + gstride(2)) * sizeof(QS);
    static constexpr unsigned tx_bytes = (unsigned)(5 * R4Y * (TX + 8) * sizeof(QS));
    static_assert(TY % 4 == 0, "4-row groups");
};

// ---------------------------------------------------------------------------
// host: cuTensorMapEncodeTiled through the runtime's driver entry point (no
// -lcuda), maps cached per (buffer, geometry)
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !f)
            throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
        fn = (EncodeTiledFn)f;
    }
    return fn;
}

template <class QS>
inline const WsTma& ws_tma_maps(const void* q, int nx, int ny, int planes, int TX, int TY) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, int, int, int, int>, WsTma> cache;
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(q, nx, ny, planes, TX, TY);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    WsTma t;
    std::memset(&t, 0, sizeof t);
    const CUtensorMapDataType dt = sizeof(QS) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                   : sizeof(QS) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                                     : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    const cuuint64_t dims[4] = {(cuuint64_t)nx, (cuuint64_t)ny, 5, (cuuint64_t)planes};
    const cuuint64_t strides[3] = {(cuuint64_t)nx * sizeof(QS), (cuuint64_t)nx * ny * sizeof(QS),
                                   (cuuint64_t)5 * nx * ny * sizeof(QS)};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    for (int m = 0; m < 2; ++m) {
        const cuuint32_t box[4] = {m ? (cuuint32_t)TX : 4u, 4, 5, 1};
        const CUresult r = encode_tiled()(&t.map[m], dt, 4, const_cast<void*>(q), dims, strides, box, es,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    }
    return cache.emplace(key, t).first->second;
}

}  // namespace mpfd_b200
