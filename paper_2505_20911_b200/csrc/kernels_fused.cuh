// kernels_fused.cuh -- fused residual + RK stage update (filled in later).
#pragma once

#include "kernels_staged.cuh"

namespace mpfd_b200 {

template <int MODE, int QK, int TK, int RK, int WK>
struct FusedPlan {
    static constexpr bool available = false;
    static void launch(const Geo&, cudaStream_t, const void*, void*, const void*, void*, void*,
                       const PrimConsts&, const ResConsts&, const StageConsts&, bool, const RkConsts&,
                       bool, DevDiv*, int, int) {}
};

}  // namespace mpfd_b200
