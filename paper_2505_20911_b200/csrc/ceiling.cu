// ceiling.cu -- measured issue ceilings of the arithmetic the residual
// kernels run (hard part 1: "verify FP64, FP32 and HFMA2 issue
// rates with a microbenchmark on the box").  The reference's arithmetic is
// unfused add/sub/mul (-ffp-contract=off, proj/CMakeLists.txt:13), so the
// ceiling that bounds the compute-heavy fused kernels is the rate of exactly
// those instructions in the forms the kernels emit: DADD/DMUL (fp64), FADD2
// and the FFMA2-with-opaque-zero product (fp32 pairs), HADD2/HMUL2 (fp16
// pairs).  Reported as lane operations per second.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>

#include "../../include/mpfd_b200.h"
#include "arith.cuh"

namespace mpfd_b200 {

template <class T>
struct Lanes {
    static constexpr int n = 1;
};
template <>
struct Lanes<float2> {
    static constexpr int n = 2;
};
template <>
struct Lanes<__half2> {
    static constexpr int n = 2;
};

// 8 independent chains per thread, alternating add and mul; the operands
// (0 and 1) are runtime values, so nothing folds and the chains stay exact
template <class T>
__global__ void __launch_bounds__(256) k_issue(T* out, T zero, T one, int iters) {
    T a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = Op<T>::add(one, zero);
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = Op<T>::add(a[i], zero);
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = Op<T>::mul(a[i], one);
    }
    T s = a[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) s = Op<T>::add(s, a[i]);
    if (iters < 0) out[threadIdx.x] = s;  // never: keeps the chains live
}

template <class T>
static double measure(T zero, T one) {
    cudaStream_t st;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return -1.0;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    k_issue<T><<<blocks, threads, 0, st>>>(nullptr, zero, one, 64);  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a, st);
        k_issue<T><<<blocks, threads, 0, st>>>(nullptr, zero, one, iters);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        best = std::min(best, ms);
    }
    const cudaError_t e = cudaGetLastError();
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaStreamDestroy(st);
    if (e != cudaSuccess) return -1.0;
    const double ops = (double)blocks * threads * iters * 16.0 * Lanes<T>::n;
    return ops / (best * 1e-3);
}

}  // namespace mpfd_b200

extern "C" int mpfd_b200_issue_ceiling(int device, double out[3]) {
    using namespace mpfd_b200;
    if (!out) return MPFD_ECONFIG;
    if (cudaSetDevice(device) != cudaSuccess) return MPFD_EDEVICE;
    out[0] = measure<double>(0.0, 1.0);
    out[1] = measure<float2>(make_float2(0.f, 0.f), make_float2(1.f, 1.f));
    out[2] = measure<__half2>(__floats2half2_rn(0.f, 0.f), __floats2half2_rn(1.f, 1.f));
    return (out[0] > 0 && out[1] > 0 && out[2] > 0) ? MPFD_OK : MPFD_EDEVICE;
}
