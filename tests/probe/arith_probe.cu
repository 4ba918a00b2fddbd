// Test-only probe (built by tests/test_arith_gpu.py): the fused kernels'
// shared-divisor primitives (arith.cuh PrimCalc) against the per-quotient
// library path on arbitrary operand bits, including zeros, subnormals,
// infinities, NaNs and overflow/underflow ranges.
#include <cuda_runtime.h>

#include "../../paper_2505_20911_b200/csrc/arith.cuh"

using namespace mpfd_b200;

template <class W>
__global__ void k_prim(const W* in, long n, W* fast, W* ref, W half, W gm1, W gM2) {
    const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const W* q = in + 5 * i;
    const PrimOut<W> a = PrimCalc<W>::run(q[0], q[1], q[2], q[3], q[4], half, gm1, gM2);
    const PrimOut<W> b = prim_generic<W>(q[0], q[1], q[2], q[3], q[4], half, gm1, gM2);
    W* f = fast + 5 * i;
    W* r = ref + 5 * i;
    f[0] = a.ux; f[1] = a.uy; f[2] = a.uz; f[3] = a.pr; f[4] = a.Tv;
    r[0] = b.ux; r[1] = b.uy; r[2] = b.uz; r[3] = b.pr; r[4] = b.Tv;
}

template <class W>
static int run(const void* host_in, long n, void* host_fast, void* host_ref, W half, W gm1, W gM2) {
    W *in, *f, *r;
    const size_t bytes = sizeof(W) * 5 * (size_t)n;
    if (cudaMalloc(&in, bytes) || cudaMalloc(&f, bytes) || cudaMalloc(&r, bytes)) return 1;
    cudaMemcpy(in, host_in, bytes, cudaMemcpyHostToDevice);
    k_prim<W><<<(unsigned)((n + 127) / 128), 128>>>(in, n, f, r, half, gm1, gM2);
    cudaMemcpy(host_fast, f, bytes, cudaMemcpyDeviceToHost);
    cudaMemcpy(host_ref, r, bytes, cudaMemcpyDeviceToHost);
    const int err = cudaDeviceSynchronize() != cudaSuccess;
    cudaFree(in);
    cudaFree(f);
    cudaFree(r);
    return err;
}

// in: n points x 5 binary64 (rho, rhou, rhov, rhow, rhoE)
extern "C" int probe_prim_f64(const double* in, long n, double* fast, double* ref, double half, double gm1,
                              double gM2) {
    return run<double>(in, n, fast, ref, half, gm1, gM2);
}
// in: n pairs x 5 float2 (lane pairs), bit patterns
extern "C" int probe_prim_f2(const float* in, long n, float* fast, float* ref, double half, double gm1, double gM2) {
    return run<float2>(in, n, fast, ref, make_float2((float)half, (float)half), make_float2((float)gm1, (float)gm1),
                       make_float2((float)gM2, (float)gM2));
}
// in: n pairs x 5 half2 words (lane pairs), bit patterns
extern "C" int probe_prim_h2(const unsigned* in, long n, unsigned* fast, unsigned* ref, double half, double gm1,
                             double gM2) {
    return run<__half2>(in, n, fast, ref, __half2half2(__double2half(half)), __half2half2(__double2half(gm1)),
                        __half2half2(__double2half(gM2)));
}
