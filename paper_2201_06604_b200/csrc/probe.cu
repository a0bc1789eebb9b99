// probe.cu -- roofline probes used by bench.py (not part of the hot path).
//
// MEASURED_PEAKS.json has the copy bandwidth and the bf16 tensor peak; the
// Fisher kernel is bound by the FP64 pipe, whose peak this probe measures:
// every thread runs 8 independent DFMA chains (enough ILP to cover the FP64
// latency), so the kernel issues DFMA at the pipe's throughput limit.
#include <cuda_runtime.h>

#include "fisher_sampler.cuh"
#include "sfb_internal.h"

namespace sfb {

__global__ void __launch_bounds__(256) fp64_probe_kernel(double *out, int iters, double a,
                                                         double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __fma_rn(x[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

// write-only HBM probe: 16-byte streaming stores, grid-stride
__global__ void __launch_bounds__(256) write_probe_kernel(double2 *out, int64_t n) {
    const double2 v = make_double2(1.0, 2.0);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        __stcs(out + i, v);
}

// div_walk (fisher_sampler.cuh) vs the IEEE __ddiv_rn on pseudo-random walk
// operands: a in [2^-970, 1] (log-uniform + uniform), b an exact integer product
// (k+1)(m+1) up to ~2^62 or small; counts mismatches
__global__ void div_probe_kernel(uint64_t seed, int64_t per_thread, unsigned long long *bad,
                                 double *example) {
    uint64_t x = seed ^ (0x9e3779b97f4a7c15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1));
    unsigned long long nbad = 0;
    for (int64_t i = 0; i < per_thread; ++i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        const uint64_t y1 = x;
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        const uint64_t y2 = x;
        double a = (double)(y1 >> 11) * 0x1p-53;
        if (i & 1) a = ldexp(a + 0.5, -(int)(y2 % 970));
        const double c = (double)((y2 >> 8) % 2000000000ull) + 1.0;
        const double d = (double)((y1 >> 3) % ((i & 2) ? 2000000000ull : 40000ull)) + 1.0;
        const double b = c * d;
        const double q = div_walk(a, b), r = __ddiv_rn(a, b);
        if (__double_as_longlong(q) != __double_as_longlong(r)) {
            ++nbad;
            example[0] = a;
            example[1] = b;
        }
    }
    if (nbad) atomicAdd(bad, nbad);
}

}  // namespace sfb

using namespace sfb;

extern "C" int sfb_probe_div(uint64_t seed, int64_t per_thread, uint64_t *d_bad, double *d_example,
                             void *stream) {
    div_probe_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(
        seed, per_thread, (unsigned long long *)d_bad, d_example);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SFB_E_CUDA, "div probe: %s", cudaGetErrorString(e));
    return SFB_OK;
}

extern "C" int sfb_probe_write(void *d_out, int64_t bytes, void *stream) {
    write_probe_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>((double2 *)d_out, bytes / 16);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SFB_E_CUDA, "write probe: %s", cudaGetErrorString(e));
    return SFB_OK;
}

extern "C" int sfb_probe_fp64(double *d_out, int64_t blocks, int iters, void *stream) {
    fp64_probe_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(d_out, iters,
                                                                          0.999999, 1e-7);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SFB_E_CUDA, "fp64 probe: %s", cudaGetErrorString(e));
    return SFB_OK;
}
