// probe.cu -- roofline probes used by bench.py (not part of the hot path).
//
// MEASURED_PEAKS.json has the copy bandwidth and the bf16 tensor peak; the
// Fisher kernel is bound by the FP64 pipe, whose peak this probe measures:
// every thread runs 8 independent DFMA chains (enough ILP to cover the FP64
// latency), so the kernel issues DFMA at the pipe's throughput limit.
#include <cuda_runtime.h>

#include "box_muller.cuh"
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

// write-only HBM probes, 16-byte streaming stores.
//   variant 0: grid-stride (the whole grid sweeps the buffer front to back);
//   variant 1: each CTA owns a contiguous segment and writes it with 4
//              independent stores in flight per thread -- the access shape of
//              fill_uniform_fast (many warps writing far-apart 512-byte runs).
__global__ void __launch_bounds__(256) write_probe_kernel(double2 *out, int64_t n) {
    const double2 v = make_double2(1.0, 2.0);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        __stcs(out + i, v);
}

__global__ void __launch_bounds__(256) write_probe_seg_kernel(double2 *out, int64_t n,
                                                              int64_t seg) {
    const double2 v = make_double2(1.0, 2.0);
    const int64_t b0 = (int64_t)blockIdx.x * seg, b1 = min(b0 + seg, n);
    int64_t i = b0 + threadIdx.x;
    for (; i + 3 * 256 < b1; i += 4 * 256) {
        __stcs(out + i, v);
        __stcs(out + i + 256, v);
        __stcs(out + i + 512, v);
        __stcs(out + i + 768, v);
    }
    for (; i < b1; i += 256) __stcs(out + i, v);
}

// rsqrt.approx.f64 seed of box_muller_pair_f32, for the accuracy test
__global__ void rsqrt_probe_kernel(const double *x, double *y, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = RsqrtSeedHw()(x[i]);
}

// variant 2: per-CTA segments with 32-byte stores (STG.E.ENL2.256)
__global__ void __launch_bounds__(256) write_probe_seg256_kernel(double *out, int64_t n4,
                                                                 int64_t seg) {
    const int64_t b0 = (int64_t)blockIdx.x * seg, b1 = min(b0 + seg, n4);
    for (int64_t i = b0 + threadIdx.x; i < b1; i += 256)
        asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(out + 4 * i), "d"(1.0),
                     "d"(2.0), "d"(3.0), "d"(4.0)
                     : "memory");
}

// TMA bulk-store probe: every warp's lane 0 streams its CTA's contiguous
// segment out of one shared-memory chunk with cp.async.bulk (no registers in
// the data path); chunks of kBulkChunk bytes interleaved across the 8 warps
constexpr int kBulkChunk = 16384;
__global__ void __launch_bounds__(256) write_probe_bulk_kernel(unsigned char *out, int64_t bytes,
                                                               int64_t seg) {
    __shared__ __align__(128) unsigned char buf[kBulkChunk];
    for (int i = threadIdx.x; i < kBulkChunk / 8; i += 256) ((double *)buf)[i] = 1.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const int64_t b0 = (int64_t)blockIdx.x * seg, b1 = min(b0 + seg, bytes);
    if ((threadIdx.x & 31) == 0) {
        const int w = threadIdx.x >> 5;
        const uint32_t src = (uint32_t)__cvta_generic_to_shared(buf);
        for (int64_t off = b0 + (int64_t)w * kBulkChunk; off < b1; off += 8LL * kBulkChunk) {
            const uint32_t n = (uint32_t)min((int64_t)kBulkChunk, b1 - off);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         ::"l"(out + off), "r"(src), "r"(n) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

// FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) issue rate: every warp runs
// 16 independent accumulators (the shape of the Cholesky tile products) on
// register operands; 512 flops per instruction
__global__ void __launch_bounds__(128) dmma_probe_kernel(double *out, int iters, double a0) {
    double acc[16][2];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q][0] = acc[q][1] = 0.0;
    double a = a0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 16; ++q)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(acc[q][0]), "+d"(acc[q][1])
                         : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 16; ++q) s += acc[q][0] + acc[q][1];
    if (s == 12345.678) out[0] = s;  // keeps the chains live
}

}  // namespace sfb

using namespace sfb;

extern "C" int sfb_probe_dmma(double *d_out, int64_t blocks, int iters, void *stream) {
    dmma_probe_kernel<<<(unsigned)blocks, 128, 0, (cudaStream_t)stream>>>(d_out, iters, 1e-3);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SFB_E_CUDA, "dmma probe: %s", cudaGetErrorString(e));
    return SFB_OK;
}

extern "C" int sfb_probe_write(void *d_out, int64_t bytes, int variant, void *stream) {
    const int64_t n = bytes / 16;
    if (variant == 3 || variant == 4) {  // TMA bulk stores; 4: 2 CTAs per SM
        const int64_t blocks = 148 * (variant == 3 ? 8 : 2);
        const int64_t seg = ((bytes + blocks - 1) / blocks + kBulkChunk - 1) / kBulkChunk *
                            kBulkChunk;
        write_probe_bulk_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
            (unsigned char *)d_out, bytes, seg);
    } else if (variant == 2) {
        const int64_t n4 = bytes / 32;
        const int64_t blocks = 148 * 64;
        const int64_t seg = (n4 + blocks - 1) / blocks;
        write_probe_seg256_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
            (double *)d_out, n4, seg);
    } else if (variant == 1) {
        const int64_t blocks = 148 * 64;
        const int64_t seg = (n + blocks - 1) / blocks;
        write_probe_seg_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
            (double2 *)d_out, n, seg);
    } else {
        write_probe_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>((double2 *)d_out, n);
    }
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

extern "C" int sfb_probe_rsqrt(const double *d_x, double *d_y, int64_t n, void *stream) {
    if (n <= 0) return SFB_OK;
    rsqrt_probe_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(d_x, d_y, n);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SFB_E_CUDA, "rsqrt probe: %s", cudaGetErrorString(e));
    return SFB_OK;
}
