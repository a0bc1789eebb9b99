// Dependent-latency microbenchmark (measurement scaffolding): cycles per
// dependent DFMA / DMUL / DADD / MUFU.RCP64H / SHFL / FFMA on one warp.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/lat/lat_probe.cu -o /tmp/lat && /tmp/lat
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double *out, long long *cyc, double x0, int n) {
    double x = x0 + threadIdx.x * 1e-9, y = 1.0000001;
    float xf = (float)x, yf = 1.0000001f;
    __syncwarp();
    long long t0 = clock64();
#pragma unroll 1
    for (int k = 0; k < n; ++k) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            if (OP == 0) x = fma(x, y, -1e-7);
            if (OP == 1) x = x * y;
            if (OP == 2) x = x + y;
            if (OP == 3) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x));
            if (OP == 4) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
            if (OP == 5) xf = fmaf(xf, yf, -1e-7f);
            if (OP == 6) asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(x));
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = x + xf;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int OP>
void run(const char *name) {
    double *o;
    long long *c, hc;
    cudaMalloc(&o, 256);
    cudaMalloc(&c, 8);
    const int n = 4096;
    chain<OP><<<1, 32>>>(o, c, 1.5, n);
    chain<OP><<<1, 32>>>(o, c, 1.5, n);
    cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("%-22s %6.1f cycles per dependent op\n", name, (double)hc / (16.0 * n));
    cudaFree(o);
    cudaFree(c);
}

int main() {
    run<0>("DFMA");
    run<1>("DMUL");
    run<2>("DADD");
    run<3>("MUFU.RCP64H (rcp.approx.f64)");
    run<6>("MUFU.RSQ64H (rsqrt.approx.f64)");
    run<4>("SHFL (double = 2 SHFL)");
    run<5>("FFMA");
    return 0;
}
