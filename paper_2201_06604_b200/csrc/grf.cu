// grf.cu -- Matern covariance kernels of the Gaussian-random-field pipeline
// (reference grf.py:116-187).
//
// The reference builds each covariance block on the host: scipy pdist of the
// anisotropically transformed cell centres, the Matern correlation
//     rho(d) = 2^(1-kappa) / Gamma(kappa) (sqrt(8 kappa) d / phi)^kappa K_kappa(.)
// through scipy.special.kv (AMOS), mirrored from the upper triangle, with the
// variance on the diagonal.  Here:
//   * matern_cov_pairs: one thread per (block, i < j) pair of arbitrary
//     coordinates, writing (i, j) and (j, i) (exactly symmetric) and the
//     diagonal;
//   * matern_cov_offsets: for a regular GridSpec the transformed distance of
//     cells i, j depends only on their index offset (dy, dx), so rho is
//     evaluated once per distinct offset ((2 nx - 1)(2 ny - 1) Bessel calls
//     instead of n^2 / 2) and the block is a gather from that table;
//   * bessel_k / matern_correlation: the elementwise API functions.
// K_nu is bessel_k.cuh (CF2 / trapezoidal integral, ~1e-13 vs AMOS): the GRF
// path is compared with the reference within tolerances, as its own tests do.
#include <cuda_runtime.h>
#include <math.h>

#include "bessel_k.cuh"
#include "sfb_internal.h"

namespace sfb {

__global__ void bessel_k_kernel(double nu, const double *__restrict__ x, double *__restrict__ out,
                                int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = bessel_k(nu, x[i]);
}

// grf.py:138-159: arg = sqrt(8 kappa) d / phi; 1 at arg == 0
__device__ __forceinline__ double matern_rho(double kappa, double lg, double s8k, double range,
                                             double d) {
    const double arg = s8k * d / range;
    return arg > 0.0 ? matern_corr_arg(kappa, lg, arg) : 1.0;
}

__global__ void matern_corr_kernel(double kappa, double lg, double s8k, double range,
                                   const double *__restrict__ d, double *__restrict__ out,
                                   int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = matern_rho(kappa, lg, s8k, range, d[i]);
}

struct MaternDev {  // one parameter set, host-prepared
    double kappa, lg, s8k, range, variance;
    double t00, t01, t10, t11;  // anisotropy transform (scale @ rot), grf.py:127-132
};

// arbitrary coordinates (n, 2): pair (i, j), i < j, of block b
__global__ void matern_cov_pairs(const double *__restrict__ coords, int64_t n,
                                 const MaternDev *__restrict__ prm, int nb,
                                 double *__restrict__ out) {
    const int64_t npairs = n * (n - 1) / 2;
    const int64_t total = npairs * nb;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(q / npairs);
        const int64_t p = q - (int64_t)b * npairs;
        // row i of the condensed upper triangle: p = i n - i (i + 1) / 2 + (j - i - 1)
        int64_t i = (int64_t)((2.0 * n - 1.0 - sqrt((2.0 * n - 1.0) * (2.0 * n - 1.0) - 8.0 * p)) / 2.0);
        while (i > 0 && i * n - i * (i + 1) / 2 > p) --i;
        while ((i + 1) * n - (i + 1) * (i + 2) / 2 <= p) ++i;
        const int64_t j = p - (i * n - i * (i + 1) / 2) + i + 1;
        const MaternDev m = prm[b];
        // transformed coordinates as the reference forms them: coords @ T^T
        const double xi = coords[2 * i], yi = coords[2 * i + 1];
        const double xj = coords[2 * j], yj = coords[2 * j + 1];
        const double ui = xi * m.t00 + yi * m.t01, vi = xi * m.t10 + yi * m.t11;
        const double uj = xj * m.t00 + yj * m.t01, vj = xj * m.t10 + yj * m.t11;
        const double du = ui - uj, dv = vi - vj;
        const double d = sqrt(du * du + dv * dv);  // scipy pdist euclidean
        const double c = m.variance * matern_rho(m.kappa, m.lg, m.s8k, m.range, d);
        double *blk = out + (int64_t)b * n * n;
        blk[i * n + j] = c;
        blk[j * n + i] = c;
    }
    // the diagonal: exactly the variance (grf.py:186)
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n * nb;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(q / n);
        const int64_t i = q - (int64_t)b * n;
        out[(int64_t)b * n * n + i * n + i] = prm[b].variance;
    }
}

// regular grid: table of variance * rho over the canonical offsets
// (dy > 0, or dy == 0 and dx >= 0); index (dy) * (2 nx - 1) + (dx + nx - 1)
__global__ void matern_offset_table(int nx, int ny, double cell, const MaternDev *__restrict__ prm,
                                    int nb, double *__restrict__ table) {
    const int w = 2 * nx - 1;
    const int64_t per = (int64_t)ny * w;
    const int64_t total = per * nb;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(q / per);
        const int64_t r = q - (int64_t)b * per;
        const int dy = (int)(r / w), dx = (int)(r - (int64_t)dy * w) - (nx - 1);
        const MaternDev m = prm[b];
        const double ex = dx * cell, ey = dy * cell;
        const double du = ex * m.t00 + ey * m.t01, dv = ex * m.t10 + ey * m.t11;
        const double d = sqrt(du * du + dv * dv);
        table[q] = (dx == 0 && dy == 0) ? m.variance
                                        : m.variance * matern_rho(m.kappa, m.lg, m.s8k, m.range, d);
    }
}

// cells row-major over (y, x): cell k = (k / nx, k % nx); block gather.  One
// CTA per output row (block b, row i): the row's cell coordinates once, then
// coalesced stores along j with 32-bit index arithmetic (the flat 64-bit
// div/mod per element made this 6x slower than its HBM write time).
__global__ void matern_cov_offsets(int nx, int ny, const double *__restrict__ table, int nb,
                                   double *__restrict__ out) {
    const int n = nx * ny, w = 2 * nx - 1;
    const int64_t per = (int64_t)ny * w;
    for (int64_t row = blockIdx.x; row < (int64_t)n * nb; row += gridDim.x) {
        const int b = (int)(row / n), i = (int)(row - (int64_t)b * n);
        const int iy = i / nx, ix = i - iy * nx;
        const double *tb = table + (int64_t)b * per + nx - 1;
        double *o = out + row * n;
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            const int jy = j / nx, jx = j - jy * nx;
            int dy = iy - jy, dx = ix - jx;
            if (dy < 0 || (dy == 0 && dx < 0)) {  // canonical half: rho(-d) == rho(d)
                dy = -dy;
                dx = -dx;
            }
            o[j] = tb[dy * w + dx];
        }
    }
}

static int launch_err(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SFB_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return SFB_OK;
}

static int prepare(const double *params, int nb, MaternDev *out) {
    for (int b = 0; b < nb; ++b) {
        const double *p = params + 5 * b;  // shape, range, variance, ratio, angle
        if (!(p[0] > 0 && p[1] > 0 && p[2] > 0) || !(p[3] >= 1.0))
            return fail(SFB_E_INVALID_PARAMS, "invalid Matern parameters in set %d", b);
        const double c = cos(p[4]), s = sin(p[4]);
        // (scale @ rot) with rot = [[c, -s], [s, c]], scale = diag(1, ratio)
        out[b] = MaternDev{p[0], lgamma(p[0]), sqrt(8.0 * p[0]), p[1], p[2],
                           c, -s, p[3] * s, p[3] * c};
    }
    return SFB_OK;
}

}  // namespace sfb

using namespace sfb;

extern "C" {

int sfb_bessel_k(double nu, const double *d_x, int64_t n, double *d_out, void *stream) {
    if (!(nu > 0)) return fail(SFB_E_INVALID_ARGUMENT, "Bessel order must be > 0");
    if (n <= 0) return SFB_OK;
    bessel_k_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(nu, d_x, d_out, n);
    return launch_err("bessel_k");
}

int sfb_matern_correlation(double kappa, double range, const double *d_dist, int64_t n,
                           double *d_out, void *stream) {
    if (!(kappa > 0 && range > 0)) return fail(SFB_E_INVALID_PARAMS, "invalid Matern parameters");
    if (n <= 0) return SFB_OK;
    matern_corr_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        kappa, lgamma(kappa), sqrt(8.0 * kappa), range, d_dist, d_out, n);
    return launch_err("matern_correlation");
}

int sfb_matern_cov(const double *params, int nb, const double *d_coords, int64_t n, int nx,
                   int ny, double cell, double *d_scratch, double *d_out, void *stream) {
    if (nb < 1) return fail(SFB_E_INVALID_PARAMS, "need at least one parameter set");
    if (n < 1) return fail(SFB_E_INVALID_ARGUMENT, "need at least one coordinate");
    MaternDev host[64];
    if (nb > 64) return fail(SFB_E_INVALID_ARGUMENT, "at most 64 parameter sets per call");
    if (int rc = prepare(params, nb, host)) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    // parameters travel in the scratch buffer's head (caller sizes it)
    MaternDev *dprm = (MaternDev *)d_scratch;
    cudaError_t e = cudaMemcpyAsync(dprm, host, sizeof(MaternDev) * nb, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return fail(SFB_E_CUDA, "matern params: %s", cudaGetErrorString(e));
    const unsigned grid = 148 * 16;
    if (nx > 0 && ny > 0 && (int64_t)nx * ny == n) {
        double *table = (double *)(dprm + 64);
        matern_offset_table<<<grid, 256, 0, st>>>(nx, ny, cell, dprm, nb, table);
        if (int rc = launch_err("matern_offset_table")) return rc;
        matern_cov_offsets<<<grid, 256, 0, st>>>(nx, ny, table, nb, d_out);
        return launch_err("matern_cov_offsets");
    }
    matern_cov_pairs<<<grid, 256, 0, st>>>(d_coords, n, dprm, nb, d_out);
    return launch_err("matern_cov_pairs");
}

int64_t sfb_matern_scratch_bytes(int nb, int nx, int ny) {
    return (int64_t)sizeof(MaternDev) * 64 +
           (int64_t)8 * nb * (int64_t)(nx > 0 ? ny : 0) * (int64_t)(nx > 0 ? 2 * nx - 1 : 0) + 64;
}

double sfb_host_bessel_k(double nu, double x) { return bessel_k(nu, x); }

}  // extern "C"
