// chol.cu -- batched FP64 Cholesky LDL^T and the L D^1/2 Z contraction of the
// Gaussian-random-field pipeline (reference
// grf.py:190-240 chol_batch / multiply_lower_diag_batch).
//
// The reference factors each covariance block with LAPACK dpotrf (C C^T,
// lower), then L = C / diag(C) (unit lower), D = diag(C)^2, and multiplies
// L diag(sqrt D) Z with numpy.  Here, per batch of B blocks of n x n (row-major,
// block b at a + b n^2), all on the device with hand-written kernels:
//
//   * blocked right-looking Cholesky on 64 x 64 tiles, every launch covering
//     all B blocks:
//       chol_diag    -- factor tile (k, k) in shared memory in 16-column
//                       blocks (warp-register factor, per-row panel solve,
//                       sub-block trailing update), the tile below riding
//                       along as extra panel rows, and invert L_kk;
//       chol_panel   -- panel tiles (I, k), I > k + 1:  A_Ik <- A_Ik L_kk^-T
//                       as a 64 x 64 x 64 product with the inverse (the
//                       TRSM-by-inverse of GPU LAPACKs), fused with the next
//                       column's update inside a super-panel;
//       chol_update  -- trailing tiles (I, J), J <= I, over a K range of
//                       panel columns: A_IJ <- A_IJ - sum_k A_Ik A_Jk^T;
//     the products run on the FP64 tensor cores (mma.sync m8n8k4 f64, DMMA;
//     tcgen05 has no FP64 kind), 64 x 64 output tile per CTA, 4 warps of
//     32 x 32, operands staged in shared memory at a padded pitch
//     (conflict-free fragment loads); the schedule (super-panels, lazy
//     per-column updates, look-ahead streams) is in sfb_chol_batch;
//   * chol_finish    -- L = C / diag(C) below the diagonal, 1 on it, 0 above;
//                       D = diag(C)^2 (grf.py:203-207);
//   * lower_diag_mul -- out = L diag(s) Z, s = sqrt(D) or D: one warp per
//                       output row, the row of L read once (HBM-bound).
// A non-positive (or NaN) pivot stops that block: info[b] = LAPACK's info (the
// 1-based order of the first non-positive leading minor), and the later
// stages skip the block.  Results match LAPACK/numpy within rounding (the
// summation order differs), which is how the reference's own tests compare.
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <vector>

#include "sfb_internal.h"

namespace sfb {

constexpr int kT = 64;        // tile
constexpr int kPitch = 68;    // shared-memory row pitch in doubles (64 + 4)
constexpr int kGemmThreads = 128;

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// acc (this warp's 32 x 32 quarter of a 64 x 64 tile, 4 x 4 DMMA tiles of
// 8 x 8, two doubles per lane each) = sa[0:64, 0:64] * sb[0:64, 0:64]^T
__device__ __forceinline__ void tile_product(const double *sa, const double *sb,
                                             double (&acc)[4][4][2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wr = (warp >> 1) * 32, wc = (warp & 1) * 32;
    const int fr = lane >> 2, fk = lane & 3;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 4
    for (int k0 = 0; k0 < kT; k0 += 4) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = sa[(wr + 8 * i + fr) * kPitch + k0 + fk];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = sb[(wc + 8 * j + fr) * kPitch + k0 + fk];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
}

// Factor tile (k, k) of every block and store the inverse of its lower factor.
// The tile's factorisation is on the critical path of every panel step, so it
// is blocked in 16-column steps to keep the number of block-wide barriers
// small (~20 instead of 3 per column):
//   (a) warp 0 factors the 16 x 16 diagonal block in registers (lane i holds
//       row i; the column is broadcast with shuffles, no barriers);
//   (b) the rows below solve against it (one thread per row, forward
//       substitution in registers);
//   (c) the trailing lower part is updated (thread (rr, cc) of every 16 x 16
//       sub-block, the sub-blocks' row/column values loaded once per column);
// then the inverse X = L^-1: the four diagonal blocks by forward substitution
// (warp p, lane c = column c of X_pp), the off-diagonal blocks in three stages
// X_ip = -X_ii sum_{p <= m < i} L_im X_mp.  (Unblocked 64-step forms with
// three barriers per column measured 50-60 us per tile under ncu;
// register-resident fully unrolled 64-column forms stalled on instruction
// fetch, 113-200 us.)
#ifdef DIAG_CLOCKS  // phase timing of chol_diag (experiment builds: -DDIAG_CLOCKS)
#define DCLK(i) do { if (threadIdx.x == 0) dclk[i] = clock64(); } while (0)
#else
#define DCLK(i) do { } while (0)
#endif
constexpr int kDiagThreads = 256;
constexpr int kDP = kT + 1;  // shared pitch (column accesses conflict-free)
// s: 128 rows (the tile, then the tile below it), x: 64, stage products, 1/L_jj
constexpr int kDiagSmem = (3 * kT * kDP + 3 * 256 + kT) * (int)sizeof(double);

// sqrt(d) and 1/sqrt(d) for d > 0 without the library's out-of-line slow paths
// (their calls made the unrolled factor loop save its row registers to the
// stack): rsqrt.approx seed and two Newton steps; within a few ulp of
// LAPACK's sqrt and 1/sqrt (tolerance-level parity).  Subnormal-range d is
// scaled by 2^600 first (the seed flushes subnormals).
__device__ __forceinline__ void sqrt_rsqrt(double d, double &l, double &r) {
    const bool tiny = d < 0x1p-900;
    const double ds = tiny ? d * 0x1p600 : d;
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(ds));
    const double h = 0.5 * ds;
    y = y * fma(-h * y, y, 1.5);
    y = y * fma(-h * y, y, 1.5);
    l = tiny ? ds * y * 0x1p-300 : ds * y;
    r = tiny ? y * 0x1p300 : y;
}

// 1/d for d > 0: rcp.approx seed and one third-order correction (relative
// error ~e^3, e <= 2^-20); subnormal-range d scaled as in sqrt_rsqrt
__device__ __forceinline__ double recip(double d) {
    const bool tiny = d < 0x1p-900;
    const double ds = tiny ? d * 0x1p600 : d;
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(ds));
    const double e = fma(-ds, r, 1.0);
    r = fma(r, fma(e, e, e), r);
    return tiny ? r * 0x1p600 : r;
}

// (a): warp 0, lanes 0..15 own rows; returns 0 or the 1-based failing column.
// The next pivot comes from the lane's own values: on lane j + 1,
// dn = a_{j+1,j+1} - a_{j+1,j}^2 / d (= l_{j+1,j}^2), so the step-to-step
// chain is one broadcast, a reciprocal and one fma (FP64 latency is what
// bounds this loop); the roots and the shuffled column updates run beside it.
__device__ __forceinline__ int factor16(double (*s)[kDP], double *rinv, int p0, int lane) {
    // lane = 16 h + i holds row i, columns c = 2 cl + h (cl < 8): both halves
    // of the warp carry distinct columns, so a step's column broadcast and
    // update is ~(16 - j) / 2 shuffles and fmas per lane instead of 15 - j
    const int i = lane & 15, h = lane >> 4;
    double v[8];
#pragma unroll
    for (int cl = 0; cl < 8; ++cl) v[cl] = s[p0 + i][p0 + 2 * cl + h];  // c > i: never read
    int fail = 0;  // no early exit: the loop stays unrolled (v in registers)
    double dn = v[0];  // pivot 0 on lane 0 (row 0, column 0)
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int hj = j & 1, jl = j >> 1;  // owner half / local index of column j
        const double raw = __shfl_sync(0xffffffffu, v[jl], hj * 16 + i);  // a_ij (unscaled)
        const double d = __shfl_sync(0xffffffffu, dn, hj * 16 + j);
        if (!(d > 0.0) && !fail) fail = j + 1;  // warp-uniform
        // next pivot on lane (j+1 & 1) 16 + j + 1: a_{j+1,j+1} - a_{j+1,j}^2 / d
        if (j + 1 < 16) dn = fma(-(raw * raw), recip(d), v[(j + 1) >> 1]);
        double l, r;
        sqrt_rsqrt(d, l, r);
        const double lij = raw * r;
        if (lane == hj * 16 + j) rinv[p0 + j] = r;
#pragma unroll
        for (int cl = 0; cl < 8; ++cl) {
            if (2 * cl + 1 > j) {  // some column 2 cl + h lies right of j
                const int c = 2 * cl + h;
                const double lc = __shfl_sync(0xffffffffu, v[jl], hj * 16 + c) * r;
                if (c > j && i >= c) v[cl] -= lij * lc;
            }
        }
        // column j itself, on its owner half (after the shuffles above read it)
        v[jl] = h != hj ? v[jl] : (i == j ? l : (i > j ? lij : v[jl]));
    }
    if (!fail) {
#pragma unroll
        for (int cl = 0; cl < 8; ++cl) s[p0 + i][p0 + 2 * cl + h] = v[cl];  // c > i: unchanged
    }
    return fail;
}

// (c): rows/columns [r0, 64) lower part, and with NEXT rows 64..127 (the tile
// below) over columns [r0, 64), -= A[:, p0:p0+16] A[:, p0:p0+16]^T;
// NB = (64 - r0) / 16 sub-blocks per side
template <int NB, bool NEXT>
__device__ __forceinline__ void trailing16(double (*s)[kDP], int p0, int r0, int t) {
    constexpr int NR = NB + (NEXT ? 4 : 0);
    const int rr = t >> 4, cc = t & 15;
    auto row = [&](int bi) { return bi < NB ? r0 + 16 * bi + rr : kT + 16 * (bi - NB) + rr; };
    double acc[NR][NB];
#pragma unroll
    for (int bi = 0; bi < NR; ++bi)
#pragma unroll
        for (int bj = 0; bj < NB; ++bj) acc[bi][bj] = 0.0;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
        double rv[NR], cv[NB];
#pragma unroll
        for (int bi = 0; bi < NR; ++bi) rv[bi] = s[row(bi)][p0 + c];
#pragma unroll
        for (int bj = 0; bj < NB; ++bj) cv[bj] = s[r0 + 16 * bj + cc][p0 + c];
#pragma unroll
        for (int bi = 0; bi < NR; ++bi)
#pragma unroll
            for (int bj = 0; bj < NB; ++bj)
                if (bi >= NB || bj <= bi) acc[bi][bj] += rv[bi] * cv[bj];
    }
#pragma unroll
    for (int bi = 0; bi < NR; ++bi)
#pragma unroll
        for (int bj = 0; bj < NB; ++bj)
            if (bi >= NB || bj <= bi) s[row(bi)][r0 + 16 * bj + cc] -= acc[bi][bj];
}

// Factor tile (k, k) of every block and store the inverse of its lower factor.
// The tile's factorisation is on the critical path of every panel step, so it
// is blocked in 16-column steps to keep the number of block-wide barriers
// small (~20 instead of 3 per column):
//   (a) warp 0 factors the 16 x 16 diagonal block in registers (lane i holds
//       row i; the column is broadcast with shuffles, no barriers);
//   (b) the rows below solve against it (one thread per row, forward
//       substitution in registers);
//   (c) the trailing lower part is updated (thread (rr, cc) of every 16 x 16
//       sub-block, the sub-blocks' row/column values loaded once per column);
// then the inverse X = L^-1: the four diagonal blocks by forward substitution
// (warp p, lane c = column c of X_pp), the off-diagonal blocks in three stages
// X_ip = -X_ii sum_{p <= m < i} L_im X_mp.  With solve_next the tile below,
// (k + 1, k), rides along as 64 more panel rows in (b) and (c), so L_{k+1,k}
// (which the next diagonal tile's update needs first) leaves with L_kk.
// (Unblocked 64-step forms with three barriers per column measured 50-60 us
// per tile under ncu; register-resident fully unrolled 64-column forms
// stalled on instruction fetch, 113-200 us.)
__global__ void __launch_bounds__(kDiagThreads) chol_diag(double *a, int64_t n, int k, int *info,
                                                          double *linv, int solve_next) {
    extern __shared__ double dsm[];
    double(*s)[kDP] = (double(*)[kDP])dsm;                    // tile + tile below -> L
    double(*x)[kDP] = (double(*)[kDP])(dsm + 2 * kT * kDP);   // X = L^-1
    double *tmp = dsm + 3 * kT * kDP;                         // stage products, 3 x 16 x 16
    double *rinv = tmp + 3 * 256;  // 1 / L[j][j] (LAPACK dpotf2 scales by the reciprocal too)
    __shared__ int bad;
#ifdef DIAG_CLOCKS
    __shared__ long long dclk[24];
#endif
    DCLK(0);
    // launched with programmatic stream serialisation: everything below reads
    // what the previous chain kernel wrote
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int b = blockIdx.y;
    if (info[b]) return;
    double *blk = a + (int64_t)b * n * n;
    const int64_t o = (int64_t)k * kT;
    const int m = (int)(n - o < kT ? n - o : kT);
    const int t = threadIdx.x, w = t >> 5, lane = t & 31;
    const int m2 = solve_next ? (int)(n - o - kT < kT ? n - o - kT : kT) : 0;  // rows of tile k+1
    const bool next = m2 > 0;
    // rows/columns past the block factor as the identity; X starts as 0.
    // Every load in flight before the first shared store.
    {
        constexpr int kPer = kT * kT / kDiagThreads;
        double v[kPer], vn[kPer];
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int e = t + q * kDiagThreads, rr = e >> 6, c = e & 63;
            v[q] = (rr < m && c < m) ? blk[(o + rr) * n + o + c] : (rr == c ? 1.0 : 0.0);
            vn[q] = rr < m2 ? blk[(o + kT + rr) * n + o + c] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int e = t + q * kDiagThreads, rr = e >> 6, c = e & 63;
            s[rr][c] = v[q];
            s[kT + rr][c] = vn[q];
            x[rr][c] = 0.0;
        }
    }
    if (t == 0) bad = 0;
    __syncthreads();
    DCLK(1);
    const int rend = next ? 2 * kT : kT;  // panel rows end
    for (int p = 0; p < 4; ++p) {
        const int p0 = 16 * p, r0 = p0 + 16;
        if (w == 0) {
            const int f = factor16(s, rinv, p0, lane);
            if (f && lane == 0) bad = p0 + f;
        }
        __syncthreads();
        DCLK(2 + 3 * p);
        if (bad) break;
        if (t < rend - r0) {  // (b) row r0 + t of the panel: Y L_pp^T = A
            const int r = r0 + t;
            double y[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) y[c] = s[r][p0 + c];
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                y[c] *= rinv[p0 + c];
#pragma unroll
                for (int q = 1; q < 16; ++q)
                    if (q > c) y[q] -= y[c] * s[p0 + q][p0 + c];
            }
#pragma unroll
            for (int c = 0; c < 16; ++c) s[r][p0 + c] = y[c];
        }
        __syncthreads();
        DCLK(3 + 3 * p);
        if (p == 3) break;
        if (next) {
            if (p == 0) trailing16<3, true>(s, p0, r0, t);
            else if (p == 1) trailing16<2, true>(s, p0, r0, t);
            else trailing16<1, true>(s, p0, r0, t);
        } else {
            if (p == 0) trailing16<3, false>(s, p0, r0, t);
            else if (p == 1) trailing16<2, false>(s, p0, r0, t);
            else trailing16<1, false>(s, p0, r0, t);
        }
        __syncthreads();
        DCLK(4 + 3 * p);
    }
    if (bad) {
        if (t == 0) info[b] = (int)(o + bad);  // LAPACK info: order of the failing minor
        return;
    }
    // L_kk and L_{k+1,k} are final: stored while the inverse is formed
    for (int e = t; e < kT * kT; e += kDiagThreads) {
        const int rr = e >> 6, c = e & 63;
        if (rr < m && c <= rr) blk[(o + rr) * n + o + c] = s[rr][c];
        if (rr < m2) blk[(o + kT + rr) * n + o + c] = s[kT + rr][c];
    }
    // X_pp = L_pp^-1: warp p, lane c computes column c (L X = I, right-looking)
    if (w < 4 && lane < 16) {
        const int p0 = 16 * w, c = lane;
        double xv[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) xv[i] = i == c ? 1.0 : 0.0;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            xv[i] *= rinv[p0 + i];
#pragma unroll
            for (int q = 1; q < 16; ++q)
                if (q > i) xv[q] -= s[p0 + q][p0 + i] * xv[i];
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) x[p0 + i][p0 + c] = xv[i];
    }
    __syncthreads();
    DCLK(14);
    // X_ip = -X_ii sum_{p <= q < i} L_iq X_qp, by distance d = i - p: the
    // 16 x 16 block products on the DMMA pipe, one 8 x 8 output tile per warp
    // (the scalar form was shared-load bound, ~9k cycles for the three stages)
    {
        const int fr = lane >> 2, fk = lane & 3;
        for (int d = 1; d < 4; ++d) {
            const int ntile = (4 - d) * 4;
            for (int tl = w; tl < ntile; tl += kDiagThreads / 32) {
                const int p = tl >> 2, i = p + d, tr = ((tl >> 1) & 1) * 8, tc = (tl & 1) * 8;
                double c0 = 0.0, c1 = 0.0;
                for (int q0 = 16 * p; q0 < 16 * i; q0 += 4)
                    dmma(c0, c1, s[16 * i + tr + fr][q0 + fk], x[q0 + fk][16 * p + tc + fr]);
                double *tp = tmp + p * 256 + (tr + fr) * 16 + tc + 2 * fk;
                tp[0] = c0;
                tp[1] = c1;
            }
            __syncthreads();
            for (int tl = w; tl < ntile; tl += kDiagThreads / 32) {
                const int p = tl >> 2, i = p + d, tr = ((tl >> 1) & 1) * 8, tc = (tl & 1) * 8;
                double c0 = 0.0, c1 = 0.0;
#pragma unroll
                for (int q0 = 0; q0 < 16; q0 += 4)
                    dmma(c0, c1, x[16 * i + tr + fr][16 * i + q0 + fk],
                         tmp[p * 256 + (q0 + fk) * 16 + tc + fr]);
                x[16 * i + tr + fr][16 * p + tc + 2 * fk] = -c0;
                x[16 * i + tr + fr][16 * p + tc + 2 * fk + 1] = -c1;
            }
            __syncthreads();
        }
    }
    DCLK(15);
    double *li = linv + (int64_t)b * kT * kT;
    for (int e = t; e < kT * kT; e += kDiagThreads) li[e] = x[e >> 6][e & 63];
    DCLK(16);
#ifdef DIAG_CLOCKS
    if (t == 0 && b == 0 && k == 5) {
        printf("diag k=5 cycles:");
        for (int q = 1; q < 17; ++q) printf(" %lld", dclk[q] - dclk[q - 1]);
        printf("\n");
    }
#endif
}

// Panel step k for the tiles below the diagonal.  CTA I (I >= k + 2) solves
// L_Ik = A_Ik L_kk^-T (a 64 x 64 x 64 DMMA product with the inverse, the
// TRSM-by-inverse of GPU LAPACKs) and stores it; with UPD (the next column
// lies in the same super-panel) it then applies that column's update
// A_{I,k+1} -= L_Ik L_{k+1,k}^T from the tile still in shared memory, and
// CTA I = k + 1 applies the diagonal tile's A_{k+1,k+1} -= L_{k+1,k}
// L_{k+1,k}^T (chol_diag already solved L_{k+1,k}).  One launch per step
// instead of a solve and an update.
constexpr int kPanelSmem = 3 * kT * kPitch * (int)sizeof(double);

template <bool UPD>
__global__ void __launch_bounds__(kGemmThreads) chol_panel(double *a, int64_t n, int k,
                                                           const int *info, const double *linv) {
    extern __shared__ double sm[];
    double *sa = sm, *sx = sm + kT * kPitch, *sb = sm + 2 * kT * kPitch;
#ifdef DIAG_CLOCKS
    __shared__ long long dclk[8];
#endif
    DCLK(0);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // see chol_diag
    const int b = blockIdx.y;
    if (info[b]) return;
    double *blk = a + (int64_t)b * n * n;
    const int64_t I = (int64_t)k + (UPD ? 1 : 2) + blockIdx.x;
    const bool own = UPD && I == k + 1;  // uniform per CTA
    const int64_t r0 = I * kT, c0 = (int64_t)k * kT, c1 = c0 + kT;
    const int rows = (int)(n - r0 < kT ? n - r0 : kT);
    const int rows1 = UPD ? (int)(n - c1 < kT ? n - c1 : kT) : 0;  // tile k + 1
    const double *li = linv + (int64_t)b * kT * kT;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wr = (warp >> 1) * 32, wc = (warp & 1) * 32;
    {
        // every load in flight before the first shared store
        constexpr int kPer = kT * kT / kGemmThreads;
        double va[kPer], vx[kPer], vb[kPer];
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int e = threadIdx.x + q * kGemmThreads, rr = e >> 6, c = e & 63;
            if (!own) {
                va[q] = rr < rows ? blk[(r0 + rr) * n + c0 + c] : 0.0;
                vx[q] = li[e];
            }
            if (UPD) vb[q] = rr < rows1 ? blk[(c1 + rr) * n + c0 + c] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int e = threadIdx.x + q * kGemmThreads, rr = e >> 6, c = e & 63;
            if (!own) {
                sa[rr * kPitch + c] = va[q];
                sx[rr * kPitch + c] = vx[q];
            }
            if (UPD) sb[rr * kPitch + c] = vb[q];
        }
    }
    __syncthreads();
    DCLK(1);
    double acc[4][4][2];
    if (!own) {
        tile_product(sa, sx, acc);  // A_Ik Linv^T: B[q][c] = Linv[c][q]
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int rr = wr + 8 * i + (lane >> 2);
            if (rr >= rows) continue;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                double *p = blk + (r0 + rr) * n + c0 + wc + 8 * j + 2 * (lane & 3);
                p[0] = acc[i][j][0];
                p[1] = acc[i][j][1];
            }
        }
    }
    DCLK(2);
    if (!UPD) return;
    double *sl = sb;
    if (!own) {
        __syncthreads();  // every warp is done reading sa
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                double *q = sa + (wr + 8 * i + (lane >> 2)) * kPitch + wc + 8 * j + 2 * (lane & 3);
                q[0] = acc[i][j][0];
                q[1] = acc[i][j][1];
            }
        sl = sa;
        __syncthreads();
    }
    DCLK(3);
    tile_product(sl, sb, acc);  // L_Ik L_{k+1,k}^T
    DCLK(4);
    // C -= acc: every load first, then the stores
    double cv[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int rr = wr + 8 * i + (lane >> 2);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int cc = wc + 8 * j + 2 * (lane & 3);
            const double *p = blk + (r0 + rr) * n + c1 + cc;
            cv[i][j][0] = (rr < rows && cc < rows1) ? p[0] : 0.0;
            cv[i][j][1] = (rr < rows && cc + 1 < rows1) ? p[1] : 0.0;
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int rr = wr + 8 * i + (lane >> 2);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int cc = wc + 8 * j + 2 * (lane & 3);
            double *p = blk + (r0 + rr) * n + c1 + cc;
            if (rr < rows && cc < rows1) p[0] = cv[i][j][0] - acc[i][j][0];
            if (rr < rows && cc + 1 < rows1) p[1] = cv[i][j][1] - acc[i][j][1];
        }
    }
#ifdef DIAG_CLOCKS
    DCLK(5);
    if (threadIdx.x == 0 && b == 0 && k == 5 && blockIdx.x == 1) {
        printf("panel k=5 I=7 cycles:");
        for (int q = 1; q < 6; ++q) printf(" %lld", dclk[q] - dclk[q - 1]);
        printf("\n");
    }
#endif
}

// Update of the tiles (I, J), J in [j_lo, j_hi), I in [J, nt):
//   A_IJ -= sum_{k in [k_lo, k_hi)} A_Ik A_Jk^T
// (the panel-local updates inside a super-panel, K = one tile, and the delayed
// trailing update after it, K = the super-panel).  K is streamed in slices of
// 32 columns through a two-stage cp.async pipeline (16-byte copies; rows past
// the block are zero-filled by the copy); VEC == false (odd n, unaligned rows)
// loads synchronously.
constexpr int kSlice = 32;
constexpr int kSPitch = kSlice + 4;  // conflict-free fragment loads
// cp.async pipeline depth: 2 (74 KB per CTA); 3 (110 KB) for the bulk update
// via SFB_CHOL_STAGES (measured slower: two CTAs per SM instead of three)
constexpr int upd_smem(int stages) { return stages * 2 * kT * kSPitch * (int)sizeof(double); }

__device__ __forceinline__ void cp_async16(void *dst, const void *src, int src_bytes) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(src_bytes)
                 : "memory");
}

template <bool VEC>
__device__ __forceinline__ void load_slice(double *sa, const double *blk, int64_t n, int64_t r0,
                                           int rows, int64_t c0) {
    if (VEC) {
        // thread t copies columns cc, cc + 1 of rows t/16 + 8q (q < 8): one
        // base pointer, the row step is a constant
        const int rr0 = threadIdx.x >> 4, cc = (threadIdx.x & 15) * 2;
        const double *src = blk + (r0 + rr0) * n + c0 + cc;
        double *dst = sa + rr0 * kSPitch + cc;
#pragma unroll
        for (int q = 0; q < kT * kSlice / 2 / kGemmThreads; ++q) {
            const bool in = rr0 + 8 * q < rows;
            cp_async16(dst + 8 * q * kSPitch, in ? src + 8 * q * n : src, in ? 16 : 0);
        }
    } else {
        for (int e = threadIdx.x; e < kT * kSlice; e += blockDim.x) {
            const int rr = e >> 5, cc = e & 31;
            sa[rr * kSPitch + cc] = rr < rows ? blk[(r0 + rr) * n + c0 + cc] : 0.0;
        }
    }
}

// CTAs stride over the linear index of the (batch, J, I >= J) tiles -- the
// lower trapezoid, column by column, so neighbouring CTAs share A_Jk -- and a
// launch can be held to a fixed number of CTAs per SM (SFB_CHOL_BULK_CTAS;
// the default launches one CTA per tile).
__device__ __forceinline__ int64_t trap_start(int64_t jj, int64_t R) {
    return jj * R - jj * (jj - 1) / 2;  // tiles in columns before jj (R - c in column c)
}

template <bool VEC, int kStages>
__global__ void __launch_bounds__(kGemmThreads) chol_update(double *a, int64_t n, int nt, int k_lo,
                                                            int k_hi, int j_lo, int j_hi,
                                                            int batch, const int *info) {
    extern __shared__ double sm[];
    const int64_t R = nt - j_lo, Wc = j_hi - j_lo, per = trap_start(Wc, R);
    for (int64_t x = blockIdx.x; x < per * batch; x += gridDim.x) {
        const int b = (int)(x / per);
        const int64_t y = x - b * per;
        const double q = (double)(2 * R + 1);
        int64_t jj = (int64_t)((q - sqrt(q * q - 8.0 * (double)y)) * 0.5);
        jj = jj < 0 ? 0 : (jj >= Wc ? Wc - 1 : jj);
        while (jj + 1 < Wc && trap_start(jj + 1, R) <= y) ++jj;
        while (jj > 0 && trap_start(jj, R) > y) --jj;
        const int64_t J = j_lo + jj, I = J + (y - trap_start(jj, R));
        if (info[b]) continue;  // uniform per CTA
        double *blk = a + (int64_t)b * n * n;
        const int64_t ri = I * kT, rj = J * kT;
        const int rows = (int)(n - ri < kT ? n - ri : kT);
        const int cols = (int)(n - rj < kT ? n - rj : kT);
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const int wr = (warp >> 1) * 32, wc = (warp & 1) * 32;
        const int fr = lane >> 2, fk = lane & 3;
        double acc[4][4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        const int nsl = (k_hi - k_lo) * (kT / kSlice);
        const int64_t kc0 = (int64_t)k_lo * kT;
        auto stage = [&](int st) { return sm + st * 2 * kT * kSPitch; };
        // prologue: slices 0 .. kStages-2 in flight; one commit group per slice
        // (empty groups past the end keep the wait_group arithmetic uniform)
#pragma unroll
        for (int q = 0; q < kStages - 1; ++q) {
            if (q < nsl) {
                load_slice<VEC>(stage(q), blk, n, ri, rows, kc0 + (int64_t)q * kSlice);
                load_slice<VEC>(stage(q) + kT * kSPitch, blk, n, rj, cols, kc0 + (int64_t)q * kSlice);
            }
            if (VEC) asm volatile("cp.async.commit_group;" ::: "memory");
        }
        for (int sl = 0; sl < nsl; ++sl) {
            const int nx = sl + kStages - 1;  // refill the stage consumed at sl - 1
            if (nx < nsl) {
                double *sg = stage(nx % kStages);
                load_slice<VEC>(sg, blk, n, ri, rows, kc0 + (int64_t)nx * kSlice);
                load_slice<VEC>(sg + kT * kSPitch, blk, n, rj, cols, kc0 + (int64_t)nx * kSlice);
            }
            if (VEC) {
                asm volatile("cp.async.commit_group;" ::: "memory");
                asm volatile("cp.async.wait_group %0;" ::"n"(kStages - 1) : "memory");
            }
            __syncthreads();
            const double *sa = stage(sl % kStages), *sb = sa + kT * kSPitch;
#pragma unroll
            for (int k0 = 0; k0 < kSlice; k0 += 4) {
                double fa[4], fb[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) fa[i] = sa[(wr + 8 * i + fr) * kSPitch + k0 + fk];
#pragma unroll
                for (int j = 0; j < 4; ++j) fb[j] = sb[(wc + 8 * j + fr) * kSPitch + k0 + fk];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
            }
            __syncthreads();  // the stage is refilled at the next iteration
        }
        // C -= acc: every load first (32 in flight), then the stores (a
        // read-modify-write per element serialises on possible aliasing:
        // measured 86 % of the stall samples)
        double cv[4][4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int rr = wr + 8 * i + fr;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int cc = wc + 8 * j + 2 * fk;
                const double *p = blk + (ri + rr) * n + rj + cc;
                cv[i][j][0] = (rr < rows && cc < cols) ? p[0] : 0.0;
                cv[i][j][1] = (rr < rows && cc + 1 < cols) ? p[1] : 0.0;
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int rr = wr + 8 * i + fr;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int cc = wc + 8 * j + 2 * fk;
                double *p = blk + (ri + rr) * n + rj + cc;
                if (rr < rows && cc < cols) p[0] = cv[i][j][0] - acc[i][j][0];
                if (rr < rows && cc + 1 < cols) p[1] = cv[i][j][1] - acc[i][j][1];
            }
        }
        __syncthreads();  // the next tile's prologue refills the stages
    }
}

// L = C / diag(C) below the diagonal, 1 on it, 0 above; D = diag(C)^2
// (grf.py:203-207), in place on the factored blocks.
__global__ void chol_finish(double *c, double *diag, int64_t n, const int *info) {
    const int b = blockIdx.y;
    if (info[b]) return;
    double *blk = c + (int64_t)b * n * n;
    const int64_t total = n * n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / n, j = e - i * n;
        if (j < i) {
            blk[e] = blk[e] / blk[j * n + j];  // reads the untouched diagonal C_jj
        } else if (j > i) {
            blk[e] = 0.0;
        }
    }
}

__global__ void chol_diag_out(double *c, double *diag, int64_t n, const int *info) {
    const int b = blockIdx.y;
    if (info[b]) return;
    double *blk = c + (int64_t)b * n * n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double d = blk[i * n + i];
        diag[(int64_t)b * n + i] = d * d;
        blk[i * n + i] = 1.0;
    }
}

// w[b][j][c] = s(D[b][j]) Z[bz][j][c], s = sqrt (transform 0) or identity
__global__ void scale_rows(const double *diag, const double *z, int z_shared, int64_t n,
                           int64_t r, int transform, double *w) {
    const int b = blockIdx.y;
    const double *zb = z + (z_shared ? 0 : (int64_t)b * n * r);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * r;
         e += (int64_t)gridDim.x * blockDim.x) {
        const double d = diag[(int64_t)b * n + e / r];
        w[(int64_t)b * n * r + e] = (transform == 0 ? sqrt(d) : d) * zb[e];
    }
}

// out[b][i][c] = sum_{j <= i} L[b][i][j] w[b][j][c]: one warp per row i,
// RC columns of w per pass
template <int RC>
__global__ void __launch_bounds__(256) lower_mul(const double *lmat, const double *w, int64_t n,
                                                 int64_t r, int64_t c0, double *out) {
    const int b = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= n) return;
    const double *li = lmat + (int64_t)b * n * n + i * n;
    const double *wb = w + (int64_t)b * n * r + c0;
    const int rc = (int)(r - c0 < RC ? r - c0 : RC);
    double acc[RC];
#pragma unroll
    for (int c = 0; c < RC; ++c) acc[c] = 0.0;
    // four row elements per lane in flight (independent loads), then the FMAs
    int64_t j = lane;
    for (; j + 96 <= i; j += 128) {
        double l[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) l[u] = __ldg(li + j + 32 * u);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double *wj = wb + (j + 32 * u) * r;
#pragma unroll
            for (int c = 0; c < RC; ++c)
                if (c < rc) acc[c] += l[u] * __ldg(wj + c);
        }
    }
    for (; j <= i; j += 32) {
        const double l = __ldg(li + j);
        const double *wj = wb + j * r;
#pragma unroll
        for (int c = 0; c < RC; ++c)
            if (c < rc) acc[c] += l * __ldg(wj + c);
    }
#pragma unroll
    for (int c = 0; c < RC; ++c)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
    if (lane == 0) {
        double *ob = out + (int64_t)b * n * r + i * r + c0;
#pragma unroll
        for (int c = 0; c < RC; ++c)
            if (c < rc) ob[c] = acc[c];
    }
}

// Grow-only per-device scratch (a cudaMallocAsync / cudaFreeAsync pair per
// call measured 0.4 -> 3.3 ms of variance: the pool hands memory back and
// re-maps it).  A reuse on another stream waits for the last use's event.
struct Scratch {
    std::mutex mu;
    void *p = nullptr;
    size_t cap = 0;
    cudaEvent_t last = nullptr;
    bool used = false;
};

static Scratch &scratch(int dev, int which) {
    static Scratch sc[64][2];
    return sc[dev & 63][which & 1];
}

// call with sc.mu held; the returned buffer is valid for work enqueued on st
// until release()
static cudaError_t acquire(Scratch &sc, size_t bytes, cudaStream_t st, void **out) {
    cudaError_t e = cudaSuccess;
    if (!sc.last) e = cudaEventCreateWithFlags(&sc.last, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
    if (bytes > sc.cap) {
        if (sc.used) e = cudaEventSynchronize(sc.last);  // the old buffer's last reader
        if (e == cudaSuccess && sc.p) e = cudaFree(sc.p);
        sc.p = nullptr;
        sc.cap = 0;
        if (e == cudaSuccess) e = cudaMalloc(&sc.p, bytes);
        if (e != cudaSuccess) return e;
        sc.cap = bytes;
        sc.used = false;
    }
    if (sc.used) e = cudaStreamWaitEvent(st, sc.last, 0);
    *out = sc.p;
    return e;
}

static void release(Scratch &sc, cudaStream_t st) {
    cudaEventRecord(sc.last, st);
    sc.used = true;
}

// chain kernels are launched with programmatic stream serialisation (PDL):
// the next one is scheduled while the previous one's CTAs drain and waits in
// griddepcontrol.wait, hiding the launch gap of the serial chain
template <typename... KArgs, typename... Args>
static cudaError_t launch_chain(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                cudaStream_t st, bool pdl, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

struct LookAhead {
    std::mutex mu;
    cudaStream_t sb = nullptr, sh = nullptr;  // bulk update (low priority), chain (high)
    cudaStream_t sr = nullptr;                // super-panel-local updates beside the chain
    cudaStream_t sc = nullptr;                // the next super-panel's later columns
    cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_s = nullptr, ev_h = nullptr, ev_r = nullptr;
    cudaEvent_t ev_x = nullptr, ev_be = nullptr;
    std::vector<cudaEvent_t> ev_col;  // per column of the next super-panel (sc)
};

static LookAhead &look_ahead(int dev) {
    static LookAhead la[64];
    return la[dev & 63];
}

}  // namespace sfb

using namespace sfb;

extern "C" {

int sfb_chol_batch(const double *d_a, int64_t n, int64_t batch, double *d_lmat, double *d_diag,
                   int32_t *d_info, void *stream) {
    if (n < 1 || batch < 1) return fail(SFB_E_INVALID_ARGUMENT, "need n >= 1 and batch >= 1");
    if (batch > 65535) return fail(SFB_E_INVALID_ARGUMENT, "at most 65535 blocks per call");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t bytes = (size_t)batch * n * n * sizeof(double);
    cudaError_t e = cudaMemsetAsync(d_info, 0, sizeof(int32_t) * batch, st);
    if (e == cudaSuccess && d_lmat != d_a)
        e = cudaMemcpyAsync(d_lmat, d_a, bytes, cudaMemcpyDeviceToDevice, st);
    int dev = 0;
    cudaGetDevice(&dev);
    Scratch &sc = scratch(dev, 0);
    std::lock_guard<std::mutex> slock(sc.mu);
    double *linv = nullptr;
    if (e == cudaSuccess) e = acquire(sc, sizeof(double) * kT * kT * batch, st, (void **)&linv);
    if (e != cudaSuccess) return fail(SFB_E_CUDA, "chol_batch setup: %s", cudaGetErrorString(e));
    // dynamic shared-memory limits, raised once per device
    static std::atomic<uint64_t> done{0};
    if (!(done.load() & (1ull << (dev & 63)))) {
        e = cudaFuncSetAttribute(chol_panel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kPanelSmem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(chol_panel<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kPanelSmem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(chol_update<true, 2>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, upd_smem(2));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(chol_update<false, 2>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, upd_smem(2));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(chol_update<true, 3>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, upd_smem(3));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(chol_update<false, 3>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, upd_smem(3));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(chol_diag, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kDiagSmem);
        if (e != cudaSuccess) return fail(SFB_E_CUDA, "chol_batch attributes: %s", cudaGetErrorString(e));
        done.fetch_or(1ull << (dev & 63));
    }
    int *info = (int *)d_info;
    const int nt = (int)((n + kT - 1) / kT);
    // right-looking over super-panels of W tiles: inside a super-panel each
    // 64-column step factors its diagonal tile, solves its whole column below
    // and updates only the super-panel's later columns; the rest of the
    // trailing matrix gets one delayed update with K = the super-panel
    const int W = std::max(1, tune_knob("SFB_CHOL_PANEL", 8));
    const bool vec = (n % 2) == 0;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int bulk_per_sm = tune_knob("SFB_CHOL_BULK_CTAS", 0);  // 0: one CTA per tile
    // cap: CTAs per launch (the bulk update: bulk_per_sm per SM)
    const int bulk_stages = tune_knob("SFB_CHOL_STAGES", 2) == 3 ? 3 : 2;
    auto update = [&](cudaStream_t us, int k_lo, int k_hi, int j_lo, int j_hi, int cap) {
        const int64_t R = nt - j_lo, Wc = j_hi - j_lo;
        const int64_t tiles = (Wc * R - Wc * (Wc - 1) / 2) * batch;  // I >= J only
        const unsigned grid = (unsigned)std::min<int64_t>(tiles, cap);
        const bool deep = cap < (1 << 30) && bulk_stages == 3;
        if (vec && deep)
            chol_update<true, 3><<<grid, kGemmThreads, upd_smem(3), us>>>(
                d_lmat, n, nt, k_lo, k_hi, j_lo, j_hi, (int)batch, info);
        else if (vec)
            chol_update<true, 2><<<grid, kGemmThreads, upd_smem(2), us>>>(
                d_lmat, n, nt, k_lo, k_hi, j_lo, j_hi, (int)batch, info);
        else if (deep)
            chol_update<false, 3><<<grid, kGemmThreads, upd_smem(3), us>>>(
                d_lmat, n, nt, k_lo, k_hi, j_lo, j_hi, (int)batch, info);
        else
            chol_update<false, 2><<<grid, kGemmThreads, upd_smem(2), us>>>(
                d_lmat, n, nt, k_lo, k_hi, j_lo, j_hi, (int)batch, info);
    };
    const int cap_all = 1 << 30, cap_bulk = bulk_per_sm > 0 ? nsm * bulk_per_sm : cap_all;
    const bool split = tune_knob("SFB_CHOL_SPLIT", 1) != 0;
    // Look-ahead: after super-panel i is factored, its update of the next
    // super-panel's columns (a_i) runs on the caller's stream, the bulk update
    // of everything beyond (b_i) on a second stream, where it overlaps the
    // factorisation of super-panel i + 1 (the serial diag/trsm chain).  a_i
    // touches the tiles b_{i-1} updated, so it waits for b_{i-1}; b_i waits for
    // super-panel i's factors.  Per device: the second stream and two events,
    // used under a lock (the enqueue sequence of one call is atomic).
    // The serial chain runs on a high-priority stream (the block scheduler
    // then dispatches its small grids ahead of the bulk update's pending CTAs).
    LookAhead &la = look_ahead(dev);
    std::lock_guard<std::mutex> lock(la.mu);
    if (!la.sb) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        e = cudaStreamCreateWithPriority(&la.sb, cudaStreamNonBlocking, lo);
        if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&la.sh, cudaStreamNonBlocking, hi);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&la.ev_a, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&la.ev_b, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&la.ev_s, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&la.sr, cudaStreamNonBlocking, hi);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&la.ev_h, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&la.ev_r, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&la.sc, cudaStreamNonBlocking, hi);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&la.ev_x, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&la.ev_be, cudaEventDisableTiming);
        if (e != cudaSuccess) return fail(SFB_E_CUDA, "chol_batch streams: %s", cudaGetErrorString(e));
    }
    while (e == cudaSuccess && (int)la.ev_col.size() < W) {
        cudaEvent_t ev = nullptr;
        e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e == cudaSuccess) la.ev_col.push_back(ev);
    }
    if (e != cudaSuccess) return fail(SFB_E_CUDA, "chol_batch events: %s", cudaGetErrorString(e));
    // Super-panel columns after the first get their update by the previous
    // super-panel (its "a" part) one column per launch on stream sc, and the
    // chain waits for each column just before it touches it: only the first
    // column's part sits on the serial path (a schedule without the bulk
    // update measured 6.5 of 9.1 ms, i.e. the chain and the whole "a" update
    // were the critical path).
    const bool split_a = split && tune_knob("SFB_CHOL_SPLIT_A", 1) != 0;
    bool col_pending = false;  // this super-panel's columns > p0 have sc events
    // The bulk update of super-panel i is split: the columns of super-panel
    // i + 2 first (what the next "a" update waits for), then the rest, which
    // keeps running beside super-panel i + 1's chain.
    const bool split_b = tune_knob("SFB_CHOL_SPLIT_B", 1) != 0;
    const bool pdl = tune_knob("SFB_CHOL_PDL", 1) != 0;
    const cudaStream_t caller = st;
    cudaEventRecord(la.ev_s, caller);  // the copy into d_lmat, the info reset, linv
    cudaStreamWaitEvent(la.sh, la.ev_s, 0);
    st = la.sh;
    bool pending_b = false;
    for (int p0 = 0; p0 < nt && e == cudaSuccess; p0 += W) {
        const int p1 = std::min(p0 + W, nt), p2 = std::min(p1 + W, nt);
        // inside a super-panel the chain only waits for the update of the
        // next column tile; the update of the super-panel's later columns runs
        // on a third stream and is waited for one step later (the next
        // column's own update touches the tiles it updated)
        bool pending_r = false;
        for (int k = p0; k < p1; ++k) {
            launch_chain(chol_diag, dim3(1, (unsigned)batch), dim3(kDiagThreads), kDiagSmem, st,
                         pdl, d_lmat, n, k, info, linv, (int)(k + 1 < nt));
            if (k + 1 >= nt) continue;
            if (k + 1 < p1) {
                // the next column's update also writes tiles the previous
                // step's panel-local update (and the previous super-panel's
                // column update on sc) wrote
                if (pending_r) cudaStreamWaitEvent(st, la.ev_r, 0);
                if (col_pending) cudaStreamWaitEvent(st, la.ev_col[k + 1 - p0], 0);
                launch_chain(chol_panel<true>, dim3((unsigned)(nt - k - 1), (unsigned)batch),
                             dim3(kGemmThreads), kPanelSmem, st, pdl, d_lmat, n, k,
                             (const int *)info, (const double *)linv);
                pending_r = false;
                if (k + 2 < p1) {
                    // column k + 2 gets the contributions of columns p0 .. k
                    // in one update (K = k + 1 - p0 tiles) beside the next
                    // diagonal tile; column k + 1's own comes with the next
                    // panel launch.  (Updating all later columns of the
                    // super-panel by column k alone, K = one tile per
                    // launch, ran the small updates at ~35 % DMMA.)
                    const int lazy = tune_knob("SFB_CHOL_LAZY", 1);
                    if (split) {
                        cudaEventRecord(la.ev_h, st);  // panel k solved
                        cudaStreamWaitEvent(la.sr, la.ev_h, 0);
                        if (col_pending) cudaStreamWaitEvent(la.sr, la.ev_col[k + 2 - p0], 0);
                        if (lazy)
                            update(la.sr, p0, k + 1, k + 2, k + 3, cap_all);
                        else
                            update(la.sr, k, k + 1, k + 2, p1, cap_all);
                        cudaEventRecord(la.ev_r, la.sr);
                        pending_r = true;
                    } else if (lazy) {
                        if (col_pending) cudaStreamWaitEvent(st, la.ev_col[k + 2 - p0], 0);
                        update(st, p0, k + 1, k + 2, k + 3, cap_all);
                    } else {
                        update(st, k, k + 1, k + 2, p1, cap_all);
                    }
                }
            } else if (k + 2 < nt) {
                launch_chain(chol_panel<false>, dim3((unsigned)(nt - k - 2), (unsigned)batch),
                             dim3(kGemmThreads), kPanelSmem, st, pdl, d_lmat, n, k,
                             (const int *)info, (const double *)linv);
            }
        }
        if (pending_r) cudaStreamWaitEvent(st, la.ev_r, 0);
        if (p1 < nt) {
            cudaEventRecord(la.ev_a, st);  // super-panel p0 factored
            if (pending_b) cudaStreamWaitEvent(st, la.ev_b, 0);  // b of the previous super-panel
            if (split_a && p2 - p1 > 1) {
                // a: the next super-panel's first column on the chain, the
                // others one launch each on sc
                cudaEventRecord(la.ev_x, st);
                cudaStreamWaitEvent(la.sc, la.ev_x, 0);
                update(st, p0, p1, p1, p1 + 1, cap_all);
                for (int c = p1 + 1; c < p2; ++c) {
                    update(la.sc, p0, p1, c, c + 1, cap_all);
                    cudaEventRecord(la.ev_col[c - p1], la.sc);
                }
                col_pending = true;
            } else {
                update(st, p0, p1, p1, p2, cap_all);  // a: the next super-panel's columns
                col_pending = false;
            }
            if (p2 < nt) {
                cudaStreamWaitEvent(la.sb, la.ev_a, 0);
#ifdef DIAG_CLOCKS  // experiment builds: time the schedule without the bulk update
                if (!getenv("SFB_CHOL_NO_BULK"))
#endif
                {
                    const int p3 = std::min(p2 + W, nt);
                    if (split_b && p3 < nt) {
                        update(la.sb, p0, p1, p2, p3, cap_bulk);  // b, near columns
                        cudaEventRecord(la.ev_b, la.sb);
                        update(la.sb, p0, p1, p3, nt, cap_bulk);  // b, the rest
                    } else {
                        update(la.sb, p0, p1, p2, nt, cap_bulk);  // b: the rest
                        cudaEventRecord(la.ev_b, la.sb);
                    }
                }
                cudaEventRecord(la.ev_be, la.sb);
                pending_b = true;
            } else {
                pending_b = false;
            }
        }
        e = cudaGetLastError();
    }
    if (pending_b) cudaStreamWaitEvent(st, la.ev_be, 0);  // every bulk update
    cudaEventRecord(la.ev_s, st);
    cudaStreamWaitEvent(caller, la.ev_s, 0);
    st = caller;
    if (e == cudaSuccess) {
        const unsigned g = (unsigned)std::min<int64_t>(1184, (n * n + 255) / 256);
        chol_finish<<<dim3(g, (unsigned)batch), 256, 0, st>>>(d_lmat, d_diag, n, info);
        chol_diag_out<<<dim3((unsigned)((n + 255) / 256), (unsigned)batch), 256, 0, st>>>(
            d_lmat, d_diag, n, info);
        e = cudaGetLastError();
    }
    release(sc, st);
    if (e != cudaSuccess) return fail(SFB_E_CUDA, "chol_batch: %s", cudaGetErrorString(e));
    return SFB_OK;
}

int sfb_lower_diag_multiply(const double *d_lmat, const double *d_diag, int64_t n, int64_t batch,
                            const double *d_z, int z_shared, int64_t r, int transform,
                            double *d_out, void *stream) {
    if (n < 1 || batch < 1 || r < 1) return fail(SFB_E_INVALID_ARGUMENT, "empty operands");
    if (transform != 0 && transform != 1)
        return fail(SFB_E_INVALID_ARGUMENT, "transform must be 'sqrt' or 'identity'");
    if (batch > 65535) return fail(SFB_E_INVALID_ARGUMENT, "at most 65535 blocks per call");
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0;
    cudaGetDevice(&dev);
    Scratch &sc = scratch(dev, 1);
    std::lock_guard<std::mutex> slock(sc.mu);
    double *w = nullptr;
    cudaError_t e = acquire(sc, sizeof(double) * batch * n * r, st, (void **)&w);
    if (e != cudaSuccess) return fail(SFB_E_CUDA, "lower_diag_multiply: %s", cudaGetErrorString(e));
    const unsigned g = (unsigned)std::min<int64_t>(1184, (n * r + 255) / 256);
    scale_rows<<<dim3(g, (unsigned)batch), 256, 0, st>>>(d_diag, d_z, z_shared, n, r, transform, w);
    const unsigned rows_per_cta = 8;
    for (int64_t c0 = 0; c0 < r; c0 += 8) {
        const dim3 grid((unsigned)((n + rows_per_cta - 1) / rows_per_cta), (unsigned)batch);
        if (r - c0 <= 2)
            lower_mul<2><<<grid, 256, 0, st>>>(d_lmat, w, n, r, c0, d_out);
        else
            lower_mul<8><<<grid, 256, 0, st>>>(d_lmat, w, n, r, c0, d_out);
    }
    e = cudaGetLastError();
    release(sc, st);
    if (e != cudaSuccess) return fail(SFB_E_CUDA, "lower_diag_multiply: %s", cudaGetErrorString(e));
    return SFB_OK;
}

}  // extern "C"
