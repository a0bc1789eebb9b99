/*
 * sfb.h -- C ABI of the B200-native streamforge hot path (libsfb.so).
 *
 * This is the drop-in seam that replaces the reference's Python->numba
 * boundary, the `_kernels` module (/root/reference/pkg/src/streamforge/
 * _kernels.py), plus the exact-integer stream arithmetic of core.py.  Every
 * entry point names the reference interface it replaces (file:line, paths
 * relative to /root/reference/pkg/src/streamforge/).
 *
 * Conventions
 *   - plain pointers and sizes only; no torch / C++ types cross the ABI;
 *   - every function returns 0 (SFB_OK) or a negative SFB_E_* code, with a
 *     thread-local message in sfb_last_error(); codes map 1:1 onto the
 *     reference exception classes (errors.py:8-32) or CUDA failures;
 *   - no C++ exception ever crosses the ABI;
 *   - "device" functions take device pointers and a cudaStream_t passed as
 *     void*; they are stream-ordered and return after enqueueing (the Python
 *     layer synchronises where the reference is synchronous);
 *   - stream states use the reference layout: int64 (n, 6) C-contiguous,
 *     row w = (g1[0..2], g2[0..2]) newest-first (core.py:161-172), mutated in
 *     place exactly where the reference kernels mutate `cur`;
 *   - results never depend on thread-block scheduling: a launch that splits a
 *     stream's draws over several threads writes no state in its sampling
 *     kernel; a second kernel on the same stream advances each stream by the
 *     draws it consumed.
 */
#ifndef SFB_H_
#define SFB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFB_OK 0
#define SFB_E_INVALID_ARGUMENT (-1)      /* errors.py:12 InvalidArgumentError */
#define SFB_E_INSUFFICIENT_STREAMS (-2)  /* errors.py:20 InsufficientStreamsError */
#define SFB_E_INVALID_GRID (-3)          /* errors.py:24 InvalidGridError */
#define SFB_E_INVALID_RATE (-4)          /* errors.py:28 InvalidRateError */
#define SFB_E_INVALID_MARGINS (-5)       /* errors.py:32 InvalidMarginsError */
#define SFB_E_INVALID_SEED (-6)          /* errors.py:8 InvalidSeedError */
#define SFB_E_CORRUPT_STREAM_FILE (-7)   /* errors.py:16 CorruptStreamFileError */
#define SFB_E_IO (-8)                    /* OSError from open()/write() */
#define SFB_E_INVALID_PARAMS (-9)        /* errors.py:36 InvalidParamsError (GRF) */
#define SFB_E_CUDA (-100)                /* CUDA runtime / launch failure */

/* output element types */
#define SFB_F64 0
#define SFB_F32 1
#define SFB_I64 2

/* ---- library ----------------------------------------------------------- */
const char *sfb_last_error(void);
int sfb_version(void);
/* 1 when the library was built for sm_100a and a device is visible */
int sfb_device_ok(void);

/* page-lock a host array in place for direct DMA of stream states (no
 * reference counterpart: the reference never leaves the host).  Returns 0 when
 * registered, 1 when the range is already page-locked (nothing done), or
 * SFB_E_CUDA (not fatal: copies stay pageable); never leaves a sticky CUDA
 * error behind. */
int sfb_host_register(void *p, int64_t bytes);
int sfb_host_unregister(void *p);

/* ---- host stream arithmetic (exact integers; core.py) -------------------- */
/* core.py:79-86 validate_seed -> SFB_E_INVALID_SEED */
int sfb_validate_seed(const int64_t seed[6]);
/* core.py:114-123 next_state: one step, z in [1, m1] */
int sfb_next_state(int64_t state[6], int64_t *z);
/* core.py:55-62 _jump_matrices(e): T1^(2^e) mod m1, T2^(2^e) mod m2 (row-major) */
int sfb_jump_matrices(int e, int64_t j1[9], int64_t j2[9]);
/* core.py:126-136 jump_ahead(s, e): advance 2^e steps */
int sfb_jump_ahead(int64_t state[6], int e);
/* generalisation used by the chunked kernels: advance n steps (any n) */
int sfb_skip(int64_t state[6], uint64_t n);
/* core.py:222-235 create_streams + core.py:139-142 _jump_seed:
 * rows[k] = J^k seed (J = T^(2^134)); next_seed = J^n seed. */
int sfb_create_streams(const int64_t seed[6], int64_t n, int64_t *rows,
                       int64_t next_seed[6]);

/* ---- stream files (core.py:238-305) ------------------------------------ */
/* bytes needed by sfb_format_streams (upper bound) */
int64_t sfb_format_streams_bound(int64_t n);
/* core.py:242-250 save_streams: writes the exact text into buf; *len = bytes */
int sfb_format_streams(const int64_t *current, const int64_t *initial, int64_t n,
                       char *buf, int64_t cap, int64_t *len);
/* core.py:238-261 save_streams / save_streams_atomic to a path
 * (atomic: temp file + fsync + rename, core.py:253-261) */
int sfb_save_streams(const char *path, const int64_t *current,
                     const int64_t *initial, int64_t n, int atomic);
/* core.py:264-305 load_streams, split in two: count from the header, then
 * the parse (same checks, same error class: SFB_E_CORRUPT_STREAM_FILE). */
int sfb_parse_streams_count(const char *text, int64_t len, int64_t *n);
int sfb_parse_streams(const char *text, int64_t len, int64_t *current,
                      int64_t *initial, int64_t n);

/* ---- device fills (grid.py:112-144 run_grid -> _kernels) --------------- */
/* _kernels.py:50-80 fill_real: mode 0 uniform (f64 out), mode 1 exponential
 * (f64 out, rate > 0).  Work item w=(i,j) = i + g0*j owns cells
 * {r = i mod g0, c = j mod g1}, row-major.  Only items with ordinal in
 * [item_lo, item_hi) run (multi-GPU shard; the whole grid is [0, g0*g1)).
 * Padding columns [ncol, npad) of every row are zeroed when zero_pad != 0.
 * d_cur: device int64 (n_streams, 6); d_out: device f64 (nrow, npad). */
int sfb_fill_real(int64_t *d_cur, int64_t n_streams, double *d_out, int64_t nrow,
                  int64_t ncol, int64_t npad, int64_t g0, int64_t g1, int mode,
                  double rate, int64_t item_lo, int64_t item_hi, int zero_pad,
                  void *stream);
/* _kernels.py:83-105 fill_integer: raw z in [1, m1] into int64 */
int sfb_fill_integer(int64_t *d_cur, int64_t n_streams, int64_t *d_out,
                     int64_t nrow, int64_t ncol, int64_t npad, int64_t g0,
                     int64_t g1, int64_t item_lo, int64_t item_hi, int zero_pad,
                     void *stream);
/* _kernels.py:108-166 fill_normal: paired-lane Box-Muller, row-major stream
 * ordinal s = i*g1 + j (pairs j even).  out_dtype SFB_F64 or SFB_F32 (the
 * float32 extension rounds the fp64 result once).  Shard range [item_lo,
 * item_hi) is in stream ordinals and must be pair aligned.  g1 must be even
 * (SFB_E_INVALID_GRID, grid.py:37-40). */
/* ---- Gaussian random fields (grf.py:116-187) -------- */
/* grf.py:116-124 bessel_k: K_nu(x) elementwise on device arrays (nu > 0, x > 0
 * validated by the caller); ~1e-13 relative to scipy.special.kv */
int sfb_bessel_k(double nu, const double *d_x, int64_t n, double *d_out, void *stream);
/* grf.py:138-159 matern_correlation at distances d (1 at d == 0) */
int sfb_matern_correlation(double kappa, double range, const double *d_dist, int64_t n,
                           double *d_out, void *stream);
/* grf.py:170-187 matern_cov: nb blocks of n x n into d_out (nb*n, n).
 * params: nb rows of (shape, range, variance, aniso_ratio, aniso_angle), host.
 * nx*ny == n: a regular GridSpec (cells row-major over (y, x), spacing `cell`)
 * -> one correlation per distinct index offset; otherwise d_coords (n, 2).
 * d_scratch: sfb_matern_scratch_bytes(nb, nx, ny) bytes of device memory. */
int sfb_matern_cov(const double *params, int nb, const double *d_coords, int64_t n, int nx,
                   int ny, double cell, double *d_scratch, double *d_out, void *stream);
int64_t sfb_matern_scratch_bytes(int nb, int nx, int ny);
/* CPU test hook: the same K_nu on the host */
double sfb_host_bessel_k(double nu, double x);
/* grf.py:190-208 chol_batch: per block LDL^T of `batch` SPD blocks of n x n
 * (d_a (batch*n, n), row-major, not modified): d_lmat receives the unit-lower
 * L = C / diag(C) (0 above the diagonal), d_diag (batch, n) D = diag(C)^2, C
 * the Cholesky factor (LAPACK dpotrf, lower).  d_info (batch) int32: 0, or
 * LAPACK's info -- the order of the first non-positive leading minor -- for a
 * block that is not positive definite (the caller raises
 * NotPositiveDefiniteError(batch, pivot)).  Hand-written FP64 tensor-core
 * (DMMA) blocked factorisation; d_lmat may alias d_a. */
int sfb_chol_batch(const double *d_a, int64_t n, int64_t batch, double *d_lmat, double *d_diag,
                   int32_t *d_info, void *stream);
/* grf.py:211-240 multiply_lower_diag_batch: d_out (batch*n, r) block b =
 * L_b diag(s(D_b)) Z_b, s = sqrt (transform 0) or identity (1); d_z (n, r)
 * shared by every block (z_shared = 1) or (batch*n, r). */
int sfb_lower_diag_multiply(const double *d_lmat, const double *d_diag, int64_t n, int64_t batch,
                            const double *d_z, int z_shared, int64_t r, int transform,
                            double *d_out, void *stream);

/* multi-GPU e2e helper (no reference counterpart: the reference has one host):
 * copy the cells of grid columns [j_lo, j_hi) -- columns c = j + g1 q of a
 * rank's uniform-kind shard -- from the (nrow, npad) device matrix into a
 * packed host array, row-major over (row, q, j).  Stream-ordered. */
int sfb_download_shard(void *dst_host, const void *src_dev, int64_t nrow, int64_t ncol,
                       int64_t npad, int64_t g1, int64_t j_lo, int64_t j_hi, int64_t elsize,
                       void *stream);
int sfb_fill_normal(int64_t *d_cur, int64_t n_streams, void *d_out, int out_dtype,
                    int64_t nrow, int64_t ncol, int64_t npad, int64_t g0,
                    int64_t g1, int64_t item_lo, int64_t item_hi, int zero_pad,
                    void *stream);

/* ---- device Fisher simulation (fisher.py:118-164 -> _kernels) ----------- */
/* _kernels.py:169-286 fisher_replicates over items [item_lo, item_hi):
 * each item runs `reps` replicates on its own stream; the hit count
 * (stat <= threshold) is ADDED to *d_count (device uint64; zero it first, or
 * pass zero_count=1).  d_stats (nullable, device f64) receives the statistic of
 * replicate rep of item w at (w - item_lo)*reps + rep (work-item major,
 * _kernels.py:277-278).  d_item_counts (nullable, device int64) receives the
 * per-item hit counts.  nrowt/ncolt/lf are HOST arrays (the margins and the
 * scipy gammaln table, fisher.py:70-72); lf_len = total + 1. */
int sfb_fisher_replicates(int64_t *d_cur, int64_t n_streams, const int64_t *nrowt,
                          int nr, const int64_t *ncolt, int nc, const double *lf,
                          int64_t lf_len, double threshold, int64_t reps,
                          int64_t item_lo, int64_t item_hi, double *d_stats,
                          int64_t *d_item_counts, uint64_t *d_count,
                          int zero_count, void *stream);
/* Host-buffer form of sfb_fisher_replicates -- the call a host-authoritative
 * fisher_sim makes (fisher.py:147-157: states, count and statistics in host
 * memory; the reference's kernel call is synchronous): uploads rows
 * [item_lo, item_hi) of h_cur (int64 (n_streams, 6), mutated in place), runs
 * the kernels on `stream`, and returns after the final states, *h_count (=
 * hits, not added) and h_stats (nullable; (w - item_lo)*reps + rep) are back
 * in host memory.  Page-locked host arrays give direct DMA. */
int sfb_fisher_replicates_host(int64_t *h_cur, int64_t n_streams, const int64_t *nrowt,
                               int nr, const int64_t *ncolt, int nc, const double *lf,
                               int64_t lf_len, double threshold, int64_t reps,
                               int64_t item_lo, int64_t item_hi, double *h_stats,
                               uint64_t *h_count, void *stream);
/* Background memo builds in flight (sfb_fisher_replicates* upgrade a capped
 * table's memo set on repeated use, on host threads; a call made while one is
 * pending runs on the current set).  No reference counterpart: lets a caller
 * that times steady-state calls wait until the set is final. */
int sfb_fisher_memo_pending(void);
/* _kernels.py:289-391 rcont2_table: one table from one 6-word state, run by
 * the same device sampler on one thread.  d_state: device int64[6] (mutated),
 * d_mat: device int64[nr*nc]. */
int sfb_rcont2_table(const int64_t *nrowt, int nr, const int64_t *ncolt, int nc,
                     const double *lf, int64_t lf_len, int64_t *d_state,
                     int64_t *d_mat, void *stream);

/* ---- measurement ---------------------------------------------------------- */
/* the rsqrt.approx.f64 seed used by the float32 Box-Muller form, elementwise
 * (accuracy test, tests/test_gpu_parity.py) */
int sfb_probe_rsqrt(const double *d_x, double *d_y, int64_t n, void *stream);
/* FP64-pipe roofline probe (bench.py): blocks x 256 threads x iters x 8 DFMA */
int sfb_probe_fp64(double *d_out, int64_t blocks, int iters, void *stream);
/* FP64 tensor-core (DMMA) probe: `blocks` CTAs of 4 warps, each warp `iters`
 * x 16 independent mma.sync.m8n8k4.f64 (512 flops each); bench.py derives the
 * DMMA roofline denominator of the GRF Cholesky from its time. */
int sfb_probe_dmma(double *d_out, int64_t blocks, int iters, void *stream);
/* write-only HBM probe: fills `bytes` (multiple of 16) with 16-byte stores;
 * variant 0 = grid-stride sweep, 1 = per-CTA contiguous segments (fill shape),
 * 2 = per-CTA segments with 32-byte stores */
int sfb_probe_write(void *d_out, int64_t bytes, int variant, void *stream);

/* ---- test hooks (host execution of the device arithmetic) --------------- */
/* runs the uint32 device step formulation on the host: n states x steps,
 * writes the outputs z and advances states (int64 (n,6)) */
int sfb_host_step_u32(int64_t *states, int64_t n, int64_t steps, int64_t *z_out);
/* the device exp() port (glibc __exp FMA variant) evaluated on the host */
double sfb_host_exp(double x);
/* the device log1p() port (glibc __log1p FMA variant) evaluated on the host */
double sfb_host_log1p(double x);
/* test hook: the branch-free log1p of the exponential fill's domain (x = -u);
 * *rare = 1 where the fill recomputes with the full port */
double sfb_host_log1p_fill(double x, int *rare);
/* the device Box-Muller pair transform (box_muller.cuh) evaluated on the host
 * for draws z1[k], z2[k] in [1, m1]: a = R cos(theta), b = R cos(theta - pi/2) */
int sfb_host_box_muller(const int64_t *z1, const int64_t *z2, int64_t n, double *a,
                        double *b);
/* the device Fisher sampler (fisher_sampler.cuh) run serially on the host over
 * items [item_lo, item_hi) (states int64 (n,6), mutated; stats nullable,
 * indexed (w - item_lo)*reps + rep; *count = hits) -- CPU test hook */
/* test hook: the float32 Box-Muller form (box_muller_pair_f32) on the host,
 * with `newton` sqrt corrections and a modelled rsqrt seed of relative error
 * seed_rel_err */
int sfb_host_box_muller_f32(const int64_t *z1, const int64_t *z2, int64_t n, int newton,
                            double seed_rel_err, float *a, float *b);
int sfb_host_fisher_replicates(int64_t *cur, const int64_t *nrowt, int nr,
                               const int64_t *ncolt, int nc, const double *lf,
                               double threshold, int64_t reps, int64_t item_lo,
                               int64_t item_hi, double *stats, int64_t *count);

#ifdef __cplusplus
}
#endif
#endif /* SFB_H_ */
