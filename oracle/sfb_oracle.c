/*
 * sfb_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * A plain-C restatement of the reference CPU hot path of `streamforge`
 * (/root/reference/pkg/src/streamforge/_kernels.py and core.py), used by
 *   - tests/ (parity oracle, pinned against tests/golden/ fixtures that were
 *     produced by importing the real reference, see tests/golden/gen_golden.py),
 *   - __graft_entry__.smoke() (checker),
 *   - bench.py's cpu_baseline / --impl reference arm (timed CPU port).
 * Nothing in the product package may load this library.
 *
 * Bit-exactness notes:
 *   - compiled with -ffp-contract=off: numba emits no FMA contraction in these
 *     loops, so neither may we;
 *   - exp/log/log1p/cos/sqrt are the host glibc libm calls, exactly what the
 *     numba kernels call, never numpy's SIMD versions;
 *   - every int64 -> double promotion mirrors numba's typing of the Python
 *     expression it restates (int64 * float64 -> sitofp + fmul).
 * Parallelism: OpenMP over work items (the reference's prange axis,
 * _kernels.py:58,87,124,186); results are thread-count invariant by
 * construction, exactly like the reference.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define M1 2147483647LL /* core.py:29 */
#define M2 2147462579LL /* core.py:30 */
static const double NORM = 1.0 / 2147483648.0; /* _kernels.py:20 */
static const double TWOPI = 2.0 * 3.141592653589793; /* _kernels.py:21 */
static const double HALFPI = 0.5 * 3.141592653589793; /* _kernels.py:22 */

static int set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_num_procs();
    return nthreads;
#else
    (void)nthreads;
    return 1;
#endif
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_num_procs();
#else
    return 1;
#endif
}

/* _kernels.py:33-47 -- one MRG31k3p step; z in [1, m1]. */
static inline int64_t step(int64_t *a0, int64_t *a1, int64_t *a2,
                           int64_t *b0, int64_t *b1, int64_t *b2) {
    int64_t y1 = (4194304LL * *a1 + 129LL * *a2) % M1;
    *a2 = *a1; *a1 = *a0; *a0 = y1;
    int64_t y2 = (32768LL * *b0 + 32769LL * *b2) % M2;
    *b2 = *b1; *b1 = *b0; *b0 = y2;
    int64_t z = y1 - y2;
    if (z <= 0) z += M1;
    return z;
}

int64_t orc_step(int64_t *st) {
    return step(&st[0], &st[1], &st[2], &st[3], &st[4], &st[5]);
}

/* _kernels.py:50-80 -- uniform (mode 0) / exponential (mode 1) fill.
 * Item w=(i,j), i = w mod g0, j = w div g0, draws from stream w. */
void orc_fill_real(int64_t *cur, double *out, int64_t nrow, int64_t ncol,
                   int64_t npad, int64_t g0, int64_t g1n, int mode,
                   double rate, int nthreads) {
    int64_t nitems = g0 * g1n;
    nthreads = set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
    for (int64_t w = 0; w < nitems; ++w) {
        int64_t i = w % g0, j = w / g0;
        int64_t *c = cur + 6 * w;
        int64_t a0 = c[0], a1 = c[1], a2 = c[2], b0 = c[3], b1 = c[4], b2 = c[5];
        for (int64_t r = i; r < nrow; r += g0) {
            for (int64_t cc = j; cc < ncol; cc += g1n) {
                int64_t z = step(&a0, &a1, &a2, &b0, &b1, &b2);
                double u = (double)z * NORM;
                if (mode == 0)
                    out[r * npad + cc] = u;
                else
                    out[r * npad + cc] = -log1p(-u) / rate;
            }
        }
        c[0] = a0; c[1] = a1; c[2] = a2; c[3] = b0; c[4] = b1; c[5] = b2;
    }
}

/* _kernels.py:83-105 -- raw integer fill, same layout as fill_real. */
void orc_fill_integer(int64_t *cur, int64_t *out, int64_t nrow, int64_t ncol,
                      int64_t npad, int64_t g0, int64_t g1n, int nthreads) {
    int64_t nitems = g0 * g1n;
    nthreads = set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
    for (int64_t w = 0; w < nitems; ++w) {
        int64_t i = w % g0, j = w / g0;
        int64_t *c = cur + 6 * w;
        int64_t a0 = c[0], a1 = c[1], a2 = c[2], b0 = c[3], b1 = c[4], b2 = c[5];
        for (int64_t r = i; r < nrow; r += g0)
            for (int64_t cc = j; cc < ncol; cc += g1n)
                out[r * npad + cc] = step(&a0, &a1, &a2, &b0, &b1, &b2);
        c[0] = a0; c[1] = a1; c[2] = a2; c[3] = b0; c[4] = b1; c[5] = b2;
    }
}

/* _kernels.py:108-166 -- paired-lane Box-Muller; row-major stream ordinal
 * s0 = i*g1n + j0, s1 = s0+1.  out_f64 or out_f32 (exactly one non-NULL):
 * the f32 variant stores (float)(reference double), the tolerance anchor for
 * the GPU float32 path. */
void orc_fill_normal(int64_t *cur, double *out_f64, float *out_f32,
                     int64_t nrow, int64_t ncol, int64_t npad, int64_t g0,
                     int64_t g1n, int nthreads) {
    int64_t half = g1n / 2;
    int64_t npairs = g0 * half;
    nthreads = set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
    for (int64_t p = 0; p < npairs; ++p) {
        int64_t i = p / half;
        int64_t j0 = 2 * (p % half);
        int64_t s0 = i * g1n + j0, s1 = s0 + 1;
        int64_t *c0p = cur + 6 * s0, *c1p = cur + 6 * s1;
        int64_t a0 = c0p[0], a1 = c0p[1], a2 = c0p[2], b0 = c0p[3], b1 = c0p[4], b2 = c0p[5];
        int64_t c0 = c1p[0], c1 = c1p[1], c2 = c1p[2], d0 = c1p[3], d1 = c1p[4], d2 = c1p[5];
        for (int64_t r = i; r < nrow; r += g0) {
            int64_t ca = j0, cb = j0 + 1;
            while (ca < ncol) {
                int64_t z1 = step(&a0, &a1, &a2, &b0, &b1, &b2);
                int64_t z2 = step(&c0, &c1, &c2, &d0, &d1, &d2);
                double u1 = (double)z1 * NORM;
                double theta = (TWOPI * NORM) * (double)z2;
                double radius = sqrt(-2.0 * log(u1));
                double va = radius * cos(theta);
                if (out_f64) out_f64[r * npad + ca] = va; else out_f32[r * npad + ca] = (float)va;
                if (cb < ncol) {
                    double vb = radius * cos(theta - HALFPI);
                    if (out_f64) out_f64[r * npad + cb] = vb; else out_f32[r * npad + cb] = (float)vb;
                }
                ca += g1n;
                cb += g1n;
            }
        }
        c0p[0] = a0; c0p[1] = a1; c0p[2] = a2; c0p[3] = b0; c0p[4] = b1; c0p[5] = b2;
        c1p[0] = c0; c1p[1] = c1; c1p[2] = c2; c1p[3] = d0; c1p[4] = d1; c1p[5] = d2;
    }
}

/* _kernels.py:147-152 for arbitrary draw pairs (z1, z2) in [1, m1]: the
 * transform alone, used to measure the device port's accuracy at scale. */
void orc_box_muller(const int64_t *z1, const int64_t *z2, int64_t n, double *a,
                    double *b) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n; ++k) {
        double u1 = (double)z1[k] * NORM;
        double theta = (TWOPI * NORM) * (double)z2[k];
        double radius = sqrt(-2.0 * log(u1));
        a[k] = radius * cos(theta);
        b[k] = radius * cos(theta - HALFPI);
    }
}

/* One conditional-hypergeometric cell draw, _kernels.py:205-261 (shared with
 * rcont2_table, _kernels.py:322-375).  Consumes exactly one step. */
static inline int64_t sample_cell(int64_t ia, int64_t idv, int64_t ie,
                                  int64_t ib, int64_t ic, int64_t ii,
                                  const double *lf, int64_t *s) {
    int64_t z = step(&s[0], &s[1], &s[2], &s[3], &s[4], &s[5]);
    double u = (double)z * NORM;
    int64_t lo = ia + idv - ie;
    if (lo < 0) lo = 0;
    int64_t hi = ia < idv ? ia : idv;
    int64_t k;
    if (hi <= lo) {
        k = lo;
    } else {
        k = (int64_t)((double)ia * ((double)idv / (double)ie) + 0.5);
        if (k < lo) k = lo;
        else if (k > hi) k = hi;
        double base = lf[ia] + lf[ib] + lf[idv] + lf[ic] - lf[ie];
        double x = exp(base - lf[k] - lf[idv - k] - lf[ia - k] - lf[ii + k]);
        if (u > x) {
            double acc = x, pu = x, pd = x;
            int64_t ku = k, kd = k;
            for (;;) {
                int moved = 0;
                if (ku < hi) {
                    pu = pu * (double)(idv - ku) * (double)(ia - ku) /
                         (((double)ku + 1.0) * ((double)(ii + ku) + 1.0));
                    ku += 1;
                    acc += pu;
                    moved = 1;
                    if (u <= acc) { k = ku; break; }
                }
                if (kd > lo) {
                    pd = pd * (double)kd * (double)(ii + kd) /
                         (((double)(idv - kd) + 1.0) * ((double)(ia - kd) + 1.0));
                    kd -= 1;
                    acc += pd;
                    moved = 1;
                    if (u <= acc) { k = kd; break; }
                }
                if (!moved) { k = ku; break; }
            }
        }
    }
    return k;
}

/* Sample one table (nr, nc >= 2) into mat; _kernels.py:196-270. */
static void sample_table(const int64_t *nrowt, int nr, const int64_t *ncolt,
                         int nc, int64_t ntot, const double *lf, int64_t *s,
                         int64_t *mat, int64_t *jwork) {
    int64_t jc = ntot;
    for (int m = 0; m < nc - 1; ++m) jwork[m] = ncolt[m];
    for (int l = 0; l < nr - 1; ++l) {
        int64_t ia = nrowt[l];
        int64_t ic = jc;
        jc -= ia;
        for (int m = 0; m < nc - 1; ++m) {
            int64_t idv = jwork[m];
            int64_t ie = ic;
            ic -= idv;
            int64_t ib = ie - ia;
            int64_t ii = ib - idv;
            int64_t k = sample_cell(ia, idv, ie, ib, ic, ii, lf, s);
            mat[(int64_t)l * nc + m] = k;
            ia -= k;
            jwork[m] -= k;
        }
        mat[(int64_t)l * nc + nc - 1] = ia;
    }
    int64_t rem = nrowt[nr - 1];
    for (int m = 0; m < nc - 1; ++m) {
        mat[(int64_t)(nr - 1) * nc + m] = jwork[m];
        rem -= jwork[m];
    }
    mat[(int64_t)(nr - 1) * nc + nc - 1] = rem;
}

/* _kernels.py:169-286 over items [item_lo, item_hi).  stats (nullable) is
 * indexed w*reps + rep with the global item index w (_kernels.py:277-278).
 * item_counts (nullable) receives per-item hit counts (test aid). */
int64_t orc_fisher_replicates(int64_t *cur, const int64_t *nrowt, int nr,
                              const int64_t *ncolt, int nc, const double *lf,
                              double threshold, int64_t reps, int64_t item_lo,
                              int64_t item_hi, double *stats,
                              int64_t *item_counts, int nthreads) {
    int64_t ntot = 0;
    for (int l = 0; l < nr; ++l) ntot += nrowt[l];
    int64_t counts = 0;
    nthreads = set_threads(nthreads);
#pragma omp parallel num_threads(nthreads) reduction(+ : counts)
    {
        int64_t *mat = (int64_t *)__builtin_alloca(sizeof(int64_t) * (size_t)nr * (size_t)nc);
        int64_t *jwork = (int64_t *)__builtin_alloca(sizeof(int64_t) * (size_t)nc);
#pragma omp for schedule(dynamic, 1)
        for (int64_t w = item_lo; w < item_hi; ++w) {
            int64_t s[6];
            memcpy(s, cur + 6 * w, sizeof s);
            int64_t hits = 0;
            for (int64_t rep = 0; rep < reps; ++rep) {
                sample_table(nrowt, nr, ncolt, nc, ntot, lf, s, mat, jwork);
                double stat = 0.0;
                for (int l = 0; l < nr; ++l)
                    for (int m = 0; m < nc; ++m) stat -= lf[mat[(int64_t)l * nc + m]];
                if (stat <= threshold) hits += 1;
                if (stats) stats[w * reps + rep] = stat;
            }
            counts += hits;
            if (item_counts) item_counts[w - item_lo] = hits;
            memcpy(cur + 6 * w, s, sizeof s);
        }
    }
    return counts;
}

/* _kernels.py:289-391 -- one table from a 6-entry state (mutated). */
void orc_rcont2_table(const int64_t *nrowt, int nr, const int64_t *ncolt,
                      int nc, const double *lf, int64_t *state, int64_t *mat) {
    int64_t ntot = 0;
    for (int l = 0; l < nr; ++l) ntot += nrowt[l];
    memset(mat, 0, sizeof(int64_t) * (size_t)nr * (size_t)nc);
    if (nr == 1) {
        for (int m = 0; m < nc; ++m) mat[m] = ncolt[m];
    } else if (nc == 1) {
        for (int l = 0; l < nr; ++l) mat[l] = nrowt[l];
    } else {
        int64_t jwork[nc];
        sample_table(nrowt, nr, ncolt, nc, ntot, lf, state, mat, jwork);
    }
}

/* ---- stream arithmetic: core.py:44-66, 126-142, 222-235 ---------------- */
static const int64_t T1[9] = {0, 1LL << 22, (1LL << 7) + 1, 1, 0, 0, 0, 1, 0};
static const int64_t T2[9] = {1LL << 15, 0, (1LL << 15) + 1, 1, 0, 0, 0, 1, 0};

static void mat_mul(const int64_t *a, const int64_t *b, int64_t m, int64_t *o) {
    int64_t t[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            unsigned __int128 acc = 0;
            for (int k = 0; k < 3; ++k)
                acc += (unsigned __int128)(uint64_t)a[3 * i + k] * (uint64_t)b[3 * k + j];
            t[3 * i + j] = (int64_t)(acc % (uint64_t)m);
        }
    memcpy(o, t, sizeof t);
}

static void mat_vec(const int64_t *a, const int64_t *v, int64_t m, int64_t *o) {
    int64_t t[3];
    for (int i = 0; i < 3; ++i) {
        unsigned __int128 acc = 0;
        for (int k = 0; k < 3; ++k)
            acc += (unsigned __int128)(uint64_t)a[3 * i + k] * (uint64_t)v[k];
        t[i] = (int64_t)(acc % (uint64_t)m);
    }
    memcpy(o, t, sizeof t);
}

/* core.py:55-62: T^(2^e) by e squarings. */
void orc_jump_matrices(int e, int64_t *j1, int64_t *j2) {
    memcpy(j1, T1, sizeof T1);
    memcpy(j2, T2, sizeof T2);
    for (int k = 0; k < e; ++k) {
        mat_mul(j1, j1, M1, j1);
        mat_mul(j2, j2, M2, j2);
    }
}

/* core.py:126-136 generalised to any step count n (binary powering of the
 * same transition matrices; jump_ahead(s, e) == skip(s, 2^e)). */
void orc_skip(int64_t *state, uint64_t n) {
    int64_t p1[9], p2[9];
    memcpy(p1, T1, sizeof T1);
    memcpy(p2, T2, sizeof T2);
    while (n) {
        if (n & 1) {
            mat_vec(p1, state, M1, state);
            mat_vec(p2, state + 3, M2, state + 3);
        }
        n >>= 1;
        if (n) {
            mat_mul(p1, p1, M1, p1);
            mat_mul(p2, p2, M2, p2);
        }
    }
}

/* core.py:222-235 (+ _jump_seed core.py:139-142): stream k = J^k seed. */
void orc_create_streams(const int64_t *seed, int64_t n, int64_t *rows,
                        int64_t *next_seed) {
    int64_t j1[9], j2[9], s[6];
    orc_jump_matrices(134, j1, j2);
    memcpy(s, seed, sizeof s);
    for (int64_t k = 0; k < n; ++k) {
        memcpy(rows + 6 * k, s, sizeof s);
        mat_vec(j1, s, M1, s);
        mat_vec(j2, s + 3, M2, s + 3);
    }
    memcpy(next_seed, s, sizeof s);
}
