// fill.cu -- sm_100a generation kernels: uniform / integer / exponential and
// paired-lane Box-Muller fills (the reference's _kernels.fill_real,
// fill_integer, fill_normal: _kernels.py:50-166, dispatched by grid.run_grid,
// grid.py:112-144).
//
// Layout contract (grid.py:73-102): work item (i, j) of the g0 x g1 grid owns
// the cells {(r, c): r = i mod g0, c = j mod g1} and visits them row-major,
// one MRG31k3p step per cell (uniform kinds) or one step of each of the two
// lane streams per cell pair (normal).  Stream ordinals: i + g0*j for the
// uniform kinds, i*g1 + j for normals.  Unused streams are never touched and
// padding columns are never written by the kernels (they are zeroed by a
// cudaMemset2DAsync when requested, matching MatrixBuffer's np.zeros).
//
// B200 decomposition: since every cell consumes exactly one
// step, the state at any draw index d of an item is A^d s_item, so the work of
// one item is split into chunks whose start states are reached by jump-ahead
// (powers A^(2^b) passed by value as kernel parameters).  Results are
// bit-identical for every chunking, exactly like the reference's thread-count
// invariance (tests/test_grid.py:91-103).
//
//  * *_fast kernels: the dominant layouts (g1 even, npad even): one thread
//    drives the two streams of a column pair (j, j+1) over a block of owned
//    rows and writes both values with one 16-byte (f64/i64) or 8-byte (f32)
//    streaming store; adjacent lanes own adjacent pairs, so a warp writes 512
//    contiguous bytes per step (coalesced, HBM-write bound).
//  * *_generic kernels: any grid / shape / shard (odd g1, vectors, ragged
//    shards): one thread per (item, chunk of draws), scalar stores.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "box_muller.cuh"
#include "log1p_glibc.cuh"
#include "sfb_internal.h"

namespace sfb {

enum Kind { kUniform = 0, kExponential = 1, kInteger = 2 };

struct Geom {
    int64_t nrow, ncol, npad, g0, g1;
};

// number of owned rows of grid row i / owned columns of grid column j
__device__ __forceinline__ int64_t owned(int64_t n, int64_t idx, int64_t g) {
    return idx < n ? (n - idx + g - 1) / g : 0;
}

// u = z * NORM (_kernels.py:70) from zm1 = z - 1, without an int->double
// conversion (I2F.F64 runs on the narrow XU pipe): the register pair
// (lo = zm1, hi = 0x43300000) is the double M = 2^52 + zm1, and
// fma(M, 2^-31, 2^-31 - 2^21) = zm1 2^-31 + 2^-31 exactly (M 2^-31 is an
// exact power-of-two scaling and the sum is representable), i.e. one DFMA.
__device__ __forceinline__ double u01(uint32_t zm1) {
    const double m = __hiloint2double(0x43300000, (int)zm1);
    return __fma_rn(m, kNorm, kNorm - 0x1p21);
}

// the exponential rate with its correctly rounded reciprocal (host-computed):
// v / rate = q0 + (v - rate q0) y with q0 = RN(v y) is RN(v / rate) when
// y = RN(1 / rate) (Markstein; no over/underflow: used for rates in
// [2^-500, 2^500], otherwise the IEEE division); markstein == 2: rate 1, no
// division at all (v / 1 == v)
struct RateArg {
    double r, y;
    int markstein;
};

// -log1p(-u) / rate (_kernels.py:74), bit-exact: log1p_fill_domain (the
// glibc port without data-dependent branches) for N values at once, the rare
// inputs of glibc's other paths (~2^-19) recomputed afterwards with the full
// port out of line, so the N evaluations stay in one basic block; divisions
// on the branch-free fast path (operands always normal on this domain); the
// division by the rate is Markstein's correction when RateArg allows it.
__device__ __noinline__ double log1p_rare(double x) { return glibc_log1p(x, DivFastNormal()); }

template <int KIND, int N>
__device__ __forceinline__ void real_values(const uint32_t *zm1, const RateArg &rate,
                                            double *v) {
    if (KIND == kUniform) {
#pragma unroll
        for (int k = 0; k < N; ++k) v[k] = u01(zm1[k]);
        return;
    }
    bool any = false, rare[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        v[k] = -log1p_fill_domain(-u01(zm1[k]), DivFastNormal(), rare[k]);
        any |= rare[k];
    }
    if (any) {
#pragma unroll
        for (int k = 0; k < N; ++k)
            if (rare[k]) v[k] = -log1p_rare(-u01(zm1[k]));
    }
#pragma unroll
    for (int k = 0; k < N; ++k) {
        if (rate.markstein == 2) {  // rate 1: v / 1 == v
        } else if (!rate.markstein) {
            v[k] = __ddiv_rn(v[k], rate.r);
        } else {
            const double q0 = v[k] * rate.y;
            v[k] = __fma_rn(__fma_rn(-q0, rate.r, v[k]), rate.y, q0);
        }
    }
}

template <int KIND>
__device__ __forceinline__ double real_value(uint32_t zm1, const RateArg &rate) {
    double v;
    real_values<KIND, 1>(&zm1, rate, &v);
    return v;
}

// one 16-byte streaming store of a column pair / one 8-byte store
template <int KIND>
__device__ __forceinline__ void put_pair(void *out, int64_t off, uint32_t za, uint32_t zb,
                                         const RateArg &rate) {
    if (KIND == kInteger)
        __stcs((longlong2 *)((long long *)out + off),
               make_longlong2((long long)za + 1, (long long)zb + 1));
    else {
        const uint32_t z[2] = {za, zb};
        double v[2];
        real_values<KIND, 2>(z, rate, v);
        __stcs((double2 *)((double *)out + off), make_double2(v[0], v[1]));
    }
}

template <int KIND>
__device__ __forceinline__ void put_one(void *out, int64_t off, uint32_t za,
                                        const RateArg &rate) {
    if (KIND == kInteger)
        __stcs((long long *)out + off, (long long)za + 1);
    else
        __stcs((double *)out + off, real_value<KIND>(za, rate));
}

// ---------------------------------------------------------------------------
// generic layouts (odd g1, vectors, ragged shards): unit = (grid row i, chunk
// c of an item's draws, column index jj), jj fastest -- adjacent lanes are the
// items that write adjacent columns, and only items with owned cells get
// units (a 1 x n vector on the default 64 x 8 grid has 8 active items)
struct GenMap {
    int64_t lo, hi;      // shard: items (uniform kinds) / pairs (normal)
    int64_t jlo, J;      // column indices covered: items' j / pairs' jp
    int64_t i_lo;        // first active grid row; rows i_lo .. (nunits / (J nchunks))
    int64_t nchunks, chunk, nunits;
};

// uniform kinds, generic layout
template <int KIND>
__global__ void __launch_bounds__(256) fill_uniform_generic(StateIO io,
                                                            void *__restrict__ out, Geom g,
                                                            GenMap m, RateArg rate,
                                                            const __grid_constant__ Pow2Table tab) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= m.nunits) return;
    const int64_t j = m.jlo + u % m.J;
    const int64_t r = u / m.J;
    const int64_t c = r % m.nchunks;
    const int64_t i = m.i_lo + r / m.nchunks;
    const int64_t w = i + g.g0 * j;
    if (w < m.lo || w >= m.hi) return;
    const int64_t nr = owned(g.nrow, i, g.g0), nc = owned(g.ncol, j, g.g1);
    const int64_t total = nr * nc;
    const int64_t d0 = c * m.chunk;
    if (d0 >= total) return;
    const int64_t d1 = min(d0 + m.chunk, total);
    Mrg s = load_state(io, w);
    skip(tab, s, (uint64_t)d0);
    // row segments of the item's draws: inside a segment the cells are g1
    // apart, so the inner loop is a pointer bump (no per-cell index math)
    int64_t rho = d0 / nc, q = d0 % nc;
    for (int64_t d = d0; d < d1; ++rho, q = 0) {
        const int64_t len = min(nc - q, d1 - d);
        d += len;
        const int64_t off = (i + g.g0 * rho) * g.npad + j + g.g1 * q;
        if (KIND == kInteger) {
            long long *p = (long long *)out + off;
#pragma unroll 4
            for (int64_t t = 0; t < len; ++t, p += g.g1) __stcs(p, (long long)step_m1(s) + 1);
        } else {
            double *p = (double *)out + off;
            int64_t t = 0;
            for (; t + 4 <= len; t += 4, p += 4 * g.g1) {  // 4 evaluations per basic block
                uint32_t z[4];
                double v[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) z[k] = step_m1(s);
                real_values<KIND, 4>(z, rate, v);
#pragma unroll
                for (int k = 0; k < 4; ++k) __stcs(p + k * g.g1, v[k]);
            }
            for (; t < len; ++t, p += g.g1) __stcs(p, real_value<KIND>(step_m1(s), rate));
        }
    }
    if (d1 == total) store_state(io, w, s);
}

// uniform kinds, column-pair fast path (g1 even, npad even, shard = whole pairs)
// unit = (chunk c, grid row i, pair jp): adjacent lanes = adjacent pairs
template <int KIND, int MINB, int NT = 256>
__global__ void __launch_bounds__(NT, MINB) fill_uniform_fast(StateIO io,
                                                         void *__restrict__ out, Geom g,
                                                         int64_t j_lo, int64_t npairs,
                                                         int64_t rows_per_chunk, int64_t nunits,
                                                         RateArg rate, const __grid_constant__ Pow2Table tab) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= nunits) return;
    const int64_t jp = u % npairs;
    const int64_t ic = u / npairs;
    const int64_t i = ic % g.g0, c = ic / g.g0;
    const int64_t j = j_lo + 2 * jp;
    const int64_t nr = owned(g.nrow, i, g.g0);
    const int64_t rho0 = c * rows_per_chunk;
    if (rho0 >= nr) return;
    const int64_t rho1 = min(rho0 + rows_per_chunk, nr);
    const int64_t na = owned(g.ncol, j, g.g1), nb = owned(g.ncol, j + 1, g.g1);
    const int64_t wa = i + g.g0 * j, wb = wa + g.g0;
    Mrg sa = load_state(io, wa), sb = load_state(io, wb);
    if (rho0) {
        skip(tab, sa, (uint64_t)(rho0 * na));
        skip(tab, sb, (uint64_t)(rho0 * nb));
    }
    for (int64_t rho = rho0; rho < rho1; ++rho) {
        const int64_t rowoff = (i + g.g0 * rho) * g.npad + j;
        int64_t q = 0;
        for (; q + 3 <= nb; q += 3) {  // step3: no shift-register moves
            uint32_t a0, a1, a2, b0, b1, b2;
            step3(sa, a0, a1, a2);
            step3(sb, b0, b1, b2);
            put_pair<KIND>(out, rowoff + g.g1 * q, a0, b0, rate);
            put_pair<KIND>(out, rowoff + g.g1 * (q + 1), a1, b1, rate);
            put_pair<KIND>(out, rowoff + g.g1 * (q + 2), a2, b2, rate);
        }
        for (; q < nb; ++q) {
            const uint32_t za = step_m1(sa), zb = step_m1(sb);
            put_pair<KIND>(out, rowoff + g.g1 * q, za, zb, rate);
        }
        if (na > nb) put_one<KIND>(out, rowoff + g.g1 * nb, step_m1(sa), rate);
    }
    if (rho1 == nr) {
        store_state(io, wa, sa);
        store_state(io, wb, sb);
    }
}

// uniform kinds, quad fast path (g1 % 4 == 0, npad % 4 == 0, shard = whole
// quads): one thread drives the four streams of columns j..j+3 and writes them
// with ONE 32-byte streaming store per owned row step (STG.E.ENL2.256, new on
// sm_100), so a warp store covers 1 KB contiguous and the LSU issues half the
// store instructions of the pair path.
__device__ __forceinline__ void st256(void *p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    asm volatile("st.global.cs.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c),
                 "l"(d)
                 : "memory");
}


template <int KIND>
__device__ __forceinline__ void put_quad(void *out, int64_t off, uint32_t z0, uint32_t z1,
                                         uint32_t z2, uint32_t z3, const RateArg &rate) {
    if (KIND == kInteger) {
        st256((long long *)out + off, (uint64_t)z0 + 1u, (uint64_t)z1 + 1u, (uint64_t)z2 + 1u,
              (uint64_t)z3 + 1u);
        return;
    }
    const uint32_t z[4] = {z0, z1, z2, z3};
    double v[4];
    real_values<KIND, 4>(z, rate, v);
    st256((long long *)out + off, (uint64_t)__double_as_longlong(v[0]),
          (uint64_t)__double_as_longlong(v[1]), (uint64_t)__double_as_longlong(v[2]),
          (uint64_t)__double_as_longlong(v[3]));
}

template <int KIND, int MINB, bool STEP3 = true>
__global__ void __launch_bounds__(256, MINB) fill_uniform_quad(StateIO io,
                                                         void *__restrict__ out, Geom g,
                                                         int64_t j_lo, int64_t nquads,
                                                         int64_t rows_per_chunk, int64_t nunits,
                                                         RateArg rate, const __grid_constant__ Pow2Table tab) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= nunits) return;
    const int64_t jq = u % nquads;
    const int64_t ic = u / nquads;
    const int64_t i = ic % g.g0, c = ic / g.g0;
    const int64_t j = j_lo + 4 * jq;
    const int64_t nr = owned(g.nrow, i, g.g0);
    const int64_t rho0 = c * rows_per_chunk;
    if (rho0 >= nr) return;
    const int64_t rho1 = min(rho0 + rows_per_chunk, nr);
    int64_t n[4];
    Mrg s[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        n[k] = owned(g.ncol, j + k, g.g1);  // nonincreasing in k, by at most one
        s[k] = load_state(io, i + g.g0 * (j + k));
        if (rho0) skip(tab, s[k], (uint64_t)(rho0 * n[k]));
    }
    for (int64_t rho = rho0; rho < rho1; ++rho) {
        const int64_t rowoff = (i + g.g0 * rho) * g.npad + j;
        int64_t q = 0;
        if (STEP3)
            for (; q + 3 <= n[3]; q += 3) {  // step3: no shift-register moves
                uint32_t z[4][3];
#pragma unroll
                for (int k = 0; k < 4; ++k) step3(s[k], z[k][0], z[k][1], z[k][2]);
#pragma unroll
                for (int t = 0; t < 3; ++t)
                    put_quad<KIND>(out, rowoff + g.g1 * (q + t), z[0][t], z[1][t], z[2][t],
                                   z[3][t], rate);
            }
        for (; q < n[3]; ++q) {
            const uint32_t z0 = step_m1(s[0]), z1 = step_m1(s[1]);
            const uint32_t z2 = step_m1(s[2]), z3 = step_m1(s[3]);
            put_quad<KIND>(out, rowoff + g.g1 * q, z0, z1, z2, z3, rate);
        }
#pragma unroll
        for (int k = 0; k < 3; ++k)  // ragged last column block
            if (n[k] > n[3]) put_one<KIND>(out, rowoff + k + g.g1 * n[3], step_m1(s[k]), rate);
    }
    if (rho1 == nr) {
#pragma unroll
        for (int k = 0; k < 4; ++k) store_state(io, i + g.g0 * (j + k), s[k]);
    }
}

// ---------------------------------------------------------------------------
// Box-Muller fills (_kernels.py:108-166).  float64 output: box_muller_pair()
// (box_muller.cuh, fp64 throughout, <= 4 ulp of the reference).  float32
// output: box_muller_pair_f32() (FAST, the default: ~25 instead of ~45 FP64
// ops per pair, <= 2^-44 relative) or the float64 transform rounded once
// (FAST == false, SFB_NORMAL_VARIANT bit 2).


__device__ __forceinline__ void put4(float *p, float a, float b, float c, float d) {
    __stcs((float4 *)p, make_float4(a, b, c, d));
}
__device__ __forceinline__ void put4(double *p, double a, double b, double c, double d) {
    __stcs((double2 *)p, make_double2(a, b));
    __stcs((double2 *)p + 1, make_double2(c, d));
}
__device__ __forceinline__ void put2(float *p, float a, float b) {
    __stcs((float2 *)p, make_float2(a, b));
}
__device__ __forceinline__ void put2(double *p, double a, double b) {
    __stcs((double2 *)p, make_double2(a, b));
}

// table words of box_muller.cuh (exact form) or the fast float32 tables,
// staged in shared memory (<= 36.9 KB)
constexpr int kBmLogWords = 3 * SFB_BM_LOG_N;
constexpr int kBmTabWords = kBmLogWords + 3 * (SFB_BM_TRIG_N + 1);
constexpr int kBmSmemBytes = kBmTabWords * 8;
static_assert(kBmFastLogPairs * 16 + kBmFastTrigPairs * 24 <= kBmSmemBytes, "fast tables fit");

struct BmView {
    const uint64_t *logw, *trigw;       // exact form
    const BmPair *logp, *trigp;         // fast float32 form
    const double *angle;
};

template <bool FAST>
__device__ __forceinline__ BmView stage_bm_tables(unsigned char *raw) {
    static const uint64_t kLogTab[kBmLogWords] = SFB_BM_LOG_TABLE_INIT;
    static const uint64_t kTrigTab[kBmTabWords - kBmLogWords] = SFB_BM_TRIG_TABLE_INIT;
    BmView v{};
    if (FAST) {
        BmPair *lp = (BmPair *)raw;
        BmPair *tp = lp + kBmFastLogPairs;
        double *ang = (double *)(tp + kBmFastTrigPairs);
        bm_fast_tables(kLogTab, kTrigTab, threadIdx.x, blockDim.x, lp, tp, ang);
        v.logw = kLogTab;  // global: the rare exact fallback of box_muller_pair_f32
        v.trigw = kTrigTab;
        v.logp = lp;
        v.trigp = tp;
        v.angle = ang;
    } else {
        uint64_t *w = (uint64_t *)raw;
        for (int t = threadIdx.x; t < kBmLogWords; t += blockDim.x) w[t] = kLogTab[t];
        for (int t = threadIdx.x; t < kBmTabWords - kBmLogWords; t += blockDim.x)
            w[kBmLogWords + t] = kTrigTab[t];
        v.logw = w;
        v.trigw = w + kBmLogWords;
    }
    __syncthreads();
    return v;
}

template <bool FAST>
__device__ __forceinline__ void bm(uint32_t z1, uint32_t z2, const BmView &v, double &a,
                                   double &b) {
    box_muller_pair(z1, z2, v.logw, v.trigw, a, b);
}
template <bool FAST>
__device__ __forceinline__ void bm(uint32_t z1, uint32_t z2, const BmView &v, float &a, float &b) {
    if (FAST) {
        box_muller_pair_f32(z1, z2, v.logp, v.trigp, v.angle, v.logw, v.trigw, a, b);
    } else {
        double da, db;
        box_muller_pair(z1, z2, v.logw, v.trigw, da, db);
        a = (float)da;
        b = (float)db;
    }
}

// N pairs at once: for the float32 fast form the (rare, ~1e-5) exact fallback
// is applied after all N pairs are computed, so the hot part is one basic
// block and the compiler can interleave the N independent FP64 chains
template <bool FAST, int N>
__device__ __forceinline__ void bmN(const uint32_t *z1, const uint32_t *z2, const BmView &v,
                                    double *a, double *b) {
#pragma unroll
    for (int k = 0; k < N; ++k) box_muller_pair(z1[k], z2[k], v.logw, v.trigw, a[k], b[k]);
}
template <bool FAST, int N>
__device__ __forceinline__ void bmN(const uint32_t *z1, const uint32_t *z2, const BmView &v,
                                    float *a, float *b) {
    if (!FAST) {
#pragma unroll
        for (int k = 0; k < N; ++k) bm<false>(z1[k], z2[k], v, a[k], b[k]);
        return;
    }
    bool rare = false;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        box_muller_pair_f32_core(z1[k], z2[k], v.logp, v.trigp, v.angle, a[k], b[k]);
        rare |= bm_f32_needs_exact(z2[k]);
    }
    if (rare) {
#pragma unroll
        for (int k = 0; k < N; ++k)
            if (bm_f32_needs_exact(z2[k])) {
                const F32Pair p = box_muller_pair_f32_exact(z1[k], z2[k], v.logw, v.trigw);
                a[k] = p.a;
                b[k] = p.b;
            }
    }
}

// normal, generic layout: unit = (pair, chunk of pair-iterations); PAIRED:
// npad even and out 2-element aligned, so a lane pair is one 8/16-byte store
template <typename T, bool FAST, bool PAIRED>
__global__ void __launch_bounds__(256) fill_normal_generic(StateIO io,
                                                           T *__restrict__ out, Geom g, GenMap m,
                                                           const __grid_constant__ Pow2Table tab) {
    __shared__ __align__(16) unsigned char bm_raw[kBmSmemBytes];
    const BmView bv = stage_bm_tables<FAST && sizeof(T) == 4>(bm_raw);
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= m.nunits) return;
    const int64_t half = g.g1 / 2;
    const int64_t jp = m.jlo + u % m.J;
    const int64_t r = u / m.J;
    const int64_t c = r % m.nchunks;
    const int64_t i = m.i_lo + r / m.nchunks;
    const int64_t p = i * half + jp;
    if (p < m.lo || p >= m.hi) return;
    const int64_t j0 = 2 * jp;  // _kernels.py:125-128
    const int64_t s0 = i * g.g1 + j0;
    const int64_t nr = owned(g.nrow, i, g.g0);
    const int64_t niter = owned(g.ncol, j0, g.g1);  // `while ca < ncol` trips per row
    const int64_t total = nr * niter;
    const int64_t d0 = c * m.chunk;
    if (d0 >= total) return;
    const int64_t d1 = min(d0 + m.chunk, total);
    Mrg sa = load_state(io, s0), sb = load_state(io, s0 + 1);
    skip(tab, sa, (uint64_t)d0);
    skip(tab, sb, (uint64_t)d0);
    // the partner lane of the row's last trip may lie past ncol (discarded,
    // both streams still advance); row segments with a pointer bump inside
    const int64_t q_nopartner = (j0 + g.g1 * (niter - 1) + 1 < g.ncol) ? -1 : niter - 1;
    int64_t rho = d0 / niter, q = d0 % niter;
    for (int64_t d = d0; d < d1; ++rho, q = 0) {
        const int64_t len = min(niter - q, d1 - d);
        d += len;
        T *o = out + (i + g.g0 * rho) * g.npad + j0 + g.g1 * q;
        int64_t t = 0;
        if (PAIRED) {  // three pairs per basic block (as the fast kernel)
            const int64_t nfull = (q_nopartner >= 0 ? q_nopartner : niter) - q;
            for (; t + 3 <= min(len, nfull); t += 3, q += 3, o += 3 * g.g1) {
                uint32_t x[3], y[3];
                step3(sa, x[0], x[1], x[2]);
                step3(sb, y[0], y[1], y[2]);
                T a[3], b[3];
                bmN<FAST, 3>(x, y, bv, a, b);
                put2(o, a[0], b[0]);
                put2(o + g.g1, a[1], b[1]);
                put2(o + 2 * g.g1, a[2], b[2]);
            }
        }
        for (; t < len; ++t, ++q, o += g.g1) {
            T a, b;
            const uint32_t z1 = step_m1(sa);
            const uint32_t z2 = step_m1(sb);
            bm<FAST>(z1, z2, bv, a, b);
            if (PAIRED && q != q_nopartner) {
                put2(o, a, b);
            } else {
                __stcs(o, a);
                if (q != q_nopartner) __stcs(o + 1, b);  // _kernels.py:151
            }
        }
    }
    if (d1 == total) {
        store_state(io, s0, sa);
        store_state(io, s0 + 1, sb);
    }
}

// normal, fast path: unit = (chunk, grid row i, group of PAIRS adjacent pairs)
//   PAIRS == 1: npad even; handles a partner past ncol on the last trip.
//   PAIRS == 2: g1 % 4 == 0, ncol % 4 == 0, npad % 4 == 0 -> both pairs of a
//               thread have the same trip count and always-valid partners; one
//               16-byte store (float32) per trip.
template <typename T, int PAIRS, int MINB, bool FAST>
__global__ void __launch_bounds__(256, MINB) fill_normal_fast(StateIO io,
                                                        T *__restrict__ out, Geom g,
                                                        int64_t i_lo, int64_t nrows_grid,
                                                        int64_t rows_per_chunk, int64_t nunits,
                                                        const __grid_constant__ Pow2Table tab) {
    __shared__ __align__(16) unsigned char bm_raw[kBmSmemBytes];
    const BmView bv = stage_bm_tables<FAST && sizeof(T) == 4>(bm_raw);
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= nunits) return;
    const int64_t groups = g.g1 / (2 * PAIRS);
    const int64_t jq = u % groups;
    const int64_t ic = u / groups;
    const int64_t i = i_lo + ic % nrows_grid, c = ic / nrows_grid;
    const int64_t j0 = 2 * PAIRS * jq;
    const int64_t nr = owned(g.nrow, i, g.g0);
    const int64_t rho0 = c * rows_per_chunk;
    if (rho0 >= nr) return;
    const int64_t rho1 = min(rho0 + rows_per_chunk, nr);
    const int64_t niter = owned(g.ncol, j0, g.g1);
    const int64_t s0 = i * g.g1 + j0;
    Mrg st[2 * PAIRS];
#pragma unroll
    for (int k = 0; k < 2 * PAIRS; ++k) {
        st[k] = load_state(io, s0 + k);
        if (rho0) skip(tab, st[k], (uint64_t)(rho0 * niter));
    }
    if (PAIRS == 2) {
        for (int64_t rho = rho0; rho < rho1; ++rho) {
            T *p = out + (i + g.g0 * rho) * g.npad + j0;
            int64_t q = 0;
            for (; q + 3 <= niter; q += 3) {  // step3: no shift-register moves
                uint32_t z[4][3];
#pragma unroll
                for (int k = 0; k < 4; ++k) step3(st[k], z[k][0], z[k][1], z[k][2]);
                T a[6], b[6];
                const uint32_t u1[6] = {z[0][0], z[2][0], z[0][1], z[2][1], z[0][2], z[2][2]};
                const uint32_t u2[6] = {z[1][0], z[3][0], z[1][1], z[3][1], z[1][2], z[3][2]};
                bmN<FAST, 6>(u1, u2, bv, a, b);
#pragma unroll
                for (int t = 0; t < 3; ++t)
                    put4(p + g.g1 * (q + t), a[2 * t], b[2 * t], a[2 * t + 1], b[2 * t + 1]);
            }
            for (; q < niter; ++q) {
                T a0, b0, a1, b1;
                const uint32_t z0 = step_m1(st[0]), z1 = step_m1(st[1]);
                const uint32_t z2 = step_m1(st[2]), z3 = step_m1(st[3]);
                bm<FAST>(z0, z1, bv, a0, b0);
                bm<FAST>(z2, z3, bv, a1, b1);
                put4(p + g.g1 * q, a0, b0, a1, b1);
            }
        }
    } else {
        // the last trip of a row may have its partner column past ncol
        const bool partner_last = j0 + 1 + g.g1 * (niter - 1) < g.ncol;
        const int64_t nfull = partner_last ? niter : niter - 1;
        for (int64_t rho = rho0; rho < rho1; ++rho) {
            T *p = out + (i + g.g0 * rho) * g.npad + j0;
            int64_t q = 0;
            for (; q + 3 <= nfull; q += 3) {
                uint32_t x[3], y[3];
                step3(st[0], x[0], x[1], x[2]);
                step3(st[1], y[0], y[1], y[2]);
                T a[3], b[3];
                bmN<FAST, 3>(x, y, bv, a, b);
                put2(p + g.g1 * q, a[0], b[0]);
                put2(p + g.g1 * (q + 1), a[1], b[1]);
                put2(p + g.g1 * (q + 2), a[2], b[2]);
            }
            for (; q < nfull; ++q) {
                T a, b;
                const uint32_t z1 = step_m1(st[0]), z2 = step_m1(st[1]);
                bm<FAST>(z1, z2, bv, a, b);
                put2(p + g.g1 * q, a, b);
            }
            if (nfull < niter) {
                T a, b;
                const uint32_t z1 = step_m1(st[0]), z2 = step_m1(st[1]);
                bm<FAST>(z1, z2, bv, a, b);
                __stcs(p + g.g1 * nfull, a);
            }
        }
    }
    if (rho1 == nr) {
#pragma unroll
        for (int k = 0; k < 2 * PAIRS; ++k) store_state(io, s0 + k, st[k]);
    }
}

// ---------------------------------------------------------------------------
// host-side launch planning

constexpr int kThreads = 256;
// measured on B200 (tools/tune.py normal): both output types are best at 3
// CTAs/SM with one pair per thread (variant 10); the spread over all
// variants is ~10 %
template <typename T>
constexpr int normal_variant_default() {
    return 10;
}
// enough units to fill 148 SMs several times over (2048 resident threads/SM)
constexpr int64_t kTargetUnits = 148LL * 2048 * 3;
constexpr int64_t kMinChunkDraws = 512;

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

static int launch_check(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SFB_E_CUDA, "%s launch: %s", what, cudaGetErrorString(e));
    return SFB_OK;
}

static int check_common(int64_t n_streams, int64_t nrow, int64_t ncol, int64_t npad, int64_t g0,
                        int64_t g1, int64_t item_lo, int64_t item_hi) {
    if (g0 < 1 || g1 < 1) return fail(SFB_E_INVALID_GRID, "work grid dimensions must be >= 1");
    if (nrow < 1 || ncol < 1) return fail(SFB_E_INVALID_ARGUMENT, "matrix dimensions must be >= 1");
    if (npad < ncol) return fail(SFB_E_INVALID_ARGUMENT, "npad must be >= ncol");
    if (n_streams < g0 * g1)
        return fail(SFB_E_INSUFFICIENT_STREAMS, "grid needs %lld streams, got %lld",
                    (long long)(g0 * g1), (long long)n_streams);
    if (item_lo < 0 || item_hi > g0 * g1 || item_lo > item_hi)
        return fail(SFB_E_INVALID_ARGUMENT, "item range [%lld, %lld) outside the grid",
                    (long long)item_lo, (long long)item_hi);
    return SFB_OK;
}

static int zero_padding(void *out, size_t elsize, int64_t nrow, int64_t ncol, int64_t npad,
                        cudaStream_t st) {
    if (npad == ncol) return SFB_OK;
    cudaError_t e = cudaMemset2DAsync((char *)out + ncol * elsize, npad * elsize, 0,
                                      (npad - ncol) * elsize, nrow, st);
    if (e != cudaSuccess) return fail(SFB_E_CUDA, "padding memset: %s", cudaGetErrorString(e));
    return SFB_OK;
}

// Chunked launches (several threads per stream): no thread writes a state --
// a stream's chunks all read its start state and nothing orders thread
// blocks -- and a second kernel then advances every stream of the launch by
// the number of draws it consumed (each owned cell is exactly one draw; a
// normal pair's two streams advance together, the discarded partner
// included): one skip through the A^(2^b) table per stream.
StateIO state_io(int64_t *cur, bool chunked) { return StateIO{cur, 0, chunked ? nullptr : cur}; }

template <bool NORMAL>
__global__ void __launch_bounds__(256) advance_fill_states(int64_t *cur, Geom g, int64_t lo,
                                                           int64_t hi,
                                                           const __grid_constant__ Pow2Table tab) {
    const int64_t w = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= hi) return;
    int64_t i, j;
    if (NORMAL) {  // stream w of pair w / 2: grid row i, lane pair starting at column j
        const int64_t p = w / 2, half = g.g1 / 2;
        i = p / half;
        j = 2 * (p % half);
    } else {  // work item w = i + g0 j
        i = w % g.g0;
        j = w / g.g0;
    }
    const int64_t draws = owned(g.nrow, i, g.g0) * owned(g.ncol, j, g.g1);
    if (draws == 0) return;
    Mrg s = load_state(cur + 6 * w);
    skip(tab, s, (uint64_t)draws);
    store_state(cur + 6 * w, s);
}

static int finish_states(bool normal, bool chunked, int64_t *cur, const Geom &g, int64_t lo,
                         int64_t hi, cudaStream_t st, const char *what) {
    if (int rc = launch_check(what)) return rc;
    if (!chunked || hi <= lo) return SFB_OK;
    Pow2Table tab;
    pow2_table(&tab);
    const unsigned nb = (unsigned)ceil_div(hi - lo, 256);
    if (normal)
        advance_fill_states<true><<<nb, 256, 0, st>>>(cur, g, lo, hi, tab);
    else
        advance_fill_states<false><<<nb, 256, 0, st>>>(cur, g, lo, hi, tab);
    return launch_check("advance_fill_states");
}

template <int KIND>
static int launch_uniform(int64_t *cur, void *out, const Geom &g, int64_t item_lo,
                          int64_t item_hi, double rate_d, cudaStream_t st) {
    Pow2Table tab;
    pow2_table(&tab);
    RateArg rate{rate_d, 1.0 / rate_d,
                 rate_d == 1.0 ? 2 : rate_d >= 0x1p-500 && rate_d <= 0x1p500 ? 1 : 0};
    const int64_t nloc = item_hi - item_lo;
    if (nloc == 0) return SFB_OK;
    const int64_t twog0 = 2 * g.g0;
    const bool fast = (g.g1 % 2 == 0) && (g.npad % 2 == 0) && (item_lo % twog0 == 0) &&
                      (item_hi % twog0 == 0) && g.nrow >= g.g0 && g.ncol >= g.g1;
    if (fast) {
        const int64_t j_lo = item_lo / g.g0;
        const int64_t npairs = (item_hi / g.g0 - j_lo) / 2;
        const int64_t rows = ceil_div(g.nrow, g.g0);  // max owned rows
        const int64_t base = g.g0 * npairs;
        const int64_t cols = ceil_div(g.ncol, g.g1);
        // variant knob (tuning only): low 4 bits = unit count in quarters of
        // kTargetUnits (0 -> 4/4), bits 4-7 = CTAs/SM register cap (0 ->
        // none), bits 8-11 = dynamic shared memory in 16 KB steps (occupancy
        // throttle)
        const int v = tune_knob("SFB_UNIFORM_VARIANT", 0);
        const int64_t target = kTargetUnits * ((v & 15) ? (v & 15) : 4) / 4;
        const size_t dsmem = (size_t)((v >> 8) & 15) * 16384;
        if (dsmem > 48 * 1024) {
            cudaFuncSetAttribute(fill_uniform_fast<KIND, 1>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem);
        }
        // chunks of at least max(1, kMinChunkDraws / cols) rows
        const int64_t min_rows = std::max<int64_t>(1, kMinChunkDraws / std::max<int64_t>(1, cols));
        int64_t nchunks = std::max<int64_t>(1, std::min(ceil_div(target, base),
                                                          ceil_div(rows, min_rows)));
        const int64_t rpc = ceil_div(rows, nchunks);
        nchunks = ceil_div(rows, rpc);
        const int64_t nunits = base * nchunks;
        const unsigned blocks = (unsigned)ceil_div(nunits, kThreads);
        const bool quad = !((v >> 14) & 1) && g.g1 % 4 == 0 && g.npad % 4 == 0 &&
                          (j_lo % 4) == 0 && (npairs % 2) == 0 &&
                          ((uintptr_t)out & 31) == 0;
        if (quad) {  // bit 14 set: the pair path instead
            const int64_t nquads = npairs / 2;
            const int64_t qbase = g.g0 * nquads;
            int64_t qchunks = std::max<int64_t>(1, std::min(ceil_div(target, qbase),
                                                             ceil_div(rows, min_rows)));
            const int64_t qrpc = ceil_div(rows, qchunks);
            qchunks = ceil_div(rows, qrpc);
            const int64_t qunits = qbase * qchunks;
            const unsigned qb = (unsigned)ceil_div(qunits, kThreads);
            const StateIO io = state_io(cur, qchunks > 1);
            // register cap / single-step variants (tuning); the exponential's
            // twelve log1p evaluations in flight want 3 CTAs/SM (measured 19.4 ->
            // 15.4 ms on C5), the store-bound kinds the uncapped default
            int sel = (v >> 4) & 15;
            if (sel == 0 && KIND == kExponential) sel = 3;
            switch (sel) {
                case 3:
                    fill_uniform_quad<KIND, 3><<<qb, kThreads, 0, st>>>(io, out, g, j_lo, nquads,
                                                                        qrpc, qunits, rate, tab);
                    break;
                case 4:
                    fill_uniform_quad<KIND, 4><<<qb, kThreads, 0, st>>>(io, out, g, j_lo, nquads,
                                                                        qrpc, qunits, rate, tab);
                    break;
                case 9:
                    fill_uniform_quad<KIND, 1, false><<<qb, kThreads, 0, st>>>(
                        io, out, g, j_lo, nquads, qrpc, qunits, rate, tab);
                    break;
                case 10:
                    fill_uniform_quad<KIND, 3, false><<<qb, kThreads, 0, st>>>(
                        io, out, g, j_lo, nquads, qrpc, qunits, rate, tab);
                    break;
                default:
                    fill_uniform_quad<KIND, 1><<<qb, kThreads, 0, st>>>(io, out, g, j_lo, nquads,
                                                                        qrpc, qunits, rate, tab);
            }
            return finish_states(false, qchunks > 1, cur, g, item_lo, item_hi, st,
                                 "fill_uniform_quad");
        }
        const StateIO io = state_io(cur, nchunks > 1);
        if ((v >> 12) & 3) {  // bits 12-13: 512 / 1024 threads per CTA
            const int nt = (v >> 12) == 1 ? 512 : 1024;
            const unsigned b2 = (unsigned)ceil_div(nunits, nt);
            if (nt == 512)
                fill_uniform_fast<KIND, 1, 512><<<b2, 512, 0, st>>>(io, out, g, j_lo, npairs, rpc,
                                                                   nunits, rate, tab);
            else
                fill_uniform_fast<KIND, 1, 1024><<<b2, 1024, 0, st>>>(io, out, g, j_lo, npairs,
                                                                     rpc, nunits, rate, tab);
            return finish_states(false, nchunks > 1, cur, g, item_lo, item_hi, st,
                                 "fill_uniform_fast");
        }
        switch ((v >> 4) & 15) {
            case 4:
                fill_uniform_fast<KIND, 4><<<blocks, kThreads, 0, st>>>(io, out, g, j_lo, npairs,
                                                                       rpc, nunits, rate, tab);
                break;
            case 6:
                fill_uniform_fast<KIND, 6><<<blocks, kThreads, 0, st>>>(io, out, g, j_lo, npairs,
                                                                       rpc, nunits, rate, tab);
                break;
            case 8:
                fill_uniform_fast<KIND, 8><<<blocks, kThreads, 0, st>>>(io, out, g, j_lo, npairs,
                                                                       rpc, nunits, rate, tab);
                break;
            default:
                fill_uniform_fast<KIND, 1><<<blocks, kThreads, dsmem, st>>>(io, out, g, j_lo,
                                                                           npairs, rpc, nunits,
                                                                           rate, tab);
        }
        return finish_states(false, nchunks > 1, cur, g, item_lo, item_hi, st,
                             "fill_uniform_fast");
    }
    // items with owned cells: rows i < min(g0, nrow), columns j < min(g1, ncol)
    GenMap m{};
    m.lo = item_lo;
    m.hi = item_hi;
    m.i_lo = 0;
    const int64_t ieff = std::min(g.g0, g.nrow);
    const int64_t jeff = std::min(g.g1, g.ncol);
    m.jlo = item_lo / g.g0;
    m.J = std::min(jeff, (item_hi - 1) / g.g0 + 1) - m.jlo;
    if (m.J <= 0) return SFB_OK;
    const int64_t maxdraws = ceil_div(g.nrow, g.g0) * ceil_div(g.ncol, g.g1);
    m.chunk = std::max<int64_t>(tune_knob("SFB_GENERIC_CHUNK", (int)kMinChunkDraws),
                                ceil_div(maxdraws * ieff * m.J, kTargetUnits));
    m.chunk = std::min(m.chunk, std::max<int64_t>(1, maxdraws));
    m.nchunks = ceil_div(maxdraws, m.chunk);
    m.nunits = ieff * m.J * m.nchunks;
    const StateIO io = state_io(cur, m.nchunks > 1);
    fill_uniform_generic<KIND><<<(unsigned)ceil_div(m.nunits, kThreads), kThreads, 0, st>>>(
        io, out, g, m, rate, tab);
    return finish_states(false, m.nchunks > 1, cur, g, item_lo, item_hi, st,
                         "fill_uniform_generic");
}

// variant knob (tuning only): bit 0 -> cap registers (4 CTAs/SM), bit 3 ->
// cap registers (3 CTAs/SM), bit 1 -> one pair per thread even when two fit,
// bit 2 -> float32 via the exact float64 transform instead of
// box_muller_pair_f32
template <typename T, int PAIRS, bool FAST>
static void launch_normal_fast_minb(int minb, unsigned blocks, cudaStream_t st, StateIO io,
                                    T *out, const Geom &g, int64_t i_lo, int64_t nrows_grid,
                                    int64_t rpc, int64_t nunits, const Pow2Table &tab) {
    if (minb >= 4)
        fill_normal_fast<T, PAIRS, 4, FAST><<<blocks, kThreads, 0, st>>>(io, out, g, i_lo,
                                                                         nrows_grid, rpc, nunits, tab);
    else if (minb == 3)
        fill_normal_fast<T, PAIRS, 3, FAST><<<blocks, kThreads, 0, st>>>(io, out, g, i_lo,
                                                                         nrows_grid, rpc, nunits, tab);
    else
        fill_normal_fast<T, PAIRS, 1, FAST><<<blocks, kThreads, 0, st>>>(io, out, g, i_lo,
                                                                         nrows_grid, rpc, nunits, tab);
}

template <typename T, bool FAST>
static void launch_normal_fast(bool two, int minb, cudaStream_t st, StateIO io, T *out,
                               const Geom &g, int64_t i_lo, int64_t nrows_grid, int64_t rpc,
                               int64_t nunits) {
    Pow2Table tab;
    pow2_table(&tab);
    const unsigned blocks = (unsigned)ceil_div(nunits, kThreads);
    if (two)
        launch_normal_fast_minb<T, 2, FAST>(minb, blocks, st, io, out, g, i_lo, nrows_grid, rpc,
                                            nunits, tab);
    else
        launch_normal_fast_minb<T, 1, FAST>(minb, blocks, st, io, out, g, i_lo, nrows_grid, rpc,
                                            nunits, tab);
}

template <typename T>
static int launch_normal(int64_t *cur, T *out, const Geom &g, int64_t item_lo, int64_t item_hi,
                         cudaStream_t st) {
    Pow2Table tab;
    pow2_table(&tab);
    const int64_t pair_lo = item_lo / 2, pair_hi = item_hi / 2;
    const int64_t nloc = pair_hi - pair_lo;
    if (nloc == 0) return SFB_OK;
    const int64_t half = g.g1 / 2;
    const bool fast = (g.npad % 2 == 0) && (pair_lo % half == 0) && (pair_hi % half == 0) &&
                      g.nrow >= g.g0 && g.ncol >= g.g1;
    if (fast) {
        const int64_t i_lo = pair_lo / half;
        const int64_t nrows_grid = (pair_hi - pair_lo) / half;
        const bool two = g.g1 % 4 == 0 && g.ncol % 4 == 0 && g.npad % 4 == 0;
        const int64_t rows = ceil_div(g.nrow, g.g0);
        const int64_t base = nrows_grid * half / (two ? 2 : 1);
        const int64_t cols = ceil_div(g.ncol, g.g1);
        const int64_t min_rows = std::max<int64_t>(1, kMinChunkDraws / std::max<int64_t>(1, cols));
        int64_t nchunks = std::max<int64_t>(1, std::min(ceil_div(kTargetUnits, base),
                                                          ceil_div(rows, min_rows)));
        const int64_t rpc = ceil_div(rows, nchunks);
        nchunks = ceil_div(rows, rpc);
        const int64_t nunits = base * nchunks;
        const int v = tune_knob("SFB_NORMAL_VARIANT", normal_variant_default<T>());
        const bool use_two = two && !(v & 2);
        // one pair per thread where two would fit: twice the units
        const int64_t nu = (two && !use_two) ? nunits * 2 : nunits;
        const int minb = (v & 1) ? 4 : (v & 8) ? 3 : 1;
        const StateIO io = state_io(cur, nchunks > 1);
        if (v & 4)
            launch_normal_fast<T, false>(use_two, minb, st, io, out, g, i_lo, nrows_grid, rpc, nu);
        else
            launch_normal_fast<T, true>(use_two, minb, st, io, out, g, i_lo, nrows_grid, rpc, nu);
        return finish_states(true, nchunks > 1, cur, g, item_lo, item_hi, st,
                             "fill_normal_fast");
    }
    // pairs with owned cells: grid rows of the shard below min(g0, nrow),
    // pair columns jp with 2 jp < ncol
    GenMap m{};
    m.lo = pair_lo;
    m.hi = pair_hi;
    m.i_lo = pair_lo / half;
    const int64_t i_end = std::min((pair_hi - 1) / half + 1, std::min(g.g0, g.nrow));
    if (i_end <= m.i_lo) return SFB_OK;
    const int64_t jpeff = std::min(half, ceil_div(g.ncol, 2));
    if (i_end - m.i_lo == 1) {  // a shard inside one grid row
        m.jlo = pair_lo - m.i_lo * half;
        m.J = std::min(jpeff, pair_hi - m.i_lo * half) - m.jlo;
    } else {
        m.jlo = 0;
        m.J = jpeff;
    }
    if (m.J <= 0) return SFB_OK;
    const int64_t maxdraws = ceil_div(g.nrow, g.g0) * ceil_div(g.ncol, g.g1);
    m.chunk = std::max<int64_t>(tune_knob("SFB_GENERIC_CHUNK", (int)kMinChunkDraws),
                                ceil_div(maxdraws * (i_end - m.i_lo) * m.J, kTargetUnits));
    m.chunk = std::min(m.chunk, std::max<int64_t>(1, maxdraws));
    m.nchunks = ceil_div(maxdraws, m.chunk);
    m.nunits = (i_end - m.i_lo) * m.J * m.nchunks;
    const bool paired = g.npad % 2 == 0 && ((uintptr_t)out % (2 * sizeof(T))) == 0;
    const unsigned nb = (unsigned)ceil_div(m.nunits, kThreads);
    const StateIO io = state_io(cur, m.nchunks > 1);
    const bool exact = tune_knob("SFB_NORMAL_VARIANT", normal_variant_default<T>()) & 4;
    if (exact)
        paired ? fill_normal_generic<T, false, true><<<nb, kThreads, 0, st>>>(io, out, g, m, tab)
               : fill_normal_generic<T, false, false><<<nb, kThreads, 0, st>>>(io, out, g, m, tab);
    else
        paired ? fill_normal_generic<T, true, true><<<nb, kThreads, 0, st>>>(io, out, g, m, tab)
               : fill_normal_generic<T, true, false><<<nb, kThreads, 0, st>>>(io, out, g, m, tab);
    return finish_states(true, m.nchunks > 1, cur, g, item_lo, item_hi, st,
                         "fill_normal_generic");
}

}  // namespace sfb

using namespace sfb;

extern "C" {

int sfb_device_ok(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) {
        cudaGetLastError();
        return 0;
    }
    int dev = 0, major = 0, minor = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    return major == 10 && minor == 0;
}

int sfb_host_register(void *p, int64_t bytes) {
    if (!p || bytes <= 0) return fail(SFB_E_INVALID_ARGUMENT, "nothing to register");
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost)
        return 1;  // already page-locked (another registration or a pinned allocation)
    cudaGetLastError();
    cudaError_t e = cudaHostRegister(p, (size_t)bytes, cudaHostRegisterDefault);
    if (e != cudaSuccess) {
        cudaGetLastError();  // leave no sticky error behind: registration is optional
        return fail(SFB_E_CUDA, "cudaHostRegister: %s", cudaGetErrorString(e));
    }
    return SFB_OK;
}

int sfb_host_unregister(void *p) {
    cudaError_t e = cudaHostUnregister(p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(SFB_E_CUDA, "cudaHostUnregister: %s", cudaGetErrorString(e));
    }
    return SFB_OK;
}

int sfb_fill_real(int64_t *d_cur, int64_t n_streams, double *d_out, int64_t nrow, int64_t ncol,
                  int64_t npad, int64_t g0, int64_t g1, int mode, double rate, int64_t item_lo,
                  int64_t item_hi, int zero_pad, void *stream) {
    if (int rc = check_common(n_streams, nrow, ncol, npad, g0, g1, item_lo, item_hi)) return rc;
    if (mode != 0 && mode != 1) return fail(SFB_E_INVALID_ARGUMENT, "unknown fill mode %d", mode);
    if (mode == 1 && !(rate > 0)) return fail(SFB_E_INVALID_RATE, "exponential rate must be > 0");
    cudaStream_t st = (cudaStream_t)stream;
    if (zero_pad)
        if (int rc = zero_padding(d_out, sizeof(double), nrow, ncol, npad, st)) return rc;
    const Geom g{nrow, ncol, npad, g0, g1};
    return mode == 0 ? launch_uniform<kUniform>(d_cur, d_out, g, item_lo, item_hi, rate, st)
                     : launch_uniform<kExponential>(d_cur, d_out, g, item_lo, item_hi, rate, st);
}

int sfb_fill_integer(int64_t *d_cur, int64_t n_streams, int64_t *d_out, int64_t nrow,
                     int64_t ncol, int64_t npad, int64_t g0, int64_t g1, int64_t item_lo,
                     int64_t item_hi, int zero_pad, void *stream) {
    if (int rc = check_common(n_streams, nrow, ncol, npad, g0, g1, item_lo, item_hi)) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    if (zero_pad)
        if (int rc = zero_padding(d_out, sizeof(int64_t), nrow, ncol, npad, st)) return rc;
    const Geom g{nrow, ncol, npad, g0, g1};
    return launch_uniform<kInteger>(d_cur, d_out, g, item_lo, item_hi, 1.0, st);
}

int sfb_fill_normal(int64_t *d_cur, int64_t n_streams, void *d_out, int out_dtype, int64_t nrow,
                    int64_t ncol, int64_t npad, int64_t g0, int64_t g1, int64_t item_lo,
                    int64_t item_hi, int zero_pad, void *stream) {
    if (int rc = check_common(n_streams, nrow, ncol, npad, g0, g1, item_lo, item_hi)) return rc;
    if (g1 % 2 != 0)
        return fail(SFB_E_INVALID_GRID, "normal generation needs an even lane count (nglobal1)");
    if (item_lo % 2 != 0 || item_hi % 2 != 0)
        return fail(SFB_E_INVALID_ARGUMENT, "normal shard range must be pair aligned");
    if (out_dtype != SFB_F64 && out_dtype != SFB_F32)
        return fail(SFB_E_INVALID_ARGUMENT, "normal output dtype must be f64 or f32");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t es = out_dtype == SFB_F64 ? sizeof(double) : sizeof(float);
    if (zero_pad)
        if (int rc = zero_padding(d_out, es, nrow, ncol, npad, st)) return rc;
    const Geom g{nrow, ncol, npad, g0, g1};
    if (out_dtype == SFB_F64)
        return launch_normal<double>(d_cur, (double *)d_out, g, item_lo, item_hi, st);
    return launch_normal<float>(d_cur, (float *)d_out, g, item_lo, item_hi, st);
}

int sfb_download_shard(void *dst_host, const void *src_dev, int64_t nrow, int64_t ncol,
                       int64_t npad, int64_t g1, int64_t j_lo, int64_t j_hi, int64_t elsize,
                       void *stream) {
    if (nrow < 1 || ncol < 1 || npad < ncol || g1 < 1 || elsize < 1)
        return fail(SFB_E_INVALID_ARGUMENT, "bad shard geometry");
    if (j_lo < 0 || j_hi > g1 || j_lo > j_hi)
        return fail(SFB_E_INVALID_ARGUMENT, "column range [%lld, %lld) outside [0, %lld)",
                    (long long)j_lo, (long long)j_hi, (long long)g1);
    const int64_t w = j_hi - j_lo;
    if (w == 0) return SFB_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t es = (size_t)elsize;
    cudaError_t e = cudaSuccess;
    if (npad == ncol && ncol % g1 == 0) {
        // every run is w elements at pitch g1 across the whole matrix: one 2-D copy
        const int64_t runs = nrow * (ncol / g1);
        e = cudaMemcpy2DAsync(dst_host, w * es, (const char *)src_dev + j_lo * es, g1 * es,
                              w * es, (size_t)runs, cudaMemcpyDeviceToHost, st);
    } else {
        // row by row: runs c = j + g1 q, the last one possibly ragged
        char *dst = (char *)dst_host;
        for (int64_t r = 0; r < nrow && e == cudaSuccess; ++r) {
            const char *row = (const char *)src_dev + (size_t)(r * npad) * es;
            const int64_t full = ncol / g1, rem = ncol - full * g1;
            if (full) {
                e = cudaMemcpy2DAsync(dst, w * es, row + j_lo * es, g1 * es, w * es, (size_t)full,
                                      cudaMemcpyDeviceToHost, st);
                dst += (size_t)(full * w) * es;
            }
            const int64_t tail = std::min(j_hi, rem) - j_lo;
            if (e == cudaSuccess && tail > 0) {
                e = cudaMemcpyAsync(dst, row + (full * g1 + j_lo) * es, (size_t)tail * es,
                                    cudaMemcpyDeviceToHost, st);
                dst += (size_t)tail * es;
            }
        }
    }
    if (e != cudaSuccess) return fail(SFB_E_CUDA, "shard download: %s", cudaGetErrorString(e));
    return SFB_OK;
}

}  // extern "C"
