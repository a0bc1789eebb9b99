// box_muller.cuh -- the paired-lane Box-Muller transform of the reference,
// rebuilt for the FP64 pipe of sm_100a (host + device, bit-identical).
//
// Reference (_kernels.py:145-152), per pair of draws z1 (lane 0), z2 (lane 1):
//   u1 = z1*NORM;  theta = (2*pi*NORM)*z2;  R = sqrt(-2*log(u1))
//   a = R*cos(theta);  b = R*cos(theta - pi/2)          (glibc log/cos/sqrt)
//
// Generic log/cos cost ~100 FP64 instructions per pair.  Both arguments are
// 31-bit integers scaled by 2^-31, which allows short table-driven forms:
//   * log: u1 = 2^k m, m in [0.5, 1) read from the bits of (double)z1;
//     512-bucket table with 1/c and -ln(c) (hi + lo); r = fma(m, 1/c, -1),
//     |r| <= 2^-10, ln(1+r) by a degree-5 Taylor polynomial.  k <= 0 and
//     ln m < 0, so nothing cancels; the last bucket has c = 1, so u1 -> 1
//     keeps full relative accuracy.
//   * trig: theta = fl(c z2) exactly as the reference rounds it (c = TWOPI
//     2^-31 is an exact power-of-two scaling of the double 2*pi).  With
//     k = round(z2 / 2^21), A_k = fl(k TWOPI/1024) is a table double with
//     cos/sin(A_k) tabulated; B = theta - A_k is EXACT (Sterbenz), |B| <=
//     pi/1024, so cos/sin(theta) = cos/sin(A_k + B) need only sin B to B^5 and
//     cos B - 1 to B^4.  No Cody-Waite reduction, and theta exactly on a
//     table point (e.g. fl(pi/2)) reproduces glibc's cos(fl(pi/2)) exactly.
//   * lane b without a second evaluation: thb = fl(theta - H), H = pi/2
//     rounded; cos(thb) = sin(theta + d) = sin(theta) + d cos(theta) (d^2
//     terms < 1e-31) where d = (thb - (theta - H)) + (pi/2 - H) is computed
//     exactly (rounding_error_minus_halfpi()).
// All polynomial coefficients live in __constant__ memory (direct c[] operands
// of DFMA; literal doubles would cost two UMOVs each per use).
// No expression here may be contracted by the compiler: the TU is built with
// -fmad=false (device) / -ffp-contract=off (host) and every fma is explicit.
// Accuracy is verified on the host against glibc (tests/test_host_lib.py::
// test_box_muller_port_against_libm): <= 3 ulp_f64, and float32(port) ==
// float32(reference) on every tested pair.
#pragma once
#include <math.h>
#include <stdint.h>

#include "bm_tables.inc"
#include "exp_glibc.cuh"  // as_f64 / as_u64 / fma_rn

namespace sfb {

enum BmCoef {
    kC_Ln2Hi, kC_Ln2Lo, kC_L5, kC_L4, kC_L3, kC_L2,  // ln(1+r) coefficients 1/5, -1/4, 1/3, -1/2
    kC_S5, kC_S3, kC_C4, kC_C2,                      // sin B, cos B - 1
    kC_TwoPiNorm, kC_HalfPi, kC_PiO2Lo, kC_Neg2, kC_Ln2, kC_Half, kC_3o8, kC_Neg2Ln2,
    kC_TwoPiNormBias, kC_M2L5, kC_M2L4, kC_M2L3, kC_One, kC_Count
};

#define SFB_BM_COEF_INIT                                                                 \
    {                                                                                    \
        6.93147180369123816490e-01, /* ln2 hi: 33 bits, k*ln2_hi exact */               \
            1.90821492927058770002e-10,  /* ln2 - ln2_hi */                              \
            1.0 / 5.0, -1.0 / 4.0, 1.0 / 3.0, -1.0 / 2.0, 1.0 / 120.0, -1.0 / 6.0,        \
            1.0 / 24.0, -1.0 / 2.0, (2.0 * 3.141592653589793) / 2147483648.0,            \
            0.5 * 3.141592653589793, /* HALFPI, _kernels.py:22 */                         \
            6.123233995736766e-17,   /* pi/2 - HALFPI */                                  \
            -2.0, 6.93147180559945286227e-01, /* ln 2 rounded */ 0.5,                    \
            0.375, -1.38629436111989057245, /* -2 ln 2 rounded */                          \
            (2.0 * 3.141592653589793) * -2097152.0, /* -2^52 TWOPI 2^-31 (exact) */      \
            -2.0 / 5.0, 2.0 / 4.0, -2.0 / 3.0, 1.0                                         \
    }

#ifdef __CUDACC__
static __constant__ double c_bm_coef[kC_Count] = SFB_BM_COEF_INIT;
#endif
static const double h_bm_coef[kC_Count] = SFB_BM_COEF_INIT;

#ifdef __CUDA_ARCH__
#define SFB_BMC(i) c_bm_coef[i]
#else
#define SFB_BMC(i) h_bm_coef[i]
#endif

SFB_EXP_HD double sel(bool p, double a, double b) { return p ? a : b; }

// ln(z * 2^-31) for integer z in [1, 2^31 - 1]; tab = SFB_BM_LOG_TABLE_INIT words
SFB_EXP_HD double log_u31(uint32_t z, const uint64_t *tab) {
    const double d = (double)z;  // exact
    const uint64_t bits = as_u64(d);
    const int k = (int)(bits >> 52) - 1053;  // z in [2^e, 2^(e+1)), k = e - 30 <= 0
    const double m = as_f64((bits & 0x000fffffffffffffull) | 0x3fe0000000000000ull);
    const uint32_t i = (uint32_t)(bits >> 43) & (SFB_BM_LOG_N - 1);
    const double invc = as_f64(tab[3 * i]);
    const double lhi = as_f64(tab[3 * i + 1]);
    const double llo = as_f64(tab[3 * i + 2]);
    const double r = fma_rn(m, invc, -1.0);
    const double kd = (double)k;
    // ln(1+r) = r + r^2 (-1/2 + r (1/3 + r (-1/4 + r/5)))   (|r| <= 2^-10)
    double p = fma_rn(r, SFB_BMC(kC_L5), SFB_BMC(kC_L4));
    p = fma_rn(r, p, SFB_BMC(kC_L3));
    p = fma_rn(r, p, SFB_BMC(kC_L2));
    const double r2 = r * r;
    // hi + err == k ln2_hi + logc_hi exactly (k ln2_hi exact; Fast2Sum since
    // |k ln2_hi| >= |logc_hi| whenever k != 0)
    const double t = kd * SFB_BMC(kC_Ln2Hi);
    const double hi = t + lhi;
    const double err = (t - hi) + lhi;
    const double lo = fma_rn(kd, SFB_BMC(kC_Ln2Lo), llo) + err;
    return hi + (r + fma_rn(r2, p, lo));
}

// d = fl(theta - H) - (theta - H), exactly (theta in (0, 2 pi], thb = fl(theta - H)):
//   theta <  H: thb + H is exact (Sterbenz) and so is (thb + H) - theta;
//   theta >= H: thb - theta is exact (theta <= 2 thb, or thb exact) and so is + H.
SFB_EXP_HD double rounding_error_minus_halfpi(double theta, double thb) {
    const double H = SFB_BMC(kC_HalfPi);
    const bool small = theta < H;
    const double a = sel(small, H, -theta);
    const double b = sel(small, -theta, H);
    return (thb + a) + b;
}

// sqrt of a positive normal double without the special-case branch of the
// library sqrt (which splits the unrolled pair loop into separate basic
// blocks): rsqrt.approx seed (MUFU.RSQ64H, <= 2^-20), one Newton step on
// 1/sqrt(x) and one residual-corrected step on sqrt(x) -- within an ulp of the
// correctly rounded root.  The host uses libm sqrt.
SFB_EXP_HD double sqrt_pos(double x) {
#ifdef __CUDA_ARCH__
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double hx = 0.5 * x;
    y = fma_rn(fma_rn(-hx, y * y, 0.5), y, y);  // y (1.5 - x y^2 / 2)
    const double s = x * y;
    return fma_rn(fma_rn(-s, s, x), 0.5 * y, s);
#else
    return sqrt(x);
#endif
}

// the pair transform; z1m1 = z1 - 1, z2m1 = z2 - 1 (see step_m1)
SFB_EXP_HD void box_muller_pair(uint32_t z1m1, uint32_t z2m1, const uint64_t *logtab,
                                const uint64_t *trigtab, double &a, double &b) {
    const double ln_u1 = log_u31(z1m1 + 1u, logtab);
    const double radius = sqrt_pos(SFB_BMC(kC_Neg2) * ln_u1);
    // theta = fl((2 pi NORM) * z2) == fma(c, z2 - 1, c): exact product + c, one rounding
    const double c = SFB_BMC(kC_TwoPiNorm);
    const double theta = fma_rn(c, (double)z2m1, c);
    const uint32_t k = (z2m1 + 1u + (1u << 20)) >> 21;  // nearest table angle, 0..1024
    const double ak = as_f64(trigtab[3 * k]);
    const double ca = as_f64(trigtab[3 * k + 1]);
    const double sa = as_f64(trigtab[3 * k + 2]);
    const double B = theta - ak;  // exact
    const double B2 = B * B;
    const double sb = fma_rn(B * B2, fma_rn(B2, SFB_BMC(kC_S5), SFB_BMC(kC_S3)), B);
    const double cm1 = B2 * fma_rn(B2, SFB_BMC(kC_C4), SFB_BMC(kC_C2));  // cos B - 1
    // cos(A+B) = cA + (cA (cB-1) - sA sB);  sin(A+B) = sA + (sA (cB-1) + cA sB)
    const double cos_t = ca + fma_rn(ca, cm1, -(sa * sb));
    const double sin_t = sa + fma_rn(sa, cm1, ca * sb);
    const double thb = theta - SFB_BMC(kC_HalfPi);  // the reference's argument of lane b
    const double d = rounding_error_minus_halfpi(theta, thb) + SFB_BMC(kC_PiO2Lo);
    a = radius * cos_t;
    b = radius * fma_rn(d, cos_t, sin_t);
}

// ---------------------------------------------------------------------------
// Float32-output form (rnormGpu with float32 output -- an extension; the
// reference is float64-only, and float32(reference) is the target).  Each
// output is rounded to float32 once, so the transform needs a relative error
// far below 2^-24, not the ~2^-52 of box_muller_pair: this form targets
// <= 2^-44, so a result can differ from float32(reference) only when the
// reference lies within ~2^-44 of a float32 rounding boundary (expected rate
// ~1e-6 of cells, by 1 ulp_f32).  FP64 work drops from ~45 to ~23 ops/pair:
//   * log: x = -2 ln u1 directly: the table holds (1/c, -2 ln c) (one
//     16-byte load), -2 k ln2 + (-2 ln c) in one fma, and -2 ln(1+r) as
//     -2r + r^2 q(r) with the degree-5 coefficients pre-scaled by -2 (the
//     scaling commutes with every rounding), so no separate -2 multiply;
//     |r| <= 2^-10 and ln u1 ~ r near u1 = 1, where r^5/5 is 2^-42 relative;
//   * sqrt: rsqrt.approx seed y0 (MUFU.RSQ64H, measured <= 2^-20.06 relative
//     on B200), e = 1 - x y0^2, R = x y0 (1 + e/2 + 3e^2/8): 6 FP64 ops,
//     truncation 5e^3/16 < 2^-58;
//   * theta: fma(2^52 + z2, c, -2^52 c) = fl(c z2) from the integer bits
//     (no I2F on the XU pipe);
//   * trig: sin B to B^3 (B^5/120 < 2.3e-15 absolute), cos B - 1 to B^4,
//     fused fma recombination; (cos A, sin A) as one 16-byte load;
//   * lane b = R sin(theta): the reference's cos(fl(theta - fl(pi/2))) differs
//     by d cos(theta), |d| <= 2^-53 pi, which is below the float32 resolution
//     except where sin(theta) itself is tiny: z2 within kBmExactWin of a
//     multiple of 2^30 (theta near 0, pi, 2 pi).  Those pairs (~1e-5 of all)
//     take the full-accuracy box_muller_pair (tables in global memory).
//   Near the zeros of cos and sin elsewhere the table points A_k sit exactly
//   on the reference's fl(k pi/2), so cos_t / sin_t stay relatively accurate.
struct alignas(16) BmPair {
    double x, y;
};
constexpr int kBmFastLogPairs = SFB_BM_LOG_N;         // (1/c, -2 ln c)
constexpr int kBmFastTrigPairs = SFB_BM_TRIG_N + 1;   // (cos A, sin A)

// fill the fast-path tables from the table words of bm_tables.inc
constexpr double kBmF32LogScale = -2.0;  // logp[i].y = -2 ln c (box_muller_pair_f32_core)
SFB_EXP_HD void bm_fast_tables(const uint64_t *logw, const uint64_t *trigw, int t, int nt,
                               BmPair *logp, BmPair *trigp, double *angle,
                               double yscale = kBmF32LogScale) {
    for (int i = t; i < kBmFastLogPairs; i += nt)
        logp[i] = BmPair{as_f64(logw[3 * i]),
                         (as_f64(logw[3 * i + 1]) + as_f64(logw[3 * i + 2])) * yscale};
    for (int i = t; i < kBmFastTrigPairs; i += nt) {
        trigp[i] = BmPair{as_f64(trigw[3 * i + 1]), as_f64(trigw[3 * i + 2])};
        angle[i] = as_f64(trigw[3 * i]);
    }
}

// 1/sqrt(x) seeds: the hardware approximation (MUFU.RSQ64H) on the device;
// on the host a model with a chosen relative error (CPU tests use the bound
// measured on the B200, tests/test_gpu_parity.py::test_rsqrt_seed_accuracy)
struct RsqrtSeedHw {
    SFB_EXP_HD double operator()(double x) const {
#ifdef __CUDA_ARCH__
        double y;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
        return y;
#else
        return 1.0 / sqrt(x);
#endif
    }
};
struct RsqrtSeedModel {
    double rel_err;  // the seed is RN(1/sqrt(x)) * (1 + rel_err)
    SFB_EXP_HD double operator()(double x) const { return (1.0 / sqrt(x)) * (1.0 + rel_err); }
};

constexpr uint32_t kBmExactWin = 1u << 12;

#ifdef __CUDACC__
#define SFB_BM_COLD static __host__ __device__ __noinline__
#else
#define SFB_BM_COLD inline
#endif
// the rare exact path, kept out of line so the hot loop stays compact
struct F32Pair {
    float a, b;
};
SFB_BM_COLD F32Pair box_muller_pair_f32_exact(uint32_t z1m1, uint32_t z2m1,
                                              const uint64_t *logw, const uint64_t *trigw) {
    double da, db;
    box_muller_pair(z1m1, z2m1, logw, trigw, da, db);
    return F32Pair{(float)da, (float)db};
}

// z2 within kBmExactWin of a multiple of 2^30 (theta near 0, pi, 2 pi): the
// pair must take the exact form
SFB_EXP_HD bool bm_f32_needs_exact(uint32_t z2m1) {
    return ((z2m1 + 1u + kBmExactWin) & ((1u << 30) - 1u)) < 2u * kBmExactWin;
}

// the fast form without the exact fallback (callers test bm_f32_needs_exact;
// keeping the rare branch out of this function lets the compiler interleave
// several pairs in one basic block).  logp[i] = (1/c, -2 ln c) as staged by
// bm_fast_tables(..., kBmF32LogScale).
template <typename SEED = RsqrtSeedHw>
SFB_EXP_HD void box_muller_pair_f32_core(uint32_t z1m1, uint32_t z2m1, const BmPair *logp,
                                         const BmPair *trigp, const double *angle, float &a,
                                         float &b, const SEED &seed = SEED()) {
    const double d = (double)(z1m1 + 1u);  // exact
    const uint64_t bits = as_u64(d);
    const int k = (int)(bits >> 52) - 1053;
    const double m = as_f64((bits & 0x000fffffffffffffull) | 0x3fe0000000000000ull);
    const BmPair lc = logp[(uint32_t)(bits >> 43) & (SFB_BM_LOG_N - 1)];
    const double r = fma_rn(m, lc.x, -1.0);
    // x = -2 ln u1 = (-2 k ln2 - 2 ln c) - 2r + r^2 (1 + r (-2/3 + r (1/2 - 2r/5))):
    // -2 ln(1+r) with the -2 folded into the table and the coefficients
    double p = fma_rn(r, SFB_BMC(kC_M2L5), SFB_BMC(kC_M2L4));
    p = fma_rn(r, p, SFB_BMC(kC_M2L3));
    p = fma_rn(r, p, SFB_BMC(kC_One));
    const double r2 = r * r;
    const double y2 = fma_rn((double)k, SFB_BMC(kC_Neg2Ln2), lc.y);
    const double x = fma_rn(r2, p, fma_rn(r, SFB_BMC(kC_Neg2), y2));
    // R = sqrt(x) = x y0 (1 - e)^-1/2 with e = 1 - x y0^2, |e| <= 2^-19 for the
    // rsqrt.approx seed y0: x y0 (1 + e/2 + 3e^2/8), truncation 5e^3/16 < 2^-58
    const double y0 = seed(x);
    const double e = fma_rn(-x, y0 * y0, 1.0);
    const double s0 = x * y0;
    const double R = fma_rn(s0 * e, fma_rn(e, SFB_BMC(kC_3o8), SFB_BMC(kC_Half)), s0);
    // theta = fl((2 pi NORM) z2) exactly as the reference rounds it:
    // fma(2^52 + z2, c, -2^52 c) is c z2 rounded once (no XU conversion)
    const double theta = fma_rn(as_f64(0x4330000000000000ull | (z2m1 + 1u)),
                                SFB_BMC(kC_TwoPiNorm), SFB_BMC(kC_TwoPiNormBias));
    const uint32_t kk = (z2m1 + 1u + (1u << 20)) >> 21;
    const BmPair cs = trigp[kk];
    const double B = theta - angle[kk];  // exact
    const double B2 = B * B;
    const double sb = fma_rn(B * B2, SFB_BMC(kC_S3), B);
    const double cm1 = B2 * fma_rn(B2, SFB_BMC(kC_C4), SFB_BMC(kC_C2));
    const double cos_t = fma_rn(cs.x, cm1, fma_rn(-cs.y, sb, cs.x));
    const double sin_t = fma_rn(cs.y, cm1, fma_rn(cs.x, sb, cs.y));
    a = (float)(R * cos_t);
    b = (float)(R * sin_t);
}

template <typename SEED = RsqrtSeedHw>
SFB_EXP_HD void box_muller_pair_f32(uint32_t z1m1, uint32_t z2m1, const BmPair *logp,
                                    const BmPair *trigp, const double *angle,
                                    const uint64_t *logw, const uint64_t *trigw, float &a,
                                    float &b, const SEED &seed = SEED()) {
    if (bm_f32_needs_exact(z2m1)) {
        const F32Pair p = box_muller_pair_f32_exact(z1m1, z2m1, logw, trigw);  // theta ~ 0, pi, 2pi
        a = p.a;
        b = p.b;
        return;
    }
    box_muller_pair_f32_core<SEED>(z1m1, z2m1, logp, trigp, angle, a, b, seed);
}

}  // namespace sfb
