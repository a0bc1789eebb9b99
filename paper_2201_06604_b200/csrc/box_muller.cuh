// box_muller.cuh -- the paired-lane Box-Muller transform of the reference,
// rebuilt for the FP64 pipe of sm_100a (host + device, bit-identical).
//
// Reference (_kernels.py:145-152), per pair of draws z1 (lane 0), z2 (lane 1):
//   u1 = z1*NORM;  theta = (2*pi*NORM)*z2;  R = sqrt(-2*log(u1))
//   a = R*cos(theta);  b = R*cos(theta - pi/2)          (glibc log/cos/sqrt)
//
// Generic libm-style log/cos cost ~100 FP64 instructions per pair on the GPU.
// Here the arguments are known to be 31-bit integers scaled by 2^-31, which
// allows a much shorter evaluation with the same accuracy class (~1 ulp):
//   * log: u1 = 2^k m, m in [0.5, 1) read straight from the exponent/fraction
//     bits of (double)z1; 128-bucket table (bm_tables.inc) with 1/c and
//     -ln(c) as hi+lo; r = fma(m, 1/c, -1), |r| <= 2^-8; ln(1+r) by a degree-6
//     Taylor polynomial.  k <= 0 and ln m < 0, so nothing cancels, and the
//     last bucket has c = 1 exactly, so u1 -> 1 keeps full relative accuracy.
//   * one Cody-Waite reduction of theta (2-part pi/2 with fma), fdlibm
//     __kernel_sin/__kernel_cos minimax polynomials, quadrant by q = rint(2 theta/pi).
//   * lane b without a second reduction: with thb = fl(theta - H), H = pi/2
//     rounded, cos(thb) = sin(theta + d) = sin(theta) + d cos(theta) (d^2 terms
//     < 1e-31) where d = (thb - (theta - H)) + (pi/2 - H) is computed exactly
//     (Sterbenz-exact differences, see rounding_error_minus_halfpi()).
//   * theta itself is rounded exactly like the reference: fl(c*z2) with
//     c = 2 pi 2^-31 (an exact power-of-two scaling of the double 2*pi).
// No expression here may be contracted by the compiler: the TU is built with
// -fmad=false and every fma is explicit.
// Accuracy is verified on the host against glibc (tests/test_host_lib.py:
// test_box_muller_port_against_libm): |err| <= 2 ulp_f64 typical, and the
// float32 rounding equals float32(reference) on >= 99.999 % of pairs.
#pragma once
#include <math.h>
#include <stdint.h>

#include "bm_tables.inc"
#include "exp_glibc.cuh"  // as_f64 / as_u64 / fma_rn

namespace sfb {

constexpr double kBmNorm = 1.0 / 2147483648.0;
constexpr double kTwoPiNorm = (2.0 * 3.141592653589793) / 2147483648.0;  // exact scaling
constexpr double kHalfPi = 0.5 * 3.141592653589793;                      // _kernels.py:22
constexpr double kPiO2Lo = 6.123233995736766e-17;  // pi/2 - kHalfPi
constexpr double kTwoOverPi = 0.6366197723675814;
constexpr double kPiO2_1 = 1.57079632673412561417e+00;   // first 33 bits of pi/2
constexpr double kPiO2_1t = 6.07710050650619224932e-11;  // pi/2 - kPiO2_1
constexpr double kLn2Hi = 6.93147180369123816490e-01;  // 33 bits: k*kLn2Hi exact
constexpr double kLn2Lo = 1.90821492927058770002e-10;

SFB_EXP_HD double sel(bool p, double a, double b) { return p ? a : b; }

// ln(z * 2^-31) for integer z in [1, 2^31 - 1]; tab = SFB_BM_LOG_TABLE_INIT words
SFB_EXP_HD double log_u31(uint32_t z, const uint64_t *tab) {
    const double d = (double)z;  // exact
    const uint64_t bits = as_u64(d);
    const int e = (int)(bits >> 52) - 1023;  // z in [2^e, 2^(e+1))
    const int k = e - 30;                    // u1 = 2^k * m, m in [0.5, 1)
    const double m = as_f64((bits & 0x000fffffffffffffull) | 0x3fe0000000000000ull);
    const uint32_t i = (uint32_t)(bits >> 45) & 127u;
    const double invc = as_f64(tab[3 * i]);
    const double lhi = as_f64(tab[3 * i + 1]);
    const double llo = as_f64(tab[3 * i + 2]);
    const double r = fma_rn(m, invc, -1.0);
    const double kd = (double)k;
    // ln(1+r) = r + r^2 * (-1/2 + r/3 - r^2/4 + r^3/5 - r^4/6 + r^5/7)
    // (truncation r^8/8 <= 2^-59 |r| for |r| <= 2^-8)
    double p = fma_rn(r, 1.0 / 7.0, -1.0 / 6.0);
    p = fma_rn(r, p, 1.0 / 5.0);
    p = fma_rn(r, p, -0.25);
    p = fma_rn(r, p, 1.0 / 3.0);
    p = fma_rn(r, p, -0.5);
    const double r2 = r * r;
    // hi + err == k*ln2_hi + logc_hi exactly (k*ln2_hi is exact; |k ln2_hi| >=
    // |logc_hi| whenever k != 0, so Fast2Sum applies)
    const double t = kd * kLn2Hi;
    const double hi = t + lhi;
    const double err = (t - hi) + lhi;
    const double lo = fma_rn(kd, kLn2Lo, llo) + err;
    return hi + (r + fma_rn(r2, p, lo));
}

// fdlibm __kernel_sin(x, y, 1) / __kernel_cos(x, y) on |x + y| <= pi/4 (+eps),
// y the tail of the reduced argument
SFB_EXP_HD void sincos_kernel(double x, double y, double &s, double &c) {
    const double S1 = -1.66666666666666324348e-01, S2 = 8.33333333332248946124e-03,
                 S3 = -1.98412698298579493134e-04, S4 = 2.75573137070700676789e-06,
                 S5 = -2.50507602534068634195e-08, S6 = 1.58969099521155010221e-10;
    const double C1 = 4.16666666666666019037e-02, C2 = -1.38888888888741095749e-03,
                 C3 = 2.48015872894767294178e-05, C4 = -2.75573143513906633035e-07,
                 C5 = 2.08757232129817482790e-09, C6 = -1.13596475577881948265e-11;
    const double z = x * x;
    // sin
    const double v = z * x;
    double rs = fma_rn(z, S6, S5);
    rs = fma_rn(z, rs, S4);
    rs = fma_rn(z, rs, S3);
    rs = fma_rn(z, rs, S2);
    // x - ((z*(y/2 - v*r) - y) - v*S1)
    s = x - ((z * (0.5 * y - v * rs) - y) - v * S1);
    // cos: w + (((1 - w) - hz) + (z*r - x*y)), r = z*(C1 + z*(C2 + ... ))
    double rc = fma_rn(z, C6, C5);
    rc = fma_rn(z, rc, C4);
    rc = fma_rn(z, rc, C3);
    rc = fma_rn(z, rc, C2);
    rc = fma_rn(z, rc, C1);
    rc = z * rc;
    const double hz = 0.5 * z;
    const double w = 1.0 - hz;
    c = w + (((1.0 - w) - hz) + (z * rc - x * y));
}

// d = fl(theta - H) - (theta - H), exactly (theta in (0, 2 pi], thb = fl(theta - H)):
//   theta <  H: thb + H is exact (Sterbenz) and so is (thb + H) - theta;
//   theta >= H: thb - theta is exact (theta <= 2 thb or thb exact) and so is + H.
SFB_EXP_HD double rounding_error_minus_halfpi(double theta, double thb) {
    const bool small = theta < kHalfPi;
    const double a = sel(small, kHalfPi, -theta);
    const double b = sel(small, -theta, kHalfPi);
    return (thb + a) + b;
}

// the pair transform; z1m1 = z1 - 1, z2m1 = z2 - 1 (see step_m1)
SFB_EXP_HD void box_muller_pair(uint32_t z1m1, uint32_t z2m1, const uint64_t *logtab,
                                double &a, double &b) {
    const double ln_u1 = log_u31(z1m1 + 1u, logtab);
    const double radius = sqrt(-2.0 * ln_u1);
    // theta = fl((2 pi NORM) * z2) == fma(c, z2 - 1, c): exact product + c, one rounding
    const double theta = fma_rn(kTwoPiNorm, (double)z2m1, kTwoPiNorm);
    const double qd = rint(theta * kTwoOverPi);
    const int q = (int)qd;
    // 3-part Cody-Waite: q*P1 is exact (33-bit P1) and so is theta - q*P1
    // (Sterbenz); (r, rt) is the reduced argument as an unevaluated sum
    const double r1 = fma_rn(-qd, kPiO2_1, theta);
    const double w = qd * kPiO2_1t;
    const double r = r1 - w;
    const double rt = (r1 - r) - w;
    double s, c;
    sincos_kernel(r, rt, s, c);
    const bool odd = (q & 1) != 0;
    const double cs = sel(odd, s, c), sn = sel(odd, c, s);
    const double cos_t = sel(((q + 1) & 2) != 0, -cs, cs);
    const double sin_t = sel((q & 2) != 0, -sn, sn);
    const double thb = theta - kHalfPi;  // the reference's argument of lane b
    const double d = rounding_error_minus_halfpi(theta, thb) + kPiO2Lo;
    a = radius * cos_t;
    b = radius * fma_rn(d, cos_t, sin_t);
}

}  // namespace sfb
