// bessel_k.cuh -- modified Bessel function of the second kind K_nu(x) in
// float64, host + device (the Matern covariance of the GRF pipeline; the
// reference calls scipy.special.kv, grf.py:116-124, 138-159).
//
// K_mu and K_{mu+1} are computed for the fractional order mu = nu - round(nu)
// in [-1/2, 1/2), then the upward recurrence (stable for K)
//     K_{m+1}(x) = K_{m-1}(x) + (2 m / x) K_m(x)
// reaches nu.  The pair comes from
//   * x >= 2: Steed's continued fraction CF2 with Temme's normalisation sum
//     (the classical algorithm, ~tens of iterations, relative error ~1e-15);
//   * x <  2: the integral K_m(x) = int_0^inf exp(-x cosh t) cosh(m t) dt by
//     the trapezoidal rule.  The integrand is analytic in the strip
//     |Im t| < pi/2, so the rule converges like exp(-pi^2 / h): h = 1/8 gives
//     ~1e-34 discretisation error; the sum stops once the terms are below
//     1e-18 of it on the decaying side.
// Accuracy vs scipy.special.kv (AMOS): ~1e-14 relative over the Matern range
// (tests/test_grf.py).  Not bit-compatible with AMOS -- the GRF pipeline is
// compared within tolerances, as the reference's own tests do.
#pragma once
#include <math.h>
#include <stdint.h>

#ifdef __CUDACC__
#define SFB_BK_HD __host__ __device__ __forceinline__
#else
#define SFB_BK_HD inline
#endif

namespace sfb {

SFB_BK_HD void bessel_k_cf2(double mu, double x, double &kmu, double &kmu1) {
    // Steed's method for CF2 with the Temme normalisation sum (x >= 2)
    const double kPi = 3.141592653589793;
    const double a1 = 0.25 - mu * mu;
    double b = 2.0 * (1.0 + x);
    double d = 1.0 / b;
    double h = d, delh = d;
    double q1 = 0.0, q2 = 1.0;
    double q = a1, c = a1, a = -a1;
    double s = 1.0 + q * delh;
    for (int i = 1; i < 2000; ++i) {
        a -= 2 * i;
        c = -a * c / (i + 1.0);
        const double qnew = (q1 - b * q2) / a;
        q1 = q2;
        q2 = qnew;
        q += c * qnew;
        b += 2.0;
        d = 1.0 / (b + a * d);
        delh = (b * d - 1.0) * delh;
        h += delh;
        const double dels = q * delh;
        s += dels;
        if (fabs(dels / s) < 1e-17) break;
    }
    h = a1 * h;
    kmu = sqrt(kPi / (2.0 * x)) * exp(-x) / s;
    kmu1 = kmu * (mu + x + 0.5 - h) / x;
}

SFB_BK_HD void bessel_k_integral(double mu, double x, double &kmu, double &kmu1) {
    // trapezoidal rule on int_0^inf exp(-x cosh t) cosh(m t) dt (x < 2)
    const double hstep = 0.125;
    double s0 = 0.5 * exp(-x), s1 = s0;  // t = 0 (half weight): cosh(0) = 1
    double c0 = 0.0, c1 = 0.0;           // Neumaier compensation of the sums
    const double m0 = mu, m1 = mu + 1.0;
    for (int k = 1; k < 4000; ++k) {
        const double t = k * hstep;
        const double et = exp(t), eti = 1.0 / et;
        const double ch = 0.5 * (et + eti);
        const double g = exp(-x * ch);
        const double f0 = g * cosh(m0 * t), f1 = g * cosh(m1 * t);
        double u = s0 + f0;
        c0 += fabs(s0) >= fabs(f0) ? (s0 - u) + f0 : (f0 - u) + s0;
        s0 = u;
        u = s1 + f1;
        c1 += fabs(s1) >= fabs(f1) ? (s1 - u) + f1 : (f1 - u) + s1;
        s1 = u;
        // past the peak of the heavier integrand (x sinh t > m1) the terms
        // decay super-exponentially: stop once negligible
        if (x * 0.5 * (et - eti) > m1 && f1 < 1e-18 * s1 && f0 < 1e-18 * s0) break;
    }
    kmu = hstep * (s0 + c0);
    kmu1 = hstep * (s1 + c1);
}

// K_nu(x), nu > 0, x > 0 (callers validate the domain)
SFB_BK_HD double bessel_k(double nu, double x) {
    const int nl = (int)(nu + 0.5);
    const double mu = nu - nl;  // in [-1/2, 1/2)
    double k0, k1;
    if (x >= 2.0)
        bessel_k_cf2(mu, x, k0, k1);
    else
        bessel_k_integral(mu, x, k0, k1);
    // k0 = K_mu, k1 = K_{mu+1}; step up to K_{mu+nl} = K_nu
    for (int i = 1; i <= nl; ++i) {
        const double k2 = k0 + 2.0 * (mu + i) / x * k1;
        k0 = k1;
        k1 = k2;
    }
    return k0;
}

// Matern correlation at distance-argument a = sqrt(8 kappa) d / range > 0:
// 2^(1-kappa) / Gamma(kappa) * a^kappa * K_kappa(a), the prefactor in logs as
// in grf.py:150-157 (lg = lgamma(kappa) supplied by the caller)
SFB_BK_HD double matern_corr_arg(double kappa, double lg, double a) {
    return exp((1.0 - kappa) * 0.6931471805599453 - lg + kappa * log(a)) * bessel_k(kappa, a);
}

}  // namespace sfb
