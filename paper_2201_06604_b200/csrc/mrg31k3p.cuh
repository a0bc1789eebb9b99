// mrg31k3p.cuh -- MRG31k3p arithmetic shared by host and device code.
//
// Reference: the int64 step `_step` (_kernels.py:33-47) and its oracle
// `next_state` (core.py:114-123):
//   y1 = (2^22*a1 + (2^7+1)*a2) mod m1, shift (a0,a1,a2) <- (y1,a0,a1)
//   y2 = (2^15*b0 + (2^15+1)*b2) mod m2, shift (b0,b1,b2) <- (y2,b0,b1)
//   z  = y1 - y2, z <= 0 => z += m1          (z in [1, m1])
//
// B200 formulation (step_m1 below): uint32 state registers, one 32x32->64
// IMAD.WIDE per component product, a single Mersenne-style fold per component
// and one conditional subtraction each; csub(v, m) = min(v, v - m) on
// unsigned values (v < 2m) compiles to one VIADDMNMX on sm_100a.
// Verified against the int64 oracle step on random and extreme states by the
// CPU test tests/test_host_lib.py (through sfb_host_step_u32).
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define SFB_HD __host__ __device__ __forceinline__
#else
#define SFB_HD inline
#endif

namespace sfb {

constexpr uint32_t kM1 = 2147483647u;  // core.py:29
constexpr uint32_t kM2 = 2147462579u;  // core.py:30
constexpr double kNorm = 1.0 / 2147483648.0;  // _kernels.py:20

SFB_HD uint32_t umin32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
    return min(a, b);
#else
    return a < b ? a : b;
#endif
}

SFB_HD uint32_t csub(uint32_t v, uint32_t m) { return umin32(v, v - m); }

struct Mrg {
    uint32_t a0, a1, a2, b0, b1, b2;
};

// one MRG31k3p step (_kernels.py:33-47); returns z - 1 in [0, m1 - 1]
// (callers fold the +1 into their next operation, e.g. u = fma(z-1, 2^-31, 2^-31)).
//   component 1: p = 2^22 a1 + 129 a2 < 2^54 (two IMAD.WIDE), and since
//     2^31 == 1 (mod m1), p == (p & m1) + (p >> 31) < 2m1: one csub.
//   component 2: p = 2^15 b0 + (2^15+1) b2 < 2^48 (two IMAD.WIDE),
//     2^31 == 21069 (mod m2): p == (p >> 31) * 21069 + (p & m1) < 2m2: one csub.
//   z - 1 = y1 - y2 - 1 (+ m1 if y1 <= y2) = min(y1 - y2 - 1 + m1, y1 - y2 - 1).
// step_core computes the new words from the lag values and writes them into
// the slots of the dropped (oldest) words; step3 runs three steps with the
// roles of the three slots rotating statically, so a loop over step3 needs no
// register moves for the shift register.
SFB_HD uint32_t step_core(uint32_t a1, uint32_t a2, uint32_t b0, uint32_t b2, uint32_t &a_out,
                          uint32_t &b_out) {
    const uint64_t p1 = (uint64_t)a1 * 4194304u + (uint64_t)a2 * 129u;
    const uint32_t y1 = csub(((uint32_t)p1 & kM1) + (uint32_t)(p1 >> 31), kM1);
    const uint64_t p2 = (uint64_t)b0 * 32768u + (uint64_t)b2 * 32769u;
    const uint32_t y2 = csub((uint32_t)(p2 >> 31) * 21069u + ((uint32_t)p2 & kM1), kM2);
    a_out = y1;
    b_out = y2;
    const uint32_t dm1 = y1 - y2 - 1u;  // IADD3 + VIADDMNMX
    return umin32(dm1 + kM1, dm1);
}

SFB_HD uint32_t step_m1(Mrg &s) {
    uint32_t y1, y2;
    const uint32_t zm1 = step_core(s.a1, s.a2, s.b0, s.b2, y1, y2);
    s.a2 = s.a1;
    s.a1 = s.a0;
    s.a0 = y1;
    s.b2 = s.b1;
    s.b1 = s.b0;
    s.b0 = y2;
    return zm1;
}

// three consecutive steps (z - 1 outputs in order); s ends in canonical order
SFB_HD void step3(Mrg &s, uint32_t &z0, uint32_t &z1, uint32_t &z2) {
    // slots (A0,A1,A2)=(a0,a1,a2), (B0,B1,B2)=(b0,b1,b2)
    z0 = step_core(s.a1, s.a2, s.b0, s.b2, s.a2, s.b2);  // newest in A2/B2
    z1 = step_core(s.a0, s.a1, s.b2, s.b1, s.a1, s.b1);  // newest in A1/B1
    z2 = step_core(s.a2, s.a0, s.b1, s.b0, s.a0, s.b0);  // newest in A0/B0
}

// one MRG31k3p step (_kernels.py:33-47); returns z in [1, m1]
SFB_HD uint32_t step(Mrg &s) { return step_m1(s) + 1u; }

SFB_HD Mrg load_state(const int64_t *row) {
    Mrg s;
    s.a0 = (uint32_t)row[0];
    s.a1 = (uint32_t)row[1];
    s.a2 = (uint32_t)row[2];
    s.b0 = (uint32_t)row[3];
    s.b1 = (uint32_t)row[4];
    s.b2 = (uint32_t)row[5];
    return s;
}

SFB_HD void store_state(int64_t *row, const Mrg &s) {
    row[0] = s.a0;
    row[1] = s.a1;
    row[2] = s.a2;
    row[3] = s.b0;
    row[4] = s.b1;
    row[5] = s.b2;
}

// 3x3 modular matrix (row-major) acting on (x[n-1], x[n-2], x[n-3]) --
// the transition matrices _T1/_T2 of core.py:44-45 and their powers.
struct Mat3 {
    uint32_t m[9];
};

// a*v0 + b*v1 + c*v2: three products < 2^62 sum below 2^64
SFB_HD uint64_t dot3(const uint32_t *row, uint32_t v0, uint32_t v1, uint32_t v2) {
    return (uint64_t)row[0] * v0 + (uint64_t)row[1] * v1 + (uint64_t)row[2] * v2;
}

// x mod m1 for any 64-bit x, without a 64-bit division: 2^31 == 1 (mod m1),
// so x == (x & m1) + (x >> 31) < 2^33 + 2^31, folded once more below 2 m1
SFB_HD uint32_t mod_m1(uint64_t x) {
    x = (x & kM1) + (x >> 31);
    const uint32_t y = (uint32_t)(x & kM1) + (uint32_t)(x >> 31);  // < 2^31 + 8
    return csub(y, kM1);
}

// x mod m2 for any 64-bit x: 2^31 == 21069 (mod m2), so
// x == (x >> 31) * 21069 + (x & m1): < 2^33 * 21069 + 2^31 < 2^49, then
// < (2^18 + 1) * 21069 + 2^31 < 2^33, then below 2 m2
SFB_HD uint32_t mod_m2(uint64_t x) {
    x = (x >> 31) * 21069u + (x & kM1);
    x = (x >> 31) * 21069u + (x & kM1);
    const uint32_t y = (uint32_t)(x >> 31) * 21069u + (uint32_t)(x & kM1);  // < 2^31 + 4 * 21069
    return csub(y, kM2);
}

SFB_HD void apply1(const Mat3 &p, uint32_t &x0, uint32_t &x1, uint32_t &x2) {
    const uint32_t y0 = mod_m1(dot3(p.m + 0, x0, x1, x2));
    const uint32_t y1 = mod_m1(dot3(p.m + 3, x0, x1, x2));
    const uint32_t y2 = mod_m1(dot3(p.m + 6, x0, x1, x2));
    x0 = y0;
    x1 = y1;
    x2 = y2;
}

SFB_HD void apply2(const Mat3 &p, uint32_t &x0, uint32_t &x1, uint32_t &x2) {
    const uint32_t y0 = mod_m2(dot3(p.m + 0, x0, x1, x2));
    const uint32_t y1 = mod_m2(dot3(p.m + 3, x0, x1, x2));
    const uint32_t y2 = mod_m2(dot3(p.m + 6, x0, x1, x2));
    x0 = y0;
    x1 = y1;
    x2 = y2;
}

// A^n for both components as one jump: state <- (P1 g1, P2 g2)
struct Jump {
    Mat3 p1, p2;
};

SFB_HD void apply(const Jump &j, Mrg &s) {
    apply1(j.p1, s.a0, s.a1, s.a2);
    apply2(j.p2, s.b0, s.b1, s.b2);
}

// Powers A^(2^b), b < kPow2Bits, for device-side arbitrary skip-ahead.
constexpr int kPow2Bits = 48;
struct Pow2Table {
    Jump p[kPow2Bits];
};

// advance s by n < 2^kPow2Bits steps (binary powering; bit-exact for any n)
SFB_HD void skip(const Pow2Table &t, Mrg &s, uint64_t n) {
#ifdef __CUDA_ARCH__
#pragma unroll 1
#endif
    for (int b = 0; n != 0 && b < kPow2Bits; ++b, n >>= 1)
        if (n & 1) apply(t.p[b], s);
}

}  // namespace sfb
