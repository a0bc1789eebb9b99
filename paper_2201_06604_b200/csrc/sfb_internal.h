// sfb_internal.h -- shared helpers of libsfb (not part of the ABI).
#pragma once
#include <stdarg.h>
#include <stdint.h>

#include "../../include/sfb.h"
#include "mrg31k3p.cuh"

namespace sfb {

// set the thread-local error message; returns code (for `return fail(...)`)
int fail(int code, const char *fmt, ...);

// transition matrices _T1/_T2 (core.py:44-45) raised to arbitrary powers
void jump_pow(uint64_t n, Jump *out);       // A^n, exact
void jump_pow2(int e, Jump *out);           // A^(2^e), exact, any e >= 0
void jump_mul(const Jump &a, const Jump &b, Jump *out);  // a*b (powers of A commute)
void pow2_table(Pow2Table *t);              // A^(2^b), b < kPow2Bits (cached)

// integer tuning knob from the environment (kernel variant selection for
// profiling sweeps; never changes results)
int tune_knob(const char *name, int dflt);

}  // namespace sfb
