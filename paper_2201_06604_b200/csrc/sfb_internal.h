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

// Stream states of one launch: start states are read from `in` (row w - in_lo
// = stream w); final states are written to `out` unless it is null (chunked
// launches: a second kernel advances the states, see fill.cu state_io).
struct StateIO {
    const int64_t *in;
    int64_t in_lo;
    int64_t *out;
};
SFB_HD Mrg load_state(const StateIO &io, int64_t w) { return load_state(io.in + 6 * (w - io.in_lo)); }
SFB_HD void store_state(const StateIO &io, int64_t w, const Mrg &s) {
    if (io.out) store_state(io.out + 6 * w, s);
}

// integer tuning knob from the environment (kernel variant selection for
// profiling sweeps; never changes results)
int tune_knob(const char *name, int dflt);

}  // namespace sfb
