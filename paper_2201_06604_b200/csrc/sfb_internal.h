// sfb_internal.h -- shared helpers of libsfb (not part of the ABI).
#pragma once
#include <cuda_runtime_api.h>
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

// Stream states of one launch: `in` holds the start states of streams
// in_lo, in_lo + 1, ...; final states go to `out` (row index = stream index).
struct StateIO {
    const int64_t *in;
    int64_t in_lo;
    int64_t *out;
};
SFB_HD Mrg load_state(const StateIO &io, int64_t w) { return load_state(io.in + 6 * (w - io.in_lo)); }
SFB_HD void store_state(const StateIO &io, int64_t w, const Mrg &s) { store_state(io.out + 6 * w, s); }

// A chunked launch (several threads per stream, each jumping to its chunk)
// reads every stream's start state in all chunks while the stream's LAST
// chunk writes the final state.  Nothing orders those thread blocks, so the
// readers get a stream-ordered snapshot of rows [lo, hi) (freed after the
// launch) -- otherwise the result would depend on block scheduling.
struct StateSnapshot {
    int64_t *buf = nullptr;
    cudaStream_t st = nullptr;
    StateSnapshot() = default;
    StateSnapshot(const StateSnapshot &) = delete;
    StateSnapshot &operator=(const StateSnapshot &) = delete;
    ~StateSnapshot();
};
int make_state_io(int64_t *cur, int64_t lo, int64_t hi, bool chunked, cudaStream_t st,
                  StateSnapshot &snap, StateIO *io);

// integer tuning knob from the environment (kernel variant selection for
// profiling sweeps; never changes results)
int tune_knob(const char *name, int dflt);

}  // namespace sfb
