// host_streams.cpp -- host side of libsfb: exact stream arithmetic, stream
// files, error plumbing and CPU test hooks.
//
// Replaces the pure-Python big-integer code of the reference (core.py):
//   _mat_mul/_jump_matrices/_mat_vec   core.py:48-66
//   next_state / jump_ahead            core.py:114-136
//   _jump_seed / create_streams        core.py:139-142, 222-235
//   save_streams / save_streams_atomic core.py:238-261
//   load_streams (+ StreamSet.validate) core.py:264-305, 204-212
// All arithmetic is exact (uint64 accumulators, entries < 2^31), so results
// equal the reference's Python ints bit for bit.
#include <errno.h>
#include <fcntl.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "box_muller.cuh"
#include "fisher_sampler.cuh"
#include "log1p_glibc.cuh"
#include "exp_glibc.cuh"
#include "sfb_internal.h"

namespace sfb {

static thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

// _T1 / _T2 of core.py:44-45 (acting on (x[n-1], x[n-2], x[n-3]))
static const uint32_t kT1[9] = {0, 1u << 22, (1u << 7) + 1, 1, 0, 0, 0, 1, 0};
static const uint32_t kT2[9] = {1u << 15, 0, (1u << 15) + 1, 1, 0, 0, 0, 1, 0};

static void mat_mul(const Mat3 &a, const Mat3 &b, uint32_t mod, Mat3 &o) {
    Mat3 t;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            uint64_t acc = 0;
            for (int k = 0; k < 3; ++k) acc += (uint64_t)a.m[3 * i + k] * b.m[3 * k + j];
            t.m[3 * i + j] = (uint32_t)(acc % mod);
        }
    o = t;
}

static Jump identity_jump() {
    Jump j;
    for (int k = 0; k < 9; ++k) j.p1.m[k] = j.p2.m[k] = (k % 4 == 0) ? 1u : 0u;
    return j;
}

static Jump base_jump() {
    Jump j;
    memcpy(j.p1.m, kT1, sizeof kT1);
    memcpy(j.p2.m, kT2, sizeof kT2);
    return j;
}

static void jump_mul(const Jump &a, const Jump &b, Jump &o) {
    mat_mul(a.p1, b.p1, kM1, o.p1);
    mat_mul(a.p2, b.p2, kM2, o.p2);
}

void jump_mul(const Jump &a, const Jump &b, Jump *o) { jump_mul(a, b, *o); }

void jump_pow2(int e, Jump *out) {  // core.py:55-62
    Jump j = base_jump();
    for (int k = 0; k < e; ++k) jump_mul(j, j, j);
    *out = j;
}

void jump_pow(uint64_t n, Jump *out) {
    Jump r = identity_jump(), p = base_jump();
    while (n) {
        if (n & 1) jump_mul(p, r, r);  // powers of A commute
        n >>= 1;
        if (n) jump_mul(p, p, p);
    }
    *out = r;
}

void pow2_table(Pow2Table *t) {
    static std::once_flag once;
    static Pow2Table cached;
    std::call_once(once, [] {
        Jump j = base_jump();
        for (int b = 0; b < kPow2Bits; ++b) {
            cached.p[b] = j;
            jump_mul(j, j, j);
        }
    });
    *t = cached;
}

static const uint64_t kExpTable[256] = SFB_EXP_TABLE_INIT;

int tune_knob(const char *name, int dflt) {
    const char *v = getenv(name);
    return (v && *v) ? atoi(v) : dflt;
}

}  // namespace sfb

using namespace sfb;

extern "C" {

const char *sfb_last_error(void) { return g_err.c_str(); }

int sfb_version(void) { return 100; }

int sfb_validate_seed(const int64_t seed[6]) {  // core.py:69-86
    for (int c = 0; c < 2; ++c) {
        const int64_t *v = seed + 3 * c;
        const int64_t m = c == 0 ? kM1 : kM2;
        for (int k = 0; k < 3; ++k)
            if (v[k] < 0 || v[k] >= m)
                return fail(SFB_E_INVALID_SEED, "component-%d seed component %lld outside [0, %lld]",
                            c + 1, (long long)v[k], (long long)(m - 1));
        if (v[0] == 0 && v[1] == 0 && v[2] == 0)
            return fail(SFB_E_INVALID_SEED, "component-%d seed must not be all zero", c + 1);
    }
    return SFB_OK;
}

int sfb_next_state(int64_t state[6], int64_t *z) {  // core.py:114-123
    // exact int64 restatement (inputs may be any valid state)
    const int64_t M1 = kM1, M2 = kM2;
    int64_t y1 = ((1LL << 22) * state[1] + 129LL * state[2]) % M1;
    int64_t y2 = ((1LL << 15) * state[3] + 32769LL * state[5]) % M2;
    state[2] = state[1];
    state[1] = state[0];
    state[0] = y1;
    state[5] = state[4];
    state[4] = state[3];
    state[3] = y2;
    int64_t zz = ((y1 - y2) % M1 + M1) % M1;
    *z = zz == 0 ? M1 : zz;
    return SFB_OK;
}

int sfb_jump_matrices(int e, int64_t j1[9], int64_t j2[9]) {
    if (e < 0) return fail(SFB_E_INVALID_ARGUMENT, "jump exponent must be >= 0");
    Jump j;
    jump_pow2(e, &j);
    for (int k = 0; k < 9; ++k) {
        j1[k] = j.p1.m[k];
        j2[k] = j.p2.m[k];
    }
    return SFB_OK;
}

static void apply_i64(const Jump &j, int64_t s[6]) {
    Mrg m = load_state(s);
    apply(j, m);
    store_state(s, m);
}

static int check_state(const int64_t s[6]) {
    for (int k = 0; k < 6; ++k) {
        const int64_t m = k < 3 ? kM1 : kM2;
        if (s[k] < 0 || s[k] >= m)
            return fail(SFB_E_INVALID_ARGUMENT, "state component %lld outside [0, %lld]",
                        (long long)s[k], (long long)(m - 1));
    }
    return SFB_OK;
}

int sfb_jump_ahead(int64_t state[6], int e) {  // core.py:126-136
    if (e < 0) return fail(SFB_E_INVALID_ARGUMENT, "jump exponent must be >= 0");
    if (int rc = check_state(state)) return rc;
    Jump j;
    jump_pow2(e, &j);
    apply_i64(j, state);
    return SFB_OK;
}

int sfb_skip(int64_t state[6], uint64_t n) {
    if (int rc = check_state(state)) return rc;
    Jump j;
    jump_pow(n, &j);
    apply_i64(j, state);
    return SFB_OK;
}

int sfb_create_streams(const int64_t seed[6], int64_t n, int64_t *rows,
                       int64_t next_seed[6]) {  // core.py:222-235
    if (n < 1) return fail(SFB_E_INVALID_ARGUMENT, "number of streams to create must be >= 1");
    if (int rc = sfb_validate_seed(seed)) return rc;
    static std::once_flag once;
    static Jump j134;
    std::call_once(once, [] { jump_pow2(134, &j134); });
    Mrg s = load_state(seed);
    for (int64_t k = 0; k < n; ++k) {
        store_state(rows + 6 * k, s);
        apply(j134, s);  // _jump_seed, core.py:139-142
    }
    store_state(next_seed, s);
    return SFB_OK;
}

/* ---- stream files -------------------------------------------------------- */
static const char kMagic[] = "streamforge-streams";  // core.py:238
static const char kVersion[] = "v1";                 // core.py:239

int64_t sfb_format_streams_bound(int64_t n) { return 96 + n * 12 * 21; }

}  // extern "C"

namespace sfb {

// Run f(t, lo, hi) over contiguous ranges of [0, n) on up to one thread per
// host core (at least `min_per` items per range).  Stream files of 2^20
// streams are 132 MB: formatting and parsing them are embarrassingly parallel
// over lines.
template <typename F>
static int parallel_ranges(int64_t n, int64_t min_per, F &&f) {
    const int64_t hw = std::max<int64_t>(1, std::min<int64_t>(std::thread::hardware_concurrency(), 64));
    const int64_t nt = std::max<int64_t>(1, std::min<int64_t>(hw, n / std::max<int64_t>(1, min_per)));
    if (nt == 1) {
        f(0, (int64_t)0, n);
        return 1;
    }
    std::vector<std::thread> pool;
    for (int64_t t = 1; t < nt; ++t)
        pool.emplace_back([&f, t, n, nt] { f(t, n * t / nt, n * (t + 1) / nt); });
    f(0, (int64_t)0, n / nt);
    for (auto &th : pool) th.join();
    return (int)nt;
}

static const char kDigits2[] =
    "00010203040506070809101112131415161718192021222324252627282930313233343536373839"
    "40414243444546474849505152535455565758596061626364656667686970717273747576777879"
    "8081828384858687888990919293949596979899";

static char *put_i64(char *p, int64_t v) {
    char tmp[24];
    int k = sizeof tmp;
    uint64_t u = v < 0 ? (uint64_t)0 - (uint64_t)v : (uint64_t)v;
    while (u >= 100) {
        const unsigned r = (unsigned)(u % 100);
        u /= 100;
        tmp[--k] = kDigits2[2 * r + 1];
        tmp[--k] = kDigits2[2 * r];
    }
    if (u >= 10) {
        tmp[--k] = kDigits2[2 * u + 1];
        tmp[--k] = kDigits2[2 * u];
    } else {
        tmp[--k] = (char)('0' + u);
    }
    if (v < 0) *p++ = '-';
    memcpy(p, tmp + k, sizeof tmp - k);
    return p + (sizeof tmp - k);
}

// lines of streams [lo, hi): "c0 .. c5 i0 .. i5\n" (core.py:242-250)
static char *format_rows(char *p, const int64_t *current, const int64_t *initial, int64_t lo,
                         int64_t hi) {
    for (int64_t k = lo; k < hi; ++k) {
        for (int c = 0; c < 12; ++c) {
            if (c) *p++ = ' ';
            p = put_i64(p, c < 6 ? current[6 * k + c] : initial[6 * k + c - 6]);
        }
        *p++ = '\n';
    }
    return p;
}

// format in parallel: one private buffer per range, in file order
struct FormattedChunks {
    std::string header;
    std::vector<std::vector<char>> parts;
};

static void format_parallel(const int64_t *current, const int64_t *initial, int64_t n,
                            FormattedChunks &out) {
    char hdr[96];
    snprintf(hdr, sizeof hdr, "%s %s count=%lld\n", kMagic, kVersion, (long long)n);
    out.header = hdr;
    const int64_t hw = std::max<int64_t>(1, std::min<int64_t>(std::thread::hardware_concurrency(), 64));
    out.parts.assign((size_t)hw, {});
    parallel_ranges(n, 16384, [&](int64_t t, int64_t lo, int64_t hi) {
        std::vector<char> &buf = out.parts[(size_t)t];
        buf.resize((size_t)(hi - lo) * 12 * 21);
        char *e = format_rows(buf.data(), current, initial, lo, hi);
        buf.resize((size_t)(e - buf.data()));
    });
}

}  // namespace sfb

extern "C" {

int sfb_format_streams(const int64_t *current, const int64_t *initial, int64_t n,
                       char *buf, int64_t cap, int64_t *len) {  // core.py:242-250
    if (cap < sfb_format_streams_bound(n))
        return fail(SFB_E_INVALID_ARGUMENT, "format buffer too small");
    FormattedChunks fc;
    format_parallel(current, initial, n, fc);
    char *p = buf;
    memcpy(p, fc.header.data(), fc.header.size());
    p += fc.header.size();
    for (auto &part : fc.parts) {
        if (!part.empty()) memcpy(p, part.data(), part.size());
        p += part.size();
    }
    *len = p - buf;
    return SFB_OK;
}

static int write_all(int fd, const char *p, size_t len, const std::string &name) {
    while (len) {
        ssize_t w = write(fd, p, len);
        if (w < 0) {
            if (errno == EINTR) continue;
            return fail(SFB_E_IO, "%s: %s", name.c_str(), strerror(errno));
        }
        p += w;
        len -= (size_t)w;
    }
    return SFB_OK;
}

int sfb_save_streams(const char *path, const int64_t *current, const int64_t *initial,
                     int64_t n, int atomic) {  // core.py:242-261
    FormattedChunks fc;
    format_parallel(current, initial, n, fc);
    std::string target = path;
    std::string tmp = atomic ? target + ".tmp" : target;
    int fd = open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
    if (fd < 0) return fail(SFB_E_IO, "%s: %s", tmp.c_str(), strerror(errno));
    int rc = write_all(fd, fc.header.data(), fc.header.size(), tmp);
    for (size_t t = 0; rc == SFB_OK && t < fc.parts.size(); ++t)
        rc = write_all(fd, fc.parts[t].data(), fc.parts[t].size(), tmp);
    if (rc) {
        close(fd);
        return rc;
    }
    if (atomic && fsync(fd) != 0) {
        int e = errno;
        close(fd);
        return fail(SFB_E_IO, "fsync %s: %s", tmp.c_str(), strerror(e));
    }
    if (close(fd) != 0) return fail(SFB_E_IO, "close %s: %s", tmp.c_str(), strerror(errno));
    if (atomic && rename(tmp.c_str(), target.c_str()) != 0)
        return fail(SFB_E_IO, "rename %s: %s", tmp.c_str(), strerror(errno));
    return SFB_OK;
}

}  // extern "C"

namespace sfb {

// Python str.split() whitespace (ASCII subset)
static inline bool is_ws(char c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f' ||
           (c >= 0x1c && c <= 0x1f);
}

struct Cursor {
    const char *p, *end;
    // next line without its '\n' terminator (file.readline semantics);
    // returns false at EOF (readline() == "")
    bool line(const char *&b, const char *&e) {
        if (p >= end) return false;
        b = p;
        const char *nl = (const char *)memchr(p, '\n', (size_t)(end - p));
        e = nl ? nl : end;
        p = nl ? nl + 1 : end;
        return true;
    }
};

// split [b, e) on whitespace into at most maxtok tokens; returns the count
// (maxtok + 1 means "more than maxtok")
static int split(const char *b, const char *e, const char **tb, const char **te, int maxtok) {
    int n = 0;
    while (b < e) {
        while (b < e && is_ws(*b)) ++b;
        if (b >= e) break;
        const char *s = b;
        while (b < e && !is_ws(*b)) ++b;
        if (n == maxtok) return maxtok + 1;
        tb[n] = s;
        te[n] = b;
        ++n;
    }
    return n;
}

// Python int(token): optional sign, digits with single '_' separators
static bool parse_int(const char *b, const char *e, int64_t *out) {
    bool neg = false;
    if (b < e && (*b == '+' || *b == '-')) neg = *b++ == '-';
    if (b >= e || *b < '0' || *b > '9') return false;
    unsigned __int128 v = 0;
    bool prev_digit = false;
    for (; b < e; ++b) {
        if (*b == '_') {
            if (!prev_digit || b + 1 >= e || b[1] < '0' || b[1] > '9') return false;
            prev_digit = false;
            continue;
        }
        if (*b < '0' || *b > '9') return false;
        v = v * 10 + (unsigned)(*b - '0');
        if (v > ((unsigned __int128)1 << 64)) return false;
        prev_digit = true;
    }
    if (neg) {
        if (v > ((unsigned __int128)1 << 63)) return false;
        *out = (int64_t)(0 - (uint64_t)v);
    } else {
        if (v >= ((unsigned __int128)1 << 63)) return false;
        *out = (int64_t)v;
    }
    return true;
}

static int parse_header(Cursor &cur, int64_t *count) {  // core.py:271-284
    const char *b, *e;
    if (!cur.line(b, e)) b = e = cur.p;
    const char *tb[4], *te[4];
    int nt = split(b, e, tb, te, 3);
    if (nt != 3 || (size_t)(te[0] - tb[0]) != strlen(kMagic) ||
        memcmp(tb[0], kMagic, strlen(kMagic)) != 0 ||
        (size_t)(te[1] - tb[1]) != strlen(kVersion) ||
        memcmp(tb[1], kVersion, strlen(kVersion)) != 0 || te[2] - tb[2] < 6 ||
        memcmp(tb[2], "count=", 6) != 0)
        return fail(SFB_E_CORRUPT_STREAM_FILE, "bad stream file header");
    int64_t n;
    if (!parse_int(tb[2] + 6, te[2], &n))
        return fail(SFB_E_CORRUPT_STREAM_FILE, "bad stream count in header");
    if (n < 1) return fail(SFB_E_CORRUPT_STREAM_FILE, "stream count must be >= 1");
    *count = n;
    return SFB_OK;
}

// the canonical line: 12 unsigned decimal tokens separated by single spaces
// (what save_streams writes); anything else takes the general tokenizer
static bool parse_line_fast(const char *b, const char *e, int64_t *vals) {
    const char *p = b;
    for (int c = 0; c < 12; ++c) {
        if (c) {
            if (p >= e || *p != ' ') return false;
            ++p;
        }
        const char *s = p;
        uint64_t v = 0;
        while (p < e && (unsigned)(*p - '0') < 10u) v = v * 10 + (uint64_t)(*p++ - '0');
        if (p == s || p - s > 18) return false;
        vals[c] = (int64_t)v;
    }
    return p == e;
}

// one stream line -> 12 values, with the reference's error for a bad line
// (returns 0 or an error code; msg receives the message)
static int parse_line(const char *b, const char *e, int64_t k, int64_t *vals, char *msg,
                      size_t msglen) {
    if (parse_line_fast(b, e, vals)) return SFB_OK;
    const char *tb[13], *te[13];
    if (split(b, e, tb, te, 12) != 12) {
        snprintf(msg, msglen, "stream %lld: expected 12 integers", (long long)(k + 1));
        return SFB_E_CORRUPT_STREAM_FILE;
    }
    for (int c = 0; c < 12; ++c)
        if (!parse_int(tb[c], te[c], &vals[c])) {
            snprintf(msg, msglen, "stream %lld: non-integer entry", (long long)(k + 1));
            return SFB_E_CORRUPT_STREAM_FILE;
        }
    return SFB_OK;
}

}  // namespace sfb

extern "C" {

int sfb_parse_streams_count(const char *text, int64_t len, int64_t *n) {
    Cursor cur{text, text + len};
    return parse_header(cur, n);
}

int sfb_parse_streams(const char *text, int64_t len, int64_t *current, int64_t *initial,
                      int64_t n) {  // core.py:264-305
    Cursor cur{text, text + len};
    int64_t count;
    if (int rc = parse_header(cur, &count)) return rc;
    if (count != n) return fail(SFB_E_INVALID_ARGUMENT, "count mismatch");
    // Parallel over byte ranges of the body: pass 1 counts the lines that start
    // in each range, pass 2 parses lines [0, count) where they start.  The
    // first error in file order wins, as in the sequential reference loop.
    const char *body = cur.p, *end = text + len;
    const int64_t nbytes = end - body;
    const int64_t hw = std::max<int64_t>(1, std::min<int64_t>(std::thread::hardware_concurrency(), 64));
    const int64_t nt = std::max<int64_t>(1, std::min<int64_t>(hw, nbytes / (1 << 20)));
    std::vector<int64_t> starts((size_t)nt + 1, 0), lines((size_t)nt, 0);
    for (int64_t t = 0; t <= nt; ++t) starts[(size_t)t] = nbytes * t / nt;
    // a line starts at body[0] or right after a '\n'; it belongs to the range
    // holding its first byte
    auto count_starts = [&](int64_t t, int64_t, int64_t) {
        const int64_t lo = starts[(size_t)t], hi = starts[(size_t)t + 1];
        int64_t c = (lo == 0 && nbytes > 0) ? 1 : 0;
        for (const char *q = body + std::max<int64_t>(lo - 1, 0); q < body + hi - 1;) {
            const char *nl = (const char *)memchr(q, '\n', (size_t)(body + hi - 1 - q));
            if (!nl) break;
            if (nl + 1 >= body + lo && nl + 1 < end) ++c;
            q = nl + 1;
        }
        lines[(size_t)t] = c;
    };
    if (nt == 1)
        count_starts(0, 0, 1);
    else
        parallel_ranges(nt, 1, [&](int64_t, int64_t lo, int64_t hi) {
            for (int64_t t = lo; t < hi; ++t) count_starts(t, 0, 0);
        });
    std::vector<int64_t> first_line((size_t)nt + 1, 0);
    for (int64_t t = 0; t < nt; ++t) first_line[(size_t)t + 1] = first_line[(size_t)t] + lines[(size_t)t];
    const int64_t total_lines = first_line[(size_t)nt];
    struct Err {
        int64_t line = INT64_MAX;
        int code = 0;
        char msg[160] = {0};
    };
    std::vector<Err> errs((size_t)nt);
    std::vector<const char *> after((size_t)nt, nullptr);  // start of line `count`, if in range t
    auto parse_range = [&](int64_t t) {
        const int64_t lo = starts[(size_t)t], hi = starts[(size_t)t + 1];
        int64_t k = first_line[(size_t)t];
        // first line start at or after lo
        const char *q = body + lo;
        if (lo > 0 && body[lo - 1] != '\n') {
            const char *nl = (const char *)memchr(q, '\n', (size_t)(end - q));
            q = nl ? nl + 1 : end;
        }
        while (q < body + hi && q < end && k < count) {
            const char *nl = (const char *)memchr(q, '\n', (size_t)(end - q));
            const char *e = nl ? nl : end;
            int64_t vals[12];
            char msg[160];
            if (int rc = parse_line(q, e, k, vals, msg, sizeof msg)) {
                Err &er = errs[(size_t)t];
                er.line = k;
                er.code = rc;
                memcpy(er.msg, msg, sizeof msg);
                return;
            }
            memcpy(current + 6 * k, vals, 6 * sizeof(int64_t));
            memcpy(initial + 6 * k, vals + 6, 6 * sizeof(int64_t));
            ++k;
            q = nl ? nl + 1 : end;
        }
        if (k == count && q < body + hi && q < end) after[(size_t)t] = q;
    };
    if (nt == 1)
        parse_range(0);
    else
        parallel_ranges(nt, 1, [&](int64_t, int64_t lo, int64_t hi) {
            for (int64_t t = lo; t < hi; ++t) parse_range(t);
        });
    const Err *first = nullptr;
    for (const Err &er : errs)
        if (er.code && (!first || er.line < first->line)) first = &er;
    if (total_lines < count && (!first || first->line >= total_lines))
        return fail(SFB_E_CORRUPT_STREAM_FILE, "truncated file: expected %lld streams",
                    (long long)count);
    if (first) return fail(first->code, "%s", first->msg);
    cur.p = end;
    for (const char *q : after)
        if (q) cur.p = q;
    const char *b, *e;
    if (cur.line(b, e)) {
        for (; b < e; ++b)
            if (!is_ws(*b)) return fail(SFB_E_CORRUPT_STREAM_FILE, "trailing data after last stream");
    }
    // StreamSet.validate (core.py:204-212): ranges first for both arrays, then
    // all-zero triplets, in the reference's order
    const int64_t *arrs[2] = {current, initial};
    const char *what[2] = {"current", "initial"};
    for (int a = 0; a < 2; ++a)
        for (int side = 0; side < 2; ++side) {
            const int64_t m = side == 0 ? kM1 : kM2;
            for (int64_t k = 0; k < count; ++k)
                for (int c = 0; c < 3; ++c) {
                    int64_t v = arrs[a][6 * k + 3 * side + c];
                    if (v < 0 || v >= m)
                        return fail(SFB_E_CORRUPT_STREAM_FILE, "%s state integer outside [0, %lld]",
                                    what[a], (long long)(m - 1));
                }
            for (int64_t k = 0; k < count; ++k) {
                const int64_t *t = arrs[a] + 6 * k + 3 * side;
                if (t[0] == 0 && t[1] == 0 && t[2] == 0)
                    return fail(SFB_E_CORRUPT_STREAM_FILE, "all-zero %s state triplet", what[a]);
            }
        }
    return SFB_OK;
}

/* ---- CPU test hooks -------------------------------------------------------- */
int sfb_host_step_u32(int64_t *states, int64_t n, int64_t steps, int64_t *z_out) {
    for (int64_t w = 0; w < n; ++w) {
        Mrg s = load_state(states + 6 * w);
        int64_t t = 0;
        for (; t + 3 <= steps; t += 3) {  // the rotating-slot form used by the kernels
            uint32_t z0, z1, z2;
            step3(s, z0, z1, z2);
            if (z_out) {
                z_out[w * steps + t] = z0 + 1;
                z_out[w * steps + t + 1] = z1 + 1;
                z_out[w * steps + t + 2] = z2 + 1;
            }
        }
        for (; t < steps; ++t) {
            uint32_t z = step(s);
            if (z_out) z_out[w * steps + t] = z;
        }
        store_state(states + 6 * w, s);
    }
    return SFB_OK;
}

double sfb_host_exp(double x) { return glibc_exp(x, kExpTable); }

double sfb_host_log1p(double x) { return glibc_log1p(x); }

double sfb_host_log1p_fill(double x, int *rare) {
    bool r = false;
    const double v = log1p_fill_domain(x, DivIeee(), r);
    *rare = r ? 1 : 0;
    return v;
}

int sfb_host_fisher_replicates(int64_t *cur, const int64_t *nrowt, int nr, const int64_t *ncolt,
                               int nc, const double *lf, double threshold, int64_t reps,
                               int64_t item_lo, int64_t item_hi, double *stats,
                               int64_t *count) {
    std::vector<int32_t> rowm(nrowt, nrowt + nr), colm(ncolt, ncolt + nc);
    std::vector<int> jw(nc > 1 ? nc - 1 : 1);
    int64_t ntot = 0;
    for (int l = 0; l < nr; ++l) ntot += nrowt[l];
    HostMemo hm;
    const bool use_memo = tune_knob("SFB_FISHER_MEMO", 1) != 0;
    if (use_memo)
        build_memo_set(rowm.data(), nr, colm.data(), nc, (int)ntot, LfPlain{lf}, kExpTable, hm,
                       (size_t)1 << tune_knob("SFB_MEMO_WORDS_LOG2", 25), kMemoSigmas,
                       tune_knob("SFB_FISHER_MEMO_INT", 1) != 0, kMemoIntRadiusMax,
                       (size_t)1 << tune_knob("SFB_MEMO_CELL_PTS_LOG2", 15));
    const MemoSet mp = use_memo ? hm.view() : MemoSet{};
    const int walk = tune_knob("SFB_FISHER_WALK", 3);
    int64_t hits = 0;
    for (int64_t w = item_lo; w < item_hi; ++w) {
        Mrg s = load_state(cur + 6 * w);
        for (int64_t rep = 0; rep < reps; ++rep) {
            const double stat =
                walk == 0 ? sample_table<0>(rowm.data(), colm.data(), nr, nc, (int)ntot,
                                            LfPlain{lf}, kExpTable, s, jw.data(), 1, nullptr, mp)
                : walk == 2 ? sample_table<2>(rowm.data(), colm.data(), nr, nc, (int)ntot,
                                              LfPlain{lf}, kExpTable, s, jw.data(), 1, nullptr, mp)
                : walk == 3 ? sample_table<3>(rowm.data(), colm.data(), nr, nc, (int)ntot,
                                              LfPlain{lf}, kExpTable, s, jw.data(), 1, nullptr, mp)
                            : sample_table<1>(rowm.data(), colm.data(), nr, nc, (int)ntot,
                                              LfPlain{lf}, kExpTable, s, jw.data(), 1, nullptr, mp);
            hits += stat <= threshold;
            if (stats) stats[(w - item_lo) * reps + rep] = stat;
        }
        store_state(cur + 6 * w, s);
    }
    *count = hits;
    return SFB_OK;
}

int sfb_host_box_muller(const int64_t *z1, const int64_t *z2, int64_t n, double *a,
                        double *b) {
    static const uint64_t kLogTab[3 * SFB_BM_LOG_N] = SFB_BM_LOG_TABLE_INIT;
    static const uint64_t kTrigTab[3 * (SFB_BM_TRIG_N + 1)] = SFB_BM_TRIG_TABLE_INIT;
    for (int64_t k = 0; k < n; ++k) {
        if (z1[k] < 1 || z1[k] > (int64_t)kM1 || z2[k] < 1 || z2[k] > (int64_t)kM1)
            return fail(SFB_E_INVALID_ARGUMENT, "draws must lie in [1, m1]");
        box_muller_pair((uint32_t)(z1[k] - 1), (uint32_t)(z2[k] - 1), kLogTab, kTrigTab,
                        a[k], b[k]);
    }
    return SFB_OK;
}

// newton: unused (kept for ABI stability; the float32 form has one sqrt path)
int sfb_host_box_muller_f32(const int64_t *z1, const int64_t *z2, int64_t n, int newton,
                            double seed_rel_err, float *a, float *b) {
    (void)newton;
    static const uint64_t kLogTab[3 * SFB_BM_LOG_N] = SFB_BM_LOG_TABLE_INIT;
    static const uint64_t kTrigTab[3 * (SFB_BM_TRIG_N + 1)] = SFB_BM_TRIG_TABLE_INIT;
    static std::vector<BmPair> logp(kBmFastLogPairs), trigp(kBmFastTrigPairs);
    static std::vector<double> angle(kBmFastTrigPairs);
    static std::once_flag once;
    std::call_once(once, [] {
        bm_fast_tables(kLogTab, kTrigTab, 0, 1, logp.data(), trigp.data(), angle.data());
    });
    const RsqrtSeedModel seed{seed_rel_err};
    for (int64_t k = 0; k < n; ++k) {
        if (z1[k] < 1 || z1[k] > (int64_t)kM1 || z2[k] < 1 || z2[k] > (int64_t)kM1)
            return fail(SFB_E_INVALID_ARGUMENT, "draws must lie in [1, m1]");
        box_muller_pair_f32(uint32_t(z1[k] - 1), uint32_t(z2[k] - 1), logp.data(), trigp.data(),
                            angle.data(), kLogTab, kTrigTab, a[k], b[k], seed);
    }
    return SFB_OK;
}

}  // extern "C"
