// Byte-exact JSON text of the planner's result types, as nlohmann::json's
// dump(indent) writes them (the reference's output files, cli.cpp:121,165-175).
//
// Doubles follow nlohmann's serializer exactly: non-finite -> "null"; +-0 ->
// "0.0"/"-0.0"; otherwise the Grisu2 digits of Loitsch's algorithm with a
// 64-bit diy_fp and the cached powers 10^k, k = -300 + 8i (nlohmann
// detail::dtoa_impl), formatted with kMinExp = -4 / kMaxExp = 15 (".0"
// appended to integral values, "e+XX" exponents with at least two digits).
// The same code runs on the host (glue, tests against nlohmann) and device.
#pragma once

#include <stdint.h>

#ifndef __CUDACC__
#ifndef __host__
#define __host__
#endif
#ifndef __device__
#define __device__
#endif
#endif

#include "cg_dtoa_tables.h"  // generated: kCachedPow{F,E,K}[_dev]

namespace cg {
namespace json {

struct Diy {
    uint64_t f;
    int e;
};

__host__ __device__ inline uint64_t umulhi(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// diyfp::mul: upper 64 bits of the 128-bit product, rounded half up.
__host__ __device__ inline Diy dmul(Diy x, Diy y) {
    const uint64_t lo = x.f * y.f;
    return Diy{umulhi(x.f, y.f) + (lo >> 63), x.e + y.e + 64};
}

__host__ __device__ inline Diy normalize(Diy x) {
    while ((x.f >> 63) == 0) {
        x.f <<= 1;
        x.e--;
    }
    return x;
}

__host__ __device__ inline int find_largest_pow10(uint32_t n, uint32_t& pow10) {
    if (n >= 1000000000u) { pow10 = 1000000000u; return 10; }
    if (n >= 100000000u) { pow10 = 100000000u; return 9; }
    if (n >= 10000000u) { pow10 = 10000000u; return 8; }
    if (n >= 1000000u) { pow10 = 1000000u; return 7; }
    if (n >= 100000u) { pow10 = 100000u; return 6; }
    if (n >= 10000u) { pow10 = 10000u; return 5; }
    if (n >= 1000u) { pow10 = 1000u; return 4; }
    if (n >= 100u) { pow10 = 100u; return 3; }
    if (n >= 10u) { pow10 = 10u; return 2; }
    pow10 = 1;
    return 1;
}

__host__ __device__ inline void grisu2_round(char* buf, int len, uint64_t dist, uint64_t delta, uint64_t rest,
                                             uint64_t ten_k) {
    while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
        buf[len - 1]--;
        rest += ten_k;
    }
}

// Digits of v (finite, > 0) into buf (<= 17 chars); returns the digit count,
// decimal_exponent such that v ~= digits * 10^decimal_exponent.
__host__ __device__ inline int grisu2(char* buf, int& decimal_exponent, double value) {
    uint64_t bits;
#ifdef __CUDA_ARCH__
    bits = (uint64_t)__double_as_longlong(value);
#else
    __builtin_memcpy(&bits, &value, 8);
#endif
    const uint64_t E = bits >> 52, F = bits & ((1ull << 52) - 1);
    const Diy v = E == 0 ? Diy{F, 1 - 1075} : Diy{F + (1ull << 52), (int)E - 1075};
    const bool lower_closer = F == 0 && E > 1;
    const Diy m_plus{2 * v.f + 1, v.e - 1};
    const Diy m_minus = lower_closer ? Diy{4 * v.f - 1, v.e - 2} : Diy{2 * v.f - 1, v.e - 1};
    const Diy w_plus = normalize(m_plus);
    const Diy w_minus{m_minus.f << (m_minus.e - w_plus.e), w_plus.e};
    const Diy vn = normalize(v);
    // cached power: -60 <= e_c + e + 64 <= -32
    const int f = -60 - w_plus.e - 1;
    const int k = (f * 78913) / (1 << 18) + (f > 0 ? 1 : 0);
    const int index = (300 + k + 7) / 8;
#ifdef __CUDA_ARCH__
    const Diy c{kCachedPowF_dev[index], kCachedPowE_dev[index]};
    const int ck = kCachedPowK_dev[index];
#else
    const Diy c{kCachedPowF[index], kCachedPowE[index]};
    const int ck = kCachedPowK[index];
#endif
    const Diy w = dmul(vn, c);
    const Diy wm = dmul(w_minus, c);
    const Diy wp = dmul(w_plus, c);
    const Diy Mm{wm.f + 1, wm.e};
    const Diy Mp{wp.f - 1, wp.e};
    decimal_exponent = -ck;
    // digit generation
    uint64_t delta = Mp.f - Mm.f;
    uint64_t dist = Mp.f - w.f;
    const int sh = -Mp.e;
    const uint64_t one_f = 1ull << sh;
    uint32_t p1 = (uint32_t)(Mp.f >> sh);
    uint64_t p2 = Mp.f & (one_f - 1);
    uint32_t pow10 = 0;
    int n = find_largest_pow10(p1, pow10);
    int len = 0;
    while (n > 0) {
        const uint32_t d = p1 / pow10;
        const uint32_t r = p1 % pow10;
        buf[len++] = (char)('0' + d);
        p1 = r;
        n--;
        const uint64_t rest = ((uint64_t)p1 << sh) + p2;
        if (rest <= delta) {
            decimal_exponent += n;
            grisu2_round(buf, len, dist, delta, rest, (uint64_t)pow10 << sh);
            return len;
        }
        pow10 /= 10;
    }
    int m = 0;
    for (;;) {
        p2 *= 10;
        const uint64_t d = p2 >> sh;
        const uint64_t r = p2 & (one_f - 1);
        buf[len++] = (char)('0' + d);
        p2 = r;
        m++;
        delta *= 10;
        dist *= 10;
        if (p2 <= delta) break;
    }
    decimal_exponent -= m;
    grisu2_round(buf, len, dist, delta, p2, one_f);
    return len;
}

// nlohmann detail::to_chars for a finite double: writes <= 25 chars, returns length.
__host__ __device__ inline int dtoa(char* out, double value) {
    int p = 0;
    uint64_t bits;
#ifdef __CUDA_ARCH__
    bits = (uint64_t)__double_as_longlong(value);
#else
    __builtin_memcpy(&bits, &value, 8);
#endif
    if (bits >> 63) {
        out[p++] = '-';
        bits &= ~(1ull << 63);
    }
    if (bits == 0) {
        out[p++] = '0';
        out[p++] = '.';
        out[p++] = '0';
        return p;
    }
    double a;
#ifdef __CUDA_ARCH__
    a = __longlong_as_double((long long)bits);
#else
    __builtin_memcpy(&a, &bits, 8);
#endif
    char d[20];
    int dexp = 0;
    const int k = grisu2(d, dexp, a);
    const int n = k + dexp;
    if (k <= n && n <= 15) {
        for (int i = 0; i < k; ++i) out[p++] = d[i];
        for (int i = k; i < n; ++i) out[p++] = '0';
        out[p++] = '.';
        out[p++] = '0';
        return p;
    }
    if (0 < n && n <= 15) {
        for (int i = 0; i < n; ++i) out[p++] = d[i];
        out[p++] = '.';
        for (int i = n; i < k; ++i) out[p++] = d[i];
        return p;
    }
    if (-4 < n && n <= 0) {
        out[p++] = '0';
        out[p++] = '.';
        for (int i = 0; i < -n; ++i) out[p++] = '0';
        for (int i = 0; i < k; ++i) out[p++] = d[i];
        return p;
    }
    out[p++] = d[0];
    if (k > 1) {
        out[p++] = '.';
        for (int i = 1; i < k; ++i) out[p++] = d[i];
    }
    out[p++] = 'e';
    int e = n - 1;
    if (e < 0) {
        e = -e;
        out[p++] = '-';
    } else {
        out[p++] = '+';
    }
    if (e < 10) {
        out[p++] = '0';
        out[p++] = (char)('0' + e);
    } else if (e < 100) {
        out[p++] = (char)('0' + e / 10);
        out[p++] = (char)('0' + e % 10);
    } else {
        out[p++] = (char)('0' + e / 100);
        out[p++] = (char)('0' + (e / 10) % 10);
        out[p++] = (char)('0' + e % 10);
    }
    return p;
}

// Text sink: counts (buf == nullptr) or writes.
struct Out {
    char* buf;
    long long n;
    __host__ __device__ inline void ch(char c) {
        if (buf) buf[n] = c;
        ++n;
    }
    __host__ __device__ inline void str(const char* s) {
        while (*s) ch(*s++);
    }
    __host__ __device__ inline void spaces(int k) {
        for (int i = 0; i < k; ++i) ch(' ');
    }
    __host__ __device__ inline void i64(long long v) {
        char t[24];
        int k = 0;
        unsigned long long u = v < 0 ? 0ull - (unsigned long long)v : (unsigned long long)v;
        do {
            t[k++] = (char)('0' + u % 10);
            u /= 10;
        } while (u);
        if (v < 0) ch('-');
        while (k) ch(t[--k]);
    }
    __host__ __device__ inline void dbl(double x) {
        uint64_t b;
#ifdef __CUDA_ARCH__
        b = (uint64_t)__double_as_longlong(x);
#else
        __builtin_memcpy(&b, &x, 8);
#endif
        if ((b & 0x7ff0000000000000ull) == 0x7ff0000000000000ull) {
            str("null");
            return;
        }
        char t[32];
        const int k = dtoa(t, x);
        for (int i = 0; i < k; ++i) ch(t[i]);
    }
    // "key": (at the object's member indentation)
    __host__ __device__ inline void key(int ind, const char* k) {
        spaces(ind);
        ch('"');
        str(k);
        str("\": ");
    }
    // member separator: ",\n" or "\n" + closing indentation handled by caller
    __host__ __device__ inline void sep(bool last) {
        if (!last) ch(',');
        ch('\n');
    }
};

// Array with nlohmann's pretty layout at indentation `ind` (the value starts
// after "key": ; elements at ind + step).  compact: "[a,b,c]" on one line --
// what the nlohmann build shipped in this image (cudnn-frontend's copy of
// 3.11.3) does for arrays whose first element is an integer; upstream 3.11.3
// prints them pretty like any other array (see cg_sweep_result_json flags).
template <class F>
__host__ __device__ inline void array_of(Out& o, int ind, int step, long long count, F&& elem,
                                         bool compact = false) {
    if (count == 0) {
        o.str("[]");
        return;
    }
    if (compact) {
        o.ch('[');
        for (long long i = 0; i < count; ++i) {
            if (i) o.ch(',');
            elem(i);
        }
        o.ch(']');
        return;
    }
    o.str("[\n");
    for (long long i = 0; i < count; ++i) {
        o.spaces(ind + step);
        elem(i);
        o.sep(i + 1 == count);
    }
    o.spaces(ind);
    o.ch(']');
}

// Flattened result view (device or host pointers).
struct ResultView {
    int C;
    int compact_ints;         // integer arrays on one line (see array_of)
    const double* thr;        // [E][C-1]
    const double* lat;        // [E]
    const double* qual;       // [E]
    const double* ratios;     // [E][C]
    const int* alloc;         // [E][C]
    const long long* eplan;   // [E][C] -1 = null
    const int* plan_gpus;     // [P]
    const int* plan_dp;       // [P]
    const long long* plan_off;  // [P]
    const int* rep_tp;        // [R]
    const int* rep_pp;        // [R]
};

// RoutingThresholds {"thresholds": [...]} as an object value at `ind`.
__host__ __device__ inline void emit_thresholds(Out& o, int ind, int step, const double* h, int D) {
    o.str("{\n");
    o.key(ind + step, "thresholds");
    array_of(o, ind + step, step, D, [&](long long i) { o.dbl(h[i]); });
    o.ch('\n');
    o.spaces(ind);
    o.ch('}');
}

// ParallelismPlan {"gpus_used", "replicas": [{"pp","tp"}]} at `ind`.
__host__ __device__ inline void emit_plan(Out& o, int ind, int step, const ResultView& r, long long p) {
    if (p < 0) {
        o.str("null");
        return;
    }
    o.str("{\n");
    o.key(ind + step, "gpus_used");
    o.i64(r.plan_gpus[p]);
    o.sep(false);
    o.key(ind + step, "replicas");
    const long long off = r.plan_off[p];
    array_of(o, ind + step, step, r.plan_dp[p], [&](long long k) {
        const int rind = ind + 2 * step;
        o.str("{\n");
        o.key(rind + step, "pp");
        o.i64(r.rep_pp[off + k]);
        o.sep(false);
        o.key(rind + step, "tp");
        o.i64(r.rep_tp[off + k]);
        o.ch('\n');
        o.spaces(rind);
        o.ch('}');
    });
    o.ch('\n');
    o.spaces(ind);
    o.ch('}');
}

// CascadePlan of evaluation e at `ind` (keys sorted as nlohmann's std::map).
__host__ __device__ inline void emit_cascade_plan(Out& o, int ind, int step, const ResultView& r, long long e) {
    const int C = r.C, D = C - 1;
    const int mi = ind + step;
    o.str("{\n");
    o.key(mi, "allocations");
    array_of(o, mi, step, C, [&](long long i) { o.i64(r.alloc[e * C + i]); }, r.compact_ints != 0);
    o.sep(false);
    o.key(mi, "plans");
    array_of(o, mi, step, C, [&](long long i) { emit_plan(o, mi + step, step, r, r.eplan[e * C + i]); });
    o.sep(false);
    o.key(mi, "predicted_max_p95_s");
    o.dbl(r.lat[e]);
    o.sep(false);
    o.key(mi, "predicted_quality");
    o.dbl(r.qual[e]);
    o.sep(false);
    o.key(mi, "processing_ratios");
    array_of(o, mi, step, C, [&](long long i) { o.dbl(r.ratios[e * C + i]); });
    o.sep(false);
    o.key(mi, "thresholds");
    emit_thresholds(o, mi, step, r.thr + e * D, D);
    o.ch('\n');
    o.spaces(ind);
    o.ch('}');
}

// ObjectivePoint of evaluation e at `ind`.
__host__ __device__ inline void emit_point(Out& o, int ind, int step, const ResultView& r, long long e) {
    const int D = r.C - 1;
    const int mi = ind + step;
    o.str("{\n");
    o.key(mi, "latency_s");
    o.dbl(r.lat[e]);
    o.sep(false);
    o.key(mi, "plan_ref");
    emit_cascade_plan(o, mi, step, r, e);
    o.sep(false);
    o.key(mi, "quality");
    o.dbl(r.qual[e]);
    o.sep(false);
    o.key(mi, "thresholds");
    emit_thresholds(o, mi, step, r.thr + e * D, D);
    o.ch('\n');
    o.spaces(ind);
    o.ch('}');
}

}  // namespace json
}  // namespace cg
