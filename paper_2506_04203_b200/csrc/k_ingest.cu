// Trace ingest on the GPU: cascade::read_trace_jsonl (proj/src/domain.cpp:361-387)
// -> SoA columns in HBM, ready for cg_sweep.
//
// Reference semantics: the file is split into lines at '\n' (std::getline;
// a final unterminated line counts, empty lines are skipped but numbered);
// each line is json::parse'd and converted with from_json(TraceRecord)
// (domain.cpp:309-315: arrival_s, input_tokens, per_stage[{output_tokens,
// score}]); require_valid(rec, C of the first record) (domain.cpp:196-209) and
// non-decreasing arrivals (domain.cpp:379-383) are enforced in line order.
//
// Device pipeline (one pass over the bytes for newlines, one parse pass):
//   k_nl_count / k_nl_write   newline positions (block-ordered compaction)
//   k_line_flags + scan        record index of every non-empty line
//   k_parse_lines              one thread per line: a strict JSON scanner for
//                              the trace schema; numbers converted exactly
//                              (integers as static_cast<double>, decimals by
//                              Eisel-Lemire with the 128-bit powers of five, =
//                              correctly rounded strtod for <= 19 digits)
//   k_validate                 require_valid + arrival order per record
// Lines the device scanner cannot decode with certainty (syntax or schema
// errors, escapes or non-ASCII bytes in strings, > 19 significant digits,
// overflow, nesting > 64) are marked and decoded on the host with the
// reference's own JSON library (ingest_host.cpp), which also produces the
// reference's exact error messages.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstring>

#include "cg_cuda.h"
#include "cg_ingest.h"
#include "cg_pow5.h"

namespace cg {

namespace {

constexpr int kIngMaxStages = 16;  // per_stage lengths stored by the device parser
constexpr int NL_THREADS = 256;
constexpr int NL_CHUNK = NL_THREADS * 64;  // bytes per block (64 per thread)
constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_PER_BLOCK = 4 * SCAN_THREADS;

enum : unsigned char { LS_OK = 0, LS_EMPTY = 1, LS_HOST = 2 };

// ---------------------------------------------------------------------------
// newline positions

__device__ __forceinline__ int nl_in_word(unsigned w) {
    const unsigned x = w ^ 0x0a0a0a0au;  // zero byte <=> '\n'
    return ((x & 0xffu) == 0) + ((x & 0xff00u) == 0) + ((x & 0xff0000u) == 0) + ((x & 0xff000000u) == 0);
}

__global__ void __launch_bounds__(NL_THREADS) k_nl_count(const uint4* __restrict__ buf, unsigned* __restrict__ bsum) {
    const uint4* p = buf + (long long)blockIdx.x * (NL_CHUNK / 16) + threadIdx.x * 4;
    int c = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint4 v = __ldg(p + j);
        c += nl_in_word(v.x) + nl_in_word(v.y) + nl_in_word(v.z) + nl_in_word(v.w);
    }
    c = __reduce_add_sync(0xffffffffu, c);
    __shared__ int ws[NL_THREADS / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int i = 0; i < NL_THREADS / 32; ++i) t += ws[i];
        bsum[blockIdx.x] = (unsigned)t;
    }
}

// block-wide exclusive scan of one int per thread (blockDim multiple of 32, <= 1024)
__device__ __forceinline__ int block_excl_scan(int v, int* ws, int& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int incl = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += t;
    }
    if (lane == 31) ws[w] = incl;
    __syncthreads();
    if (w == 0) {
        int s = lane < nw ? ws[lane] : 0;
        int si = s;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, si, off);
            if (lane >= off) si += t;
        }
        if (lane < nw) ws[lane] = si - s;
        if (lane == 31) ws[32] = si;
    }
    __syncthreads();
    const int r = ws[w] + incl - v;
    total = ws[32];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(NL_THREADS) k_nl_write(const uint4* __restrict__ buf, const unsigned* __restrict__ boff,
                                                         long long len, long long* __restrict__ nl) {
    const long long base = (long long)blockIdx.x * NL_CHUNK + threadIdx.x * 64;
    const uint4* p = buf + base / 16;
    unsigned wd[16];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint4 v = __ldg(p + j);
        wd[4 * j] = v.x;
        wd[4 * j + 1] = v.y;
        wd[4 * j + 2] = v.z;
        wd[4 * j + 3] = v.w;
    }
    int c = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) c += nl_in_word(wd[j]);
    __shared__ int ws[33];
    int total;
    long long o = (long long)boff[blockIdx.x] + block_excl_scan(c, ws, total);
    if (!c) return;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            if (((wd[j] >> (8 * b)) & 0xffu) == 0x0au) {
                const long long pos = base + 4 * j + b;
                if (pos < len) nl[o] = pos;
                ++o;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// multi-block exclusive scan of u32

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_blocks(unsigned* __restrict__ a, long long n,
                                                               unsigned* __restrict__ bsum) {
    const long long base = (long long)blockIdx.x * SCAN_PER_BLOCK + threadIdx.x * 4;
    unsigned v[4];
    int s = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        v[j] = base + j < n ? a[base + j] : 0u;
        s += (int)v[j];
    }
    __shared__ int ws[33];
    int total;
    unsigned run = (unsigned)block_excl_scan(s, ws, total);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (base + j < n) a[base + j] = run;
        run += v[j];
    }
    if (threadIdx.x == 0 && bsum) bsum[blockIdx.x] = (unsigned)total;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_single(unsigned* __restrict__ a, long long n,
                                                               unsigned* __restrict__ total_out) {
    __shared__ int ws[33];
    unsigned carry = 0;
    for (long long b0 = 0; b0 < n; b0 += SCAN_THREADS) {
        const long long i = b0 + threadIdx.x;
        const unsigned v = i < n ? a[i] : 0u;
        int tot;
        const unsigned e = (unsigned)block_excl_scan((int)v, ws, tot);
        if (i < n) a[i] = carry + e;
        carry += (unsigned)tot;
    }
    if (threadIdx.x == 0 && total_out) *total_out = carry;
}

__global__ void k_scan_add(unsigned* __restrict__ a, long long n, const unsigned* __restrict__ bsum) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) a[i] += bsum[i / SCAN_PER_BLOCK];
}

void scan_u32(unsigned* a, long long n, unsigned* tmp, unsigned* total, cudaStream_t s, int* launches) {
    const long long nb = (n + SCAN_PER_BLOCK - 1) / SCAN_PER_BLOCK;
    if (nb <= 1) {
        k_scan_single<<<1, SCAN_THREADS, 0, s>>>(a, n, total);
        CG_LAUNCH_CHECK();
        ++*launches;
        return;
    }
    k_scan_blocks<<<(unsigned)nb, SCAN_THREADS, 0, s>>>(a, n, tmp);
    k_scan_single<<<1, SCAN_THREADS, 0, s>>>(tmp, nb, total);
    k_scan_add<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, n, tmp);
    CG_LAUNCH_CHECK();
    *launches += 3;
}

// ---------------------------------------------------------------------------
// per-line JSON scanner

struct Rd {
    const uint4* base;
    long long pos, end;
    long long wa;
    uint4 w;
    __device__ __forceinline__ int peek() {
        if (pos >= end) return -1;
        const long long a = pos >> 4;
        if (a != wa) {
            wa = a;
            w = __ldg(base + a);
        }
        const int q = (int)((pos >> 2) & 3);
        const unsigned word = q == 0 ? w.x : (q == 1 ? w.y : (q == 2 ? w.z : w.w));
        return (int)((word >> ((pos & 3) * 8)) & 0xffu);
    }
    __device__ __forceinline__ void adv() { ++pos; }
    __device__ __forceinline__ void ws() {
        while (true) {
            const int c = peek();
            if (c == ' ' || c == '\t' || c == '\r' || c == '\n') adv();
            else return;
        }
    }
    __device__ __forceinline__ bool eat(int ch) {
        if (peek() != ch) return false;
        adv();
        return true;
    }
};

// Keys of the trace schema, matched while scanning (ASCII, no escapes).
__constant__ char kKeys[5][16] = {"arrival_s", "input_tokens", "per_stage", "output_tokens", "score"};
__constant__ int kKeyLen[5] = {9, 12, 9, 13, 5};

// After the opening quote: scan a string of printable ASCII without escapes.
// Returns -2 when the device leaves the line to the host, else the index of
// the matched schema key among `mask` (bit k = key k allowed) or -1.
__device__ int scan_string(Rd& r, unsigned mask) {
    unsigned viable = mask;
    int i = 0;
    while (true) {
        const int c = r.peek();
        if (c < 0) return -2;
        r.adv();
        if (c == '"') break;
        if (c == '\\' || c < 0x20 || c >= 0x80) return -2;
        if (viable) {
#pragma unroll
            for (int k = 0; k < 5; ++k)
                if ((viable >> k) & 1u)
                    if (i >= kKeyLen[k] || kKeys[k][i] != (char)c) viable &= ~(1u << k);
        }
        ++i;
    }
#pragma unroll
    for (int k = 0; k < 5; ++k)
        if (((viable >> k) & 1u) && kKeyLen[k] == i) return k;
    return -1;
}

__device__ __forceinline__ bool is_digit(int c) { return c >= '0' && c <= '9'; }

// JSON number token -> double with nlohmann's conversion rules.  Returns
// false when the line must go to the host (syntax error, overflow, > 19
// significant digits).
__device__ bool eisel_lemire(unsigned long long w, long long q, unsigned long long& bits);

__device__ bool scan_number(Rd& r, double& out) {
    bool neg = false;
    if (r.peek() == '-') {
        neg = true;
        r.adv();
    }
    unsigned long long w = 0;
    int sig = 0;
    bool big = false, u64_ovf = false;
    long long q = 0;
    int c = r.peek();
    if (c == '0') {
        r.adv();
        if (is_digit(r.peek())) return false;  // leading zero: syntax error
    } else if (c >= '1' && c <= '9') {
        while (is_digit(c = r.peek())) {
            r.adv();
            const unsigned d = (unsigned)(c - '0');
            if (sig < 19) {
                w = w * 10 + d;
                ++sig;
            } else {
                big = true;  // keep exact u64 for 20-digit integers below
                if (sig == 19) {
                    // 20th digit: exact u64 if it fits
                    const unsigned long long hi = __umul64hi(w, 10ull);
                    const unsigned long long lo = w * 10ull;
                    if (hi != 0 || lo + d < lo) u64_ovf = true;
                    else w = lo + d;
                    ++sig;
                } else {
                    u64_ovf = true;
                    ++sig;
                }
            }
        }
    } else {
        return false;
    }
    bool is_int = true;
    if (r.peek() == '.') {
        r.adv();
        is_int = false;
        if (!is_digit(r.peek())) return false;
        while (is_digit(c = r.peek())) {
            r.adv();
            const unsigned d = (unsigned)(c - '0');
            if (big) continue;  // host decodes anyway
            if (w == 0 && d == 0) {
                --q;
            } else if (sig < 19) {
                w = w * 10 + d;
                ++sig;
                --q;
            } else {
                big = true;
            }
        }
    }
    c = r.peek();
    if (c == 'e' || c == 'E') {
        r.adv();
        is_int = false;
        bool eneg = false;
        c = r.peek();
        if (c == '+' || c == '-') {
            eneg = c == '-';
            r.adv();
        }
        if (!is_digit(r.peek())) return false;
        long long e = 0;
        while (is_digit(c = r.peek())) {
            r.adv();
            if (e < 1000000) e = e * 10 + (c - '0');
        }
        q += eneg ? -e : e;
    }
    if (is_int) {
        // strtoull / strtoll semantics (nlohmann lexer), then static_cast<double>
        if (u64_ovf) return false;
        if (!neg) {
            out = __ull2double_rn(w);
        } else {
            if (w > 0x8000000000000000ull) return false;
            out = w == 0 ? 0.0 : -__ull2double_rn(w);  // "-0" is the integer 0
        }
        return true;
    }
    if (big) return false;
    if (w == 0) {
        out = neg ? -0.0 : 0.0;
        return true;
    }
    unsigned long long bits;
    if (!eisel_lemire(w, q, bits)) return false;
    if ((bits & 0x7ff0000000000000ull) == 0x7ff0000000000000ull) return false;  // overflow: parse error 406
    out = __longlong_as_double((long long)(bits | (neg ? 0x8000000000000000ull : 0ull)));
    return true;
}

// Eisel-Lemire (Lemire, "Number Parsing at a Gigabyte per Second", 2021):
// w * 10^q correctly rounded to binary64 for w < 10^19 (w != 0).  The
// 128-bit truncated powers of five kPow5 are generated at build time.
__device__ bool eisel_lemire(unsigned long long w, long long q, unsigned long long& bits) {
    if (q < -342) {
        bits = 0;
        return true;
    }
    if (q > 308) {
        bits = 0x7ff0000000000000ull;
        return true;
    }
    const int lz = __clzll((long long)w);
    w <<= lz;
    const int idx = 2 * (int)(q + 342);
    const unsigned long long t_hi = __ldg(&kPow5[idx]), t_lo = __ldg(&kPow5[idx + 1]);
    unsigned long long lo = w * t_hi;
    unsigned long long hi = __umul64hi(w, t_hi);
    if ((hi & 0x1ffull) == 0x1ffull) {
        const unsigned long long s_hi = __umul64hi(w, t_lo);
        lo += s_hi;
        if (s_hi > lo) ++hi;
    }
    const int upper = (int)(hi >> 63);
    const int shift = upper + 64 - 52 - 3;
    unsigned long long m = hi >> shift;
    int p2 = (int)((((152170 + 65536) * q) >> 16) + 63) + upper - lz + 1023;
    if (p2 <= 0) {  // subnormal
        if (-p2 + 1 >= 64) {
            bits = 0;
            return true;
        }
        m >>= -p2 + 1;
        m += (m & 1ull);
        m >>= 1;
        p2 = (m < (1ull << 52)) ? 0 : 1;
        bits = (m & ((1ull << 52) - 1)) | ((unsigned long long)p2 << 52);
        return true;
    }
    if (lo <= 1 && q >= -4 && q <= 23 && (m & 3ull) == 1ull) {
        if ((m << shift) == hi) m &= ~1ull;  // exactly halfway: round to even
    }
    m += (m & 1ull);
    m >>= 1;
    if (m >= (2ull << 52)) {
        m = 1ull << 52;
        ++p2;
    }
    m &= ~(1ull << 52);
    if (p2 >= 0x7ff) {
        bits = 0x7ff0000000000000ull;
        return true;
    }
    bits = m | ((unsigned long long)p2 << 52);
    return true;
}

// Validating skip of any JSON value (values of keys outside the schema).
__device__ bool skip_value(Rd& r) {
    unsigned long long kinds = 0;  // bit d: container at depth d is an object
    int depth = 0;
    int state = 0;  // 0 value, 1 key, 2 after value
    while (true) {
        if (state == 0) {
            r.ws();
            const int c = r.peek();
            if (c == '"') {
                r.adv();
                if (scan_string(r, 0u) == -2) return false;
                state = 2;
            } else if (c == '-' || is_digit(c)) {
                double d;
                if (!scan_number(r, d)) return false;
                state = 2;
            } else if (c == 't' || c == 'f' || c == 'n') {
                const char* lit = c == 't' ? "true" : (c == 'f' ? "false" : "null");
                for (int i = 0; lit[i]; ++i)
                    if (!r.eat(lit[i])) return false;
                state = 2;
            } else if (c == '[' || c == '{') {
                r.adv();
                r.ws();
                if (r.eat(c == '[' ? ']' : '}')) {
                    state = 2;
                } else {
                    if (depth >= 64) return false;
                    if (c == '{') kinds |= 1ull << depth;
                    else kinds &= ~(1ull << depth);
                    ++depth;
                    state = c == '{' ? 1 : 0;
                }
            } else {
                return false;
            }
        } else if (state == 1) {
            r.ws();
            if (!r.eat('"')) return false;
            if (scan_string(r, 0u) == -2) return false;
            r.ws();
            if (!r.eat(':')) return false;
            state = 0;
        } else {
            if (depth == 0) return true;
            r.ws();
            const bool obj = (kinds >> (depth - 1)) & 1ull;
            if (r.eat(',')) {
                state = obj ? 1 : 0;
            } else if (r.eat(obj ? '}' : ']')) {
                --depth;
            } else {
                return false;
            }
        }
    }
}

// A number in a schema position (anything else is a type error: host).
__device__ __forceinline__ bool schema_number(Rd& r, double& v) {
    r.ws();
    const int c = r.peek();
    if (!(c == '-' || is_digit(c))) return false;
    return scan_number(r, v);
}

struct LineOut {
    long long n;     // record stride of the stage-major columns
    int C0;          // stages stored (first record's per_stage length)
    double* arrival;
    double* in;
    double* out;
    double* scores;
    unsigned char* nst;
};

// One trace line -> record `rec`.  LS_OK or LS_HOST.
__device__ unsigned char parse_record(Rd& r, long long rec, const LineOut& o) {
    // UTF-8 byte order mark (nlohmann skips it at the start of the input)
    if (r.peek() == 0xEF) {
        if (!(r.eat(0xEF) && r.eat(0xBB) && r.eat(0xBF))) return LS_HOST;
    }
    r.ws();
    if (!r.eat('{')) return LS_HOST;
    bool has_arr = false, has_in = false, has_ps = false;
    double arr = 0, in = 0;
    int nst = 0;
    r.ws();
    if (r.peek() == '}') return LS_HOST;  // no keys: out_of_range 403
    while (true) {
        r.ws();
        if (!r.eat('"')) return LS_HOST;
        const int key = scan_string(r, 0x7u);
        if (key == -2) return LS_HOST;
        r.ws();
        if (!r.eat(':')) return LS_HOST;
        if (key == 0) {
            if (!schema_number(r, arr)) return LS_HOST;
            has_arr = true;
        } else if (key == 1) {
            if (!schema_number(r, in)) return LS_HOST;
            has_in = true;
        } else if (key == 2) {
            r.ws();
            if (!r.eat('[')) return LS_HOST;
            has_ps = true;
            nst = 0;
            r.ws();
            if (!r.eat(']')) {
                while (true) {
                    r.ws();
                    if (!r.eat('{')) return LS_HOST;
                    bool ho = false, hs = false;
                    double ov = 0, sv = 0;
                    r.ws();
                    if (r.peek() == '}') return LS_HOST;
                    while (true) {
                        r.ws();
                        if (!r.eat('"')) return LS_HOST;
                        const int k2 = scan_string(r, 0x18u);
                        if (k2 == -2) return LS_HOST;
                        r.ws();
                        if (!r.eat(':')) return LS_HOST;
                        if (k2 == 3) {
                            if (!schema_number(r, ov)) return LS_HOST;
                            ho = true;
                        } else if (k2 == 4) {
                            if (!schema_number(r, sv)) return LS_HOST;
                            hs = true;
                        } else {
                            if (!skip_value(r)) return LS_HOST;
                        }
                        r.ws();
                        if (r.eat(',')) continue;
                        if (r.eat('}')) break;
                        return LS_HOST;
                    }
                    if (!(ho && hs)) return LS_HOST;
                    if (nst >= kIngMaxStages * 16) return LS_HOST;
                    if (nst < o.C0) {
                        o.out[(long long)nst * o.n + rec] = ov;
                        o.scores[(long long)nst * o.n + rec] = sv;
                    }
                    ++nst;
                    r.ws();
                    if (r.eat(',')) continue;
                    if (r.eat(']')) break;
                    return LS_HOST;
                }
            }
        } else {
            if (!skip_value(r)) return LS_HOST;
        }
        r.ws();
        if (r.eat(',')) continue;
        if (r.eat('}')) break;
        return LS_HOST;
    }
    r.ws();
    if (r.peek() != -1) return LS_HOST;  // trailing content
    if (!(has_arr && has_in && has_ps)) return LS_HOST;
    if (o.arrival) {
        o.arrival[rec] = arr;
        o.in[rec] = in;
        o.nst[rec] = (unsigned char)(nst > 255 ? 255 : nst);
    } else {
        o.nst[0] = (unsigned char)(nst > 255 ? 255 : nst);
    }
    return LS_OK;
}

__device__ __forceinline__ void line_span(const long long* __restrict__ nl, long long total_nl, long long len,
                                          long long i, long long& b, long long& e) {
    b = i == 0 ? 0 : nl[i - 1] + 1;
    e = i < total_nl ? nl[i] : len;
}

__global__ void k_line_flags(const long long* __restrict__ nl, long long total_nl, long long len, long long L,
                             unsigned* __restrict__ flag) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= L) return;
    long long b, e;
    line_span(nl, total_nl, len, i, b, e);
    flag[i] = e > b ? 1u : 0u;
}

__global__ void __launch_bounds__(128) k_parse_lines(const uint4* __restrict__ buf, const long long* __restrict__ nl,
                                                    long long total_nl, long long len, long long L0, long long L1,
                                                    const unsigned* __restrict__ lrec, LineOut o,
                                                    unsigned char* __restrict__ status,
                                                    unsigned long long* __restrict__ recline,
                                                    unsigned long long* __restrict__ hostlist,
                                                    unsigned long long* __restrict__ hostcount) {
    const long long i = L0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= L1) return;
    long long b, e;
    line_span(nl, total_nl, len, i, b, e);
    unsigned char st;
    if (e <= b) {
        st = LS_EMPTY;
    } else {
        Rd r{buf, b, e, -1, make_uint4(0, 0, 0, 0)};
        const long long rec = lrec[i];
        st = parse_record(r, rec, o);
        if (recline) recline[rec] = (unsigned long long)i;
        if (st == LS_HOST && hostlist) {
            const unsigned long long k = atomicAdd(hostcount, 1ull);
            hostlist[k] = (unsigned long long)i;
        }
    }
    if (status) status[i] = st;
}

// require_valid(TraceRecord, C0) and the arrival order, per record; the first
// offending line (file order) wins.
__global__ void k_validate(LineOut o, const unsigned long long* __restrict__ recline,
                           unsigned long long* __restrict__ first_bad) {
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= o.n) return;
    bool bad = o.in[r] < 0.0;
    const int ns = o.nst[r];
    if (r > 0 && ns != o.C0) bad = true;
    const int m = ns < o.C0 ? ns : o.C0;
    for (int k = 0; k < m; ++k) {
        const double ov = o.out[(long long)k * o.n + r], sv = o.scores[(long long)k * o.n + r];
        bad |= ov < 0.0 || sv < 0.0 || sv > 100.0;
    }
    if (r > 0 && o.arrival[r] < o.arrival[r - 1]) bad = true;
    if (bad) atomicMin(first_bad, recline[r]);
}

double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

void ingest_jsonl(IngestBuffers& B, cudaStream_t s, const char* bytes, long long len, const std::string& path,
                  IngestOut& out) {
    const auto t0 = std::chrono::steady_clock::now();
    out = IngestOut{};
    int& launches = out.launches;
    if (len <= 0) return;  // empty file: empty trace
    const long long nchunks = (len + NL_CHUNK - 1) / NL_CHUNK;
    const size_t padded = (size_t)nchunks * NL_CHUNK + 16;
    char* dbytes = static_cast<char*>(B.bytes.reserve(padded));
    CG_CUDA(cudaMemcpyAsync(dbytes, bytes, (size_t)len, cudaMemcpyHostToDevice, s));
    CG_CUDA(cudaMemsetAsync(dbytes + len, 0, padded - (size_t)len, s));
    const uint4* buf = reinterpret_cast<const uint4*>(dbytes);

    // ---- newlines
    unsigned* bsum = B.bsum.as<unsigned>((size_t)nchunks + 64);
    unsigned* misc = B.misc.as<unsigned>(64);
    k_nl_count<<<(unsigned)nchunks, NL_THREADS, 0, s>>>(buf, bsum);
    CG_LAUNCH_CHECK();
    ++launches;
    k_scan_single<<<1, SCAN_THREADS, 0, s>>>(bsum, nchunks, misc);
    CG_LAUNCH_CHECK();
    ++launches;
    unsigned total_nl_u = 0;
    char last = 0;
    CG_CUDA(cudaMemcpyAsync(&total_nl_u, misc, 4, cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaStreamSynchronize(s));
    last = bytes[len - 1];
    const long long total_nl = total_nl_u;
    long long* nl = B.nl.as<long long>((size_t)total_nl + 1);
    k_nl_write<<<(unsigned)nchunks, NL_THREADS, 0, s>>>(buf, bsum, len, nl);
    CG_LAUNCH_CHECK();
    ++launches;
    const long long L = total_nl + (last != '\n' ? 1 : 0);
    out.lines = L;
    if (L == 0) return;

    // ---- record index of every line
    unsigned* lrec = B.lrec.as<unsigned>((size_t)L);
    k_line_flags<<<(unsigned)((L + 255) / 256), 256, 0, s>>>(nl, total_nl, len, L, lrec);
    CG_LAUNCH_CHECK();
    ++launches;
    unsigned* stmp = B.misc.as<unsigned>((size_t)(L + SCAN_PER_BLOCK - 1) / SCAN_PER_BLOCK + 64);
    misc = stmp;  // B.misc may have moved
    unsigned* ntot = stmp + (L + SCAN_PER_BLOCK - 1) / SCAN_PER_BLOCK + 8;
    scan_u32(lrec, L, stmp, ntot, s, &launches);
    unsigned n_u = 0;
    CG_CUDA(cudaMemcpyAsync(&n_u, ntot, 4, cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaStreamSynchronize(s));
    const long long n = n_u;
    if (n == 0) return;  // only empty lines

    // ---- first record: its per_stage length is C (require_valid, domain.cpp:198-200)
    long long first_line = 0;
    {
        // first non-empty line: scan the host bytes (cheap, stops at the first non-'\n')
        long long p = 0;
        while (p < len && bytes[p] == '\n') {
            ++p;
            ++first_line;
        }
    }
    unsigned char* status = B.status.as<unsigned char>((size_t)L);
    unsigned char* nst = B.nst.as<unsigned char>((size_t)n);
    unsigned long long* recline = B.recline.as<unsigned long long>((size_t)n);
    unsigned long long* hostlist = B.hostlist.as<unsigned long long>((size_t)L + 2);
    unsigned long long* hostcount = hostlist + L;
    unsigned long long* first_bad = hostlist + L + 1;
    int C0 = 0;
    {
        LineOut o1{};
        o1.nst = nst;
        k_parse_lines<<<1, 1, 0, s>>>(buf, nl, total_nl, len, first_line, first_line + 1, lrec, o1, status, nullptr,
                                      nullptr, nullptr);
        CG_LAUNCH_CHECK();
        ++launches;
        unsigned char h[2];
        CG_CUDA(cudaMemcpyAsync(&h[0], status + first_line, 1, cudaMemcpyDeviceToHost, s));
        CG_CUDA(cudaMemcpyAsync(&h[1], nst, 1, cudaMemcpyDeviceToHost, s));
        CG_CUDA(cudaStreamSynchronize(s));
        if (h[0] == LS_OK && h[1] <= kIngMaxStages) {
            C0 = h[1];
        } else {
            // host decode of the first record (or its error)
            long long b = 0, e = 0;
            {
                const char* nlp = static_cast<const char*>(std::memchr(bytes + first_line, '\n', (size_t)(len - first_line)));
                b = first_line;
                e = nlp ? (long long)(nlp - bytes) : len;
            }
            HostRecord rec;
            std::string msg;
            if (!host_parse_trace_line(bytes + b, (size_t)(e - b), path, first_line + 1, rec, msg))
                throw EngineError(0, msg);
            C0 = (int)rec.score.size();
            if (C0 > kIngMaxStages)
                throw EngineError(101, "trace ingest: more than 16 cascade stages per record");
        }
    }
    out.n = n;
    out.stages = C0;

    // ---- all lines
    double* d_arr = B.arrival.as<double>((size_t)n);
    double* d_in = B.in.as<double>((size_t)n);
    double* d_out = B.out.as<double>((size_t)std::max(1, C0) * n);
    double* d_sc = B.scores.as<double>((size_t)std::max(1, C0) * n);
    LineOut o{n, C0, d_arr, d_in, d_out, d_sc, nst};
    CG_CUDA(cudaMemsetAsync(hostcount, 0, 8, s));
    CG_CUDA(cudaMemsetAsync(first_bad, 0xff, 8, s));
    k_parse_lines<<<(unsigned)((L + 127) / 128), 128, 0, s>>>(buf, nl, total_nl, len, 0, L, lrec, o, status, recline,
                                                              hostlist, hostcount);
    CG_LAUNCH_CHECK();
    ++launches;
    unsigned long long nhost = 0;
    CG_CUDA(cudaMemcpyAsync(&nhost, hostcount, 8, cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaStreamSynchronize(s));
    out.host_lines = (long long)nhost;

    // ---- lines left to the host: decode in file order until the first error
    long long host_err_line = -1;
    std::string host_err;
    if (nhost) {
        std::vector<unsigned long long> hl(nhost);
        CG_CUDA(cudaMemcpyAsync(hl.data(), hostlist, nhost * 8, cudaMemcpyDeviceToHost, s));
        std::vector<long long> starts(nhost), ends(nhost);
        std::vector<unsigned> recs(nhost);
        CG_CUDA(cudaStreamSynchronize(s));
        std::sort(hl.begin(), hl.end());
        for (size_t k = 0; k < nhost; ++k) {
            const long long i = (long long)hl[k];
            long long b = 0, e = len;
            if (i > 0) CG_CUDA(cudaMemcpyAsync(&b, nl + i - 1, 8, cudaMemcpyDeviceToHost, s));
            if (i < total_nl) CG_CUDA(cudaMemcpyAsync(&e, nl + i, 8, cudaMemcpyDeviceToHost, s));
            CG_CUDA(cudaMemcpyAsync(&recs[k], lrec + i, 4, cudaMemcpyDeviceToHost, s));
            CG_CUDA(cudaStreamSynchronize(s));
            if (i > 0) b += 1;
            HostRecord rec;
            std::string msg;
            if (!host_parse_trace_line(bytes + b, (size_t)(e - b), path, i + 1, rec, msg)) {
                host_err_line = i;
                host_err = msg;
                break;
            }
            // patch the record into the device columns (stages beyond C0 are
            // irrelevant: a length mismatch fails validation)
            const long long r = recs[k];
            const unsigned char ns = (unsigned char)std::min<size_t>(rec.score.size(), 255);
            CG_CUDA(cudaMemcpyAsync(d_arr + r, &rec.arrival_s, 8, cudaMemcpyHostToDevice, s));
            CG_CUDA(cudaMemcpyAsync(d_in + r, &rec.input_tokens, 8, cudaMemcpyHostToDevice, s));
            CG_CUDA(cudaMemcpyAsync(nst + r, &ns, 1, cudaMemcpyHostToDevice, s));
            for (int st = 0; st < C0 && st < (int)rec.score.size(); ++st) {
                CG_CUDA(cudaMemcpyAsync(d_out + (long long)st * n + r, &rec.output_tokens[st], 8,
                                        cudaMemcpyHostToDevice, s));
                CG_CUDA(cudaMemcpyAsync(d_sc + (long long)st * n + r, &rec.score[st], 8, cudaMemcpyHostToDevice, s));
            }
            CG_CUDA(cudaStreamSynchronize(s));  // the host record dies here
        }
    }

    // ---- validation + order, first offending line
    k_validate<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(o, recline, first_bad);
    CG_LAUNCH_CHECK();
    ++launches;
    unsigned long long fb = ~0ull;
    CG_CUDA(cudaMemcpyAsync(&fb, first_bad, 8, cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaStreamSynchronize(s));
    long long err_line = fb == ~0ull ? -1 : (long long)fb;
    if (host_err_line >= 0 && (err_line < 0 || host_err_line < err_line)) throw EngineError(0, host_err);
    if (err_line >= 0) {
        // the reference's message for this line (host decode of one line)
        long long b = 0, e = len;
        unsigned r = 0;
        if (err_line > 0) CG_CUDA(cudaMemcpyAsync(&b, nl + err_line - 1, 8, cudaMemcpyDeviceToHost, s));
        if (err_line < total_nl) CG_CUDA(cudaMemcpyAsync(&e, nl + err_line, 8, cudaMemcpyDeviceToHost, s));
        CG_CUDA(cudaMemcpyAsync(&r, lrec + err_line, 4, cudaMemcpyDeviceToHost, s));
        CG_CUDA(cudaStreamSynchronize(s));
        if (err_line > 0) b += 1;
        HostRecord rec;
        std::string msg;
        if (!host_parse_trace_line(bytes + b, (size_t)(e - b), path, err_line + 1, rec, msg))
            throw EngineError(0, msg);
        const std::string prob = host_record_problems(rec, r == 0 ? -1 : C0);
        if (!prob.empty()) throw EngineError(0, prob);
        throw EngineError(0, path + ":" + std::to_string(err_line + 1) + ": arrival times must be non-decreasing");
    }
    out.d_arrival = d_arr;
    out.d_in = d_in;
    out.d_out = d_out;
    out.d_scores = d_sc;
    out.ms_total = ms_since(t0);
}

}  // namespace cg
