// K1-K3 and K2: threshold routing, aggregation, nearest-rank p95 and
// trace-order quality for every threshold candidate of a sweep at once.
//
// Reference semantics (proj/src/routing.cpp:42-93, util.cpp:11-29):
//   a request accepts at the first stage i < C-1 with score_i >= h_i, else at
//   the last stage; stage i is reached by every request accepting at >= i;
//   ratios_i = |reached_i| / n; WorkloadStats_i = (rate * ratio_i, trace-order
//   means of input / stage-i output tokens, nearest-rank p95 of both);
//   quality = (trace-order sum of accepted scores) / n.
//
// Batched formulation: per threshold dimension d the distinct grid values
// V_d (sorted) induce rank_d(r) = #{v in V_d : v <= score_d(r)}; request r
// reaches stage i under distinct-index prefix (m_0..m_{i-1}) iff
// rank_d(r) <= m_d for all d < i.  So every stage workload of every candidate
// is a dominance region of the (C-1)-dim rank histogram:
//   K1  one streaming pass: ranks + histogram of (count, sum_in, sum_out_i)
//   dominance prefix sums over the histogram (tiny)
//   K3  p95: token columns radix-sorted once (k_sort.cu); each workload scans
//       its column from the top, counting members with ballot/popc, until the
//       nearest-rank position is reached (selection by value, H4)
//   K2  quality is NOT order-independent in fp64 (H1): one thread per
//       distinct threshold tuple adds the accepted scores in trace order over
//       shared-memory staged request tiles (bit-exact with the reference).
// Token sums are exact int64 when every token is an integer in [0, 2^32)
// and the column totals are < 2^53 (then the reference's sequential double
// sum is exact too); otherwise a trace-order fp64 fallback is used.
#include <cuda_runtime.h>

#include "cg_cuda.h"
#include "cg_internal.h"
#include "cg_kernels.h"

namespace cg {

namespace {

__device__ __forceinline__ int rank_of(const double* __restrict__ v, int g, double s) {
    // #{v <= s}: upper_bound with predicate (v <= s); NaN scores rank 0.
    int lo = 0, hi = g;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (v[mid] <= s) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ bool token_ok(double x) {
    return x >= 0.0 && x < 4294967296.0 && x == trunc(x);
}

template <int D>
__global__ void __launch_bounds__(256) k_route_aggregate(RouteArgs a) {
    extern __shared__ double s_grid[];
    const double* gv = a.gvals;
    if (a.grid_in_smem) {
        for (int i = threadIdx.x; i < a.gtotal; i += blockDim.x) s_grid[i] = a.gvals[i];
        __syncthreads();
        gv = s_grid;
    }
    const int C = D + 1;
    const int Q = 2 + C;
    bool bad = false;
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < a.n;
         r += (long long)gridDim.x * blockDim.x) {
        unsigned long long packed = 0;
        long long cell = 0;
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const double s = __ldg(&a.scores[(long long)d * a.n + r]);
            const int rk = rank_of(gv + a.goff[d], a.G[d], s);
            packed |= (unsigned long long)rk << (16 * d);
            cell += (long long)rk * a.stride[d];
        }
        a.ranks[r] = packed;
        const double xin = __ldg(&a.in[r]);
        bad |= !token_ok(xin);
        unsigned long long* h = a.hist + cell * Q;
        atomicAdd(&h[0], 1ull);
        atomicAdd(&h[1], (unsigned long long)(xin >= 0.0 && xin < 4294967296.0 ? xin : 0.0));
#pragma unroll
        for (int i = 0; i < C; ++i) {
            const double xo = __ldg(&a.out[(long long)i * a.n + r]);
            bad |= !token_ok(xo);
            atomicAdd(&h[2 + i], (unsigned long long)(xo >= 0.0 && xo < 4294967296.0 ? xo : 0.0));
        }
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(a.flags, 1u);
}

// Inclusive prefix sums along dimension d of the (G_d+1)-extent histogram.
__global__ void k_hist_scan_dim(unsigned long long* __restrict__ hist, long long cells, int Q,
                                long long stride, int extent) {
    const long long lines = cells / extent;
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= lines * Q) return;
    const int q = (int)(t % Q);
    const long long line = t / Q;
    const long long low = line % stride, high = line / stride;
    const long long base = high * stride * extent + low;
    unsigned long long run = 0;
    for (int k = 0; k < extent; ++k) {
        unsigned long long* p = hist + (base + (long long)k * stride) * Q + q;
        run += *p;
        *p = run;
    }
}

// Per (stage i, workload w): count and integer token sums from the
// dominance-summed histogram.
__global__ void k_workload_counts(WorkloadArgs a) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= a.total) return;
    int i = 0;
    while (i + 1 < a.C && t >= a.wl_off[i + 1]) ++i;
    long long w = t - a.wl_off[i];
    long long cell = 0;
    for (int d = 0; d < a.C - 1; ++d) {
        long long m;
        if (d < i) {
            m = w % a.G[d];
            w /= a.G[d];
        } else {
            m = a.G[d];  // any rank
        }
        cell += m * a.stride[d];
    }
    const int Q = 2 + a.C;
    const unsigned long long* h = a.hist + cell * Q;
    a.count[t] = h[0];
    a.sum_in[t] = h[1];
    a.sum_out[t] = h[2 + i];
}

// Trace-order fp64 token sums for non-integral traces (fallback path).
__global__ void k_workload_seq_sums(WorkloadArgs a, const unsigned long long* __restrict__ ranks,
                                    const double* __restrict__ in, const double* __restrict__ out,
                                    long long n, double* __restrict__ sum_in_f,
                                    double* __restrict__ sum_out_f) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= a.total) return;
    int i = 0;
    while (i + 1 < a.C && t >= a.wl_off[i + 1]) ++i;
    long long w = t - a.wl_off[i];
    unsigned m[4] = {0, 0, 0, 0};
    for (int d = 0; d < i; ++d) {
        m[d] = (unsigned)(w % a.G[d]);
        w /= a.G[d];
    }
    double si = 0.0, so = 0.0;
    const double* oc = out + (long long)i * n;
    for (long long r = 0; r < n; ++r) {
        const unsigned long long pk = ranks[r];
        bool member = true;
        for (int d = 0; d < i; ++d) member &= ((unsigned)((pk >> (16 * d)) & 0xffffu) <= m[d]);
        if (member) {
            si = __dadd_rn(si, in[r]);
            so = __dadd_rn(so, oc[r]);
        }
    }
    sum_in_f[t] = si;
    sum_out_f[t] = so;
}

// Sort keys/payloads for the (C+1) token columns: list 0 = input tokens,
// list 1+i = stage-i output tokens; payload = packed ranks.
__global__ void k_make_lists(const double* __restrict__ in, const double* __restrict__ out,
                             const unsigned long long* __restrict__ ranks, long long n, int C,
                             unsigned long long* __restrict__ keys,
                             unsigned long long* __restrict__ vals) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n;
         r += (long long)gridDim.x * blockDim.x) {
        const unsigned long long pk = ranks[r];
        keys[r] = dbl_to_key(in[r]);
        vals[r] = pk;
        for (int i = 0; i < C; ++i) {
            keys[(long long)(1 + i) * n + r] = dbl_to_key(out[(long long)i * n + r]);
            vals[(long long)(1 + i) * n + r] = pk;
        }
    }
}

// K3: one warp per (workload, column); nearest-rank p95 by scanning the
// ascending-sorted column from the top.
__global__ void k_p95_scan(WorkloadArgs a, const unsigned long long* __restrict__ keys,
                           const unsigned long long* __restrict__ vals, long long n,
                           double* __restrict__ p95_in, double* __restrict__ p95_out) {
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= 2 * a.total) return;
    const long long t = warp >> 1;
    const int which = (int)(warp & 1);
    const unsigned long long cnt = a.count[t];
    double* dst = which ? p95_out : p95_in;
    if (cnt == 0) {
        if (lane == 0) dst[t] = 0.0;
        return;
    }
    int i = 0;
    while (i + 1 < a.C && t >= a.wl_off[i + 1]) ++i;
    long long w = t - a.wl_off[i];
    unsigned m[4] = {0, 0, 0, 0};
    for (int d = 0; d < i; ++d) {
        m[d] = (unsigned)(w % a.G[d]);
        w /= a.G[d];
    }
    const int list = which ? 1 + i : 0;
    const unsigned long long* K = keys + (long long)list * n;
    const unsigned long long* V = vals + (long long)list * n;
    const long long idx = p95_index((long long)cnt);
    long long need = (long long)cnt - idx;  // the need-th largest member
    if (i == 0) {
        if (lane == 0) dst[t] = key_to_dbl(K[n - need]);
        return;
    }
    for (long long base = 0; base < n; base += 32) {
        const long long pos = n - 1 - base - lane;
        bool member = false;
        if (pos >= 0) {
            const unsigned long long pk = V[pos];
            member = true;
            for (int d = 0; d < i; ++d) member &= ((unsigned)((pk >> (16 * d)) & 0xffffu) <= m[d]);
        }
        const unsigned b = __ballot_sync(0xffffffffu, member);
        const int c = __popc(b);
        if (c >= need) {
            const int L = __fns(b, 0, (int)need);
            if (lane == 0) dst[t] = key_to_dbl(K[n - 1 - base - L]);
            return;
        }
        need -= c;
    }
}

// WorkloadStats per (stage, prefix): stats_over (routing.cpp:19-38) plus the
// rate scaling of route_trace (routing.cpp:84-90).
__global__ void k_workload_stats(WorkloadArgs a, long long n, double rate, int integral,
                                 const double* __restrict__ sum_in_f,
                                 const double* __restrict__ sum_out_f,
                                 const double* __restrict__ p95_in,
                                 const double* __restrict__ p95_out, double* __restrict__ stats) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= a.total) return;
    const unsigned long long cnt = a.count[t];
    const double ratio = __ddiv_rn((double)cnt, (double)n);
    double* o = stats + t * 5;
    o[0] = __dmul_rn(rate, ratio);
    if (cnt == 0) {
        o[1] = o[2] = o[3] = o[4] = 0.0;
        return;
    }
    const double si = integral ? (double)a.sum_in[t] : sum_in_f[t];
    const double so = integral ? (double)a.sum_out[t] : sum_out_f[t];
    o[1] = __ddiv_rn(si, (double)cnt);
    o[2] = __ddiv_rn(so, (double)cnt);
    o[3] = p95_in[t];
    o[4] = p95_out[t];
}

// K2: trace-order quality sums, one thread per threshold tuple.
constexpr int QT_THREADS = 128;
constexpr int QT_TILE = 512;

template <int D>
__global__ void __launch_bounds__(QT_THREADS) k_quality(const double* __restrict__ scores, long long n,
                                                        const double* __restrict__ thr, long long ncand,
                                                        double* __restrict__ qsum) {
    constexpr int C = D + 1;
    __shared__ double tile[C][QT_TILE];
    const long long c = blockIdx.x * (long long)QT_THREADS + threadIdx.x;
    double h[D > 0 ? D : 1];
#pragma unroll
    for (int d = 0; d < D; ++d) h[d] = c < ncand ? thr[c * D + d] : 0.0;
    double sum = 0.0;
    for (long long base = 0; base < n; base += QT_TILE) {
        const int len = (int)((n - base) < QT_TILE ? (n - base) : QT_TILE);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < C; ++i)
            for (int k = threadIdx.x; k < len; k += QT_THREADS)
                tile[i][k] = scores[(long long)i * n + base + k];
        __syncthreads();
        for (int k = 0; k < len; ++k) {
            double acc = tile[C - 1][k];
#pragma unroll
            for (int d = D - 1; d >= 0; --d) {
                const double s = tile[d][k];
                acc = (s >= h[d]) ? s : acc;
            }
            sum = __dadd_rn(sum, acc);
        }
    }
    if (c < ncand) qsum[c] = sum;
}

}  // namespace

void launch_route_aggregate(const RouteArgs& a, int D, int sm_count, cudaStream_t s, int* launches) {
    long long blocks = (a.n + 255) / 256;
    long long cap = (long long)sm_count * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    size_t smem = a.grid_in_smem ? (size_t)a.gtotal * sizeof(double) : 0;
    switch (D) {
        case 0: k_route_aggregate<0><<<(unsigned)blocks, 256, smem, s>>>(a); break;
        case 1: k_route_aggregate<1><<<(unsigned)blocks, 256, smem, s>>>(a); break;
        case 2: k_route_aggregate<2><<<(unsigned)blocks, 256, smem, s>>>(a); break;
        case 3: k_route_aggregate<3><<<(unsigned)blocks, 256, smem, s>>>(a); break;
        case 4: k_route_aggregate<4><<<(unsigned)blocks, 256, smem, s>>>(a); break;
        default: throw EngineError(101, "GPU engine supports up to 5 cascade stages");
    }
    CG_LAUNCH_CHECK();
    if (launches) ++*launches;
}

void launch_hist_scan(unsigned long long* hist, long long cells, int Q, const long long* stride,
                      const int* G, int D, cudaStream_t s, int* launches) {
    for (int d = 0; d < D; ++d) {
        const int extent = G[d] + 1;
        const long long work = cells / extent * Q;
        k_hist_scan_dim<<<(unsigned)((work + 255) / 256), 256, 0, s>>>(hist, cells, Q, stride[d],
                                                                       extent);
        CG_LAUNCH_CHECK();
        if (launches) ++*launches;
    }
}

void launch_workload_counts(const WorkloadArgs& a, cudaStream_t s, int* launches) {
    k_workload_counts<<<(unsigned)((a.total + 255) / 256), 256, 0, s>>>(a);
    CG_LAUNCH_CHECK();
    if (launches) ++*launches;
}

void launch_workload_seq_sums(const WorkloadArgs& a, const unsigned long long* ranks,
                              const double* in, const double* out, long long n, double* sum_in_f,
                              double* sum_out_f, cudaStream_t s, int* launches) {
    k_workload_seq_sums<<<(unsigned)((a.total + 127) / 128), 128, 0, s>>>(a, ranks, in, out, n,
                                                                         sum_in_f, sum_out_f);
    CG_LAUNCH_CHECK();
    if (launches) ++*launches;
}

void launch_make_lists(const double* in, const double* out, const unsigned long long* ranks,
                       long long n, int C, unsigned long long* keys, unsigned long long* vals,
                       int sm_count, cudaStream_t s, int* launches) {
    long long blocks = (n + 255) / 256;
    if (blocks > (long long)sm_count * 8) blocks = (long long)sm_count * 8;
    if (blocks < 1) blocks = 1;
    k_make_lists<<<(unsigned)blocks, 256, 0, s>>>(in, out, ranks, n, C, keys, vals);
    CG_LAUNCH_CHECK();
    if (launches) ++*launches;
}

void launch_p95_scan(const WorkloadArgs& a, const unsigned long long* keys,
                     const unsigned long long* vals, long long n, double* p95_in, double* p95_out,
                     cudaStream_t s, int* launches) {
    const long long warps = 2 * a.total;
    k_p95_scan<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(a, keys, vals, n, p95_in, p95_out);
    CG_LAUNCH_CHECK();
    if (launches) ++*launches;
}

void launch_workload_stats(const WorkloadArgs& a, long long n, double rate, int integral,
                           const double* sum_in_f, const double* sum_out_f, const double* p95_in,
                           const double* p95_out, double* stats, cudaStream_t s, int* launches) {
    k_workload_stats<<<(unsigned)((a.total + 255) / 256), 256, 0, s>>>(a, n, rate, integral, sum_in_f,
                                                                      sum_out_f, p95_in, p95_out, stats);
    CG_LAUNCH_CHECK();
    if (launches) ++*launches;
}

void launch_quality(const double* scores, long long n, int D, const double* thr, long long ncand,
                    double* qsum, cudaStream_t s, int* launches) {
    const unsigned blocks = (unsigned)((ncand + QT_THREADS - 1) / QT_THREADS);
    switch (D) {
        case 0: k_quality<0><<<blocks, QT_THREADS, 0, s>>>(scores, n, thr, ncand, qsum); break;
        case 1: k_quality<1><<<blocks, QT_THREADS, 0, s>>>(scores, n, thr, ncand, qsum); break;
        case 2: k_quality<2><<<blocks, QT_THREADS, 0, s>>>(scores, n, thr, ncand, qsum); break;
        case 3: k_quality<3><<<blocks, QT_THREADS, 0, s>>>(scores, n, thr, ncand, qsum); break;
        case 4: k_quality<4><<<blocks, QT_THREADS, 0, s>>>(scores, n, thr, ncand, qsum); break;
        default: throw EngineError(101, "GPU engine supports up to 5 cascade stages");
    }
    CG_LAUNCH_CHECK();
    if (launches) ++*launches;
}

}  // namespace cg
