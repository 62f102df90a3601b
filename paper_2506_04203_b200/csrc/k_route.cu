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

// #{v <= s} over the sorted distinct values v[0..g): upper_bound with the
// predicate (v <= s), NaN scores rank 0.  Branch-free: the step sequence
// depends only on g (warp-uniform), so lanes never diverge.
__device__ __forceinline__ int rank_of(const double* __restrict__ v, int g, int top, double s) {
    int pos = 0;
    for (int b = top; b > 0; b >>= 1) {
        const int q = pos + b;
        pos = (q <= g && v[q - 1] <= s) ? q : pos;
    }
    return pos;
}

__device__ __forceinline__ bool token_ok(double x) {
    return x >= 0.0 && x < 4294967296.0 && x == trunc(x);
}

// Warp-aggregated histogram update of NQ u64 words per cell: lanes with the
// same cell are merged with __match_any_sync; each group's token sums are
// reduced with two 16-bit-split __reduce_add_sync (exact for u32 tokens) and
// its leader issues one atomic per word.  Words: [count?] then the sums.
template <int NQ, bool COUNT>
__device__ __forceinline__ void hist_add(unsigned long long* __restrict__ h, bool valid, unsigned cell,
                                         const unsigned* v /*[NQ - COUNT]*/) {
    constexpr int NV = NQ - (COUNT ? 1 : 0);
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    if (!valid) return;
    const int lane = threadIdx.x & 31;
    const unsigned peers = __match_any_sync(act, cell);
    unsigned long long* p = h + (unsigned long long)cell * NQ;
    if (__all_sync(act, peers == (1u << lane))) {
        if (COUNT) atomicAdd(&p[0], 1ull);
#pragma unroll
        for (int q = 0; q < NV; ++q) atomicAdd(&p[q + (COUNT ? 1 : 0)], (unsigned long long)v[q]);
        return;
    }
    unsigned long long sums[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        const unsigned lo = __reduce_add_sync(peers, v[q] & 0xffffu);
        const unsigned hi = __reduce_add_sync(peers, v[q] >> 16);
        sums[q] = ((unsigned long long)hi << 16) + lo;
    }
    if (lane == __ffs(peers) - 1) {
        if (COUNT) atomicAdd(&p[0], (unsigned long long)__popc(peers));
#pragma unroll
        for (int q = 0; q < NV; ++q) atomicAdd(&p[q + (COUNT ? 1 : 0)], sums[q]);
    }
}

__device__ __forceinline__ unsigned tok32(double x, bool& bad) {
    const bool ok = token_ok(x);
    bad |= !ok;
    return ok ? (unsigned)x : 0u;
}

// K1: one streaming pass over the trace.  Each thread routes two consecutive
// requests per iteration with 128-bit loads of every SoA column (scores of
// the C-1 threshold stages, input tokens, C output-token columns) and writes
// the packed ranks with one 128-bit store.  Aggregation (block-private in
// shared memory when it fits, PRIV, else global): full rank cells carry
// (count, sum_in, sum_out_{C-1}); the stage-i output sums (i < C-1) only
// depend on dims < i and go to small marginal histograms over those dims.
template <int D, bool PRIV>
__global__ void __launch_bounds__(256) k_route_aggregate(RouteArgs a) {
    constexpr int C = D + 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned long long* sh_hist = reinterpret_cast<unsigned long long*>(smem_raw);
    double* s_grid = reinterpret_cast<double*>(smem_raw + (PRIV ? (size_t)a.priv_words * 8 : 0));
    const double* gv = a.gvals;
    if (a.grid_in_smem) {
        for (int i = threadIdx.x; i < a.gtotal; i += blockDim.x) s_grid[i] = a.gvals[i];
        gv = s_grid;
    }
    if (PRIV)
        for (long long i = threadIdx.x; i < a.priv_words; i += blockDim.x) sh_hist[i] = 0ull;
    __syncthreads();
    unsigned long long* full = PRIV ? sh_hist : a.acc;
    bool bad = false;
    const long long n = a.n;
    const long long npairs = (n + 1) >> 1;
    const bool vec = (n & 1) == 0 && ((reinterpret_cast<unsigned long long>(a.scores) |
                                        reinterpret_cast<unsigned long long>(a.in) |
                                        reinterpret_cast<unsigned long long>(a.out) |
                                        reinterpret_cast<unsigned long long>(a.ranks)) & 15ull) == 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    // uniform trip count so every lane reaches the warp collectives
    const long long first = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long iters = (npairs + stride - 1) / stride;
    // software pipeline: the loads of iteration it+1 are in flight while
    // iteration it is ranked and aggregated
    double nsc[D > 0 ? D : 1][2], nxin[2], nxo[C][2];
    auto load_pair = [&](long long r0, double (&sc)[D > 0 ? D : 1][2], double (&xin)[2], double (&xo)[C][2]) {
        const bool v1 = r0 + 1 < n;
        if (v1 && vec) {
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const double2 t = __ldcs(reinterpret_cast<const double2*>(a.scores + (long long)d * n + r0));
                sc[d][0] = t.x;
                sc[d][1] = t.y;
            }
            const double2 ti = __ldcs(reinterpret_cast<const double2*>(a.in + r0));
            xin[0] = ti.x;
            xin[1] = ti.y;
#pragma unroll
            for (int i = 0; i < C; ++i) {
                const double2 t = __ldcs(reinterpret_cast<const double2*>(a.out + (long long)i * n + r0));
                xo[i][0] = t.x;
                xo[i][1] = t.y;
            }
        } else {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const long long r = r0 + e;
                const bool ve = r < n;
#pragma unroll
                for (int d = 0; d < D; ++d) sc[d][e] = ve ? a.scores[(long long)d * n + r] : 0.0;
                xin[e] = ve ? a.in[r] : 0.0;
#pragma unroll
                for (int i = 0; i < C; ++i) xo[i][e] = ve ? a.out[(long long)i * n + r] : 0.0;
            }
        }
    };
    if (iters > 0) load_pair(2 * first, nsc, nxin, nxo);
    for (long long it = 0; it < iters; ++it) {
        const long long p = first + it * stride;
        const long long r0 = 2 * p;
        const bool v0 = r0 < n, v1 = r0 + 1 < n;
        double sc[D > 0 ? D : 1][2], xin[2], xo[C][2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
#pragma unroll
            for (int d = 0; d < D; ++d) sc[d][e] = nsc[d][e];
            xin[e] = nxin[e];
#pragma unroll
            for (int i = 0; i < C; ++i) xo[i][e] = nxo[i][e];
        }
        if (it + 1 < iters) load_pair(r0 + 2 * stride, nsc, nxin, nxo);
        unsigned long long pk[2] = {0ull, 0ull};
        unsigned cell[2] = {0u, 0u};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const int rk = rank_of(gv + a.goff[d], a.G[d], a.gtop[d], sc[d][e]);
                pk[e] |= (unsigned long long)rk << (16 * d);
                cell[e] += (unsigned)rk * (unsigned)a.stride[d];
            }
        }
        if (v1 && vec) {
            *reinterpret_cast<ulonglong2*>(a.ranks + r0) = make_ulonglong2(pk[0], pk[1]);
        } else {
            if (v0) a.ranks[r0] = pk[0];
            if (v1) a.ranks[r0 + 1] = pk[1];
        }
        // per-lane shared-memory atomics (hardware-serialised only on real
        // address conflicts); the one-bin stage-0 marginal is a warp REDUX
        unsigned s0lo = 0, s0hi = 0;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const bool ve = e == 0 ? v0 : v1;
            if (ve) {
                unsigned long long* pf = full + (unsigned long long)cell[e] * 3;
                atomicAdd(&pf[0], 1ull);
                atomicAdd(&pf[1], (unsigned long long)tok32(xin[e], bad));
                atomicAdd(&pf[2], (unsigned long long)tok32(xo[C - 1][e], bad));
            }
            if (C > 1) {
                const unsigned v0t = ve ? tok32(xo[0][e], bad) : 0u;
                s0lo += v0t & 0xffffu;
                s0hi += v0t >> 16;
            }
#pragma unroll
            for (int i = 1; i < C - 1; ++i) {
                if (ve) {
                    const unsigned mcell = cell[e] % (unsigned)a.stride[i];
                    atomicAdd(full + a.marg_off[i] + mcell, (unsigned long long)tok32(xo[i][e], bad));
                }
            }
        }
        if (C > 1) {
            const unsigned lo = __reduce_add_sync(0xffffffffu, s0lo);
            const unsigned hi = __reduce_add_sync(0xffffffffu, s0hi);
            if ((threadIdx.x & 31) == 0)
                atomicAdd(full + a.marg_off[0], ((unsigned long long)hi << 16) + (unsigned long long)lo);
        }
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(a.flags, 1u);
    if (PRIV) {
        __syncthreads();
        unsigned long long* part = a.partials + (long long)blockIdx.x * a.priv_words;
        for (long long i = threadIdx.x; i < a.priv_words; i += blockDim.x) part[i] = sh_hist[i];
    }
}

// K1 (tiled form, used when the rank histogram fits in shared memory): per
// tile of 2048 requests the block (512 threads, 4 requests each, 128-bit
// loads) computes the rank cells, stores the packed ranks, stages the u32
// tokens in shared memory and counting-sorts the tile by cell -- ONE 32-bit
// shared atomic per request -- after which the owner thread of each cell adds
// the cell's segment (count, sum_in, sum_out_0..C-1) into the block-private
// u64 histogram without atomics.  The next tile's loads are issued before the
// sort phases so HBM traffic overlaps them.
constexpr int KT_THREADS = 512;
constexpr int KT_TILE = 4 * KT_THREADS;

template <int D, bool GHIST>
__global__ void __launch_bounds__(KT_THREADS, 1) k_route_tile(RouteArgs a) {
    constexpr int C = D + 1;
    constexpr int Q = 2 + C;
    constexpr int NV = D + 1 + C;  // raw doubles per request
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const long long cells = a.cells;
    // block-private histogram: shared memory, or (GHIST, large grids) the
    // block's own L2-resident slice of the partials -- owner-thread RMW, no atomics
    unsigned long long* hist = GHIST ? a.tile_partials + (long long)blockIdx.x * cells * Q
                                     : reinterpret_cast<unsigned long long*>(smem_raw);     // [cells][Q]
    unsigned* start = reinterpret_cast<unsigned*>(smem_raw + (GHIST ? 0 : cells * Q * 8));   // [cells+1]
    unsigned* tcell = start + ((cells + 1 + 3) & ~3ll);                                      // [TILE]
    unsigned* ttok = tcell + KT_TILE;                                                        // [C+1][TILE]
    unsigned short* order = reinterpret_cast<unsigned short*>(ttok + (C + 1) * KT_TILE);    // [TILE]
    double* s_grid = reinterpret_cast<double*>(order + KT_TILE + 8);
    __shared__ unsigned wsum[KT_THREADS / 32];

    for (int i = threadIdx.x; i < a.gtotal; i += KT_THREADS) s_grid[i] = a.gvals[i];
    if (!GHIST)
        for (long long i = threadIdx.x; i < cells * Q; i += KT_THREADS) hist[i] = 0ull;
    const long long n = a.n;
    const bool vec = (n & 1) == 0 && ((reinterpret_cast<unsigned long long>(a.scores) |
                                        reinterpret_cast<unsigned long long>(a.in) |
                                        reinterpret_cast<unsigned long long>(a.out) |
                                        reinterpret_cast<unsigned long long>(a.ranks)) & 15ull) == 0;
    const long long ntiles = (n + KT_TILE - 1) / KT_TILE;
    bool bad = false;
    // raw values of this thread's 4 requests: pairs at tile offsets 2*tid and 2*(tid+512)
    double raw[4][NV];
    auto load = [&](long long tile) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const long long r0 = tile * KT_TILE + 2 * (threadIdx.x + h * KT_THREADS);
            if (vec && r0 + 1 < n) {
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const double* col = v < D ? a.scores + (long long)v * n
                                              : (v == D ? a.in : a.out + (long long)(v - D - 1) * n);
                    const double2 t = __ldcs(reinterpret_cast<const double2*>(col + r0));
                    raw[2 * h][v] = t.x;
                    raw[2 * h + 1][v] = t.y;
                }
            } else {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const long long r = r0 + e;
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        const double* col = v < D ? a.scores + (long long)v * n
                                                  : (v == D ? a.in : a.out + (long long)(v - D - 1) * n);
                        raw[2 * h + e][v] = r < n ? col[r] : 0.0;
                    }
                }
            }
        }
    };
    long long tile = blockIdx.x;
    if (tile < ntiles) load(tile);
    __syncthreads();
    for (; tile < ntiles; tile += gridDim.x) {
        const long long tbase = tile * KT_TILE;
        const int tlen = (int)((n - tbase) < KT_TILE ? (n - tbase) : KT_TILE);
        // ---- ranks, cells, staged tokens
        unsigned cell[4];
        int li[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            li[q] = 2 * (threadIdx.x + (q >> 1) * KT_THREADS) + (q & 1);
            unsigned long long pk = 0;
            unsigned c = 0;
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const int rk = rank_of(s_grid + a.goff[d], a.G[d], a.gtop[d], raw[q][d]);
                pk |= (unsigned long long)rk << (16 * d);
                c += (unsigned)rk * (unsigned)a.stride[d];
            }
            cell[q] = c;
            const bool ve = li[q] < tlen;
            if (ve) {
                tcell[li[q]] = c;
#pragma unroll
                for (int v = 0; v <= C; ++v) ttok[v * KT_TILE + li[q]] = tok32(raw[q][D + v], bad);
            }
            raw[q][0] = __longlong_as_double((long long)pk);  // keep packed ranks for the store
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const long long r0 = tbase + 2 * (threadIdx.x + h * KT_THREADS);
            const unsigned long long p0 = (unsigned long long)__double_as_longlong(raw[2 * h][0]);
            const unsigned long long p1 = (unsigned long long)__double_as_longlong(raw[2 * h + 1][0]);
            if (vec && r0 + 1 < n) {
                *reinterpret_cast<ulonglong2*>(a.ranks + r0) = make_ulonglong2(p0, p1);
            } else {
                if (r0 < n) a.ranks[r0] = p0;
                if (r0 + 1 < n) a.ranks[r0 + 1] = p1;
            }
        }
        // ---- prefetch the next tile while this one is sorted and summed
        if (tile + gridDim.x < ntiles) load(tile + gridDim.x);
        for (long long i = threadIdx.x; i <= cells; i += KT_THREADS) start[i] = 0u;
        __syncthreads();
        unsigned rnk[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            rnk[q] = li[q] < tlen ? atomicAdd(&start[cell[q]], 1u) : 0u;
        __syncthreads();
        // ---- exclusive scan of the per-cell counts (block-wide)
        {
            const long long per = (cells + KT_THREADS - 1) / KT_THREADS;
            const long long lo = threadIdx.x * per;
            const long long hi = lo + per < cells ? lo + per : cells;
            unsigned tsum = 0;
            for (long long i = lo; i < hi; ++i) tsum += start[i];
            const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
            unsigned incl = tsum;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const unsigned v = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += v;
            }
            if (lane == 31) wsum[w] = incl;
            __syncthreads();
            unsigned wbase = 0;
            for (int k = 0; k < w; ++k) wbase += wsum[k];
            unsigned run = wbase + incl - tsum;
            for (long long i = lo; i < hi; ++i) {
                const unsigned v = start[i];
                start[i] = run;
                run += v;
            }
            if (threadIdx.x == KT_THREADS - 1) start[cells] = (unsigned)tlen;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (li[q] < tlen) order[start[cell[q]] + rnk[q]] = (unsigned short)li[q];
        __syncthreads();
        // ---- owner thread per cell: segmented sums, no atomics
        for (long long c = threadIdx.x; c < cells; c += KT_THREADS) {
            const unsigned b = start[c], e = start[c + 1];
            if (b == e) continue;
            unsigned long long acc[Q];
            acc[0] = e - b;
#pragma unroll
            for (int v = 0; v <= C; ++v) acc[1 + v] = 0ull;
            for (unsigned j = b; j < e; ++j) {
                const int r = order[j];
#pragma unroll
                for (int v = 0; v <= C; ++v) acc[1 + v] += ttok[v * KT_TILE + r];
            }
            unsigned long long* hp = hist + c * Q;
#pragma unroll
            for (int v = 0; v < Q; ++v) hp[v] += acc[v];
        }
        __syncthreads();
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(a.flags, 1u);
    if (!GHIST) {
        unsigned long long* part = a.tile_partials + (long long)blockIdx.x * cells * Q;
        for (long long i = threadIdx.x; i < cells * Q; i += KT_THREADS) part[i] = hist[i];
    }
}

// Tiled form: partials are already [cells][Q]; sum over blocks.
__global__ void k_hist_sum(const unsigned long long* __restrict__ part, long long len, int nblocks,
                           unsigned long long* __restrict__ hist) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= len) return;
    unsigned long long s = 0;
    for (int b = 0; b < nblocks; ++b) s += part[(long long)b * len + i];
    hist[i] = s;
}

// Sum the block-private partials (or take the global accumulator) and expand
// into the [cells][2+C] layout the dominance scan expects: the marginal sums
// of stage i (i < C-1) sit at the cells whose dims >= i are at their maximum
// rank, so the dominance prefix sum reproduces them at every stage-i query.
__global__ void k_hist_expand(RouteArgs a, int C, int nblocks) {
    const long long cell = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (cell >= a.cells) return;
    const int Q = 2 + C;
    auto acc = [&](long long w) -> unsigned long long {
        if (nblocks == 0) return a.acc[w];
        unsigned long long s = 0;
        for (int b = 0; b < nblocks; ++b) s += a.partials[(long long)b * a.priv_words + w];
        return s;
    };
    unsigned long long* h = a.hist + cell * Q;
    h[0] = acc(cell * 3 + 0);
    h[1] = acc(cell * 3 + 1);
    h[2 + (C - 1)] = acc(cell * 3 + 2);
    for (int i = 0; i < C - 1; ++i) {
        bool at_max = true;
        long long rem = cell;
        for (int d = 0; d < C - 1; ++d) {
            const long long coord = rem % (a.G[d] + 1);
            rem /= (a.G[d] + 1);
            if (d >= i && coord != a.G[d]) at_max = false;
        }
        h[2 + i] = at_max ? acc(a.marg_off[i] + (i == 0 ? 0 : cell % a.stride[i])) : 0ull;
    }
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

size_t tile_smem_bytes(long long cells, int D, int gtotal, bool ghist) {
    const int C = D + 1, Q = 2 + C;
    return (ghist ? 0 : (size_t)cells * Q * 8) + (size_t)((cells + 1 + 3) & ~3ll) * 4 + (size_t)KT_TILE * 4 +
           (size_t)(C + 1) * KT_TILE * 4 + (size_t)(KT_TILE + 8) * 2 + (size_t)gtotal * 8 + 64;
}

// The histogram stays in shared memory while it is small; beyond that it moves
// to the block's global (L2-resident) slice so more blocks fit per SM.
bool tile_hist_global(long long cells, int D) { return (size_t)cells * (3 + D) * 8 > 120 * 1024; }

size_t tile_smem_bytes(long long cells, int D, int gtotal) {
    return tile_smem_bytes(cells, D, gtotal, tile_hist_global(cells, D));
}

template <int D>
void launch_k1(const RouteArgs& a, int sm_count, cudaStream_t s, int* launches, int* nblocks_out) {
    const size_t tsm = tile_smem_bytes(a.cells, D, a.gtotal);
    if (a.tile_partials && tsm <= 200 * 1024) {
        const bool ghist = tile_hist_global(a.cells, D);
        auto kern = ghist ? k_route_tile<D, true> : k_route_tile<D, false>;
        CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
        int per_sm = 0;
        CG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, KT_THREADS, tsm));
        const long long ntiles = (a.n + KT_TILE - 1) / KT_TILE;
        long long blocks = (long long)sm_count * (per_sm < 1 ? 1 : per_sm);
        if (blocks > ntiles) blocks = ntiles;
        if (blocks > a.max_partials) blocks = a.max_partials;
        if (blocks < 1) blocks = 1;
        if (ghist)
            CG_CUDA(cudaMemsetAsync(a.tile_partials, 0, (size_t)blocks * a.cells * (3 + D) * 8, s));
        kern<<<(unsigned)blocks, KT_THREADS, tsm, s>>>(a);
        CG_LAUNCH_CHECK();
        if (launches) *launches += 1;
        if (nblocks_out) *nblocks_out = -(int)blocks;  // negative: tiled partial layout
        return;
    }
    const size_t grid_smem = a.grid_in_smem ? (size_t)a.gtotal * sizeof(double) : 0;
    const size_t hist_smem = (size_t)a.priv_words * 8;
    const bool priv = a.partials != nullptr && hist_smem + grid_smem <= 96 * 1024;
    const long long npairs = (a.n + 1) / 2;
    long long blocks = (npairs + 255) / 256;
    int nb = 0;
    if (priv) {
        auto kern = k_route_aggregate<D, true>;
        const size_t smem = hist_smem + grid_smem;
        CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        CG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
        const long long cap = (long long)sm_count * (per_sm < 1 ? 1 : per_sm);
        if (blocks > cap) blocks = cap;
        if (blocks > a.max_partials) blocks = a.max_partials;
        if (blocks < 1) blocks = 1;
        kern<<<(unsigned)blocks, 256, smem, s>>>(a);
        nb = (int)blocks;
    } else {
        CG_CUDA(cudaMemsetAsync(a.acc, 0, (size_t)a.priv_words * 8, s));
        const long long cap = (long long)sm_count * 8;
        if (blocks > cap) blocks = cap;
        if (blocks < 1) blocks = 1;
        k_route_aggregate<D, false><<<(unsigned)blocks, 256, grid_smem, s>>>(a);
    }
    CG_LAUNCH_CHECK();
    if (launches) *launches += 1;
    if (nblocks_out) *nblocks_out = nb;
}

void launch_route_aggregate(const RouteArgs& a, int D, int sm_count, cudaStream_t s, int* launches,
                            int* nblocks_out) {
    switch (D) {
        case 0: launch_k1<0>(a, sm_count, s, launches, nblocks_out); break;
        case 1: launch_k1<1>(a, sm_count, s, launches, nblocks_out); break;
        case 2: launch_k1<2>(a, sm_count, s, launches, nblocks_out); break;
        case 3: launch_k1<3>(a, sm_count, s, launches, nblocks_out); break;
        case 4: launch_k1<4>(a, sm_count, s, launches, nblocks_out); break;
        default: throw EngineError(101, "GPU engine supports up to 5 cascade stages");
    }
}

void launch_hist_expand(const RouteArgs& a, int C, int nblocks, cudaStream_t s, int* launches) {
    if (nblocks < 0) {  // tiled form: [blocks][cells][2+C] partials -> hist
        const long long len = a.cells * (2 + C);
        k_hist_sum<<<(unsigned)((len + 255) / 256), 256, 0, s>>>(a.tile_partials, len, -nblocks, a.hist);
        CG_LAUNCH_CHECK();
        if (launches) ++*launches;
        return;
    }
    k_hist_expand<<<(unsigned)((a.cells + 255) / 256), 256, 0, s>>>(a, C, nblocks);
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
