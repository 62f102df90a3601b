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
#include "cg_ptx.cuh"

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

// K1 (u32 form, used whenever the u32 cell histogram fits in shared memory).
//
// Rank search: per threshold dimension a 1024-bin table over the float image
// of the distinct grid values.  bin(s) = clamp(floor((float(s) - lo) * sc))
// is a composition of correctly rounded monotone operations, hence monotone
// non-decreasing in s; so every grid value in a lower bin is <= s, every one
// in a higher bin is > s, and only the values sharing s's bin need an exact
// fp64 compare (normally at most one).  NaN scores land in bin 0 and compare
// false: rank 0, as in the reference (`score >= h` is false).
//
// Aggregation: block-private u32 histogram [cells][2+C] (count, input sum,
// output sums) in shared memory with native 32-bit shared atomics (64-bit
// shared atomicAdd is a CAS loop on sm_100).  A block handles at most 2^16
// requests, so counts and sums of the low 16 bits of every token are exact in
// u32; the (rare) high parts of tokens >= 2^16 go to a global u64 accumulator.
constexpr int KH_THREADS = 512;
constexpr int KH_NB = 1024;                         // bins per dimension
constexpr int KH_MAX_REQ = 65536;                   // requests per block
constexpr int KH_MAX_ITERS = KH_MAX_REQ / (2 * KH_THREADS);

__device__ __forceinline__ int bin_of(double s, float lo, float sc) {
    const float f = __double2float_rn(s);
    const int b = __float2int_rd(__fmul_rn(__fsub_rn(f, lo), sc));  // NaN -> 0
    return min(max(b, 0), KH_NB - 1);
}

__device__ __forceinline__ void bin_params(const double* v, int g, float& lo, float& sc) {
    if (g <= 0) {
        lo = 0.f;
        sc = 0.f;
        return;
    }
    lo = __double2float_rn(v[0]);
    const float hi = __double2float_rn(v[g - 1]);
    const float span = __fsub_rn(hi, lo);
    sc = span > 0.f ? __fdiv_rn((float)(KH_NB - 1), span) : 0.f;
    if (!(sc == sc) || sc < 0.f) sc = 0.f;  // inf span etc.: one bin (still exact)
}

__device__ __forceinline__ int rank_binned(const double* __restrict__ v, const unsigned* __restrict__ tab,
                                           int g, float lo, float sc, double s) {
    const unsigned e = tab[bin_of(s, lo, sc)];
    const int j0 = (int)(e & 0xffffu);
    const int c = (int)(e >> 16);
    int r = j0;
    if (c > 0) r += (v[j0] <= s) ? 1 : 0;
    if (c > 1) {
        for (int k = 1; k < c; ++k) r += (v[j0 + k] <= s) ? 1 : 0;
    }
    return r;
}

// Per-dimension bin tables (all threads of the block call this; s_grid must
// be filled and visible): tab[d][b] = j0(b) | (j0(b+1) - j0(b)) << 16 with
// j0(b) = #{j : bin(v_j) < b}.
template <int D>
__device__ __forceinline__ void build_bin_tables(const RouteArgs& a, const double* s_grid, unsigned* tab,
                                                 int* s_bin /*[32]*/, float* lo, float* sc, int nthreads) {
#pragma unroll
    for (int d = 0; d < D; ++d) bin_params(a.gvals + a.goff[d], a.G[d], lo[d], sc[d]);
    __syncthreads();
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const double* v = s_grid + a.goff[d];
        const int g = a.G[d];
        unsigned* t = tab + d * (KH_NB + 1);
        if (g <= 32) {
            for (int j = threadIdx.x; j < g; j += nthreads) s_bin[j] = bin_of(v[j], lo[d], sc[d]);
            __syncthreads();
            for (int b = threadIdx.x; b < KH_NB; b += nthreads) {
                int j0 = 0, j1 = 0;
                for (int j = 0; j < g; ++j) {
                    j0 += s_bin[j] < b ? 1 : 0;
                    j1 += s_bin[j] <= b ? 1 : 0;
                }
                t[b] = (unsigned)j0 | ((unsigned)(j1 - j0) << 16);
            }
            __syncthreads();
        } else {
            for (int b = threadIdx.x; b < KH_NB; b += nthreads) {
                // binary searches over the monotone bins of the sorted values
                int l0 = 0, h0 = g;
                while (l0 < h0) {
                    const int m = (l0 + h0) >> 1;
                    if (bin_of(v[m], lo[d], sc[d]) < b) l0 = m + 1; else h0 = m;
                }
                int l1 = l0, h1 = g;
                while (l1 < h1) {
                    const int m = (l1 + h1) >> 1;
                    if (bin_of(v[m], lo[d], sc[d]) <= b) l1 = m + 1; else h1 = m;
                }
                t[b] = (unsigned)l0 | ((unsigned)(l1 - l0) << 16);
            }
        }
    }
    __syncthreads();
}

// One request into the block-private u32 histogram (see k_route_hist).
template <int C>
__device__ __forceinline__ void hist32_add(unsigned* __restrict__ hist, unsigned long long* __restrict__ hi_acc,
                                           unsigned cell, const double* tokd /*[C+1]: in, out_0..*/, bool& bad) {
    constexpr int Q = 2 + C;
    unsigned* hp = hist + (unsigned long long)cell * Q;
    unsigned tk[C + 1];
#pragma unroll
    for (int v = 0; v <= C; ++v) tk[v] = tok32(tokd[v], bad);
    atomicAdd(&hp[0], 1u);
#pragma unroll
    for (int v = 0; v <= C; ++v) {
        atomicAdd(&hp[1 + v], tk[v] & 0xffffu);
        if (tk[v] >> 16)
            atomicAdd(&hi_acc[(unsigned long long)cell * Q + 1 + v], (unsigned long long)(tk[v] & 0xffff0000u));
    }
}

template <int D, int MINB>
__global__ void __launch_bounds__(KH_THREADS, MINB) k_route_hist(RouteArgs a) {
    constexpr int C = D + 1;
    constexpr int Q = 2 + C;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const long long cells = a.cells;
    unsigned* hist = reinterpret_cast<unsigned*>(smem_raw);                       // [cells][Q]
    const long long hw = (cells * Q + 3) & ~3ll;
    unsigned* tab = hist + hw;                                                    // [D][NB+1]
    double* s_grid = reinterpret_cast<double*>(tab + ((D * (KH_NB + 1) + 3) & ~3));  // [gtotal]
    __shared__ int s_bin[32];  // scratch: bins of grid values while building a table

    for (int i = threadIdx.x; i < a.gtotal; i += KH_THREADS) s_grid[i] = a.gvals[i];
    for (long long i = threadIdx.x; i < hw; i += KH_THREADS) hist[i] = 0u;
    float lo[D > 0 ? D : 1], sc[D > 0 ? D : 1];
    build_bin_tables<D>(a, s_grid, tab, s_bin, lo, sc, KH_THREADS);

    bool bad = false;
    const long long n = a.n;
    const long long npairs = (n + 1) >> 1;
    const bool vec = (n & 1) == 0 && ((reinterpret_cast<unsigned long long>(a.scores) |
                                        reinterpret_cast<unsigned long long>(a.in) |
                                        reinterpret_cast<unsigned long long>(a.out) |
                                        reinterpret_cast<unsigned long long>(a.ranks)) & 15ull) == 0;
    const long long stride = (long long)gridDim.x * KH_THREADS;
    const long long first = blockIdx.x * (long long)KH_THREADS + threadIdx.x;
    const long long iters = (npairs - first + stride - 1) / stride;  // this thread's pairs (may be <= 0)
    double nsc[D > 0 ? D : 1][2], nxin[2], nxo[C][2];
    auto load_pair = [&](long long r0) {
        if (vec && r0 + 1 < n) {
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const double2 t = __ldcs(reinterpret_cast<const double2*>(a.scores + (long long)d * n + r0));
                nsc[d][0] = t.x;
                nsc[d][1] = t.y;
            }
            const double2 ti = __ldcs(reinterpret_cast<const double2*>(a.in + r0));
            nxin[0] = ti.x;
            nxin[1] = ti.y;
#pragma unroll
            for (int i = 0; i < C; ++i) {
                const double2 t = __ldcs(reinterpret_cast<const double2*>(a.out + (long long)i * n + r0));
                nxo[i][0] = t.x;
                nxo[i][1] = t.y;
            }
        } else {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const long long r = r0 + e;
                const bool ve = r < n;
#pragma unroll
                for (int d = 0; d < D; ++d) nsc[d][e] = ve ? a.scores[(long long)d * n + r] : 0.0;
                nxin[e] = ve ? a.in[r] : 0.0;
#pragma unroll
                for (int i = 0; i < C; ++i) nxo[i][e] = ve ? a.out[(long long)i * n + r] : 0.0;
            }
        }
    };
    if (iters > 0) load_pair(2 * first);
    for (long long it = 0; it < iters; ++it) {
        const long long r0 = 2 * (first + it * stride);
        double sc_[D > 0 ? D : 1][2], xin[2], xo[C][2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
#pragma unroll
            for (int d = 0; d < D; ++d) sc_[d][e] = nsc[d][e];
            xin[e] = nxin[e];
#pragma unroll
            for (int i = 0; i < C; ++i) xo[i][e] = nxo[i][e];
        }
        if (it + 1 < iters) load_pair(r0 + 2 * stride);
        unsigned long long pk[2] = {0ull, 0ull};
        unsigned cell[2] = {0u, 0u};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const int rk = a.bin_ok ? rank_binned(s_grid + a.goff[d], tab + d * (KH_NB + 1), a.G[d], lo[d],
                                                      sc[d], sc_[d][e])
                                        : rank_of(s_grid + a.goff[d], a.G[d], a.gtop[d], sc_[d][e]);
                pk[e] |= (unsigned long long)rk << (16 * d);
                cell[e] += (unsigned)rk * (unsigned)a.stride[d];
            }
        }
        const bool v1 = r0 + 1 < n;
        if (v1 && vec) {
            __stcs(reinterpret_cast<ulonglong2*>(a.ranks + r0), make_ulonglong2(pk[0], pk[1]));
        } else {
            a.ranks[r0] = pk[0];
            if (v1) a.ranks[r0 + 1] = pk[1];
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            if (e == 1 && !v1) break;
            unsigned* hp = hist + (unsigned long long)cell[e] * Q;
            unsigned tk[C + 1];
            tk[0] = tok32(xin[e], bad);
#pragma unroll
            for (int i = 0; i < C; ++i) tk[1 + i] = tok32(xo[i][e], bad);
            atomicAdd(&hp[0], 1u);
#pragma unroll
            for (int v = 0; v <= C; ++v) {
                atomicAdd(&hp[1 + v], tk[v] & 0xffffu);
                if (tk[v] >> 16)
                    atomicAdd(&a.hi_acc[(unsigned long long)cell[e] * Q + 1 + v],
                              (unsigned long long)(tk[v] & 0xffff0000u));
            }
        }
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(a.flags, 1u);
    __syncthreads();
    unsigned* part = a.part32 + (long long)blockIdx.x * cells * Q;
    for (long long i = threadIdx.x; i < cells * Q; i += KH_THREADS) __stcg(part + i, hist[i]);
}


// K1, TMA-ring form (the default when the trace columns are 16-byte aligned
// and n is even).  One producer warp streams tiles of KR_T requests of every
// SoA column (C-1 score columns, input, C output columns) into a KR_STAGES
// shared-memory ring with cp.async.bulk (UBLKCP) and mbarrier transaction
// counts; KR_NWC consumer warps route one request per thread per tile from
// shared memory, release the slot as soon as the values are in registers, and
// aggregate into the block-private u32 histogram exactly as k_route_hist.  No
// register double-buffering: the bytes in flight live in the ring.
constexpr int KR_NWC = 8;
constexpr int KR_T = 32 * KR_NWC;
constexpr int KR_STAGES = 3;
constexpr int KR_THREADS = 32 * (KR_NWC + 1);
constexpr int KR_MAX_TILES = KH_MAX_REQ / KR_T;     // per block: u32 sums stay exact

template <int D>
struct KRLayout {
    static constexpr int C = D + 1;
    static constexpr int NV = D + 1 + C;            // columns per request
    static constexpr size_t ring_bytes = (size_t)KR_STAGES * NV * KR_T * 8;
};

template <int D>
__global__ void __launch_bounds__(KR_THREADS, 1) k_route_tma(RouteArgs a, long long tiles_per_block) {
    constexpr int C = D + 1;
    constexpr int Q = 2 + C;
    constexpr int NV = KRLayout<D>::NV;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* ring = reinterpret_cast<double*>(smem_raw);                            // [S][NV][T]
    const long long cells = a.cells;
    unsigned* hist = reinterpret_cast<unsigned*>(smem_raw + KRLayout<D>::ring_bytes);  // [cells][Q]
    const long long hw = (cells * Q + 3) & ~3ll;
    unsigned* tab = hist + hw;                                                     // [D][NB+1]
    double* s_grid = reinterpret_cast<double*>(tab + ((D * (KH_NB + 1) + 3) & ~3));   // [gtotal]
    __shared__ __align__(8) unsigned long long full_bar[KR_STAGES], empty_bar[KR_STAGES];
    __shared__ int s_bin[32];

    const long long n = a.n;
    const long long ntiles = (n + KR_T - 1) / KR_T;
    const long long t0 = blockIdx.x * tiles_per_block;
    const long long t1 = min(ntiles, t0 + tiles_per_block);
    const long long my_tiles = t1 > t0 ? t1 - t0 : 0;

    if (threadIdx.x == 0) {
        for (int st = 0; st < KR_STAGES; ++st) {
            mbar_init(&full_bar[st], 1);
            mbar_init(&empty_bar[st], KR_NWC);
        }
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < a.gtotal; i += KR_THREADS) s_grid[i] = a.gvals[i];
    for (long long i = threadIdx.x; i < hw; i += KR_THREADS) hist[i] = 0u;
    float lo[D > 0 ? D : 1], sc[D > 0 ? D : 1];
    build_bin_tables<D>(a, s_grid, tab, s_bin, lo, sc, KR_THREADS);  // ends with __syncthreads

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == KR_NWC) {
        // ---------------- producer
        if (lane == 0) {
            const unsigned long long pol = l2_evict_first_policy();
            for (long long i = 0; i < my_tiles; ++i) {
                const int st = (int)(i % KR_STAGES);
                if (i >= KR_STAGES) mbar_wait(&empty_bar[st], (unsigned)(((i / KR_STAGES) - 1) & 1));
                const long long base = (t0 + i) * KR_T;
                const long long len = min((long long)KR_T, n - base);
                const unsigned bytes = (unsigned)(len * 8);
                mbar_arrive_expect_tx(&full_bar[st], bytes * NV);
                double* dst = ring + (size_t)st * NV * KR_T;
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const double* col = v < D ? a.scores + (long long)v * n
                                              : (v == D ? a.in : a.out + (long long)(v - D - 1) * n);
                    bulk_g2s(dst + v * KR_T, col + base, bytes, &full_bar[st], pol);
                }
            }
        }
        return;
    }
    // ---------------- consumers
    bool bad = false;
    for (long long i = 0; i < my_tiles; ++i) {
        const int st = (int)(i % KR_STAGES);
        const long long base = (t0 + i) * KR_T;
        const int len = (int)min((long long)KR_T, n - base);
        mbar_wait(&full_bar[st], (unsigned)((i / KR_STAGES) & 1));
        const double* src = ring + (size_t)st * NV * KR_T + threadIdx.x;
        double x[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) x[v] = src[v * KR_T];
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[st]);
        if ((int)threadIdx.x < len) {
            unsigned long long pk = 0;
            unsigned cell = 0;
#pragma unroll
            for (int d = 0; d < D; ++d) {
                const int rk = a.bin_ok ? rank_binned(s_grid + a.goff[d], tab + d * (KH_NB + 1), a.G[d], lo[d],
                                                      sc[d], x[d])
                                        : rank_of(s_grid + a.goff[d], a.G[d], a.gtop[d], x[d]);
                pk |= (unsigned long long)rk << (16 * d);
                cell += (unsigned)rk * (unsigned)a.stride[d];
            }
            a.ranks[base + threadIdx.x] = pk;
            hist32_add<C>(hist, a.hi_acc, cell, x + D, bad);
        }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.flags, 1u);
    named_bar_sync(1, KR_NWC * 32);
    unsigned* part = a.part32 + (long long)blockIdx.x * cells * Q;
    for (long long i = threadIdx.x; i < cells * Q; i += KR_NWC * 32) __stcg(part + i, hist[i]);
}

// u32 form: hist = sum over blocks of the u32 partials + the high-part accumulator.
__global__ void k_hist_sum32(const unsigned* __restrict__ part, long long len, int nblocks,
                             const unsigned long long* __restrict__ hi, unsigned long long* __restrict__ hist) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= len) return;
    unsigned long long s = hi[i];
    for (int b = 0; b < nblocks; ++b) s += __ldcs(part + (long long)b * len + i);
    hist[i] = s;
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

// K3 with chunk tables (large traces): the sorted columns are cut into
// chunks of P95_CHUNK positions from the top; per chunk a dominance table over
// the rank cells gives every workload's member count in that chunk
// (count(m_0..m_{i-1}, top..top) = members of the stage-i workload with prefix
// m).  A query walks the chunk counts to the chunk holding its need-th largest
// member and scans only that chunk, instead of ~5% of the column.
constexpr int P95_CHUNK = 1024;

__global__ void __launch_bounds__(256) k_p95_tables(const unsigned long long* __restrict__ vals, long long n,
                                                    int D, WorkloadArgs a, long long cells, int nch,
                                                    unsigned short* __restrict__ tab) {
    extern __shared__ unsigned int cnt[];
    const int k = blockIdx.x, tl = blockIdx.y;
    const int list = tl == 0 ? 0 : 1 + tl;
    const unsigned long long* V = vals + (long long)list * n;
    for (long long c = threadIdx.x; c < cells; c += blockDim.x) cnt[c] = 0u;
    __syncthreads();
    const long long hi = n - (long long)k * P95_CHUNK;
    const long long lo = hi - P95_CHUNK > 0 ? hi - P95_CHUNK : 0;
    for (long long pos = lo + threadIdx.x; pos < hi; pos += blockDim.x) {
        const unsigned long long pk = V[pos];
        long long cell = 0;
        for (int d = 0; d < D; ++d) cell += (long long)((pk >> (16 * d)) & 0xffffull) * a.stride[d];
        atomicAdd(&cnt[cell], 1u);
    }
    __syncthreads();
    for (int d = 0; d < D; ++d) {  // dominance prefix along each dimension
        const long long len = a.G[d] + 1;
        const long long lines = cells / len;
        for (long long L = threadIdx.x; L < lines; L += blockDim.x) {
            const long long base = (L / a.stride[d]) * a.stride[d] * len + L % a.stride[d];
            unsigned run = 0;
            for (long long j = 0; j < len; ++j) {
                run += cnt[base + j * a.stride[d]];
                cnt[base + j * a.stride[d]] = run;
            }
        }
        __syncthreads();
    }
    unsigned short* out = tab + ((long long)tl * nch + k) * cells;
    for (long long c = threadIdx.x; c < cells; c += blockDim.x) out[c] = (unsigned short)cnt[c];
}

__global__ void k_p95_query(WorkloadArgs a, const unsigned long long* __restrict__ keys,
                            const unsigned long long* __restrict__ vals, long long n, int D, long long cells,
                            int nch, const unsigned short* __restrict__ tab, double* __restrict__ p95_in,
                            double* __restrict__ p95_out) {
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
    long long cell = 0;
    for (int d = 0; d < D; ++d) {
        if (d < i) {
            m[d] = (unsigned)(w % a.G[d]);
            w /= a.G[d];
            cell += (long long)m[d] * a.stride[d];
        } else {
            cell += (long long)a.G[d] * a.stride[d];
        }
    }
    const int list = which ? 1 + i : 0;
    const unsigned long long* K = keys + (long long)list * n;
    const unsigned long long* V = vals + (long long)list * n;
    long long need = (long long)cnt - p95_index((long long)cnt);  // the need-th largest member
    if (i == 0) {
        if (lane == 0) dst[t] = key_to_dbl(K[n - need]);
        return;
    }
    const int tl = which ? i : 0;
    const unsigned short* T = tab + (long long)tl * nch * cells + cell;
    int kc = -1;
    for (int k0 = 0; k0 < nch && kc < 0; k0 += 32) {
        const int k = k0 + lane;
        unsigned c = k < nch ? (unsigned)T[(long long)k * cells] : 0u;
        unsigned incl = c;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += y;
        }
        const unsigned hit = __ballot_sync(0xffffffffu, (long long)incl >= need);
        if (hit) {
            const int L = __ffs(hit) - 1;
            need -= (long long)__shfl_sync(0xffffffffu, incl - c, L);
            kc = k0 + L;
        } else {
            need -= (long long)__shfl_sync(0xffffffffu, incl, 31);
        }
    }
    const long long top = n - 1 - (long long)kc * P95_CHUNK;  // first position of the chunk, descending
    for (long long base = 0; base < P95_CHUNK; base += 32) {
        const long long pos = top - base - lane;
        bool member = false;
        if (pos >= 0 && base + lane < P95_CHUNK) {
            const unsigned long long pk = V[pos];
            member = true;
            for (int d = 0; d < i; ++d) member &= ((unsigned)((pk >> (16 * d)) & 0xffffu) <= m[d]);
        }
        const unsigned b = __ballot_sync(0xffffffffu, member);
        const int c = __popc(b);
        if (c >= need) {
            const int L = __fns(b, 0, (int)need);
            if (lane == 0) dst[t] = key_to_dbl(K[top - base - L]);
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
        // accepted scores of 16 requests first (independent of the sum), then
        // the trace-order chain of 16 adds: the chain is the only serial part
        constexpr int QB = 16;
        int k = 0;
        for (; k + QB <= len; k += QB) {
            double acc[QB];
#pragma unroll
            for (int j = 0; j < QB; ++j) {
                acc[j] = tile[C - 1][k + j];
#pragma unroll
                for (int d = D - 1; d >= 0; --d) {
                    const double s = tile[d][k + j];
                    acc[j] = (s >= h[d]) ? s : acc[j];
                }
            }
#pragma unroll
            for (int j = 0; j < QB; ++j) sum = __dadd_rn(sum, acc[j]);
        }
        for (; k < len; ++k) {
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


// ---------------------------------------------------------------------------
// K2, block-parallel and still bit-exact.  The reference's quality is the
// trace-order fold s <- fl(s + a_r) of each tuple's accepted scores
// (routing.cpp:79).  While s stays in one binade [2^e, 2^(e+1)) every partial
// sum is a multiple of u = 2^(e-52), so for a_r >= 0 each step adds exactly
// u * rn(a_r / u) -- unless a_r / u is a tie (then the parity of s decides).
// A block of requests therefore advances s by an integer D(e) of units that
// does not depend on s, and the fold over blocks is an integer chain:
//   Q1  per (tuple, block): approximate block sum (any order) and a flag for
//       negative / non-finite scores;
//   Q2  per tuple: approximate prefix -> the binade each block will run in,
//       or "sequential" when a block may cross a binade (or s = 0, or flagged);
//   Q3  per (tuple, block) in one binade: D = sum of rn(a_r / u) (integer
//       shifts of the scores' bits), "sequential" on any tie or a_r >= s;
//   Q4  per tuple: the exact chain -- fast blocks check that s is in the
//       binade and stays below 2^(e+1) (partial sums are monotone), then
//       s += u * D exactly; every other block is folded request by request
//       with __dadd_rn, as the reference does.
// Sequential blocks are the first (s = 0), ~log2(blocks) binade crossings and
// the rare ties, so the fp64 add chain shrinks from n to a few blocks.
constexpr int QX_THREADS = 256;   // tuples per CTA of Q1 / Q3
constexpr int QX_TILE = 1024;     // requests staged per shared-memory tile
constexpr short QX_SEQ = -1;      // block folded sequentially in Q4

template <int D>
__device__ __forceinline__ double accepted_score(const double* __restrict__ row, const double* h) {
    double a = row[D];
#pragma unroll
    for (int d = D - 1; d >= 0; --d) a = (row[d] >= h[d]) ? row[d] : a;
    return a;
}

template <int D>
__device__ __forceinline__ void stage_tile(const double* __restrict__ scores, long long n, long long base, int len,
                                           double* tile) {
    constexpr int C = D + 1;
    for (int i = 0; i < C; ++i)
        for (int k = threadIdx.x; k < len; k += blockDim.x) tile[k * C + i] = scores[(long long)i * n + base + k];
}

// Q1: grid (blocks, tuple groups); approximate block sums, NaN marks a block
// with a negative, -0.0 or non-finite accepted score.
template <int D>
__global__ void __launch_bounds__(QX_THREADS) k_qx_approx(const double* __restrict__ scores, long long n, int B,
                                                          const double* __restrict__ thr, long long ncand, int nb,
                                                          double* __restrict__ A) {
    constexpr int C = D + 1;
    extern __shared__ double qtile[];
    const int b = blockIdx.x;
    const long long c = (long long)blockIdx.y * QX_THREADS + threadIdx.x;
    double h[D > 0 ? D : 1];
#pragma unroll
    for (int d = 0; d < D; ++d) h[d] = c < ncand ? thr[c * D + d] : 0.0;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    bool bad = false;
    const long long b0 = (long long)b * B;
    const long long b1 = b0 + B < n ? b0 + B : n;
    for (long long base = b0; base < b1; base += QX_TILE) {
        const int len = (int)(b1 - base < QX_TILE ? b1 - base : QX_TILE);
        __syncthreads();
        stage_tile<D>(scores, n, base, len, qtile);
        __syncthreads();
        int k = 0;
        for (; k + 4 <= len; k += 4) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const double a = accepted_score<D>(qtile + (k + j) * C, h);
                const unsigned long long bits = (unsigned long long)__double_as_longlong(a);
                bad |= (bits >> 63) != 0ull || (bits >> 52) == 2047ull;
                acc[j] += a;
            }
        }
        for (; k < len; ++k) {
            const double a = accepted_score<D>(qtile + k * C, h);
            const unsigned long long bits = (unsigned long long)__double_as_longlong(a);
            bad |= (bits >> 63) != 0ull || (bits >> 52) == 2047ull;
            acc[0] += a;
        }
    }
    if (c < ncand) A[c * nb + b] = bad ? __longlong_as_double(0x7ff8000000000000ll) : (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// Q2: one warp per tuple; the binade (biased exponent) each block runs in.
__global__ void k_qx_binades(const double* __restrict__ A, long long ncand, int nb, short* __restrict__ E) {
    const long long c = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (c >= ncand) return;
    double run = 0.0;  // approximate prefix before this chunk
    for (int b0 = 0; b0 < nb; b0 += 32) {
        const int b = b0 + lane;
        const double a = b < nb ? A[c * nb + b] : 0.0;
        const bool bad = a != a;
        double incl = bad ? 0.0 : a;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const double v = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += v;
        }
        const double lo = (run + incl - (bad ? 0.0 : a)) * (1.0 - 1e-9);
        const double hi = (run + incl) * (1.0 + 1e-9);
        short e = QX_SEQ;
        if (!bad && lo > 0.0) {
            const int elo = (int)(((unsigned long long)__double_as_longlong(lo) >> 52) & 2047ull);
            const int ehi = (int)(((unsigned long long)__double_as_longlong(hi) >> 52) & 2047ull);
            if (elo == ehi && elo > 52 && elo < 2047) e = (short)elo;  // u = 2^(e-52) normal
        }
        if (b < nb) E[c * nb + b] = e;
        run += __shfl_sync(0xffffffffu, incl, 31);
    }
}

// Q3: grid (blocks, tuple groups); units of u = 2^(e-52) added by each block.
template <int D>
__global__ void __launch_bounds__(QX_THREADS) k_qx_units(const double* __restrict__ scores, long long n, int B,
                                                         const double* __restrict__ thr, long long ncand, int nb,
                                                         short* __restrict__ E, unsigned long long* __restrict__ U) {
    constexpr int C = D + 1;
    extern __shared__ double qtile[];
    const int b = blockIdx.x;
    const long long c = (long long)blockIdx.y * QX_THREADS + threadIdx.x;
    const bool live = c < ncand;
    const int eb = live ? (int)E[c * nb + b] : QX_SEQ;
    if (__syncthreads_and(eb == QX_SEQ)) return;  // the whole CTA folds this block sequentially
    double h[D > 0 ? D : 1];
#pragma unroll
    for (int d = 0; d < D; ++d) h[d] = live ? thr[c * D + d] : 0.0;
    unsigned long long sum = 0ull;
    bool seq = eb == QX_SEQ;
    const long long b0 = (long long)b * B;
    const long long b1 = b0 + B < n ? b0 + B : n;
    for (long long base = b0; base < b1; base += QX_TILE) {
        const int len = (int)(b1 - base < QX_TILE ? b1 - base : QX_TILE);
        __syncthreads();
        stage_tile<D>(scores, n, base, len, qtile);
        __syncthreads();
        if (seq) continue;
        for (int k = 0; k < len; ++k) {
            const double a = accepted_score<D>(qtile + k * C, h);
            const unsigned long long bits = (unsigned long long)__double_as_longlong(a);
            const int ea = (int)(bits >> 52);  // sign bit is 0 here (Q1 checked)
            const unsigned long long m = (bits & 0xfffffffffffffull) | (ea ? (1ull << 52) : 0ull);
            const int sh = eb - (ea ? ea : 1);
            seq |= sh <= 0;  // a >= 2^e: s + a leaves the binade
            if (sh > 0 && sh < 64) {
                const unsigned long long r = m << (64 - sh);
                seq |= r == (1ull << 63);  // tie: the parity of s decides
                sum += (m >> sh) + (r > (1ull << 63) ? 1ull : 0ull);
            }
        }
    }
    if (!live) return;
    if (seq) E[c * nb + b] = QX_SEQ;
    else U[c * nb + b] = sum;
}

// Q4: one warp per tuple, the exact chain over blocks.  The warp reads 32
// blocks' (binade, units) at once; a chunk whose blocks all run in the
// current binade advances s by the warp's integer sum of their units in one
// step.  Otherwise the chunk is walked block by block: fast blocks as integer
// steps, the rest folded request by request -- the lanes load and select 32
// accepted scores at a time (independent of s), lane 0's chain adds them in
// trace order with __dadd_rn.
template <int D>
__device__ double qx_fold_block(const double* __restrict__ scores, long long n, long long b0, long long b1,
                                const double* h, double s, int lane) {
    constexpr int C = D + 1;
    for (long long r0 = b0; r0 < b1; r0 += 32) {
        const long long r = r0 + lane;
        double a = 0.0;
        if (r < b1) {
            double row[C];
#pragma unroll
            for (int i = 0; i < C; ++i) row[i] = scores[(long long)i * n + r];
            a = accepted_score<D>(row, h);
        }
        const int cnt = (int)(b1 - r0 < 32 ? b1 - r0 : 32);
        if (cnt == 32) {
            double v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __shfl_sync(0xffffffffu, a, j);
#pragma unroll
            for (int j = 0; j < 32; ++j) s = __dadd_rn(s, v[j]);
        } else {
            for (int j = 0; j < cnt; ++j) s = __dadd_rn(s, __shfl_sync(0xffffffffu, a, j));
        }
    }
    return s;
}

// s in [2^e, 2^(e+1)) (biased e) and s + units * 2^(e-52) < 2^(e+1): the exact
// result, else a negative value.
__device__ __forceinline__ double qx_units_step(double s, int eb, unsigned long long units) {
    const double u = __longlong_as_double((long long)(eb - 52) << 52);
    const double lo = __longlong_as_double((long long)eb << 52);
    if (!(s >= lo && s < 2.0 * lo)) return -1.0;
    const unsigned long long su = (unsigned long long)__double2ll_rn(__ddiv_rn(s, u));  // exact
    const unsigned long long t = su + units;
    if (t >= (1ull << 53) || t < su) return -1.0;
    return __dmul_rn((double)(long long)t, u);  // exact: t < 2^53
}

template <int D>
__global__ void k_qx_chain(const double* __restrict__ scores, long long n, int B,
                           const double* __restrict__ thr, long long ncand, int nb,
                           const short* __restrict__ E, const unsigned long long* __restrict__ U,
                           double* __restrict__ qsum, unsigned long long* __restrict__ seq_blocks) {
    const long long c = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (c >= ncand) return;
    double h[D > 0 ? D : 1];
#pragma unroll
    for (int d = 0; d < D; ++d) h[d] = thr[c * D + d];
    double s = 0.0;
    unsigned long long nseq = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
        const int b = b0 + lane;
        const int eb = b < nb ? (int)E[c * nb + b] : -2;  // -2: past the end
        const unsigned long long uu = (b < nb && eb >= 0) ? U[c * nb + b] : 0ull;
        // fast chunk: every live block in the binade of s
        const int es = s > 0.0 ? (int)(((unsigned long long)__double_as_longlong(s) >> 52) & 2047ull) : -3;
        if (__all_sync(0xffffffffu, eb == es || eb == -2)) {
            unsigned long long tot = uu;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
            const double t = qx_units_step(s, es, tot);  // every live unit sum < 2^53: no wrap
            if (t >= 0.0) {
                s = t;
                continue;
            }
        }
        const int cnt = nb - b0 < 32 ? nb - b0 : 32;
        for (int j = 0; j < cnt; ++j) {
            const int ej = __shfl_sync(0xffffffffu, eb, j);
            const unsigned long long uj = __shfl_sync(0xffffffffu, uu, j);
            if (ej >= 0) {
                const double t = qx_units_step(s, ej, uj);
                if (t >= 0.0) {
                    s = t;
                    continue;
                }
            }
            ++nseq;
            const long long r0 = (long long)(b0 + j) * B;
            s = qx_fold_block<D>(scores, n, r0, r0 + B < n ? r0 + B : n, h, s, lane);
        }
    }
    if (lane == 0) {
        qsum[c] = s;
        if (seq_blocks) atomicAdd(seq_blocks, nseq);
    }
}

template <int D>
void launch_qx(const double* scores, long long n, const double* thr, long long ncand, double* qsum,
               const QualityScratch& q, cudaStream_t s, int* launches) {
    const int nb = (int)((n + q.B - 1) / q.B);
    const dim3 grid((unsigned)nb, (unsigned)((ncand + QX_THREADS - 1) / QX_THREADS));
    const size_t smem = (size_t)QX_TILE * (D + 1) * sizeof(double);
    CG_CUDA(cudaFuncSetAttribute(k_qx_approx<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CG_CUDA(cudaFuncSetAttribute(k_qx_units<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_qx_approx<D><<<grid, QX_THREADS, smem, s>>>(scores, n, q.B, thr, ncand, nb, q.A);
    CG_LAUNCH_CHECK();
    k_qx_binades<<<(unsigned)((ncand * 32 + 255) / 256), 256, 0, s>>>(q.A, ncand, nb, q.E);
    CG_LAUNCH_CHECK();
    k_qx_units<D><<<grid, QX_THREADS, smem, s>>>(scores, n, q.B, thr, ncand, nb, q.E, q.U);
    CG_LAUNCH_CHECK();
    k_qx_chain<D><<<(unsigned)((ncand * 32 + 127) / 128), 128, 0, s>>>(scores, n, q.B, thr, ncand, nb, q.E, q.U,
                                                                       qsum, q.seq_blocks);
    CG_LAUNCH_CHECK();
    if (launches) *launches += 4;
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

size_t hist32_smem_bytes(long long cells, int D, int gtotal) {
    const int Q = 3 + D;
    return (size_t)((cells * Q + 3) & ~3ll) * 4 + (size_t)((D * (KH_NB + 1) + 3) & ~3) * 4 + (size_t)gtotal * 8;
}

template <int D>
void launch_k1(const RouteArgs& a, int sm_count, cudaStream_t s, int* launches, int* nblocks_out) {
    const size_t hsm = hist32_smem_bytes(a.cells, D, a.gtotal);
    const size_t tsm_r = KRLayout<D>::ring_bytes + hsm;
    const bool aligned = (a.n & 1) == 0 && ((reinterpret_cast<unsigned long long>(a.scores) |
                                             reinterpret_cast<unsigned long long>(a.in) |
                                             reinterpret_cast<unsigned long long>(a.out)) & 15ull) == 0;
    if (a.part32 && a.hi_acc && aligned && a.k1_form == 0 && tsm_r <= 200 * 1024 && a.n > 0) {
        auto kern = k_route_tma<D>;
        CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm_r));
        int per_sm = 0;
        CG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, KR_THREADS, tsm_r));
        const long long cap = (long long)sm_count * (per_sm < 1 ? 1 : per_sm);
        const long long ntiles = (a.n + KR_T - 1) / KR_T;
        long long tpb = (ntiles + cap - 1) / cap;
        if (tpb > KR_MAX_TILES) {  // more than one wave: equal waves of full-size blocks
            const long long waves = (ntiles + cap * KR_MAX_TILES - 1) / (cap * KR_MAX_TILES);
            tpb = (ntiles + cap * waves - 1) / (cap * waves);
        }
        if (tpb < 1) tpb = 1;
        const long long blocks = (ntiles + tpb - 1) / tpb;
        const long long Q = 3 + D;
        if (blocks * a.cells * Q <= a.part32_words) {  // hi_acc is zeroed by the caller
            kern<<<(unsigned)blocks, KR_THREADS, tsm_r, s>>>(a, tpb);
            CG_LAUNCH_CHECK();
            if (launches) *launches += 1;
            if (nblocks_out) *nblocks_out = -(int)blocks - (1 << 24);  // u32 partial layout
            return;
        }
    }
    if (a.part32 && a.hi_acc && hsm <= 110 * 1024) {
        auto kern = a.k1_form == 3 ? k_route_hist<D, 1> : k_route_hist<D, 2>;
        CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm));
        int per_sm = 0;
        CG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, KH_THREADS, hsm));
        const long long npairs = (a.n + 1) / 2;
        long long blocks = (long long)sm_count * (per_sm < 1 ? 1 : per_sm);
        const long long need = (npairs + (long long)KH_MAX_ITERS * KH_THREADS - 1) / ((long long)KH_MAX_ITERS * KH_THREADS);
        const long long useful = (npairs + KH_THREADS - 1) / KH_THREADS;
        if (blocks > useful) blocks = useful;
        if (blocks < need) blocks = need;
        if (blocks < 1) blocks = 1;
        const long long Q = 3 + D;
        if (blocks * a.cells * Q <= a.part32_words) {  // hi_acc is zeroed by the caller
            kern<<<(unsigned)blocks, KH_THREADS, hsm, s>>>(a);
            CG_LAUNCH_CHECK();
            if (launches) *launches += 1;
            if (nblocks_out) *nblocks_out = -(int)blocks - (1 << 24);  // u32 partial layout
            return;
        }
    }
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
    if (nblocks <= -(1 << 24)) {  // u32 form: [blocks][cells][2+C] u32 partials + high parts -> hist
        const long long len = a.cells * (2 + C);
        const int nb = -(nblocks + (1 << 24));
        k_hist_sum32<<<(unsigned)((len + 255) / 256), 256, 0, s>>>(a.part32, len, nb, a.hi_acc, a.hist);
        CG_LAUNCH_CHECK();
        if (launches) ++*launches;
        return;
    }
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

long long p95_table_entries(const WorkloadArgs& a, long long n) {
    const int D = a.C - 1;
    long long cells = 1;
    for (int d = 0; d < D; ++d) cells *= a.G[d] + 1;
    if (D == 0 || cells > 16384 || n < 65536) return 0;  // the direct scan
    return (long long)a.C * ((n + P95_CHUNK - 1) / P95_CHUNK) * cells;
}

void launch_p95_scan(const WorkloadArgs& a, const unsigned long long* keys,
                     const unsigned long long* vals, long long n, double* p95_in, double* p95_out,
                     unsigned short* tables, cudaStream_t s, int* launches) {
    const long long warps = 2 * a.total;
    if (tables && p95_table_entries(a, n) > 0) {
        const int D = a.C - 1;
        long long cells = 1;
        for (int d = 0; d < D; ++d) cells *= a.G[d] + 1;
        const int nch = (int)((n + P95_CHUNK - 1) / P95_CHUNK);
        const size_t smem = (size_t)cells * 4;
        CG_CUDA(cudaFuncSetAttribute(k_p95_tables, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_p95_tables<<<dim3((unsigned)nch, (unsigned)a.C), 256, smem, s>>>(vals, n, D, a, cells, nch, tables);
        CG_LAUNCH_CHECK();
        k_p95_query<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(a, keys, vals, n, D, cells, nch, tables,
                                                                         p95_in, p95_out);
        CG_LAUNCH_CHECK();
        if (launches) *launches += 2;
        return;
    }
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

int quality_block(long long n, long long ncand) {
    // requests per block: entries (tuples x blocks) stay <= 2^24 (~300 MB of scratch)
    int B = QX_TILE;
    while ((double)ncand * (double)((n + B - 1) / B) > (double)(1 << 24) && B < (1 << 30)) B *= 2;
    return B;
}

void launch_quality(const double* scores, long long n, int D, const double* thr, long long ncand,
                    double* qsum, const QualityScratch* q, cudaStream_t s, int* launches) {
    if (ncand <= 0 || n <= 0) return;
    if (q) {  // block-parallel exact form
        switch (D) {
            case 0: launch_qx<0>(scores, n, thr, ncand, qsum, *q, s, launches); return;
            case 1: launch_qx<1>(scores, n, thr, ncand, qsum, *q, s, launches); return;
            case 2: launch_qx<2>(scores, n, thr, ncand, qsum, *q, s, launches); return;
            case 3: launch_qx<3>(scores, n, thr, ncand, qsum, *q, s, launches); return;
            case 4: launch_qx<4>(scores, n, thr, ncand, qsum, *q, s, launches); return;
            default: throw EngineError(101, "GPU engine supports up to 5 cascade stages");
        }
    }
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
