// K6-K7: inner min-max allocation per threshold candidate, candidate
// expansion to grid order, weighted-Tchebycheff argmin per weight, Pareto front.
//
// Reference:
//   innerplan::solve_min_max   proj/src/innerplan.cpp:123-194
//   sweep's per-candidate table proj/src/outerplan.cpp:229-289 (cell [0] = INF for live stages)
//   tchebycheff_score + argmin proj/src/outerplan.cpp:61-65, 295-315
//   pareto_filter              proj/src/outerplan.cpp:93-112
//
// solve_min_max binary-searches the sorted distinct finite cells for the
// smallest L with sum_i min{f : l_i(f) <= L} <= N.  Feasibility is monotone
// in L and every row is non-increasing over its feasible suffix, so the
// optimum is min over live rows i of (the smallest feasible value in row i),
// found by a binary search per row -- no per-candidate sort.
#include <cuda_runtime.h>

#include "cg_cuda.h"
#include "cg_internal.h"
#include "cg_kernels.h"

namespace cg {

namespace {

constexpr unsigned long long kInfBits = 0x7ff0000000000000ull;

__device__ __forceinline__ double cell_at(const double* row_lat, int f, int raw_f0) {
    return (f == 0 && !raw_f0) ? __longlong_as_double((long long)kInfBits) : row_lat[f];
}

// smallest f in [0, N] with finite cell <= v, or -1 (min_budget_within, innerplan.cpp:123-127)
__device__ int min_f_within(const double* row_lat, int N, int raw_f0, double v) {
    if (!(cell_at(row_lat, N, raw_f0) <= v)) return -1;
    int lo = 0, hi = N;  // predicate cell(f) <= v is monotone (false..true) on validated rows
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cell_at(row_lat, mid, raw_f0) <= v) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

__global__ void k_solve(SolveArgs a) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= a.ntuples) return;
    const double INF = __longlong_as_double((long long)kInfBits);
    const double* rows[kMaxStages];
    int live[kMaxStages];
    int nl = 0;
    for (int i = 0; i < a.C; ++i) {
        const long long w = (i == 0) ? 0 : t % a.wl_P[i];
        const long long idx = a.wl_off[i] + w;
        if (a.wl_count[idx] > 0) {
            const int r = a.wl_row[idx];
            rows[nl] = a.final_lat + (long long)r * (a.N + 1);
            live[nl] = i;
            ++nl;
        }
        a.alloc[t * a.C + i] = 0;
        a.plan[t * a.C + i] = -1;
    }
    auto feasible = [&](double v) {
        long long need = 0;
        for (int q = 0; q < nl; ++q) {
            const int f = min_f_within(rows[q], a.N, a.raw_f0, v);
            if (f < 0) return false;
            need += f;
        }
        return need <= a.total_gpus;
    };
    // candidates = finite cells with f <= total_gpus; optimum = min over rows of
    // the smallest feasible candidate of that row (feasibility monotone in v).
    const int fmax = a.total_gpus < a.N ? a.total_gpus : a.N;
    const int flo = a.raw_f0 ? 0 : 1;
    double best = INF;
    for (int q = 0; q < nl; ++q) {
        const double* rl = rows[q];
        if (fmax < flo || cell_at(rl, fmax, a.raw_f0) == INF) continue;
        int lo = flo, hi = fmax;  // first finite cell
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (cell_at(rl, mid, a.raw_f0) != INF) hi = mid;
            else lo = mid + 1;
        }
        const int first = lo;
        if (!feasible(cell_at(rl, first, a.raw_f0))) continue;
        lo = first;
        hi = fmax;  // largest f with feasible(cell(f))
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (feasible(cell_at(rl, mid, a.raw_f0))) lo = mid;
            else hi = mid - 1;
        }
        const double v = cell_at(rl, lo, a.raw_f0);
        if (v < best) best = v;
    }
    if (nl == 0 || best == INF) {
        a.feasible[t] = 0;
        a.L[t] = INF;
        return;
    }
    int used = 0;
    int fs[kMaxStages];
    for (int q = 0; q < nl; ++q) {
        fs[q] = min_f_within(rows[q], a.N, a.raw_f0, best);
        used += fs[q];
    }
    fs[nl - 1] += a.total_gpus - used;  // the last live stage absorbs the slack
    double L = 0.0;
    for (int q = 0; q < nl; ++q) {
        const int i = live[q];
        const double c = cell_at(rows[q], fs[q], a.raw_f0);
        L = (L < c) ? c : L;  // std::max
        a.alloc[t * a.C + i] = fs[q];
        const long long idx = a.wl_off[i] + ((i == 0) ? 0 : t % a.wl_P[i]);
        const int r = a.wl_row[idx];
        a.plan[t * a.C + i] = (fs[q] == 0 && !a.raw_f0) ? -1 : a.final_plan[(long long)r * (a.N + 1) + fs[q]];
    }
    a.feasible[t] = 1;
    a.L[t] = L;
}

// grid order (first dimension outermost) -> distinct tuple, feasibility flag
__global__ void k_expand(ExpandArgs a) {
    const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (c >= a.ncand) return;
    long long rem = c;
    long long tuple = 0;
    long long tstride[4];
    long long s = 1;
    for (int d = 0; d < a.D; ++d) {
        tstride[d] = s;
        s *= a.Gd[d];
    }
    for (int d = a.D - 1; d >= 0; --d) {
        const long long gi = rem % a.Gg[d];
        rem /= a.Gg[d];
        tuple += (long long)a.g2d[a.goff[d] + gi] * tstride[d];
    }
    a.cand_tuple[c] = tuple;
    a.flag[c] = a.tuple_feasible[tuple] ? 1u : 0u;
}

__global__ void k_compact_evals(ExpandArgs a, const unsigned* __restrict__ pos,
                                const double* __restrict__ tuple_L, const double* __restrict__ tuple_qsum,
                                double n, long long* __restrict__ eval_cand, double* __restrict__ eval_L,
                                double* __restrict__ eval_Q, long long* __restrict__ skip_cand) {
    const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (c >= a.ncand) return;
    const long long t = a.cand_tuple[c];
    if (a.flag[c]) {
        const unsigned e = pos[c];
        eval_cand[e] = c;
        eval_L[e] = tuple_L[t];
        eval_Q[e] = __ddiv_rn(tuple_qsum[t], n);
    } else {
        skip_cand[c - pos[c]] = c;
    }
}

// K7: per weight, argmin over evaluations of (T, L, -Q, index).
struct Best {
    double T, L, Q;
    long long e;
};

__device__ __forceinline__ bool better(const Best& x, const Best& y) {
    if (y.e < 0) return x.e >= 0;
    if (x.e < 0) return false;
    if (x.T != y.T) return x.T < y.T;
    if (x.L != y.L) return x.L < y.L;
    if (x.Q != y.Q) return x.Q > y.Q;
    return x.e < y.e;
}

__global__ void __launch_bounds__(256) k_tchebycheff(const double* __restrict__ L,
                                                     const double* __restrict__ Q, long long E,
                                                     const double* __restrict__ weights, double z1,
                                                     double z2, int* __restrict__ sel) {
    const int wi = blockIdx.x;
    const double l1 = weights[2 * wi], l2 = weights[2 * wi + 1];
    Best b{0, 0, 0, -1};
    for (long long e = threadIdx.x; e < E; e += blockDim.x) {
        const double a1 = __dmul_rn(l1, __dsub_rn(L[e], z1));
        const double a2 = __dmul_rn(l2, __dsub_rn(z2, Q[e]));
        const Best c{(a1 < a2) ? a2 : a1, L[e], Q[e], e};  // std::max(a1, a2)
        if (better(c, b)) b = c;
    }
    for (int off = 16; off > 0; off >>= 1) {
        Best o;
        o.T = __shfl_down_sync(0xffffffffu, b.T, off);
        o.L = __shfl_down_sync(0xffffffffu, b.L, off);
        o.Q = __shfl_down_sync(0xffffffffu, b.Q, off);
        o.e = __shfl_down_sync(0xffffffffu, b.e, off);
        if (better(o, b)) b = o;
    }
    __shared__ Best sb[8];
    if ((threadIdx.x & 31) == 0) sb[threadIdx.x >> 5] = b;
    __syncthreads();
    if (threadIdx.x == 0) {
        Best r = sb[0];
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i)
            if (better(sb[i], r)) r = sb[i];
        sel[wi] = (int)r.e;
    }
}

__global__ void k_pareto_keys(const double* __restrict__ L, const double* __restrict__ Q, long long E,
                              unsigned long long* __restrict__ kq, unsigned long long* __restrict__ kl,
                              unsigned long long* __restrict__ idx) {
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= E) return;
    kq[e] = ~dbl_to_key(Q[e]);  // quality descending
    kl[e] = dbl_to_key(L[e]);
    idx[e] = (unsigned long long)e;
}

__global__ void k_gather_keys(const unsigned long long* __restrict__ src,
                              const unsigned long long* __restrict__ order, long long E,
                              unsigned long long* __restrict__ dst) {
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= E) return;
    dst[e] = src[order[e]];
}

// Single block: keep a point iff Q > max Q of all points before it in the
// (L asc, Q desc, index asc) order (pareto_filter, outerplan.cpp:105-111).
__global__ void __launch_bounds__(1024) k_pareto_mark(const unsigned long long* __restrict__ order,
                                                      const double* __restrict__ Q, long long E,
                                                      long long* __restrict__ front,
                                                      long long* __restrict__ front_size) {
    __shared__ double smax[1024];
    __shared__ long long scnt[1024];
    const long long per = (E + 1023) / 1024;
    const long long lo = threadIdx.x * per;
    const long long hi = lo + per < E ? lo + per : E;
    const double NEG = -__longlong_as_double((long long)kInfBits);
    double m = NEG;
    for (long long i = lo; i < hi; ++i) {
        const double q = Q[order[i]];
        m = (q > m) ? q : m;
    }
    smax[threadIdx.x] = m;
    __syncthreads();
    // exclusive max-scan of chunk maxima (Hillis-Steele on inclusive then shift)
    for (int off = 1; off < 1024; off <<= 1) {
        const double v = threadIdx.x >= off ? smax[threadIdx.x - off] : NEG;
        __syncthreads();
        smax[threadIdx.x] = (v > smax[threadIdx.x]) ? v : smax[threadIdx.x];
        __syncthreads();
    }
    double run = threadIdx.x > 0 ? smax[threadIdx.x - 1] : NEG;
    long long c = 0;
    for (long long i = lo; i < hi; ++i) {
        const double q = Q[order[i]];
        if (q > run) {
            ++c;
            run = q;
        }
    }
    scnt[threadIdx.x] = c;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const long long v = threadIdx.x >= off ? scnt[threadIdx.x - off] : 0;
        __syncthreads();
        scnt[threadIdx.x] += v;
        __syncthreads();
    }
    long long w = scnt[threadIdx.x] - c;
    run = threadIdx.x > 0 ? smax[threadIdx.x - 1] : NEG;
    for (long long i = lo; i < hi; ++i) {
        const double q = Q[order[i]];
        if (q > run) {
            front[w++] = (long long)order[i];
            run = q;
        }
    }
    if (threadIdx.x == 1023) *front_size = scnt[1023];
}

// single-block exclusive scan of u32 flags -> u32 positions
__global__ void __launch_bounds__(1024) k_scan_flags(const unsigned* __restrict__ flag, long long n,
                                                     unsigned* __restrict__ pos,
                                                     unsigned long long* __restrict__ total) {
    __shared__ unsigned long long part[1024];
    const long long per = (n + 1023) / 1024;
    const long long lo = threadIdx.x * per;
    const long long hi = lo + per < n ? lo + per : n;
    unsigned long long s = 0;
    for (long long i = lo; i < hi; ++i) s += flag[i];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const unsigned long long v = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    unsigned long long run = part[threadIdx.x] - s;
    for (long long i = lo; i < hi; ++i) {
        pos[i] = (unsigned)run;
        run += flag[i];
    }
    if (threadIdx.x == 1023) *total = part[1023];
}

}  // namespace

void launch_solve(const SolveArgs& a, cudaStream_t s, int* launches) {
    if (a.ntuples <= 0) return;
    k_solve<<<(unsigned)((a.ntuples + 127) / 128), 128, 0, s>>>(a);
    CG_LAUNCH_CHECK();
    if (launches) ++*launches;
}

void launch_expand(const ExpandArgs& a, unsigned* pos, unsigned long long* total,
                   const double* tuple_L, const double* tuple_qsum, double n, long long* eval_cand,
                   double* eval_L, double* eval_Q, long long* skip_cand, cudaStream_t s, int* launches) {
    const unsigned blocks = (unsigned)((a.ncand + 255) / 256);
    k_expand<<<blocks, 256, 0, s>>>(a);
    CG_LAUNCH_CHECK();
    k_scan_flags<<<1, 1024, 0, s>>>(a.flag, a.ncand, pos, total);
    CG_LAUNCH_CHECK();
    k_compact_evals<<<blocks, 256, 0, s>>>(a, pos, tuple_L, tuple_qsum, n, eval_cand, eval_L, eval_Q,
                                         skip_cand);
    CG_LAUNCH_CHECK();
    if (launches) *launches += 3;
}

void launch_tchebycheff(const double* L, const double* Q, long long E, const double* weights, int nw,
                        double z1, double z2, int* sel, cudaStream_t s, int* launches) {
    if (nw <= 0 || E <= 0) return;
    k_tchebycheff<<<nw, 256, 0, s>>>(L, Q, E, weights, z1, z2, sel);
    CG_LAUNCH_CHECK();
    if (launches) ++*launches;
}

void launch_pareto(const double* L, const double* Q, long long E, unsigned long long* k0,
                   unsigned long long* k1, unsigned long long* v0, unsigned long long* v1,
                   unsigned long long* kl, unsigned long long* orax, unsigned int* hist,
                   long long* front, long long* front_size, cudaStream_t s, int* launches) {
    if (E <= 0) return;
    const unsigned blocks = (unsigned)((E + 255) / 256);
    k_pareto_keys<<<blocks, 256, 0, s>>>(L, Q, E, k0, kl, v0);
    CG_LAUNCH_CHECK();
    if (launches) ++*launches;
    // pass 1: stable sort by quality descending (payload = evaluation index)
    unsigned long long h[2];
    launch_or_and(k0, E, orax, s, launches);
    CG_CUDA(cudaMemcpyAsync(h, orax, sizeof(h), cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaStreamSynchronize(s));
    int par = radix_sort_u64(k0, v0, k1, v1, E, h[0] ^ h[1], hist, s, launches);
    unsigned long long* order = par ? v1 : v0;
    unsigned long long* spare = par ? v0 : v1;
    // pass 2: stable sort by latency ascending
    k_gather_keys<<<blocks, 256, 0, s>>>(kl, order, E, k0);
    CG_LAUNCH_CHECK();
    if (launches) ++*launches;
    launch_or_and(k0, E, orax, s, launches);
    CG_CUDA(cudaMemcpyAsync(h, orax, sizeof(h), cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaStreamSynchronize(s));
    par = radix_sort_u64(k0, order, k1, spare, E, h[0] ^ h[1], hist, s, launches);
    unsigned long long* final_order = par ? spare : order;
    k_pareto_mark<<<1, 1024, 0, s>>>(final_order, Q, E, front, front_size);
    CG_LAUNCH_CHECK();
    if (launches) ++*launches;
}

}  // namespace cg
