// K4-K5: the analytical cost model over the allocation x parallelism space.
//
// Reference: proj/src/costmodel.cpp
//   memory_feasible        :79-88     service_time        :176-194
//   enumerate_multisets    :132-146   plan_set            :205-229
//   simulate_plan_p95      :248-292   StageEvaluator::row :296-414
//
// One "row" = one (stage model, WorkloadStats) pair; its value is
// latency[f] = min over stable plans using <= f GPUs of the simulated p95
// sojourn of a 2000-request FCFS join-shortest-queue replay, with the
// reference's deterministic tie-breaks (parts-lexicographic at equal
// latency, smaller budget on prefix ties).
//
// Design (B200):
//   * plans are never materialised: a plan index is unranked from the
//     multiset counting table ways[i][b] and successors come from a
//     lexicographic odometer -- exactly the reference's recursion order;
//   * one plan per group of W lanes, one replica per lane (R replicas per
//     lane beyond 32).  The JSQ choice for a request is a ballot over idle
//     replicas (lowest index wins, the reference's early break) and, only
//     when every replica is busy, a butterfly min over (queue length, index);
//   * per-replica FIFO of waiting finish times in a shared-memory ring with
//     the in-service finish time in a register; a ring overflow re-runs the
//     plan in the DEEP instantiation whose rings live in global memory;
//   * sojourns stream to a per-group scratch column; the exact p95 (the K-th
//     largest, K = n - (ceil(0.95 n) - 1)) is a group-cooperative 8-bit radix
//     select, run only for plans that complete;
//   * exact pruning: once K sojourns of a plan exceed the best latency already
//     found at a budget <= its GPU count, its p95 is strictly larger, so it
//     can never appear in the row (neither as best-at-g nor as a prefix
//     minimum) and the simulation stops.  Row results do not depend on it;
//   * fp64 uses explicit _rn intrinsics, TU compiled with --fmad=false (H2).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "cg_cuda.h"
#include "cg_internal.h"
#include "cg_kernels.h"
#include "plan_dev.cuh"
#include "cg_ptx.cuh"

namespace cg {

namespace {

constexpr double kClampedExpMeanFactor = 0.98168436111126578;  // costmodel.hpp:25
constexpr unsigned long long kInfBits = 0x7ff0000000000000ull;
constexpr unsigned long long kEmpty = ~0ull;
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int class_of_dp(int dp) {
    return dp <= 4 ? 0 : dp <= 8 ? 1 : dp <= 16 ? 2 : dp <= 32 ? 3 : dp <= 64 ? 4 : dp <= 128 ? 5 : 6;
}

// ---------------------------------------------------------------------------
// Row setup

__device__ bool dev_memory_feasible(int tp, int pp, const ModelArgs& m, const HwArgs& hw,
                                    const ParamArgs& p, double kv_tokens) {
    const double gpus = (double)(tp * pp);
    const double weights = __dmul_rn(m.param_count, m.bytes_per_param);
    if (__ddiv_rn(weights, gpus) > hw.mem_capacity) return false;
    const double kv_budget =
        __dmul_rn(p.kv_memory_fraction, __dsub_rn(__dmul_rn(gpus, hw.mem_capacity), weights));
    return kv_budget >= __dmul_rn(m.kv_bytes_per_token, kv_tokens);
}

__global__ void k_row_shapes(RowSetupArgs a) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)a.nrows * kMaxShapes) return;
    const int row = (int)(t / kMaxShapes), s = (int)(t % kMaxShapes);
    const RowDesc rd = a.rows[row];
    const PlanSpace& sp = a.spaces[rd.space];
    const long long o = (long long)row * kMaxShapes + s;
    if (s >= sp.S) {  // no such shape: defined values all the same (tables are read per row, 32 wide)
        a.tab.shape_ok[o] = 0;
        a.tab.prefill[o] = a.tab.decode[o] = a.tab.mean_service[o] = 0.0;
        a.tab.inv_service[o] = __longlong_as_double(0x7ff8000000000000ll);
        return;
    }
    const ModelArgs m = a.models[rd.stage];
    const int tp = sp.shapes[s].tp, pp = sp.shapes[s].pp;
    const double kv_tokens = __dadd_rn(rd.p95_in, rd.p95_out);
    const bool ok = dev_memory_feasible(tp, pp, m, a.hw, a.p, kv_tokens);
    a.tab.shape_ok[o] = ok ? 1 : 0;
    if (!ok) {
        a.tab.prefill[o] = a.tab.decode[o] = a.tab.mean_service[o] = 0.0;
        a.tab.inv_service[o] = __longlong_as_double(0x7ff8000000000000ll);  // any plan using it is unstable
        return;
    }
    // service_time (costmodel.cpp:176-194) with the reference's op order
    const double gpus = (double)(tp * pp);
    const double bubble = __dadd_rn(1.0, __dmul_rn(a.p.pipeline_bubble_factor, (double)(pp - 1)));
    const double flops = __dmul_rn(__dmul_rn(2.0, m.param_count), rd.mean_in);
    const double denom = __dmul_rn(__dmul_rn(gpus, a.hw.flops), a.p.prefill_efficiency);
    const double comm = __dmul_rn((double)pp, a.p.comm_overhead_per_stage);
    const double prefill = __dmul_rn(__dadd_rn(__ddiv_rn(flops, denom), comm), bubble);
    const double weights = __dmul_rn(m.param_count, m.bytes_per_param);
    const double bw = __dmul_rn(__dmul_rn((double)tp, a.hw.mem_bandwidth), a.p.decode_bw_efficiency);
    const double decode = __dadd_rn(__ddiv_rn(weights, bw), comm);
    const double clamped_mean_out = __dmul_rn(rd.mean_out, kClampedExpMeanFactor);
    a.tab.prefill[o] = prefill;
    a.tab.decode[o] = decode;
    a.tab.mean_service[o] = __dadd_rn(prefill, __dmul_rn(clamped_mean_out, decode));
    a.tab.inv_service[o] = __drcp_rn(a.tab.mean_service[o]);
}

// Common random numbers (costmodel.cpp:331-342).  L[k] = log1p(-u_k) comes
// from glibc on the host (hazard H3); exponential_mean(m) = (-m) * L.
__global__ void k_row_crn(RowSetupArgs a, const double* __restrict__ L) {
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= a.nrows) return;
    const RowDesc rd = a.rows[row];
    double* T = a.tab.T + (long long)row * a.tab.ld;
    double* O = a.tab.O + (long long)row * a.tab.ld;
    const double cap = __dmul_rn(4.0, rd.mean_out);
    const double neg_mean = -rd.mean_out;
    double t = 0.0;
    for (int k = 0; k < a.n_req; ++k) {
        t = __dadd_rn(t, __ddiv_rn(-L[2 * k], rd.rate));
        T[k] = t;
        const double x = __dmul_rn(neg_mean, L[2 * k + 1]);
        O[k] = (cap < x) ? cap : x;  // std::min(x, cap)
    }
    for (int i = 0; i < a.tab.nc; ++i) a.tab.Pv[(long long)row * a.tab.nc + i] = O[a.tab.probe_req[i]];
}

// ---------------------------------------------------------------------------
// K4

enum : int { ST_NEED = 0, ST_RUN = 1, ST_DONE = 2, ST_FINISH = 3 };

#ifndef CG_PF
#define CG_PF 1
#endif
#ifndef CG_SELBIT
#define CG_SELBIT 1
#endif
#ifndef CG_AS_MIN
#define CG_AS_MIN 32
#endif
constexpr int kGsParts = 16;  // parts held in GroupShared (>= kRecMaxParts; more: counts[] stay authoritative)

struct GroupShared {
    unsigned long long plan;  // current plan index
    unsigned long long hi;    // k_lane: the pre-claimed next record's item (cp.async target)
    double lbk;   // the plan's service bound: sojourns below it never reach the p95
    int row;
    int used;                // GPUs of the current count vector
    unsigned short dp;       // replicas (<= 255)
    unsigned short qi;       // future-bound blocks of the plan (SimArgs::qtab, a u16 count)
    unsigned char nparts;    // > 0: the plan's (shape, count) parts below, in shape order
    unsigned char status;
    unsigned ps;             // k_lane: bit j set when replica j starts a part (parts listed)
    unsigned char pshape[kGsParts], pcount[kGsParts];
    union {
        unsigned char counts[kMaxShapes];  // k_sim: count vector of the current plan
        unsigned long long pfw[4];         // k_lane: the next record's parts words and service bound
    };
};
static_assert(sizeof(GroupShared) == 112, "GroupShared layout (k_lane shared-memory budget)");

// ItemRec part stream (cg_kernels.h): header (np, used) then 13-bit parts.
__device__ __forceinline__ void encode_rec(ItemRec& r, const unsigned char* c, int S, int used) {
    unsigned long long w0 = 0ull, w1 = 0ull, w2 = 0ull;
    int np = 0;
    for (int s = 0; s < S; ++s) {
        if (!c[s]) continue;
        if (np == kRecMaxParts) {
            np = -1;
            break;
        }
        const unsigned long long f = (unsigned long long)s | ((unsigned long long)c[s] << 5);
        const int off = 13 + 13 * np;
        const int sh = off & 63;
        const unsigned long long lo = f << sh, hi = sh > 51 ? f >> (64 - sh) : 0ull;
        if (off < 64) {
            w0 |= lo;
            w1 |= hi;
        } else if (off < 128) {
            w1 |= lo;
            w2 |= hi;
        } else {
            w2 |= lo;
        }
        ++np;
    }
    if (np < 0 || used > 511) w0 = w1 = w2 = 0ull;
    else w0 |= (unsigned long long)np | ((unsigned long long)used << 4);
    r.w[0] = w0;
    r.w[1] = w1;
    r.w[2] = w2;
}
__device__ __forceinline__ unsigned rec_part(unsigned long long w0, unsigned long long w1, unsigned long long w2,
                                             int q) {
    const int off = 13 + 13 * q;
    const int sh = off & 63;
    const unsigned long long a = off < 64 ? w0 : (off < 128 ? w1 : w2);
    const unsigned long long b = off < 64 ? w1 : w2;
    unsigned long long v = a >> sh;
    if (sh > 51) v |= b << (64 - sh);
    return (unsigned)v & 0x1fffu;
}

// MODE: 0 = plan-index ranges (smem rings), 1 = explicit plan list (smem
// rings; bound seeding), 2 = explicit list with global-memory rings (deep
// re-runs of ring overflows).
enum : int { MODE_LIST = 1, MODE_DEEP = 2 };

template <int W, int R, int MODE>
struct Traits {
    static constexpr bool DEEP = MODE == MODE_DEEP;
    static constexpr int G = 32 / W;
    static constexpr int CAP = R == 1 ? 32 : (R == 2 ? 16 : 8);
    // non-DEEP: the finished group's ring columns double as its radix-select
    // histogram (W*R*CAP*2 >= 256 words); DEEP keeps a 256-word histogram.
    static constexpr size_t ring_bytes_per_warp = DEEP ? 256 * sizeof(unsigned)
                                                       : (size_t)32 * R * CAP * sizeof(double);
    static constexpr size_t bytes_per_warp = ring_bytes_per_warp + G * sizeof(GroupShared);
};

__device__ __forceinline__ void count_add(unsigned long long* ctr, unsigned long long v) {
    if (v) atomicAdd(ctr, v);
}

// Exact service-time lower bound of a plan's p95 (see the header comment of
// k_plan_filter); `counts` over the row's shapes.
__device__ __forceinline__ double service_bound(const SimArgs& a, int row, const PlanSpace& sp,
                                                const unsigned char* counts) {
    const long long rb = (long long)row * kMaxShapes;
    const double o_k = a.tab.O[(long long)row * a.tab.ld + a.kstar];
    const double t_max = a.tab.T[(long long)row * a.tab.ld + a.n_req - 1];
    double lb = __longlong_as_double(0x7ff0000000000000ll);
    for (int s = 0; s < sp.S; ++s) {
        if (!counts[s]) continue;
        const double v = a.tab.prefill[rb + s] + o_k * a.tab.decode[rb + s];
        lb = v < lb ? v : lb;
    }
    return lb * (1.0 - 1e-12) - 1e-12 * t_max;
}

// Future-service bound: the number of output-ranked blocks whose every
// request has a service lower bound > U on every shape of the plan (the
// qualifying blocks are a prefix, see RowTables).  Group-cooperative: lanes
// take the blocks round-robin, the plan's shapes come from its parts (or
// counts) in the group state.
template <int W>
__device__ __forceinline__ int future_blocks(const SimArgs& a, const GroupShared& gs, int row, bool active,
                                             double U, int gl, int gshift, unsigned wmask, int lo0) {
    const long long rb = (long long)row * kMaxShapes;
    const double t_max = active ? a.tab.T[(long long)row * a.tab.ld + a.n_req - 1] : 0.0;
    const int S = active ? a.spaces[a.rows[row].space].S : 0;
    const bool bounded = active && U < __longlong_as_double(0x7ff0000000000000ll);
    // W-ary search for the end of the qualifying prefix in [lo, hi)
    int lo = active ? lo0 : 0, hi = active ? a.tab.nc : 0;
    if (!bounded) hi = lo;
    while (__any_sync(0xffffffffu, lo < hi)) {
        const int len = hi - lo;
        const int i = lo + (int)(((long long)(gl + 1) * len) / (W + 1));
        bool qual = false;
        if (lo < hi) {
            const double o = a.tab.Pv[(long long)row * a.tab.nc + i];
            double lb = __longlong_as_double(0x7ff0000000000000ll);
            if (gs.nparts > 0) {
                for (int p = 0; p < gs.nparts; ++p) {
                    const int s = gs.pshape[p];
                    const double v = a.tab.prefill[rb + s] + o * a.tab.decode[rb + s];
                    lb = v < lb ? v : lb;
                }
            } else {
                for (int s = 0; s < S; ++s) {
                    if (!gs.counts[s]) continue;
                    const double v = a.tab.prefill[rb + s] + o * a.tab.decode[rb + s];
                    lb = v < lb ? v : lb;
                }
            }
            qual = lb * (1.0 - 1e-12) - 1e-12 * t_max > U;
        }
        const unsigned b = (__ballot_sync(0xffffffffu, qual) >> gshift) & wmask;
        const int t = __popc(b);  // qualifying probes form a prefix of the lanes
        if (lo < hi) {
            const int plo = lo + (int)(((long long)t * len) / (W + 1));        // probe t-1 position + 1 ...
            const int phi = lo + (int)(((long long)(t + 1) * len) / (W + 1));  // ... probe t position
            const int nlo = t > 0 ? plo + 1 : lo;
            const int nhi = t < W ? phi : hi;
            lo = nlo;
            hi = nhi < nlo ? nlo : nhi;
        }
    }
    return lo;
}

// Leader lane: pop the next (row, plan) work item of this kernel's list and
// unrank it; items come from k_plan_filter (already stable, class-matched) or
// are seeds / overflow re-runs.  The service-time bound is re-checked against
// the live bound (it tightens while the kernel runs).
template <int MODE>
__device__ void acquire_plan(const SimArgs& a, GroupShared& gs, unsigned long long& bound) {
    while (true) {
        const unsigned long long it = atomicAdd(a.item_counter, 1ull);
        if (it >= a.nitems) {
            gs.status = ST_DONE;
            return;
        }
        const unsigned long long slot = a.perm ? (unsigned long long)a.perm[it] : it;
        unsigned long long item, w0 = 0ull, w1 = 0ull, w2 = 0ull;
        if (a.recs) {
            const ItemRec& rec = a.recs[slot];
            item = rec.item;
            w0 = rec.w[0];
            w1 = rec.w[1];
            w2 = rec.w[2];
        } else {
            item = a.items[slot];
        }
        const int row = (int)(item >> kItemPlanBits);
        const unsigned long long plan = item & kItemPlanMask;
        const RowDesc& rd = a.rows[row];
        const PlanSpace& sp = a.spaces[rd.space];
        int dp = 0;
        const int np = (int)(w0 & 15ull);
        if (np > 0) {
            for (int s = 0; s < sp.S; ++s) gs.counts[s] = 0;
            for (int q = 0; q < np; ++q) {
                const unsigned v = rec_part(w0, w1, w2, q);
                gs.pshape[q] = (unsigned char)(v & 31u);
                gs.pcount[q] = (unsigned char)(v >> 5);
                gs.counts[v & 31u] = (unsigned char)(v >> 5);
                dp += (int)(v >> 5);
            }
            gs.used = (int)((w0 >> 4) & 511ull);
        } else {
            gs.used = unrank_plan(sp, plan, gs.counts);
            for (int s = 0; s < sp.S; ++s) dp += gs.counts[s];
        }
        gs.nparts = np;
        if (a.check_stable) {  // seeds are not pre-filtered
            const long long rb = (long long)row * kMaxShapes;
            bool good = true;
            double capacity = 0.0;
            for (int s = 0; s < sp.S; ++s) {
                const int c = gs.counts[s];
                if (!c) continue;
                if (!a.tab.shape_ok[rb + s]) {
                    good = false;
                    break;
                }
                capacity = __dadd_rn(capacity, __ddiv_rn((double)c, a.tab.mean_service[rb + s]));
            }
            if (!good || rd.rate >= capacity) continue;
        }
        if (a.prune && MODE != MODE_DEEP && !a.check_stable) {
            const double U = __longlong_as_double(
                (long long)*(volatile unsigned long long*)&a.ub[(long long)row * (a.N + 1) + gs.used]);
            if (service_bound(a, row, sp, gs.counts) > U) {
                ++bound;
                continue;
            }
        }
        gs.row = row;
        gs.plan = plan;
        gs.dp = dp;
        gs.status = ST_RUN;
        return;
    }
}

// Group-cooperative exact K-th largest of n non-negative doubles (8-bit
// radix select on the IEEE bit patterns, constant bytes skipped).
// hist word b of a group: contiguous 256 words (DEEP) or the group's ring
// columns (slot-major, W lanes x 2 words per slot).
template <int W, bool CONTIG>
__device__ __forceinline__ unsigned* hword(unsigned* base, int gshift, int b) {
    if (CONTIG) return base + b;
    return base + ((b / (2 * W)) * 32 + gshift) * 2 + (b % (2 * W));
}

template <int W, bool CONTIG>
__device__ unsigned long long group_kth_largest(const double* __restrict__ buf, int n, int K, int gl,
                                                unsigned gm, int gshift, unsigned* hist) {
    unsigned long long o = 0, an = ~0ull;
    for (int i = gl; i < n; i += W) {
        const unsigned long long k = (unsigned long long)__double_as_longlong(buf[i]);
        o |= k;
        an &= k;
    }
#pragma unroll
    for (int off = W / 2; off > 0; off >>= 1) {
        o |= __shfl_xor_sync(gm, o, off, W);
        an &= __shfl_xor_sync(gm, an, off, W);
    }
    const unsigned long long varying = o ^ an;
    unsigned long long prefix = 0, pmask = 0;
    int need = K;
    for (int byte = 7; byte >= 0; --byte) {
        const int shift = 8 * byte;
        const unsigned long long dm = 255ull << shift;
        if ((varying & dm) == 0) {
            prefix |= an & dm;
            pmask |= dm;
            continue;
        }
        for (int b = gl; b < 256; b += W) *hword<W, CONTIG>(hist, gshift, b) = 0;
        __syncwarp(gm);
        for (int i = gl; i < n; i += W) {
            const unsigned long long k = (unsigned long long)__double_as_longlong(buf[i]);
            if ((k & pmask) == prefix) atomicAdd(hword<W, CONTIG>(hist, gshift, (int)((k >> shift) & 255ull)), 1u);
        }
        __syncwarp(gm);
        constexpr int B = 256 / W;
        const int top = 255 - gl * B;
        int seg = 0;
#pragma unroll 4
        for (int j = 0; j < B; ++j) seg += *hword<W, CONTIG>(hist, gshift, top - j);
        int incl = seg;
#pragma unroll
        for (int off = 1; off < W; off <<= 1) {
            const int v = __shfl_up_sync(gm, incl, off, W);
            if (gl >= off) incl += v;
        }
        int excl = incl - seg;
        const bool mine = excl < need && need <= incl;
        int digit = 0, before = 0;
        if (mine) {
            for (int j = 0; j < B; ++j) {
                const int c = *hword<W, CONTIG>(hist, gshift, top - j);
                if (excl + c >= need) {
                    digit = top - j;
                    before = excl;
                    break;
                }
                excl += c;
            }
        }
        const unsigned ob = __ballot_sync(gm, mine);
        const int owner = (__ffs(ob) - 1) - gshift;
        digit = __shfl_sync(gm, digit, owner, W);
        before = __shfl_sync(gm, before, owner, W);
        const int cnt = *hword<W, CONTIG>(hist, gshift, digit);
        prefix |= (unsigned long long)digit << shift;
        pmask |= dm;
        need -= before;
        __syncwarp(gm);
        if (byte > 0 && (need == 1 || need == cnt)) {
            // the answer is the largest (need == 1) or the smallest (need ==
            // cnt) element under the prefix: one scan instead of more passes
            const bool want_max = need == 1;
            unsigned long long best = want_max ? 0ull : ~0ull;
            for (int i = gl; i < n; i += W) {
                const unsigned long long k = (unsigned long long)__double_as_longlong(buf[i]);
                if ((k & pmask) == prefix) best = want_max ? (k > best ? k : best) : (k < best ? k : best);
            }
#pragma unroll
            for (int off = W / 2; off > 0; off >>= 1) {
                const unsigned long long v = __shfl_xor_sync(gm, best, off, W);
                best = want_max ? (v > best ? v : best) : (v < best ? v : best);
            }
            return best;
        }
    }
    return prefix;
}

template <int W, int R, int MODE>
__global__ void __launch_bounds__(128, R <= 2 ? 6 : 3) k_sim(SimArgs a) {
    using TR = Traits<W, R, MODE>;
    constexpr bool DEEP = TR::DEEP;
    constexpr int UNROLL = 4;
    constexpr int G = TR::G;
    constexpr int CAP = TR::CAP;
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int gid = lane / W;
    const int gl = lane % W;
    const int gshift = gid * W;
    const unsigned wmask = (W == 32) ? FULL : ((1u << W) - 1u);
    const unsigned gm = wmask << gshift;

    unsigned char* wbase = smem + (size_t)warp * TR::bytes_per_warp;
    double* ring = reinterpret_cast<double*>(wbase);
    GroupShared* gsa = reinterpret_cast<GroupShared*>(wbase + TR::ring_bytes_per_warp);
    GroupShared& gs = gsa[gid];

    const long long gwarp = (long long)blockIdx.x * (blockDim.x >> 5) + warp;
    const long long slot = gwarp * G + gid;
    double* scratch = a.scratch + slot * (long long)a.sld;
    double* gring = DEEP ? a.ring_global + gwarp * (long long)32 * R * a.ring_cap : nullptr;
    const int ring_mask = DEEP ? a.ring_cap - 1 : CAP - 1;
    const int ring_cap = DEEP ? a.ring_cap : CAP;

    if (gl == 0) gs.status = ST_NEED;
    __syncwarp();

    const int n_req = a.n_req;
    int status = ST_NEED;
    int row = 0, dp = 0, gpus = 0, k = 0, ab = 0;
    unsigned long long plan = 0;
    bool ovf = false;
    double U = __longlong_as_double((long long)kInfBits);
    const double* Trow = a.tab.T;  // valid dummies until a plan is acquired
    const double* Orow = a.tab.O;
    double nd[R], avail[R], pre[R], dec[R];
    int cnt[R], head[R], tail[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        nd[r] = avail[r] = pre[r] = dec[r] = 0.0;
        cnt[r] = head[r] = tail[r] = 0;
    }
    unsigned long long steps = 0, full = 0, pruned = 0, bound = 0;
    int qi = 0;  // output-ranked blocks whose requests all exceed U on service alone
    const double INF = __longlong_as_double((long long)kInfBits);

    for (unsigned it = 0;; ++it) {
        // ---- phase A: groups without a plan acquire one
        const bool need = status == ST_NEED;
        if (__any_sync(FULL, need)) {
            if (need && gl == 0) acquire_plan<MODE>(a, gs, bound);
            __syncwarp();
            if (need) {
                status = gs.status;
                if (status == ST_RUN) {
                    row = gs.row;
                    dp = gs.dp;
                    gpus = gs.used;
                    plan = gs.plan;
                    const PlanSpace& sp = a.spaces[a.rows[row].space];
                    Trow = a.tab.T + (long long)row * a.tab.ld;
                    Orow = a.tab.O + (long long)row * a.tab.ld;
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int j = r * W + gl;
                        nd[r] = INF;
                        avail[r] = 0.0;
                        cnt[r] = head[r] = tail[r] = 0;
                        if (j < dp) {
                            int cum = 0, s = 0;
                            if (gs.nparts > 0) {
                                for (int q = 0; q < gs.nparts; ++q) {
                                    s = gs.pshape[q];
                                    cum += gs.pcount[q];
                                    if (j < cum) break;
                                }
                            } else {
                                for (; s < sp.S; ++s) {
                                    cum += gs.counts[s];
                                    if (j < cum) break;
                                }
                            }
                            pre[r] = a.tab.prefill[(long long)row * kMaxShapes + s];
                            dec[r] = a.tab.decode[(long long)row * kMaxShapes + s];
                        }
                    }
                    k = 0;
                    ab = 0;
                    ovf = false;
                    U = a.prune ? __longlong_as_double((long long)*(volatile unsigned long long*)&a.ub[(long long)row * (a.N + 1) + gpus])
                                : INF;
                }
            }
            __syncwarp();
        }
        if (__all_sync(FULL, status == ST_DONE)) break;
        {
            // the bound U is read by every lane from a concurrently tightened
            // ub: make the group agree on one value (its leader's) so that
            // every prune decision is group-uniform
            U = __shfl_sync(FULL, U, gshift);
            const bool fresh = need && status == ST_RUN;
            if (a.prune && a.tab.nc > 0 && __any_sync(FULL, fresh)) {
                const int q = future_blocks<W>(a, gs, row, fresh, U, gl, gshift, wmask, 0);
                if (fresh) qi = q;
            }
        }

        // ---- phase B: UNROLL JSQ dispatch steps per running group.
        // k is a multiple of UNROLL here (plans start at k = 0 and advance
        // UNROLL per trip), so the next arrivals/outputs come in with vector
        // loads.  A replica is idle at t iff its last finish time avail <= t
        // (FCFS: every job it holds is done by then), so the common case --
        // some replica idle -- needs no queue bookkeeping at all: the winner
        // is the lowest idle index (the reference's early break), its start
        // is t and its FIFO is reset to the new job.  Only when every replica
        // of a group is busy are the FIFOs popped up to t (lazily -- pops are
        // idempotent in t) and the winner taken as the group minimum of
        // (queue length << 9 | replica index), the reference's argmin.
        {
            const bool run0 = status == ST_RUN;
            const double2* T2 = reinterpret_cast<const double2*>(Trow + (run0 ? k : 0));
            const double2* O2 = reinterpret_cast<const double2*>(Orow + (run0 ? k : 0));
            const double2 ta = __ldg(T2), tb = __ldg(T2 + 1), oa = __ldg(O2), ob = __ldg(O2 + 1);
            const double tt[4] = {ta.x, ta.y, tb.x, tb.y};
            const double oo[4] = {oa.x, oa.y, ob.x, ob.y};
            double* const srow = scratch + k;
#pragma unroll
            for (int u = 0; u < UNROLL; ++u) {
                const bool run = status == ST_RUN;
                const double t = tt[u];
                const double o = oo[u];
                // fast path: lowest idle replica of the group
                int win = -1;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const bool idle = run && (r * W + gl) < dp && avail[r] <= t;
                    const unsigned gb = (__ballot_sync(FULL, idle) >> gshift) & wmask;
                    if (win < 0 && gb) win = r * W + (__ffs(gb) - 1);
                }
                const bool busy = run && win < 0;
                if (__any_sync(FULL, busy)) {
                    // slow path (groups whose replicas are all busy): pop the
                    // FIFOs up to t, then the (length, index) group minimum
                    bool dep[R];
                    bool anydep = false;
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        dep[r] = busy && nd[r] <= t;
                        anydep |= dep[r];
                    }
                    while (__any_sync(FULL, anydep)) {
                        anydep = false;
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            const int slotr = head[r] & ring_mask;
                            const double nx = DEEP ? gring[((long long)r * ring_cap + slotr) * 32 + lane]
                                                   : ring[(r * CAP + slotr) * 32 + lane];
                            const int c1 = cnt[r] - (dep[r] ? 1 : 0);
                            nd[r] = dep[r] ? (c1 > 0 ? nx : INF) : nd[r];
                            head[r] += (dep[r] && c1 > 0) ? 1 : 0;
                            cnt[r] = c1;
                            dep[r] = busy && nd[r] <= t;
                            anydep |= dep[r];
                        }
                    }
                    unsigned key = 0xffffffffu;
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int j = r * W + gl;
                        const unsigned kr = ((unsigned)cnt[r] << 9) | (unsigned)j;
                        key = (busy && j < dp && kr < key) ? kr : key;
                    }
#pragma unroll
                    for (int off = W / 2; off > 0; off >>= 1) {
                        const unsigned v = __shfl_xor_sync(FULL, key, off);
                        key = v < key ? v : key;
                    }
                    if (busy) win = (int)(key & 511u);
                }
                const int wl = win & (W - 1), wr = win / W;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const bool me = run && gl == wl && r == wr;
                    const bool was_idle = avail[r] <= t;
                    const double start = was_idle ? t : avail[r];  // std::max(t, avail)
                    const double fin = __dadd_rn(__dadd_rn(start, pre[r]), __dmul_rn(o, dec[r]));
                    const double soj = __dsub_rn(fin, t);
                    if (me) {
                        if (was_idle) {  // empty FIFO: the new job is in service
                            head[r] = tail[r];
                            cnt[r] = 1;
                            nd[r] = fin;
                        } else {         // joins the queue behind the busy server
                            const int slotr = tail[r] & ring_mask;
                            if (DEEP) gring[((long long)r * ring_cap + slotr) * 32 + lane] = fin;
                            else ring[(r * CAP + slotr) * 32 + lane] = fin;
                            ++tail[r];
                            ovf |= (tail[r] - head[r] > ring_cap);
                            ++cnt[r];
                        }
                        avail[r] = fin;
                        srow[u] = soj;
                        ab += soj > U ? 1 : 0;
                    }
                }
                k += run ? 1 : 0;
                status = (run && k == n_req) ? ST_FINISH : status;
            }
        }

        // ---- phase C: periodic exact-bound pruning and overflow checks
        if ((it & (32u / UNROLL - 1u)) == (32u / UNROLL - 1u)) {
            int tot = ab;
            int ov = ovf ? 1 : 0;
#pragma unroll
            for (int off = W / 2; off > 0; off >>= 1) {
                tot += __shfl_xor_sync(FULL, tot, off);
                ov |= __shfl_xor_sync(FULL, ov, off);
            }
            bool urefresh = false;
            if (status == ST_RUN) {
                // requests still to come whose service alone exceeds U
                const int fut = qi > 0 ? (int)a.tab.fut[(long long)((k + a.tab.fut_ab - 1) >> a.tab.fut_sh) * a.tab.nc + (qi - 1)] : 0;
                if (ov) {
                    if (gl == 0) {
                        const unsigned long long idx = atomicAdd(a.ovf_count, 1ull);
                        if (idx < a.ovf_cap) a.ovf[idx] = ((unsigned long long)row << kItemPlanBits) | plan;
                    }
                    steps += k;
                    status = ST_NEED;
                } else if (a.prune && tot + fut >= a.K) {
                    pruned += 1;
                    steps += k;
                    status = ST_NEED;
                } else if (a.prune) {
                    const double U2 = __longlong_as_double(
                        (long long)*(volatile unsigned long long*)&a.ub[(long long)row * (a.N + 1) + gpus]);
                    urefresh = U2 < U;
                    U = U2;
                }
            }
            U = __shfl_sync(FULL, U, gshift);
            urefresh = __shfl_sync(FULL, urefresh ? 1 : 0, gshift) != 0;
            if (a.tab.nc > 0 && __any_sync(FULL, urefresh)) {
                const int q = future_blocks<W>(a, gs, row, urefresh, U, gl, gshift, wmask, qi);
                if (urefresh) qi = q;
            }
            if (status == ST_NEED && gl == 0) gs.status = ST_NEED;
        }

        // ---- phase D: completed plans -> exact p95 and row bookkeeping
        if (__any_sync(FULL, status == ST_FINISH)) {
            if (status == ST_FINISH) {
                int tot = ab;
                int ov = ovf ? 1 : 0;
#pragma unroll
                for (int off = W / 2; off > 0; off >>= 1) {
                    tot += __shfl_xor_sync(gm, tot, off, W);
                    ov |= __shfl_xor_sync(gm, ov, off, W);
                }
                steps += k;
                if (ov) {
                    if (gl == 0) {
                        const unsigned long long idx = atomicAdd(a.ovf_count, 1ull);
                        if (idx < a.ovf_cap) a.ovf[idx] = ((unsigned long long)row << kItemPlanBits) | plan;
                    }
                } else if (a.prune && tot >= a.K) {
                    pruned += 1;
                } else {
                    __syncwarp(gm);
                    const unsigned long long xb = group_kth_largest<W, DEEP>(
                        scratch, a.n_req, a.K, gl, gm, gshift, reinterpret_cast<unsigned*>(wbase));
                    full += 1;
                    if (gl == 0) {
                        const long long base = (long long)row * (a.N + 1);
                        const unsigned long long old = atomicMin(&a.lat_min[base + gpus], xb);
                        if (xb <= old) {
                            const unsigned long long idx = atomicAdd(a.tie_count, 1ull);
                            if (idx < a.tie_cap) a.ties[idx] = TieEntry{row, gpus, xb, plan};
                        }
                        for (int g2 = gpus; g2 <= a.N; ++g2) {
                            unsigned long long* ub = &a.ub[base + g2];
                            if (*(volatile unsigned long long*)ub <= xb) break;
                            atomicMin(ub, xb);
                        }
                    }
                }
                status = ST_NEED;
                if (gl == 0) gs.status = ST_NEED;
            }
            __syncwarp();
        }
    }
    // per-lane counters -> global (leaders only to avoid double counting)
    if (gl == 0) {
        count_add(&a.counters[CTR_BOUND], bound);
        count_add(&a.counters[CTR_STEPS], steps);
        count_add(&a.counters[a.seeds ? CTR_SEED : CTR_FULL], full);
        count_add(&a.counters[a.seeds ? CTR_SEED : CTR_PRUNED], pruned);
    }
}

// ---------------------------------------------------------------------------
// K4, lane-major form (replica-count classes 0-3).  A plan lives on W = 1, 2
// or 4 lanes with R = 4 or 8 replicas per lane held in registers (replica
// j = gl*R + r), so a warp carries 32/W plans and a request-step is a handful
// of lane instructions instead of a group-wide exchange:
//   * idle fast path: the lowest idle replica (avail <= t) wins, start = t;
//     its FIFO is reset lazily (bit r of `lazy`: the replica holds exactly the
//     job in service, finishing at avail[r]);
//   * busy path (every replica of the plan busy): lazy FIFOs materialised,
//     pops up to t, then the (in-system count, index) minimum -- the
//     reference's argmin (costmodel.cpp:262-276);
//   * prefill/decode of the lane's replicas in shared memory [r][lane]; the
//     waiting jobs in shared-memory rings [r][slot][lane] of 16-bit request
//     indices: a waiting job starts when its predecessor finishes, so its
//     finish time is recomputed at pop time from the predecessor's,
//     (nd + prefill) + out[k] * decode -- the same operands and operations as
//     at dispatch, hence the same double.  Head/tail are packed 16+16 bits per
//     replica (differences taken mod 2^16);
//   * plans are claimed with one warp-aggregated atomic per round; the K-th
//     largest selection is warp-cooperative, one finished plan at a time.
// Exactness is that of k_sim: same operations in the same order per request.
#ifdef CG_K4_PROF
// development counters (CG_BUILD_VARIANT=prof): per R class (4/8/16/32) of the
// one-lane-per-plan kernels: cycles per phase and event counts, summed over warps
__device__ unsigned long long g_k4prof[4][16];
#define K4P_DECL unsigned long long p_[16] = {}; long long pt_ = clock64(), pt0_ = pt_;
#define K4P_MARK(i) do { const long long c_ = clock64(); p_[i] += (unsigned long long)(c_ - pt_); pt_ = c_; } while (0)
#define K4P_ADD(i, v) (p_[i] += (unsigned long long)(v))
#define K4P_FLUSH(ri) do { p_[0] = (unsigned long long)(clock64() - pt0_); p_[11] = 1; if (lane == 0) \
    for (int i_ = 0; i_ < 16; ++i_) atomicAdd(&g_k4prof[ri][i_], p_[i_]); } while (0)
#else
#define K4P_DECL
#define K4P_MARK(i) do {} while (0)
#define K4P_ADD(i, v) do {} while (0)
#define K4P_FLUSH(ri) do {} while (0)
#endif

template <int W, int R>
struct LaneTraits {
    static constexpr int G = 32 / W;
    // waiting-job ring slots per replica (W = 1, R = 8: 8 slots keep three
    // 128-thread blocks per SM within shared memory); deeper queues overflow
    // to the DEEP re-run.  (Four blocks per SM -- 128 registers, half the
    // slots -- measured slower: C3 K4 746 -> 795 ms.)
    // R = 16 / 32 (one lane holds a whole dp <= 32 plan): 4 slots, deeper
    // queues overflow to the DEEP re-run; 2-warp blocks pack shared memory
    static constexpr int CAP = R <= 4 ? 32 : (R <= 8 ? (W == 1 ? 8 : 16) : 4);
    // warps per block: R = 32 five 1-warp blocks per SM, R = 16 four 2-warp blocks (1-warp blocks when its
    // finish times are in shared memory, CG_AS_MIN = 16)
    static constexpr int WPB = R >= 32 ? 1 : (R >= 16 ? (W == 1 && R >= CG_AS_MIN ? 1 : 2) : 4);
    // SA (R = 32): replica finish times in shared memory -- the idle mask is a
    // fully unrolled scan of loads and compares, the winner's update one store
    // (in registers it is a compare and two selects per replica per step) --
    // and prefill/decode per part of the plan (<= kGsParts) so the footprint
    // still fits two 2-warp blocks per SM
    static constexpr bool SA = W == 1 && R >= 32;
    // AS: replica finish times in shared memory (SA, and R >= CG_AS_MIN)
    static constexpr bool AS = W == 1 && R >= CG_AS_MIN;
    // prefill/decode slots per lane (SA: per part, up to 16 parts -- plans of up to 16 parts run here; with
    // 13 slots the dp 17-32 kernel fits five blocks per SM, but 14-16-part plans then all go to the DEEP
    // re-run and exhaust its list on wide shape sets such as C5's)
    static constexpr int PD = SA ? kGsParts : R;
    static constexpr int MIN_BLOCKS = 1;
    static constexpr size_t ring_bytes = (size_t)R * CAP * 32 * sizeof(unsigned short);
    // prefill, decode, head-job finish, previous-job finish (per replica slot)
    static constexpr size_t pd_bytes = (size_t)(2 * PD + (AS ? 3 : 2) * R) * 32 * sizeof(double);
    // ring head | tail << HS, both mod HM + 1: one byte per replica when the
    // ring holds <= 4 jobs (lengths up to CAP + 1 < 16 stay distinguishable)
    using HT = typename std::conditional<CAP <= 4, unsigned char, unsigned>::type;
    static constexpr unsigned HS = CAP <= 4 ? 4u : 16u;
    static constexpr unsigned HM = CAP <= 4 ? 0xfu : 0xffffu;
    static constexpr size_t ht_bytes = (size_t)R * 32 * sizeof(HT);
    static constexpr size_t hist_bytes = 256 * sizeof(unsigned);
    static constexpr size_t bytes_per_warp = ring_bytes + pd_bytes + ht_bytes + hist_bytes + G * sizeof(GroupShared);
    static_assert(hist_bytes >= (size_t)G * kMaxShapes, "count-vector scratch in the histogram area");
};

// Claims work item `it` into gs; false when the item is rejected (an unstable
// seed, or a service bound above the live bound).  Filtered items (recs)
// carry their parts and service bound, so a claim is one round of
// independent loads (the record) and one dependent one (the live bound and
// the plan's future-bound blocks, SimArgs::qtab).
// `counts`: the lane's count-vector scratch (unranked plans with more parts
// than a record lists).
__device__ bool lane_take_r(const SimArgs& a, GroupShared& gs, unsigned char* counts, unsigned long long item,
                            unsigned long long w0, unsigned long long w1, unsigned long long w2, double lb,
                            const bool rec, unsigned long long& bound) {
    const int row = (int)(item >> kItemPlanBits);
    const unsigned long long plan = item & kItemPlanMask;
    const RowDesc& rd = a.rows[row];
    const PlanSpace& sp = a.spaces[rd.space];
    const long long rb = (long long)row * kMaxShapes;
    int np = (int)(w0 & 15ull);
    int dp = 0, used = 0;
    if (rec && np > 0 && !a.check_stable) {
        // filtered item with its parts: decode them into registers (unrolled, so
        // the part offsets are constants) and issue the live bound and every
        // part's bound-snapshot entry at once -- independent loads, one latency
        unsigned shp[kRecMaxParts];
        unsigned ps = 0u;  // part starts, from the counts in registers
#pragma unroll
        for (int q = 0; q < kRecMaxParts; ++q) {
            shp[q] = 0u;
            if (q < np) {
                const unsigned v = rec_part(w0, w1, w2, q);
                shp[q] = v & 31u;
                gs.pshape[q] = (unsigned char)(v & 31u);
                gs.pcount[q] = (unsigned char)(v >> 5);
                if (dp < 32) ps |= 1u << dp;
                dp += (int)(v >> 5);
            }
        }
        gs.ps = ps;
        used = (int)((w0 >> 4) & 511ull);
        const long long cell = (long long)row * (a.N + 1) + used;
        const double U = a.prune ? __longlong_as_double((long long)*(volatile unsigned long long*)&a.ub[cell])
                                 : __longlong_as_double(0x7ff0000000000000ll);
        const bool useq = a.prune && a.qtab && a.tab.nc > 0;
        const unsigned short* qt = useq ? a.qtab + cell * kMaxShapes : nullptr;
        int qv[kRecMaxParts];
#pragma unroll
        for (int q = 0; q < kRecMaxParts; ++q) qv[q] = (useq && q < np) ? (int)qt[shp[q]] : (1 << 30);
        if (a.prune && lb > U) {
            ++bound;
            return false;
        }
        int qi = 1 << 30;
#pragma unroll
        for (int q = 0; q < kRecMaxParts; ++q) qi = qv[q] < qi ? qv[q] : qi;
        gs.nparts = np;
        gs.row = row;
        gs.plan = plan;
        gs.dp = dp;
        gs.used = used;
        gs.qi = (useq && qi != (1 << 30)) ? qi : 0;
        gs.lbk = lb;
        return true;
    }
    unsigned ps = 0u;
    if (np > 0) {
        for (int q = 0; q < np; ++q) {
            const unsigned v = rec_part(w0, w1, w2, q);
            gs.pshape[q] = (unsigned char)(v & 31u);
            gs.pcount[q] = (unsigned char)(v >> 5);
            if (dp < 32) ps |= 1u << dp;
            dp += (int)(v >> 5);
        }
        used = (int)((w0 >> 4) & 511ull);
    } else {
        used = unrank_plan(sp, plan, counts);
        for (int s = 0; s < sp.S; ++s) {
            const int c = counts[s];
            if (!c) continue;
            if (np < kGsParts) {
                gs.pshape[np] = (unsigned char)s;
                gs.pcount[np] = (unsigned char)c;
            }
            if (dp < 32) ps |= 1u << dp;
            ++np;
            dp += c;
        }
        if (np > kGsParts) np = 0;  // counts[] stay authoritative
    }
    gs.ps = ps;
    if (a.check_stable) {  // seeds are not pre-filtered (costmodel.cpp:366-376)
        double capacity = 0.0;
        for (int q = 0, s = 0; np > 0 ? q < np : s < sp.S; np > 0 ? ++q : ++s) {
            const int sh = np > 0 ? gs.pshape[q] : s;
            const int c = np > 0 ? gs.pcount[q] : counts[s];
            if (!c) continue;
            if (!a.tab.shape_ok[rb + sh]) return false;
            capacity = __dadd_rn(capacity, __ddiv_rn((double)c, a.tab.mean_service[rb + sh]));
        }
        if (rd.rate >= capacity) return false;
    }
    if (!rec) {  // the service bound (k_plan_filter computes it for filtered items)
        const double o_k = a.tab.O[(long long)row * a.tab.ld + a.kstar];
        const double t_max = a.tab.T[(long long)row * a.tab.ld + a.n_req - 1];
        double m = __longlong_as_double(0x7ff0000000000000ll);
        for (int q = 0, s = 0; np > 0 ? q < np : s < sp.S; np > 0 ? ++q : ++s) {
            const int sh = np > 0 ? gs.pshape[q] : s;
            if (np == 0 && !counts[s]) continue;
            const double v = a.tab.prefill[rb + sh] + o_k * a.tab.decode[rb + sh];
            m = v < m ? v : m;
        }
        lb = m * (1.0 - 1e-12) - 1e-12 * t_max;
    }
    if (a.prune && !a.check_stable) {
        const double U = __longlong_as_double(
            (long long)*(volatile unsigned long long*)&a.ub[(long long)row * (a.N + 1) + used]);
        if (lb > U) {
            ++bound;
            return false;
        }
    }
    int qi = 0;
    if (a.prune && a.qtab && a.tab.nc > 0) {
        const unsigned short* qt = a.qtab + ((long long)row * (a.N + 1) + used) * kMaxShapes;
        qi = 1 << 30;
        for (int q = 0, s = 0; np > 0 ? q < np : s < sp.S; np > 0 ? ++q : ++s) {
            const int sh = np > 0 ? gs.pshape[q] : s;
            if (np == 0 && !counts[s]) continue;
            const int v = qt[sh];
            qi = v < qi ? v : qi;
        }
        qi = qi == (1 << 30) ? 0 : qi;
    }
    gs.nparts = np;
    gs.row = row;
    gs.plan = plan;
    gs.dp = dp;
    gs.used = used;
    gs.qi = qi;
    gs.lbk = lb;
    return true;
}

// (mask & bit) ? a : b as a predicate from one bit test and a selp: opaque to
// the front end, so it is not re-derived into compare-and-select chains
__device__ __forceinline__ double sel_bit(unsigned mask, unsigned bit, double a, double b) {
    double r;
    asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\tand.b32 t, %1, %2;\n\tsetp.ne.b32 p, t, 0;\n\t"
        "selp.f64 %0, %3, %4, p;\n\t}"
        : "=d"(r)
        : "r"(mask), "r"(bit), "d"(a), "d"(b));
    return r;
}

__device__ __forceinline__ bool lane_take(const SimArgs& a, GroupShared& gs, unsigned char* counts,
                                          unsigned long long slot, unsigned long long& bound) {
    if (a.recs) {
        const ItemRec& r = a.recs[slot];
        return lane_take_r(a, gs, counts, r.item, r.w[0], r.w[1], r.w[2], r.lb, true, bound);
    }
    return lane_take_r(a, gs, counts, a.items[slot], 0ull, 0ull, 0ull, 0.0, false, bound);
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// request-steps between exact-bound prune checks: SimArgs::lane_check (engine option lane_check)

template <int W, int R>
__global__ void __launch_bounds__(LaneTraits<W, R>::WPB * 32, LaneTraits<W, R>::MIN_BLOCKS) k_lane(SimArgs a) {
    using TR = LaneTraits<W, R>;
    constexpr int G = TR::G;
    constexpr int CAP = TR::CAP;
    constexpr int UNROLL = kLaneUnroll;
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int gid = lane / W;
    const int gl = lane % W;
    const int gshift = gid * W;
    const unsigned wmask = (W == 32) ? FULL : ((1u << W) - 1u);

    unsigned char* wbase = smem + (size_t)warp * TR::bytes_per_warp;
    unsigned short* ring = reinterpret_cast<unsigned short*>(wbase);
    double* pre_s = reinterpret_cast<double*>(wbase + TR::ring_bytes);
    constexpr int PD = TR::PD;
    constexpr bool SA = TR::SA;
    constexpr bool AS = TR::AS;
    double* dec_s = pre_s + PD * 32;
    double* nd_s = dec_s + PD * 32;  // finish time of each replica's head job (INF: none)
    // finish of the job before each replica's last one (INF: no replica; a
    // value <= t means the replica holds exactly one job at t).  Only the
    // winner's slot changes per step, so prev and the ring heads live in
    // shared memory (one predicated store) rather than in registers (a
    // select per replica per step).
    double* prev_s = nd_s + R * 32;
    double* avail_s = prev_s + R * 32;  // SA: finish of each replica's last job
    using HT = typename TR::HT;
    constexpr unsigned HS = TR::HS, HM = TR::HM;
    HT* ht_s = reinterpret_cast<HT*>(wbase + TR::ring_bytes + TR::pd_bytes);
    unsigned* hist = reinterpret_cast<unsigned*>(wbase + TR::ring_bytes + TR::pd_bytes + TR::ht_bytes);
    GroupShared* gsa = reinterpret_cast<GroupShared*>(wbase + TR::ring_bytes + TR::pd_bytes + TR::ht_bytes +
                                                      TR::hist_bytes);
    GroupShared& gs = gsa[gid];
    // the group's count-vector scratch lives in the warp's histogram area (used
    // only by the phase-D selection; phase A is done with it by then), so the
    // GroupShared count bytes can hold the prefetched next record
    unsigned char* const lcounts = reinterpret_cast<unsigned char*>(hist) + gid * kMaxShapes;
    // record prefetch (W = 1 lists of filtered records in list order)
    const bool pfm = CG_PF && W == 1 && a.recs != nullptr && a.perm == nullptr && !a.check_stable;
    int pf_st = 0;  // 0: no next record claimed yet, 1: next record copied into gs, 2: list exhausted

    const long long gwarp = (long long)blockIdx.x * (blockDim.x >> 5) + warp;
    double* const scratch = a.scratch + (gwarp * G + gid) * (long long)a.sld;
    const int n_req = a.n_req;
    const double INF = __longlong_as_double((long long)kInfBits);

    if (gl == 0) gs.status = ST_NEED;
    __syncwarp();

    int status = ST_NEED;
    int row = 0, dp = 0, gpus = 0, k = 0, ab = 0, qi = 0;
    int ns = 0;          // sojourns recorded in the plan's scratch column (those >= lbk)
    double lbk = 0.0;    // the plan's service bound: smaller sojourns are never the p95
    unsigned long long plan = 0;
    bool ovf = false;
    unsigned lazy = 0;
    unsigned valid = 0;  // replicas of the current plan on this lane
    unsigned fresh = 0;  // AS: replicas not dispatched since the claim (their slots are stale)
    unsigned mcur = 0;  // this step's idle mask (avail[r] <= t), computed one step ahead
    double U = INF;
    const double* Trow = a.tab.T;  // valid dummies until a plan is acquired
    const double* Orow = a.tab.O;
    // arrivals / outputs of the pair holding step k and of the next pair (prefetched)
    double2 tq = make_double2(0.0, 0.0), oq = tq, tq2 = tq, oq2 = tq;
    // per replica: avail = finish of its last job (registers: every step's
    // idle mask reads them all); the head job's finish (nd_s), the previous
    // job's finish (prev_s) and the ring head/tail (ht_s) live in shared memory
    double avail[AS ? 1 : R];
    // finish of replica r's last job
    auto av_get = [&](int r) -> double {
        if constexpr (AS) return avail_s[r * 32 + lane];
        else return avail[r];
    };
    auto av_set = [&](int r, double v) {
        if constexpr (AS) avail_s[r * 32 + lane] = v;
        else avail[r] = v;
    };
    unsigned pstart = 0;  // SA: bit r set when replica r starts a new part
    // shared-memory slot of replica r's prefill/decode
    auto pd_slot = [&](int r) -> int {
        if constexpr (SA) {
            const int q = __popc(pstart & ((2u << r) - 1u)) - 1;
            return (q > 0 ? q : 0) * 32 + lane;
        } else {
            return r * 32 + lane;
        }
    };
    // W == 1: output tokens of the job at the ring head, loaded one pop ahead
    // (the lanes' rows differ, so a load at pop time would stall on L2)
    constexpr bool HO = W == 1 && R <= 8;
    double ho[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        av_set(r, INF);
        ho[r] = 0.0;
        ht_s[r * 32 + lane] = 0u;
        prev_s[r * 32 + lane] = INF;
    }
    unsigned long long steps = 0, full = 0, pruned = 0, bound = 0;
    K4P_DECL

    for (unsigned it = 0;; ++it) {
        // ---- phase A: groups without a plan claim one (one atomic per round)
        const bool need = status == ST_NEED;
        K4P_MARK(2);
        if (__any_sync(FULL, need)) {
            K4P_ADD(5, 1);
            bool want = need && gl == 0;
            unsigned m = __ballot_sync(FULL, want);
            while (m) {
                K4P_ADD(6, 1);
                K4P_ADD(8, __popc(m));
                bool again = false;
                if (pfm) {
                    // record prefetch: a lane takes its pre-claimed record (copied
                    // into shared memory during its previous plan) and claims the
                    // next one; a lane without one (its first claim) claims two.
                    // The atomic's result is needed only to issue the next copy,
                    // after the take, so neither the atomic nor the record load is
                    // on the claim's critical path.
                    const unsigned c1 = __ballot_sync(FULL, want && pf_st == 1);
                    const unsigned c2 = __ballot_sync(FULL, want && pf_st == 0);
                    const unsigned call = c1 | c2;
                    const int ldr = call ? __ffs(call) - 1 : 0;
                    unsigned long long base = 0;
                    if (call && lane == ldr)
                        base = atomicAdd(a.item_counter, (unsigned long long)(__popc(c1) + 2 * __popc(c2)));
                    const unsigned lt = (1u << lane) - 1u;
                    const unsigned long long off = (unsigned long long)(__popc(c1 & lt) + 2 * __popc(c2 & lt));
                    if (c2) base = __shfl_sync(FULL, base, ldr);  // first claims only
                    if (want) {
                        bool have = false;
                        unsigned long long it0 = 0ull, w0 = 0ull, w1 = 0ull, w2 = 0ull;
                        double lb = 0.0;
                        if (pf_st == 1) {
                            cp_async_wait_all();
                            it0 = gs.hi;
                            w0 = gs.pfw[0];
                            w1 = gs.pfw[1];
                            w2 = gs.pfw[2];
                            lb = __longlong_as_double((long long)gs.pfw[3]);
                            have = true;
                        } else if (pf_st == 0 && base + off < a.nitems) {
                            const ItemRec& r = a.recs[base + off];
                            it0 = r.item;
                            w0 = r.w[0];
                            w1 = r.w[1];
                            w2 = r.w[2];
                            lb = r.lb;
                            have = true;
                        }
                        if (!have) gs.status = ST_DONE;
                        else if (lane_take_r(a, gs, lcounts, it0, w0, w1, w2, lb, true, bound)) gs.status = ST_RUN;
                        else again = true;
                    }
                    if (c1) base = __shfl_sync(FULL, base, ldr);
                    if ((call >> lane) & 1u) {
                        const unsigned long long nx = base + off + ((c2 >> lane) & 1u);
                        if (nx < a.nitems) {
                            const ItemRec* r = a.recs + nx;
                            cp_async8(&gs.hi, &r->item);
                            cp_async8(&gs.pfw[0], &r->w[0]);
                            cp_async8(&gs.pfw[1], &r->w[1]);
                            cp_async8(&gs.pfw[2], &r->w[2]);
                            cp_async8(&gs.pfw[3], &r->lb);
                            pf_st = 1;
                        } else {
                            pf_st = 2;
                        }
                    }
                } else {
                    const int ldr = __ffs(m) - 1;
                    unsigned long long base = 0;
                    if (lane == ldr) base = atomicAdd(a.item_counter, (unsigned long long)__popc(m));
                    base = __shfl_sync(FULL, base, ldr);
                    if (want) {
                        const unsigned long long item = base + __popc(m & ((1u << lane) - 1u));
                        if (item >= a.nitems) gs.status = ST_DONE;
                        else if (lane_take(a, gs, lcounts, a.perm ? (unsigned long long)a.perm[item] : item, bound))
                            gs.status = ST_RUN;
                        else again = true;
                    }
                }
                want = again;
                m = __ballot_sync(FULL, want);
            }
            __syncwarp();
            K4P_MARK(1);
            if (need) {
                status = gs.status;
                if (SA && status == ST_RUN && (gs.nparts == 0 || gs.nparts > TR::PD)) {
                    // more parts than the per-part tables hold: the DEEP re-run takes it
                    const unsigned long long idx = atomicAdd(a.ovf_count, 1ull);
                    if (idx < a.ovf_cap) a.ovf[idx] = ((unsigned long long)gs.row << kItemPlanBits) | gs.plan;
                    status = ST_NEED;
                    gs.status = ST_NEED;
                }
                if (status == ST_RUN) {
                    row = gs.row;
                    dp = gs.dp;
                    gpus = gs.used;
                    plan = gs.plan;
                    pstart = 0u;
                    const long long rb = (long long)row * kMaxShapes;
                    Trow = a.tab.T + (long long)row * a.tab.ld;
                    Orow = a.tab.O + (long long)row * a.tab.ld;
                    // the new row's first arrivals/outputs and live bound depend on the
                    // row alone: issue them before the replica set-up so their L2
                    // latency overlaps it
                    tq = *reinterpret_cast<const double2*>(Trow);
                    oq = *reinterpret_cast<const double2*>(Orow);
                    tq2 = *reinterpret_cast<const double2*>(Trow + (n_req > 2 ? 2 : 0));
                    oq2 = *reinterpret_cast<const double2*>(Orow + (n_req > 2 ? 2 : 0));
                    U = a.prune ? __longlong_as_double((long long)*(volatile unsigned long long*)&a.ub[(long long)row * (a.N + 1) + gpus])
                                : INF;
                    // replicas j = gl*R + r in parts order.  With the parts listed
                    // (np > 0) replica j's part is the number of part starts <= j:
                    // independent shared-memory reads instead of a serial walk
                    int q = 0, cum = 0, sh = -1;
                    const int np = gs.nparts;
                    unsigned ps = 0u;  // bit j: replica j starts a part
                    if (np > 0) {
                        ps = gs.ps;  // the claim built it from the counts in registers
                        if (SA) {
#pragma unroll
                            for (int qq = 0; qq < kGsParts; ++qq)
                                if (qq < np) {
                                    const int shq = gs.pshape[qq];
                                    pre_s[qq * 32 + lane] = a.tab.prefill[rb + shq];
                                    dec_s[qq * 32 + lane] = a.tab.decode[rb + shq];
                                }
                            pstart = ps;
                        }
                    }
                    // no per-replica reset of the shared-memory state (head-job
                    // finish, ring head/tail, previous finish, and with AS the
                    // finish times): a replica's slots are written when it is first
                    // dispatched, every read of them is masked by `valid`, and with
                    // AS the idle scan treats `fresh` (never dispatched) replicas as
                    // idle.  Until a replica is dispatched it is idle, so the busy
                    // and FIFO paths only ever see dispatched replicas.
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int j = gl * R + r;
                        if constexpr (!AS) av_set(r, INF);
                        if (j < dp) {
                            if (np > 0) {
                                sh = gs.pshape[__popc(ps & ((2u << j) - 1u)) - 1];
                            } else {
                                while (j >= cum) {
                                    ++sh;
                                    cum += lcounts[sh];
                                }
                            }
                            if (!SA) {
                                pre_s[r * 32 + lane] = a.tab.prefill[rb + sh];
                                dec_s[r * 32 + lane] = a.tab.decode[rb + sh];
                            }
                            if constexpr (!AS) av_set(r, 0.0);
                        }
                    }
                    mcur = 0;  // every replica starts idle (avail 0 <= T[0])
#pragma unroll
                    for (int r = 0; r < R; ++r) mcur |= (gl * R + r < dp) ? (1u << r) : 0u;
                    valid = mcur;
                    fresh = AS ? mcur : 0u;
                    k = 0;
                    ab = 0;
                    ns = 0;
                    qi = gs.qi;
                    lbk = gs.lbk;
                    ovf = false;
                    lazy = 0;
                }
            }
            __syncwarp();
            K4P_ADD(7, __popc(__ballot_sync(FULL, need && status == ST_RUN)));
            K4P_MARK(12);
        }
        if (__all_sync(FULL, status == ST_DONE)) break;
        U = __shfl_sync(FULL, U, gshift);  // one bound per group (leader's)
        K4P_ADD(9, 1);
        K4P_ADD(10, __popc(__ballot_sync(FULL, status == ST_RUN)));

        // a trip that ends with a prune check issues the check's loads now (the
        // future-bound count at the trip's end step and the live bound), so their
        // L2 latency overlaps the trip's steps; an earlier bound is a larger one,
        // still valid (sojourns above it exceed every later bound as well)
        const bool check_trip = (it & a.lane_check) == a.lane_check;
        int fut_pre = 0;
        double U_pre = U;
        if (check_trip && status == ST_RUN) {
            if (qi > 0)
                fut_pre = (int)a.tab.fut[(long long)((k + UNROLL + a.tab.fut_ab - 1) >> a.tab.fut_sh) * a.tab.nc + (qi - 1)];
            if (a.prune)
                U_pre = __longlong_as_double(
                    (long long)*(volatile unsigned long long*)&a.ub[(long long)row * (a.N + 1) + gpus]);
        }

        // ---- phase B: UNROLL request-steps per running plan, as pairs (rows
        // and k are even-aligned) with the next pair's arrivals/outputs
        // prefetched -- the lanes' rows differ, so they come from L2
        auto step = [&](const double t, const double o, const double tn1) {
            const bool run = status == ST_RUN;
            const unsigned m = run ? mcur : 0u;
            // next step's idle mask from the current avail (tn1 = next arrival),
            // off the critical path; the winner's bit is fixed once its finish
            // time is known
            unsigned mn = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) mn |= (av_get(r) <= tn1) ? (1u << r) : 0u;
            if constexpr (AS) mn = (mn & valid & ~fresh) | fresh;
            // a sojourn counts toward the prune test only while the FIFOs are
            // intact (no ring overflow in the group so far)
            const bool intact = W == 1 ? !ovf : ((__ballot_sync(FULL, ovf) >> gshift) & wmask) == 0u;
            bool idle;
            int wlane;
            if (W == 1) {
                idle = m != 0u;
                wlane = gl;
            } else {
                const unsigned gb = (__ballot_sync(FULL, m != 0u) >> gshift) & wmask;
                idle = gb != 0u;
                wlane = __ffs(gb) - 1;
            }
            const bool busy = run && !idle;
            int rr = __ffs(m) - 1;
            // the idle candidate's finish (start = t), issued before the busy
            // block so its shared-memory loads and fp64 chain overlap it
            const int pidx0 = pd_slot(rr > 0 ? rr : 0);
            double fin = __dadd_rn(__dadd_rn(t, pre_s[pidx0]), __dmul_rn(o, dec_s[pidx0]));
            double start = t;
            unsigned H = 0;
            bool one = false;  // count-1 dispatch: the replica holds only its last job
            if (W == 1 ? busy : __any_sync(FULL, busy)) {
                // Every replica busy.  A replica with exactly one job in system
                // (every earlier job finished: prev <= t) has the minimum count,
                // so the lowest such replica is the reference's argmin
                // (costmodel.cpp:262-276) -- no FIFO walk needed.
                unsigned m1 = 0;
#pragma unroll
                for (int r = 0; r < R; ++r) m1 |= (busy && prev_s[r * 32 + lane] <= t) ? (1u << r) : 0u;
                m1 = busy ? (m1 & valid) : 0u;
                bool has1;
                if (W == 1) {
                    has1 = m1 != 0u;
                } else {
                    const unsigned g1 = (__ballot_sync(FULL, m1 != 0u) >> gshift) & wmask;
                    has1 = g1 != 0u;
                    if (busy && has1) wlane = __ffs(g1) - 1;
                }
                if (busy && has1) {
                    rr = __ffs(m1) - 1;
                    one = true;
                }
                const bool slow = busy && !has1;
                if (W == 1 ? slow : __any_sync(FULL, slow)) {
                    // every replica holds >= 2 jobs: materialise the lazy FIFOs,
                    // pop up to t, then the (in-system count, index) minimum
                    if (slow && lazy) {
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            const bool lz = (lazy >> r) & 1u;
                            if (lz) {
                                nd_s[r * 32 + lane] = av_get(r);
                                const unsigned hr = ht_s[r * 32 + lane];
                                ht_s[r * 32 + lane] = (HT)((hr & (HM << HS)) | ((hr >> HS) & HM));
                            }
                        }
                        lazy = 0;
                    }
                    unsigned dep = 0;
#pragma unroll
                    for (int r = 0; r < R; ++r) dep |= (slow && nd_s[r * 32 + lane] <= t) ? (1u << r) : 0u;
                    dep &= valid;
                    while (W == 1 ? dep != 0u : __any_sync(FULL, dep != 0u)) {
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            if (!((dep >> r) & 1u)) continue;
                            const unsigned hr = ht_s[r * 32 + lane];
                            const unsigned h = hr & HM;
                            const unsigned tl = (hr >> HS) & HM;
                            const bool more = h != tl;  // the head waiting job enters service
                            double oh = 0.0;
                            if (HO) oh = ho[r];
                            else if (more) oh = Orow[ring[(r * CAP + (int)(h & (CAP - 1))) * 32 + lane]];
                            const double ndr = nd_s[r * 32 + lane];
                            const int pr = pd_slot(r);
                            const double nx = __dadd_rn(__dadd_rn(ndr, pre_s[pr]), __dmul_rn(oh, dec_s[pr]));
                            const double nn = more ? nx : INF;
                            nd_s[r * 32 + lane] = nn;
                            const unsigned h1 = (h + 1u) & HM;
                            if (more) ht_s[r * 32 + lane] = (HT)((hr & (HM << HS)) | h1);
                            if (HO && more && h1 != tl) ho[r] = Orow[ring[(r * CAP + (int)(h1 & (CAP - 1))) * 32 + lane]];
                            dep = (nn <= t) ? dep : (dep & ~(1u << r));
                        }
                    }
                    // (in-system count << 9 | replica) minimum, as a tree
                    unsigned kk[R];
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int j = gl * R + r;
                        const unsigned hr = ht_s[r * 32 + lane];
                        const unsigned c = (((hr >> HS) - hr) & HM) + (nd_s[r * 32 + lane] < INF ? 1u : 0u);
                        kk[r] = (j < dp) ? ((c << 9) | (unsigned)j) : 0xffffffffu;
                    }
#pragma unroll
                    for (int w = 1; w < R; w <<= 1)
#pragma unroll
                        for (int r = 0; r + w < R; r += 2 * w) kk[r] = kk[r + w] < kk[r] ? kk[r + w] : kk[r];
                    unsigned key = slow ? kk[0] : 0xffffffffu;
#pragma unroll
                    for (int off = W / 2; off > 0; off >>= 1) {
                        const unsigned v = __shfl_xor_sync(FULL, key, off);
                        key = v < key ? v : key;
                    }
                    if (slow) {
                        const int win = (int)(key & 511u);
                        wlane = win / R;
                        rr = win % R;
                    }
                }
                if (busy) {
                    // avail of replica rr: select tree on rr's bits; its ring state from shared memory
                    H = ht_s[rr * 32 + lane];
                    if constexpr (AS) {
                        start = avail_s[rr * 32 + lane];  // > t: std::max(t, avail)
                    } else {
                        double av[R];
#pragma unroll
                        for (int r = 0; r < R; ++r) av[r] = av_get(r);
#pragma unroll
                        for (int w = 1; w < R; w <<= 1) {
                            const bool hi = (rr & w) != 0;
#pragma unroll
                            for (int r = 0; r + w < R; r += 2 * w) av[r] = hi ? av[r + w] : av[r];
                        }
                        start = av[0];  // > t: std::max(t, avail)
                    }
                    const int pidx = pd_slot(rr);
                    fin = __dadd_rn(__dadd_rn(start, pre_s[pidx]), __dmul_rn(o, dec_s[pidx]));
                }
            }
            const bool me = run && gl == wlane;
            const double soj = __dsub_rn(fin, t);
            {
                // predicated on `me` throughout.  Idle: the FIFO now holds just
                // this job (lazy reset; H = 0 is an empty ring).  Count-1: the
                // job in service (finishing at start) and this one waiting --
                // the ring restarts empty.  Otherwise the job joins the queue.
                if (me && one) {
                    H = (H & (HM << HS)) | ((H >> HS) & HM);
                    nd_s[rr * 32 + lane] = start;
                    lazy &= ~(1u << rr);
                }
                const bool push = me && !idle;
                const bool first = push && (((H >> HS) & HM) == (H & HM));  // the ring was empty
                if (push) ring[(rr * CAP + (int)((H >> HS) & (CAP - 1))) * 32 + lane] = (unsigned short)k;
                H += push ? (1u << HS) : 0u;
                ovf |= push && ((((H >> HS) - H) & HM) > (unsigned)CAP);
                lazy |= (me && idle) ? (1u << rr) : 0u;
                // prev = start: the old finish when busy; when idle any value
                // <= t (every later test is prev <= t' with t' >= t)
                if (me) {
                    prev_s[rr * 32 + lane] = start;
                    ht_s[rr * 32 + lane] = (HT)H;
                }
                if constexpr (AS) {
                    if (me) avail_s[rr * 32 + lane] = fin;
                    fresh &= me ? ~(1u << rr) : ~0u;
                } else {
                    // one-hot winner mask: a bit test and one 64-bit select per
                    // replica (written as (me && r == rr) the compiler built the
                    // new value and then selected it again: five instructions)
                    const unsigned oh = me ? (1u << rr) : 0u;
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        avail[r] = CG_SELBIT ? sel_bit(oh, 1u << r, fin, avail[r]) : ((me && r == rr) ? fin : avail[r]);
                }
                if (HO && first) {  // the job is the head of an empty ring (rarer than a step)
#pragma unroll
                    for (int r = 0; r < R; ++r) ho[r] = sel_bit(1u << rr, 1u << r, o, ho[r]);
                }
                ab += (me && intact && soj > U) ? 1 : 0;
                // only sojourns >= the service bound can be among the K largest
                const bool keep = me && !(soj < lbk);
                if (keep) scratch[ns] = soj;
                if (W == 1) ns += keep ? 1 : 0;
                else ns += ((__ballot_sync(FULL, keep) >> gshift) & wmask) ? 1 : 0;
                const unsigned rb = me ? (1u << rr) : 0u;
                mcur = (mn & ~rb) | ((fin <= tn1) ? rb : 0u);
            }
            k += run ? 1 : 0;
            status = (run && k == n_req) ? ST_FINISH : status;
        };
        // k == u (mod 4) on every running lane: steps come in (even, odd)
        // pairs; after the even step the pair registers shift and the pair
        // after next is prefetched
        if constexpr (R >= 16) {
            // one inlined step (these step bodies are large: instruction-cache
            // footprint over select savings); the parity is warp-uniform
#pragma unroll 1
            for (int u = 0; u < UNROLL; ++u) {
                const bool odd = (u & 1) != 0;
                const double t = odd ? tq.y : tq.x;
                const double o = odd ? oq.y : oq.x;
                const double tn1 = odd ? tq2.x : tq.y;  // the next request's arrival
                if (odd) {
                    tq = tq2;
                    oq = oq2;
                    const int kp = (status == ST_RUN && k + 3 < n_req) ? k + 3 : 0;
                    tq2 = *reinterpret_cast<const double2*>(Trow + kp);
                    oq2 = *reinterpret_cast<const double2*>(Orow + kp);
                }
                step(t, o, tn1);
            }
        } else {
#pragma unroll 1
            for (int u = 0; u < UNROLL; u += 2) {
                step(tq.x, oq.x, tq.y);
                const double t1 = tq.y, o1 = oq.y, tn1 = tq2.x;  // tn1: the next request's arrival
                tq = tq2;
                oq = oq2;
                const int kp = (status == ST_RUN && k + 3 < n_req) ? k + 3 : 0;
                tq2 = *reinterpret_cast<const double2*>(Trow + kp);
                oq2 = *reinterpret_cast<const double2*>(Orow + kp);
                step(t1, o1, tn1);
            }
        }

        K4P_MARK(2);
        // ---- phase C: periodic exact-bound pruning and overflow checks
        if (check_trip) {
            int tot = ab;
            int ov = ovf ? 1 : 0;
#pragma unroll
            for (int off = W / 2; off > 0; off >>= 1) {
                tot += __shfl_xor_sync(FULL, tot, off);
                ov |= __shfl_xor_sync(FULL, ov, off);
            }
            if (status == ST_RUN) {
                // qi comes from the launch's bound snapshot (>= the live bound):
                // sojourns counted against any of the bounds seen exceed the
                // smallest of them, itself a latency found at <= gpus
                // fut_pre counts the plan's future requests from step k0 + UNROLL
                // on (k0: k at the trip's start); k <= k0 + UNROLL here, so it
                // counts only requests still to come
                const int fut = fut_pre;
                if (a.prune && tot + fut >= a.K) {  // tot: sojourns of intact steps only
                    pruned += 1;
                    steps += k;
                    status = ST_NEED;
                } else if (ov) {
                    if (gl == 0) {
                        const unsigned long long idx = atomicAdd(a.ovf_count, 1ull);
                        if (idx < a.ovf_cap) a.ovf[idx] = ((unsigned long long)row << kItemPlanBits) | plan;
                    }
                    steps += k;
                    status = ST_NEED;
                } else if (a.prune) {
                    U = U_pre;
                }
            }
            U = __shfl_sync(FULL, U, gshift);
            if (status == ST_NEED && gl == 0) gs.status = ST_NEED;
        }

        K4P_MARK(3);
        // ---- phase D: completed plans -> exact p95 (warp-cooperative) and row bookkeeping
        if (__any_sync(FULL, status == ST_FINISH)) {
            int tot = ab;
            int ov = ovf ? 1 : 0;
#pragma unroll
            for (int off = W / 2; off > 0; off >>= 1) {
                tot += __shfl_xor_sync(FULL, tot, off);
                ov |= __shfl_xor_sync(FULL, ov, off);
            }
            bool sel = false;
            if (status == ST_FINISH) {
                steps += k;
                ov |= ns < a.K ? 1 : 0;  // cannot happen (lbk <= p95); the DEEP re-run keeps every sojourn
                if (a.prune && tot >= a.K) {
                    pruned += 1;
                } else if (ov) {
                    if (gl == 0) {
                        const unsigned long long idx = atomicAdd(a.ovf_count, 1ull);
                        if (idx < a.ovf_cap) a.ovf[idx] = ((unsigned long long)row << kItemPlanBits) | plan;
                    }
                } else {
                    sel = true;
                }
            }
            __syncwarp();  // the columns' stores are visible to the whole warp
            unsigned fm = __ballot_sync(FULL, sel && gl == 0);
            while (fm) {
                const int ldr = __ffs(fm) - 1;
                fm &= fm - 1u;
                const double* col = a.scratch + (gwarp * G + ldr / W) * (long long)a.sld;
                const int nsel = __shfl_sync(FULL, ns, ldr);
                const unsigned long long xb = group_kth_largest<32, true>(col, nsel, a.K, lane, FULL, 0, hist);
                if (lane == ldr) {
                    full += 1;
                    const long long base = (long long)row * (a.N + 1);
                    const unsigned long long old = atomicMin(&a.lat_min[base + gpus], xb);
                    if (xb <= old) {
                        const unsigned long long idx = atomicAdd(a.tie_count, 1ull);
                        if (idx < a.tie_cap) a.ties[idx] = TieEntry{row, gpus, xb, plan};
                    }
                    for (int g2 = gpus; g2 <= a.N; ++g2) {
                        unsigned long long* ub = &a.ub[base + g2];
                        if (*(volatile unsigned long long*)ub <= xb) break;
                        atomicMin(ub, xb);
                    }
                }
                __syncwarp();
            }
            if (status == ST_FINISH) {
                status = ST_NEED;
                if (gl == 0) gs.status = ST_NEED;
            }
            __syncwarp();
        }
        K4P_MARK(4);
    }
    if constexpr (W == 1) K4P_FLUSH(R == 4 ? 0 : R == 8 ? 1 : R == 16 ? 2 : 3);
    if (gl == 0) {
        count_add(&a.counters[CTR_BOUND], bound);
        count_add(&a.counters[CTR_STEPS], steps);
        count_add(&a.counters[a.seeds ? CTR_SEED : CTR_FULL], full);
        count_add(&a.counters[a.seeds ? CTR_SEED : CTR_PRUNED], pruned);
    }
}

template <int W, int R>
void launch_lane_t(const SimArgs& a, int sm_count, cudaStream_t s, int* launches, int* grid_out) {
    using TR = LaneTraits<W, R>;
    const size_t smem = TR::bytes_per_warp * TR::WPB;
    auto kern = k_lane<W, R>;
    CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TR::WPB * 32, smem));
    if (per_sm < 1) per_sm = 1;
    const int grid = sm_count * per_sm;
    if (grid_out) *grid_out = grid;
    if (a.nitems == 0) return;
    kern<<<grid, TR::WPB * 32, smem, s>>>(a);
    CG_LAUNCH_CHECK();
    if (launches) ++*launches;
}

// ---------------------------------------------------------------------------
// K5: tie resolution and the prefix minimum over budgets

__global__ void k_resolve_ties(ResolveArgs a) {
    const unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    if (e >= a.nties) return;
    const TieEntry te = a.ties[e];
    const long long cell = (long long)te.row * (a.N + 1) + te.g;
    if (te.lat_bits != a.lat_min[cell]) return;
    const PlanSpace& sp = a.spaces[a.rows[te.row].space];
    unsigned char A[kMaxShapes], B[kMaxShapes];
    unrank_plan(sp, te.plan, A);
    unsigned long long cur = *(volatile unsigned long long*)&a.best_plan[cell];
    while (true) {
        if (cur != kEmpty) {
            if (cur == te.plan) return;
            unrank_plan(sp, cur, B);
            if (!parts_less(A, B, sp.S)) return;
        }
        const unsigned long long prev = atomicCAS(&a.best_plan[cell], cur, te.plan);
        if (prev == cur) return;
        cur = prev;
    }
}

// StageEvaluator::row prefix minimum (costmodel.cpp:398-412): strict '<' so
// ties keep the smaller budget; f = 0 is never assigned for live rows.
__global__ void k_row_prefix(ResolveArgs a) {
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= a.nrows) return;
    const long long base = (long long)row * (a.N + 1);
    double running = __longlong_as_double((long long)kInfBits);
    long long running_plan = -1;
    a.final_lat[base] = running;
    a.final_plan[base] = -1;
    for (int f = 1; f <= a.N; ++f) {
        const unsigned long long p = a.best_plan[base + f];
        if (p != kEmpty) {
            const double l = __longlong_as_double((long long)a.lat_min[base + f]);
            if (l < running) {
                running = l;
                running_plan = (long long)p;
            }
        }
        a.final_lat[base + f] = running;
        a.final_plan[base + f] = running_plan;
    }
}

// ---------------------------------------------------------------------------
// Plan filter: every plan of every row is enumerated exactly once, by a thread
// per chunk of consecutive plan indices (unrank the first, lexicographic
// successor for the rest).  A plan survives if it is stable
// (costmodel.cpp:366-376) and its exact service-time bound does not exceed the
// best latency already known at <= its budget: every sojourn on shape s is >=
// fl(fl(fl(t+p_s)+fl(o d_s))-t) >= (p_s+o d_s)(1-5u) - 2u t (u = 2^-53), and
// min_s(p_s + o d_s) is increasing in o, so the K-th largest sojourn is >=
// min_{s in plan}(p_s + o_(K) d_s)(1-1e-12) - 1e-12 T_max where o_(K) is the
// K-th largest CRN output.  Survivors go to the work list of their
// replica-count class (warp-aggregated appends).
__global__ void __launch_bounds__(128) k_plan_filter(FilterArgs a) {
    const unsigned long long chunk = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    const bool active = chunk < a.nchunks;
    int row = 0;
    unsigned long long lo = 0, hi = 0;
    if (active) {
        // this rank's chunks interleave with the other ranks' (chunk g belongs
        // to rank g mod world): every rank sees every row's plan mix
        const unsigned long long g = shard_global_chunk(chunk + a.chunk_base, a.shard_rank, a.shard_world);
        int l = 0, h = a.nrows - 1;  // chunk_prefix[l] <= g < chunk_prefix[l+1]
        while (l < h) {
            const int mid = (l + h + 1) >> 1;
            if (a.chunk_prefix[mid] <= g) l = mid;
            else h = mid - 1;
        }
        row = a.row_ids[l];
        // reversed within the row: large-shape plans (best bounds) first
        const unsigned long long nrc = a.chunk_prefix[l + 1] - a.chunk_prefix[l];
        const unsigned long long j = nrc - 1 - (g - a.chunk_prefix[l]);
        const unsigned long long P = a.spaces[a.rows[row].space].num_plans;
        lo = j * (unsigned long long)a.chunk;
        hi = lo + a.chunk < P ? lo + a.chunk : P;
    }
    const RowDesc rd = a.rows[active ? row : 0];
    const PlanSpace& sp = a.spaces[rd.space];
    const long long rb = (long long)row * kMaxShapes;
    unsigned char c[kMaxShapes];
    int used = 0, dp = 0;
    unsigned nz = 0;  // bit s: c[s] > 0 (the loops below visit the plan's parts only)
    if (active) {
        used = unrank_plan(sp, lo, c);
        for (int s = 0; s < sp.S; ++s) {
            dp += c[s];
            nz |= c[s] ? (1u << s) : 0u;
        }
    }
    const double o_k = active ? a.tab.O[(long long)row * a.tab.ld + a.kstar] : 0.0;
    const double t_max = active ? a.tab.T[(long long)row * a.tab.ld + a.n_req - 1] : 0.0;
    unsigned long long stable = 0, skipped = 0;
    const unsigned long long trips = a.chunk;
    for (unsigned long long k = 0; k < trips; ++k) {
        const unsigned long long p = lo + k;
        const bool live = active && p < hi;
        if (live && k > 0) {
            // lexicographic successor (plan_dev.cuh next_plan) keeping nz
            for (int i = sp.S - 1; i >= 0; --i) {
                const int size = sp.shapes[i].gpus;
                if (used + size <= sp.N) {
                    c[i] = (unsigned char)(c[i] + 1);
                    used += size;
                    dp += 1;
                    nz |= 1u << i;
                    break;
                }
                used -= c[i] * size;
                dp -= c[i];
                c[i] = 0;
                nz &= ~(1u << i);
            }
        }
        int cls = -1;
        unsigned long long key = 0;
        double lbs = 0.0;  // the listed plan's service bound (ItemRec::lb)
        if (live) {
            // Stability (costmodel.cpp:366-376): rate < sum over parts of cnt /
            // mean_service, summed in parts order.  Fast test first: each term
            // cnt * fl(1/ms) is within 2u(1+u) of cnt/ms and both sums carry at
            // most S roundings, so the two capacities differ by < 2(S+3)u <
            // 1e-13 relative; only rates inside that band take the exact path.
            // an infeasible shape has inv_service NaN: the capacity is NaN and
            // both stability tests below fail, as the reference's `ok` does
            double capacity = 0.0, lb = __longlong_as_double(0x7ff0000000000000ll), slow = 0.0;
            for (unsigned m = nz; m; m &= m - 1u) {
                const int s = __ffs(m) - 1;
                capacity += (double)c[s] * a.tab.inv_service[rb + s];
                const double v = a.tab.svc_k[rb + s];  // prefill + o_(K) decode
                lb = v < lb ? v : lb;
                slow = v > slow ? v : slow;
            }
            const bool good = capacity == capacity;
            bool stable_plan = good && rd.rate < capacity * (1.0 - 1e-13);
            if (good && !stable_plan && rd.rate < capacity * (1.0 + 1e-13)) {  // the exact reference sum
                double exact = 0.0;
                for (unsigned m = nz; m; m &= m - 1u) {  // parts order (ascending shape)
                    const int s = __ffs(m) - 1;
                    exact = __dadd_rn(exact, __ddiv_rn((double)c[s], a.tab.mean_service[rb + s]));
                }
                stable_plan = rd.rate < exact;
            }
            if (stable_plan) {
                ++stable;
                bool keep = true;
                lb = lb * (1.0 - 1e-12) - 1e-12 * t_max;
                lbs = lb;
                // coarse order key, likely-good plans first: the service bound,
                // or (sort_key 1) the heuristic estimate service bound / (1 - utilisation)
                // order heuristics (results never depend on them): 1 fast-shape
                // bound / (1 - rho), 3 (default) mean of the fastest and slowest
                // shapes' bounds / (1 - rho), ...
                // (order only: the default key is computed in float)
                double est = lb;
                if (a.sort_key == 3) {
                    const float rho = __fdividef((float)rd.rate, (float)capacity);
                    est = (double)__fdividef(0.5f * ((float)lb + (float)slow), 1.0f - rho);
                }
                const double rho = a.sort_key == 3 ? 0.0 : rd.rate / capacity;
                if (a.sort_key == 1) est = lb / (1.0 - rho);
                else if (a.sort_key == 2) est = lb / ((1.0 - rho) * (1.0 - rho));
                else if (a.sort_key == 4) est = slow / (1.0 - rho);
                else if (a.sort_key == 5) est = 0.25 * (lb + 3.0 * slow) / (1.0 - rho);
                else if (a.sort_key == 6) est = slow / ((1.0 - rho) * (1.0 - rho));
                est = est > 0.0 ? est : 0.0;
                key = dbl_to_key(a.sort_key ? est : lb) >> (64 - kListKeyBits);
                if (a.prune) {
                    const double U = __longlong_as_double(
                        (long long)*(volatile unsigned long long*)&a.ub[(long long)row * (a.N + 1) + used]);
                    if (lb > U) {
                        keep = false;
                        ++skipped;
                    }
                }
                if (keep && !a.pilot_only) cls = class_of_dp(dp);
                if (keep && a.pilot && sp.num_plans >= a.pilot_min_plans) {
                    // heuristic p95 estimate (order only): service bound / (1 - utilisation)
                    const unsigned long long v =
                        (((unsigned long long)__double_as_longlong(est) >> 44) << kItemPlanBits) | p;
                    unsigned long long* cell = &a.pilot[(long long)row * (a.N + 1) + used];
                    if (v < *(volatile unsigned long long*)cell) atomicMin(cell, v);
                }
            }
        }
        // warp-aggregated append into the class lists
        const unsigned want = __ballot_sync(0xffffffffu, cls >= 0);
        if (want) {
            const unsigned peers = __match_any_sync(0xffffffffu, cls);
            if (cls >= 0) {
                const int lane = threadIdx.x & 31;
                const int leader = __ffs(peers) - 1;
                unsigned long long base = 0;
                if (lane == leader) base = atomicAdd(&a.list_count[cls], (unsigned long long)__popc(peers));
                base = __shfl_sync(peers, base, leader);
                const unsigned long long slot = base + __popc(peers & ((1u << lane) - 1u));
                if (slot < a.list_caps[cls]) {
                    ItemRec r;
                    r.item = ((unsigned long long)row << kItemPlanBits) | p;
                    encode_rec(r, c, sp.S, used);
                    r.lb = lbs;
                    a.recs[cls][slot] = r;
                    a.keys[cls][slot] = key;
                }
            }
        }
    }
    if (a.pilot_only) return;
    if (stable) atomicAdd(&a.counters[CTR_STABLE], stable);
    if (skipped) atomicAdd(&a.counters[CTR_BOUND], skipped);
}

// Future-bound snapshot: per (row, budget g, shape s) the number of leading
// output-ranked request blocks i whose smallest output Pv[row][i] still gives
// a service lower bound above ub[row][g] on shape s -- the same predicate the
// plan-level bound applies to min over the plan's shapes, which is the
// minimum of these per-shape counts (the predicate is monotone in the
// bound, and min_s commutes with the monotone margin transform).  Pv is
// non-increasing in i, so the qualifying blocks form a prefix: binary search.
__global__ void k_fut_snapshot(FutSnapArgs a) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long cells = (long long)a.nrows * (a.N + 1);
    if (t >= cells * kMaxShapes) return;
    const long long cell = t / kMaxShapes;
    const int s = (int)(t % kMaxShapes);
    const int row = (int)(cell / (a.N + 1));
    const PlanSpace& sp = a.spaces[a.rows[row].space];
    unsigned short q = 0;
    const double U = __longlong_as_double((long long)*(volatile const unsigned long long*)&a.ub[cell]);
    if (s < sp.S && a.tab.nc > 0 && U < __longlong_as_double(0x7ff0000000000000ll)) {
        const long long rb = (long long)row * kMaxShapes;
        const double p = a.tab.prefill[rb + s], d = a.tab.decode[rb + s];
        const double t_max = a.tab.T[(long long)row * a.tab.ld + a.n_req - 1];
        const double* Pv = a.tab.Pv + (long long)row * a.tab.nc;
        int lo = 0, hi = a.tab.nc;  // answer in [lo, hi]: blocks [0, lo) qualify, [hi, nc) do not
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            const double v = p + Pv[mid] * d;
            if (v * (1.0 - 1e-12) - 1e-12 * t_max > U) lo = mid + 1;
            else hi = mid;
        }
        q = (unsigned short)lo;
    }
    a.qtab[t] = q;
}

__global__ void k_pilot_lists(PilotArgs a) {
    const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (c >= a.cells) return;
    const unsigned long long v = a.pilot[c];
    if (v == ~0ull) return;
    const int row = (int)(c / (a.N + 1));
    const unsigned long long plan = v & kItemPlanMask;
    const PlanSpace& sp = a.spaces[a.rows[row].space];
    unsigned char cn[kMaxShapes];
    unrank_plan(sp, plan, cn);
    int dp = 0;
    for (int s = 0; s < sp.S; ++s) dp += cn[s];
    int cls = class_of_dp(dp);
    // fewer, larger launches: class 3's kernel covers every dp <= 32
    if (a.merge == 2 && cls < 3) cls = 3;
    if (a.merge == 1 && cls >= 1 && cls < 3) cls = 3;
    const unsigned long long slot = atomicAdd(&a.list_count[cls], 1ull);
    a.lists[cls][slot] = ((unsigned long long)row << kItemPlanBits) | plan;
    a.keys[cls][slot] = 1ull + (v >> kItemPlanBits);  // 20-bit estimate + 1 (seeds carry key 0)
}

template <int W, int R, int MODE>
void launch_sim_t(const SimArgs& a, int sm_count, cudaStream_t s, int* launches, int* grid_out) {
    using TR = Traits<W, R, MODE>;
    const size_t smem = TR::bytes_per_warp * 4;
    auto kern = k_sim<W, R, MODE>;
    CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem));
    if (per_sm < 1) per_sm = 1;
    int grid = sm_count * per_sm;
    if (MODE == MODE_DEEP && grid > sm_count) grid = sm_count;
    if (grid_out) *grid_out = grid;
    if (a.nitems == 0) return;
    kern<<<grid, 128, smem, s>>>(a);
    CG_LAUNCH_CHECK();
    if (launches) ++*launches;
}

}  // namespace

SimGeometry sim_geometry(int cls, int mode, int sm_count) {
    // must mirror launch_sim's grid choice: slots = grid * 4 warps * G
    SimGeometry g{};
    int W = 32, R = 1;
    class_shape(cls, &W, &R);
    if (mode == MODE_DEEP) W = 32;
    g.W = W;
    g.R = R;
    g.G = 32 / W;
    int grid = 0;
    SimArgs dummy{};
    dummy.nitems = 0;
    launch_sim(dummy, cls, mode, sm_count, nullptr, nullptr, &grid);
    g.grid = grid;
    g.slots = (long long)grid * 4 * g.G;
    g.warps = (long long)grid * 4;
    return g;
}

// Lane packing of the replica-count classes (engine option k4_pack):
//   0: one replica per lane, W = 4/8/16/32 lanes for dp <= 4/8/16/32
//   1: two replicas per lane from dp > 4 on (more plans per warp)
//   2: up to four replicas per lane
//   3: lane-major kernels (k_lane) for dp <= 32, one lane per plan: R = 4/8/16/32
//      replicas per lane (default; C3 K4 890 -> 670 ms against 5)
//   4: k_lane with W = 1/1/2/1 lanes per plan, R = 4/8/8/32
//   5: k_lane with W = 1/1/2/4, R = 4/8/8/8 (round 1)
static thread_local int g_pack = 0;  // per host thread: engines of a multi-device group run concurrently
void set_k4_pack(int p) { g_pack = p < 0 ? 0 : (p > 5 ? 5 : p); }

void class_shape(int cls, int* W, int* R) {
    static const int Ws[6][7] = {{4, 8, 16, 32, 32, 32, 32}, {4, 4, 8, 16, 32, 32, 32}, {4, 4, 4, 8, 32, 32, 32},
                                 {1, 1, 1, 1, 32, 32, 32}, {1, 1, 2, 1, 32, 32, 32}, {1, 1, 2, 4, 32, 32, 32}};
    static const int Rs[6][7] = {{1, 1, 1, 1, 2, 4, 8}, {1, 2, 2, 2, 2, 4, 8}, {1, 2, 4, 4, 2, 4, 8},
                                 {4, 8, 16, 32, 2, 4, 8}, {4, 8, 8, 32, 2, 4, 8}, {4, 8, 8, 8, 2, 4, 8}};
    *W = Ws[g_pack][cls];
    *R = Rs[g_pack][cls];
}

void class_dp_range(int cls, int* lo, int* hi) {
    static const int His[7] = {4, 8, 16, 32, 64, 128, 256};
    *lo = cls == 0 ? 0 : His[cls - 1];
    *hi = His[cls];
}

int class_for_dp(int dpmax) {
    if (dpmax <= 4) return 0;
    if (dpmax <= 8) return 1;
    if (dpmax <= 16) return 2;
    if (dpmax <= 32) return 3;
    if (dpmax <= 64) return 4;
    if (dpmax <= 128) return 5;
    if (dpmax <= 255) return 6;  // replica counts are 8-bit (filter, packed parts, unrank)
    return -1;
}

static void launch_sim_impl(const SimArgs& a, int cls, int mode, int sm_count, cudaStream_t s, int* launches,
                            int* grid_out);

// Diagnostic (CG_TRACE_K4=1): per launch, the class, items, request-steps,
// completed / pruned plans and the launch time (synchronising: not for timing
// runs).
void launch_sim(const SimArgs& a, int cls, int mode, int sm_count, cudaStream_t s, int* launches,
                int* grid_out) {
    static const bool trace = std::getenv("CG_TRACE_K4") != nullptr;
    if (!trace || a.nitems == 0 || !a.counters) {
        launch_sim_impl(a, cls, mode, sm_count, s, launches, grid_out);
        return;
    }
    unsigned long long c0[CTR_COUNT], c1[CTR_COUNT];
    CG_CUDA(cudaStreamSynchronize(s));
    CG_CUDA(cudaMemcpy(c0, a.counters, sizeof(c0), cudaMemcpyDeviceToHost));
    cudaEvent_t e0, e1;
    CG_CUDA(cudaEventCreate(&e0));
    CG_CUDA(cudaEventCreate(&e1));
    CG_CUDA(cudaEventRecord(e0, s));
    launch_sim_impl(a, cls, mode, sm_count, s, launches, grid_out);
    CG_CUDA(cudaEventRecord(e1, s));
    CG_CUDA(cudaStreamSynchronize(s));
    float ms = 0.f;
    CG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    CG_CUDA(cudaMemcpy(c1, a.counters, sizeof(c1), cudaMemcpyDeviceToHost));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    std::fprintf(stderr, "[k4] cls=%d mode=%d seeds=%d items=%llu steps=%llu full=%llu pruned=%llu bound=%llu ms=%.3f\n",
                 cls, mode, a.seeds, (unsigned long long)a.nitems, c1[CTR_STEPS] - c0[CTR_STEPS],
                 c1[CTR_FULL] - c0[CTR_FULL], c1[CTR_PRUNED] - c0[CTR_PRUNED], c1[CTR_BOUND] - c0[CTR_BOUND], ms);
    std::fflush(stderr);
}

static void launch_sim_impl(const SimArgs& a, int cls, int mode, int sm_count, cudaStream_t s, int* launches,
                            int* grid_out) {
    if (mode == MODE_DEEP) {
        switch (cls) {
            case 0: case 1: case 2: case 3: launch_sim_t<32, 1, MODE_DEEP>(a, sm_count, s, launches, grid_out); return;
            case 4: launch_sim_t<32, 2, MODE_DEEP>(a, sm_count, s, launches, grid_out); return;
            case 5: launch_sim_t<32, 4, MODE_DEEP>(a, sm_count, s, launches, grid_out); return;
            case 6: launch_sim_t<32, 8, MODE_DEEP>(a, sm_count, s, launches, grid_out); return;
        }
    } else if (g_pack >= 3 && cls <= 3) {
        switch (cls) {
            case 0: launch_lane_t<1, 4>(a, sm_count, s, launches, grid_out); return;
            case 1: launch_lane_t<1, 8>(a, sm_count, s, launches, grid_out); return;
            case 2:
                if (g_pack == 3) launch_lane_t<1, 16>(a, sm_count, s, launches, grid_out);
                else launch_lane_t<2, 8>(a, sm_count, s, launches, grid_out);
                return;
            case 3:
                if (g_pack == 5) launch_lane_t<4, 8>(a, sm_count, s, launches, grid_out);
                else launch_lane_t<1, 32>(a, sm_count, s, launches, grid_out);
                return;
        }
    } else {
        switch (cls) {
            case 0: launch_sim_t<4, 1, MODE_LIST>(a, sm_count, s, launches, grid_out); return;
            case 1:
                if (g_pack == 0) launch_sim_t<8, 1, MODE_LIST>(a, sm_count, s, launches, grid_out);
                else launch_sim_t<4, 2, MODE_LIST>(a, sm_count, s, launches, grid_out);
                return;
            case 2:
                if (g_pack == 0) launch_sim_t<16, 1, MODE_LIST>(a, sm_count, s, launches, grid_out);
                else if (g_pack == 1) launch_sim_t<8, 2, MODE_LIST>(a, sm_count, s, launches, grid_out);
                else launch_sim_t<4, 4, MODE_LIST>(a, sm_count, s, launches, grid_out);
                return;
            case 3:
                if (g_pack == 0) launch_sim_t<32, 1, MODE_LIST>(a, sm_count, s, launches, grid_out);
                else if (g_pack == 1) launch_sim_t<16, 2, MODE_LIST>(a, sm_count, s, launches, grid_out);
                else launch_sim_t<8, 4, MODE_LIST>(a, sm_count, s, launches, grid_out);
                return;
            case 4: launch_sim_t<32, 2, MODE_LIST>(a, sm_count, s, launches, grid_out); return;
            case 5: launch_sim_t<32, 4, MODE_LIST>(a, sm_count, s, launches, grid_out); return;
            case 6: launch_sim_t<32, 8, MODE_LIST>(a, sm_count, s, launches, grid_out); return;
        }
    }
    throw EngineError(101, "unsupported JSQ kernel class");
}

void launch_fut_snapshot(const FutSnapArgs& a, cudaStream_t s, int* launches) {
    const long long work = (long long)a.nrows * (a.N + 1) * kMaxShapes;
    if (work == 0 || !a.qtab) return;
    k_fut_snapshot<<<(unsigned)((work + 255) / 256), 256, 0, s>>>(a);
    CG_LAUNCH_CHECK();
    if (launches) ++*launches;
}

void launch_pilot_lists(const PilotArgs& a, cudaStream_t s, int* launches) {
    if (a.cells == 0) return;
    k_pilot_lists<<<(unsigned)((a.cells + 127) / 128), 128, 0, s>>>(a);
    CG_LAUNCH_CHECK();
    if (launches) ++*launches;
}

void launch_plan_filter(const FilterArgs& a, cudaStream_t s, int* launches) {
    if (a.nchunks == 0) return;
    k_plan_filter<<<(unsigned)((a.nchunks + 127) / 128), 128, 0, s>>>(a);
    CG_LAUNCH_CHECK();
    if (launches) ++*launches;
}

// The filter's per-(row, shape) service term prefill + o_(K) decode (o_(K):
// the K-th largest CRN output, the same request index for every row).
__global__ void k_row_svck(RowTables tab, int nrows, int kstar) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)nrows * kMaxShapes) return;
    const long long row = t / kMaxShapes;
    const double o_k = tab.O[row * tab.ld + kstar];
    tab.svc_k[t] = tab.prefill[t] + o_k * tab.decode[t];
}

void launch_row_svck(const RowTables& tab, int nrows, int kstar, cudaStream_t s, int* launches) {
    if (nrows == 0) return;
    const long long work = (long long)nrows * kMaxShapes;
    k_row_svck<<<(unsigned)((work + 255) / 256), 256, 0, s>>>(tab, nrows, kstar);
    CG_LAUNCH_CHECK();
    if (launches) ++*launches;
}

void launch_row_setup(const RowSetupArgs& a, const double* L, cudaStream_t s, int* launches) {
    if (a.nrows == 0) return;
    const long long work = (long long)a.nrows * kMaxShapes;
    k_row_shapes<<<(unsigned)((work + 127) / 128), 128, 0, s>>>(a);
    CG_LAUNCH_CHECK();
    k_row_crn<<<(unsigned)((a.nrows + 63) / 64), 64, 0, s>>>(a, L);
    CG_LAUNCH_CHECK();
    if (launches) *launches += 2;
}

void launch_resolve(const ResolveArgs& a, cudaStream_t s, int* launches) {
    if (a.nties > 0) {
        k_resolve_ties<<<(unsigned)((a.nties + 127) / 128), 128, 0, s>>>(a);
        CG_LAUNCH_CHECK();
        if (launches) ++*launches;
    }
    if (a.nrows > 0) {
        k_row_prefix<<<(unsigned)((a.nrows + 127) / 128), 128, 0, s>>>(a);
        CG_LAUNCH_CHECK();
        if (launches) ++*launches;
    }
}

#ifdef CG_K4_PROF
extern "C" int cg_k4prof_read(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, cg::g_k4prof, sizeof(cg::g_k4prof)) == cudaSuccess ? 0 : 1;
}
extern "C" int cg_k4prof_reset() {
    static unsigned long long z[4][16] = {};
    return cudaMemcpyToSymbol(cg::g_k4prof, z, sizeof(z)) == cudaSuccess ? 0 : 1;
}
#endif
}  // namespace cg
