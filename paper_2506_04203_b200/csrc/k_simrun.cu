// Validation simulator on the GPU: cascade::sim::run
// and sim::compare (proj/src/simulator.cpp:177-299, 318-334) for a batch of
// cascade plans at once.
//
// The reference replays the real trace through one plan with a global event
// queue ordered by (time, seq).  Events reach a stage only from the previous
// deployed stage, and escalations are pushed in the order the previous stage
// processed them, so the queue order restricted to a stage is: the entry
// stage in (arrival, trace index) order; every later stage in (finish time at
// the previous stage, processing order there).  The simulation is therefore
// exactly a sequence of per-stage passes with a stable sort by finish time in
// between -- which is how it runs here:
//   k_sr_stage   one warp per plan: the stage's events in order, 32 at a time
//                (lanes gather the next 32 events' trace fields, then the warp
//                walks them with shuffles); replicas on lanes; join-shortest-
//                expected-work = lowest idle replica (ballot) or the (backlog,
//                index) minimum; per-stage wait / service sums in order
//   radix sort   stable, by finish time (k_sort.cu)
//   k_sr_metrics one block per plan: p95 (radix select), throughput span,
//                attainment counts
// fp64 with explicit _rn ops in the reference's expression order (H2).
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "cg_cuda.h"
#include "cg_internal.h"
#include "cg_kernels.h"
#include "cg_simrun.h"

namespace cg {

namespace {

constexpr int SR_WARPS = 4;

__global__ void k_sr_keys(const double* __restrict__ arrival, long long n, unsigned long long* __restrict__ keys,
                          unsigned long long* __restrict__ vals) {
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= n) return;
    keys[r] = dbl_to_key(arrival[r]);
    vals[r] = (unsigned long long)r;
}

// dry_run_base (simulator.cpp:161-173): per-request no-contention latency on
// the first replica of every stage of the accept path ...
__global__ void k_sr_dry(SimRunArgs a, const SimPlanDesc* __restrict__ plan, double* __restrict__ lat) {
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= a.n) return;
    const SimPlanDesc& p = *plan;
    double latency = 0.0;
    for (int s = p.entry; s >= 0; s = p.next[s]) {
        const int q = p.roff[s];  // replicas.front()
        const double svc = __dadd_rn(__dadd_rn(__dmul_rn(a.ppt[q], a.in[r]), a.pf[q]),
                                     __dmul_rn(a.out[(long long)s * a.n + r], a.dpt[q]));
        latency = __dadd_rn(latency, svc);
        if (s == p.last || a.scores[(long long)s * a.n + r] >= p.thr[s]) break;
    }
    lat[r] = latency;
}

// ... summed in trace order and divided by n: the block stages tiles in shared
// memory, thread 0 adds them sequentially (one block per plan)
__global__ void __launch_bounds__(1024) k_sr_mean(const double* __restrict__ lat, long long n,
                                                  double* __restrict__ out) {
    constexpr int TILE = 2048;
    __shared__ double tile[2][TILE];
    const double* x = lat + (long long)blockIdx.x * n;
    double sum = 0.0;
    int buf = 0;
    for (long long i = threadIdx.x; i < TILE && i < n; i += blockDim.x) tile[0][i] = x[i];
    __syncthreads();
    for (long long b0 = 0; b0 < n; b0 += TILE) {
        const long long nb = b0 + TILE;
        for (long long i = threadIdx.x; i < TILE && nb + i < n; i += blockDim.x) tile[buf ^ 1][i] = x[nb + i];
        if (threadIdx.x == 0) {
            const int len = (int)(n - b0 < TILE ? n - b0 : TILE);
            for (int i = 0; i < len; ++i) sum = __dadd_rn(sum, tile[buf][i]);
        }
        __syncthreads();
        buf ^= 1;
    }
    if (threadIdx.x == 0) out[blockIdx.x] = __ddiv_rn(sum, (double)n);
}

// One stage pass of every plan of the batch (warp per plan).
template <int R>
__global__ void __launch_bounds__(32 * SR_WARPS) k_sr_stage(SimRunArgs a, int step) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pi = blockIdx.x * SR_WARPS + warp;
    if (pi >= a.nplans) return;
    const SimPlanDesc& p = a.plans[pi];
    const int s = p.chain[step];
    if (s < 0) return;
    const long long n = a.n;
    const long long m = a.ev_count[pi];
    const unsigned long long* ek = a.ev_keys + (long long)pi * n;
    const unsigned long long* ev = a.ev_vals + (long long)pi * n;
    unsigned long long* nk = a.nx_keys + (long long)pi * n;
    unsigned long long* nv = a.nx_vals + (long long)pi * n;
    double* e2e = a.e2e + (long long)pi * n;
    int* ast = a.astage + (long long)pi * n;
    const int dp = p.dp[s];
    const bool last = s == p.last;
    const double thr = last ? 0.0 : p.thr[s];
    double avail[R], ppt[R], pf[R], dpt[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int j = r * 32 + lane;
        avail[r] = 0.0;
        const int q = p.roff[s] + (j < dp ? j : 0);
        ppt[r] = a.ppt[q];
        pf[r] = a.pf[q];
        dpt[r] = a.dpt[q];
    }
    const long long half = m / 2;
    double w1 = 0.0, w2 = 0.0, ssum = 0.0;
    long long nesc = 0;
    const double* out_s = a.out + (long long)s * n;
    const double* sc_s = a.scores + (long long)s * n;
    __shared__ double s_t[SR_WARPS][32], s_in[SR_WARPS][32], s_o[SR_WARPS][32];
    for (long long b = 0; b < m; b += 32) {
        // lanes gather the next 32 events (time, request, trace fields) ...
        const long long e = b + lane;
        double bt = 0.0, bin = 0.0, bout = 0.0, bsc = 0.0, barr = 0.0;
        long long br = 0;
        if (e < m) {
            bt = key_to_dbl(ek[e]);
            br = (long long)ev[e];
            bin = a.in[br];
            bout = out_s[br];
            bsc = sc_s[br];
            barr = a.arrival[br];
        }
        __syncwarp();
        s_t[warp][lane] = bt;
        s_in[warp][lane] = bin;
        s_o[warp][lane] = bout;
        __syncwarp();
        // ... and the warp walks them in order; event i's finish time ends up
        // in lane i, outputs are written in parallel after the walk
        const int cnt = (int)(m - b < 32 ? m - b : 32);
        double my_fin = 0.0;
#pragma unroll 2
        for (int i = 0; i < cnt; ++i) {
            const double t = s_t[warp][i];
            const double in = s_in[warp][i];
            const double o = s_o[warp][i];
            // join shortest expected work (simulator.cpp:215-224): the lowest
            // idle replica (backlog max(0, avail - t) == 0), else the minimum
            // (backlog, index) -- backlogs > 0, so their bit patterns order
            // like the values: hi word, lo word, then index, by warp reductions
            int win = -1;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const bool idle = (r * 32 + lane) < dp && avail[r] <= t;
                const unsigned bal = __ballot_sync(0xffffffffu, idle);
                if (win < 0 && bal) win = r * 32 + (__ffs(bal) - 1);
            }
            if (win < 0) {
                unsigned long long kw = ~0ull;
                int kj = 0x7fffffff;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int j = r * 32 + lane;
                    const unsigned long long w = (unsigned long long)__double_as_longlong(__dsub_rn(avail[r], t));
                    if (j < dp && w < kw) {
                        kw = w;
                        kj = j;
                    }
                }
                const unsigned hi = (unsigned)(kw >> 32);
                const unsigned mhi = __reduce_min_sync(0xffffffffu, hi);
                const unsigned lo = hi == mhi ? (unsigned)kw : 0xffffffffu;
                const unsigned mlo = __reduce_min_sync(0xffffffffu, lo);
                const unsigned jj = (hi == mhi && lo == mlo) ? (unsigned)kj : 0xffffffffu;
                win = (int)__reduce_min_sync(0xffffffffu, jj);
            }
            // every lane prices its own replicas (off the selection's critical
            // path); the winner keeps its finish time, the rest is broadcast
            const int wl = win & 31, wr = win >> 5;
            double wstart = 0.0, wservice = 0.0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double st_r = (t < avail[r]) ? avail[r] : t;  // std::max(ev.time, avail)
                const double sv_r = __dadd_rn(__dadd_rn(__dmul_rn(ppt[r], in), pf[r]), __dmul_rn(o, dpt[r]));
                if (r == wr) {
                    wstart = st_r;
                    wservice = sv_r;
                    if (lane == wl) avail[r] = __dadd_rn(st_r, sv_r);
                }
            }
            const double start = __shfl_sync(0xffffffffu, wstart, wl);
            const double service = __shfl_sync(0xffffffffu, wservice, wl);
            const double fin = __dadd_rn(start, service);
            if (lane == i) my_fin = fin;
            const double wait = __dsub_rn(start, t);
            if (b + i < half) w1 = __dadd_rn(w1, wait);
            else w2 = __dadd_rn(w2, wait);
            ssum = __dadd_rn(ssum, service);
        }
        // outputs of the 32 events: accepted -> per-request result, else an
        // escalation appended in processing order (ballot compaction)
        const bool valid = lane < cnt;
        const bool acc = valid && (last || bsc >= thr);
        if (acc) {
            e2e[br] = __dsub_rn(my_fin, barr);
            ast[br] = s + 1;
        }
        const bool esc = valid && !acc;
        const unsigned eb = __ballot_sync(0xffffffffu, esc);
        if (esc) {
            const long long pos = nesc + __popc(eb & ((1u << lane) - 1u));
            nk[pos] = dbl_to_key(my_fin);
            nv[pos] = (unsigned long long)br;
        }
        nesc += __popc(eb);
    }
    if (lane == 0) {
        a.nx_count[pi] = nesc;
        double* st = a.stage_stats + ((long long)pi * kSimMaxStages + s) * 4;
        st[0] = w1;
        st[1] = w2;
        st[2] = ssum;
        st[3] = (double)m;
    }
}

// Per plan: p95 over the non-warmup requests (nearest rank: radix select of
// the rank-th smallest non-negative double), last completion, attainment.
__global__ void __launch_bounds__(1024) k_sr_metrics(SimRunArgs a) {
    const int pi = blockIdx.x;
    const long long n = a.n, w0 = a.warmup, m = n - a.warmup;
    const double* e2e = a.e2e + (long long)pi * n;
    const double base = a.base[pi];
    __shared__ unsigned hist[256];
    __shared__ unsigned long long s_ok[32];
    __shared__ double s_max[32];
    __shared__ unsigned long long s_prefix, s_need;
    // last completion and attainment counts
    double mx = 0.0;  // last_completion starts at 0 (simulator.cpp:268)
    unsigned long long ok[32];
    for (int q = 0; q < a.nscales; ++q) ok[q] = 0;
    for (long long r = w0 + threadIdx.x; r < n; r += blockDim.x) {
        const double x = e2e[r];
        const double c = __dadd_rn(a.arrival[r], x);
        mx = c > mx ? c : mx;
        for (int q = 0; q < a.nscales; ++q) ok[q] += x <= __dmul_rn(a.scales[q], base) ? 1ull : 0ull;
    }
    for (int off = 16; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, mx, off);
        mx = o > mx ? o : mx;
    }
    if (threadIdx.x < 32) {
        s_max[threadIdx.x] = 0.0;
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = mx;
    __syncthreads();
    for (int q = 0; q < a.nscales; ++q) {
        unsigned long long v = ok[q];
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (threadIdx.x == 0) s_ok[0] = 0;
        __syncthreads();
        if ((threadIdx.x & 31) == 0) atomicAdd(&s_ok[0], v);
        __syncthreads();
        if (threadIdx.x == 0) a.attain_ok[(long long)pi * 32 + q] = s_ok[0];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double best = 0.0;
        for (int w = 0; w < 32; ++w) best = s_max[w] > best ? s_max[w] : best;
        a.last_completion[pi] = best;
    }
    if (m <= 0) return;
    // nearest-rank p95: rank = clamp(ceil(0.95 m), 1, m); rank-th smallest
    if (threadIdx.x == 0) {
        const long long rank = p95_index(m) + 1;
        s_need = (unsigned long long)rank;
        s_prefix = 0;
    }
    __syncthreads();
    unsigned long long pmask = 0;
    for (int byte = 7; byte >= 0; --byte) {
        const int shift = 8 * byte;
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        const unsigned long long prefix = s_prefix;
        for (long long r = w0 + threadIdx.x; r < n; r += blockDim.x) {
            const unsigned long long k = (unsigned long long)__double_as_longlong(e2e[r]);
            if ((k & pmask) == prefix) atomicAdd(&hist[(k >> shift) & 255ull], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long need = s_need, run = 0;
            int d = 0;
            for (; d < 256; ++d) {
                if (run + hist[d] >= need) break;
                run += hist[d];
            }
            s_need = need - run;
            s_prefix = prefix | ((unsigned long long)d << shift);
        }
        pmask |= 255ull << shift;
        __syncthreads();
    }
    if (threadIdx.x == 0) a.p95[pi] = __longlong_as_double((long long)s_prefix);
}

}  // namespace

void sim_run_batch(SimRunBuffers& B, cudaStream_t s, SimRunArgs a, std::vector<SimPlanDesc>& plans,
                   int max_steps, int base_mode, double cfg_base, int* launches, std::vector<SimPlanOut>& out) {
    const long long n = a.n;
    const int P = (int)plans.size();
    a.nplans = P;
    SimPlanDesc* dplans = B.plans.as<SimPlanDesc>((size_t)P);
    CG_CUDA(cudaMemcpyAsync(dplans, plans.data(), sizeof(SimPlanDesc) * P, cudaMemcpyHostToDevice, s));
    a.plans = dplans;
    // base: the configured one, each plan's dry run, or the first plan's (compare())
    double* dbase = B.base.as<double>((size_t)P);
    std::vector<double> hbase(P, cfg_base);
    if (base_mode != 0) {
        const int nb = base_mode == 2 ? 1 : P;
        double* lat = B.lat.as<double>((size_t)nb * n);
        std::vector<double> b(nb);
        for (int pi = 0; pi < nb; ++pi) {
            k_sr_dry<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, dplans + pi, lat + (long long)pi * n);
            CG_LAUNCH_CHECK();
            ++*launches;
        }
        k_sr_mean<<<nb, 1024, 0, s>>>(lat, n, dbase);
        CG_LAUNCH_CHECK();
        ++*launches;
        CG_CUDA(cudaMemcpyAsync(b.data(), dbase, 8 * nb, cudaMemcpyDeviceToHost, s));
        CG_CUDA(cudaStreamSynchronize(s));
        for (int pi = 0; pi < P; ++pi) hbase[pi] = base_mode == 2 ? b[0] : b[pi];
    }
    CG_CUDA(cudaMemcpyAsync(dbase, hbase.data(), 8 * P, cudaMemcpyHostToDevice, s));
    a.base = dbase;

    // entry events: (arrival, trace index), stable by arrival -- shared by every plan
    unsigned long long* k0 = B.k0.as<unsigned long long>((size_t)n);
    unsigned long long* v0 = B.v0.as<unsigned long long>((size_t)n);
    unsigned long long* k1 = B.k1.as<unsigned long long>((size_t)n);
    unsigned long long* v1 = B.v1.as<unsigned long long>((size_t)n);
    unsigned int* rsh = B.rsh.as<unsigned int>(radix_hist_entries(n));
    k_sr_keys<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a.arrival, n, k0, v0);
    CG_LAUNCH_CHECK();
    ++*launches;
    const int par0 = radix_sort_u64(k0, v0, k1, v1, n, ~0ull, rsh, s, launches);
    unsigned long long* sk = par0 ? k1 : k0;
    unsigned long long* sv = par0 ? v1 : v0;
    // per-plan event lists (current / next) and outputs
    a.ev_keys = B.ek.as<unsigned long long>((size_t)P * n);
    a.ev_vals = B.ev.as<unsigned long long>((size_t)P * n);
    a.nx_keys = B.nk.as<unsigned long long>((size_t)P * n);
    a.nx_vals = B.nv.as<unsigned long long>((size_t)P * n);
    a.ev_count = B.ec.as<long long>((size_t)P);
    a.nx_count = B.nc.as<long long>((size_t)P);
    a.e2e = B.e2e.as<double>((size_t)P * n);
    a.astage = B.ast.as<int>((size_t)P * n);
    a.stage_stats = B.stats.as<double>((size_t)P * kSimMaxStages * 4);
    CG_CUDA(cudaMemsetAsync(a.stage_stats, 0, sizeof(double) * P * kSimMaxStages * 4, s));
    CG_CUDA(cudaMemsetAsync(a.e2e, 0, sizeof(double) * P * n, s));
    CG_CUDA(cudaMemsetAsync(a.astage, 0, sizeof(int) * P * n, s));
    std::vector<long long> cnt(P, n);
    for (int pi = 0; pi < P; ++pi) {
        CG_CUDA(cudaMemcpyAsync(a.ev_keys + (long long)pi * n, sk, 8 * n, cudaMemcpyDeviceToDevice, s));
        CG_CUDA(cudaMemcpyAsync(a.ev_vals + (long long)pi * n, sv, 8 * n, cudaMemcpyDeviceToDevice, s));
    }
    int maxR = 1;
    for (const auto& p : plans)
        for (int st = 0; st < p.C; ++st) maxR = std::max(maxR, (p.dp[st] + 31) / 32);
    for (int step = 0; step < max_steps; ++step) {
        CG_CUDA(cudaMemcpyAsync(a.ev_count, cnt.data(), 8 * P, cudaMemcpyHostToDevice, s));
        const unsigned grid = (unsigned)((P + SR_WARPS - 1) / SR_WARPS);
        if (maxR <= 1) k_sr_stage<1><<<grid, 32 * SR_WARPS, 0, s>>>(a, step);
        else if (maxR <= 2) k_sr_stage<2><<<grid, 32 * SR_WARPS, 0, s>>>(a, step);
        else if (maxR <= 4) k_sr_stage<4><<<grid, 32 * SR_WARPS, 0, s>>>(a, step);
        else k_sr_stage<8><<<grid, 32 * SR_WARPS, 0, s>>>(a, step);
        CG_LAUNCH_CHECK();
        ++*launches;
        std::vector<long long> nxt(P, 0);
        CG_CUDA(cudaMemcpyAsync(nxt.data(), a.nx_count, 8 * P, cudaMemcpyDeviceToHost, s));
        CG_CUDA(cudaStreamSynchronize(s));
        bool more = false;
        for (int pi = 0; pi < P; ++pi) {
            const bool active = plans[pi].chain[step] >= 0;
            cnt[pi] = active ? nxt[pi] : 0;
            if (step + 1 < max_steps && plans[pi].chain[step + 1] >= 0 && cnt[pi] > 0) {
                // stable sort of the escalations by finish time -> next stage's order
                unsigned long long* kk = a.nx_keys + (long long)pi * n;
                unsigned long long* vv = a.nx_vals + (long long)pi * n;
                const int par = radix_sort_u64(kk, vv, k1, v1, cnt[pi], ~0ull, rsh, s, launches);
                CG_CUDA(cudaMemcpyAsync(a.ev_keys + (long long)pi * n, par ? k1 : kk, 8 * cnt[pi],
                                        cudaMemcpyDeviceToDevice, s));
                CG_CUDA(cudaMemcpyAsync(a.ev_vals + (long long)pi * n, par ? v1 : vv, 8 * cnt[pi],
                                        cudaMemcpyDeviceToDevice, s));
                more = true;
            } else {
                cnt[pi] = 0;
            }
        }
        if (!more) break;
    }
    // metrics
    a.p95 = B.p95.as<double>((size_t)P);
    a.last_completion = B.lastc.as<double>((size_t)P);
    a.attain_ok = B.ok.as<unsigned long long>((size_t)P * 32);
    CG_CUDA(cudaMemsetAsync(a.p95, 0, 8 * P, s));
    k_sr_metrics<<<P, 1024, 0, s>>>(a);
    CG_LAUNCH_CHECK();
    ++*launches;
    out.assign(P, SimPlanOut{});
    std::vector<double> p95(P), lastc(P), stats((size_t)P * kSimMaxStages * 4);
    std::vector<unsigned long long> ok((size_t)P * 32);
    CG_CUDA(cudaMemcpyAsync(p95.data(), a.p95, 8 * P, cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaMemcpyAsync(lastc.data(), a.last_completion, 8 * P, cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaMemcpyAsync(ok.data(), a.attain_ok, 8 * ok.size(), cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaMemcpyAsync(stats.data(), a.stage_stats, 8 * stats.size(), cudaMemcpyDeviceToHost, s));
    for (int pi = 0; pi < P; ++pi) {
        SimPlanOut& o = out[pi];
        o.e2e.resize((size_t)n);
        o.stage.resize((size_t)n);
        CG_CUDA(cudaMemcpyAsync(o.e2e.data(), a.e2e + (long long)pi * n, 8 * n, cudaMemcpyDeviceToHost, s));
        CG_CUDA(cudaMemcpyAsync(o.stage.data(), a.astage + (long long)pi * n, 4 * n, cudaMemcpyDeviceToHost, s));
    }
    CG_CUDA(cudaStreamSynchronize(s));
    for (int pi = 0; pi < P; ++pi) {
        SimPlanOut& o = out[pi];
        o.base = hbase[pi];
        o.p95 = p95[pi];
        o.last_completion = lastc[pi];
        o.ok.assign(ok.begin() + (long long)pi * 32, ok.begin() + (long long)pi * 32 + a.nscales);
        for (int st = 0; st < kSimMaxStages; ++st) {
            const double* q = &stats[((size_t)pi * kSimMaxStages + st) * 4];
            o.w1[st] = q[0];
            o.w2[st] = q[1];
            o.service_sum[st] = q[2];
            o.served[st] = (long long)q[3];
        }
    }
}

}  // namespace cg
