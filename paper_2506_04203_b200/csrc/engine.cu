// Host orchestration of the plan-search engine behind the C ABI
// (include/cascade_gpu.h).  Mirrors cascade::outerplan::sweep
// (proj/src/outerplan.cpp:166-319) phase by phase:
//
//   validation (same order and messages as the reference)
//   -> trace to HBM -> threshold grid (explicit, or default deciles on GPU)
//   -> K1-K3 routing of every (stage, threshold-prefix) workload at once
//   -> K2 trace-order quality of every distinct threshold tuple
//   -> workload validation in candidate order + row-cache dedup (host, exact bits)
//   -> K4-K5 latency rows for every unique workload (sharded over ranks,
//      merged with one all-gather)
//   -> utopia check -> K6 min-max solve per tuple -> grid-order expansion
//   -> K7 Tchebycheff argmin per weight, Pareto front -> SweepResult.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <future>
#include <mutex>
#include <thread>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <string>
#include <unordered_map>
#include <vector>

#include "cascade_gpu.h"
#include "cg_cuda.h"
#include "cg_ingest.h"
#include "cg_drift.h"
#include "cg_json.h"
#include "cg_simrun.h"
#include "cg_internal.h"
#include "cg_kernels.h"
#include "host_model.h"
#include "plan_dev.cuh"

using namespace cg;

namespace {

constexpr unsigned long long kInfBits = 0x7ff0000000000000ull;
constexpr double kThresholdSentinel = 101.0;  // domain.hpp:21

double dinf() { return std::numeric_limits<double>::infinity(); }

cg_status ok_status() {
    cg_status s;
    s.code = CG_OK;
    s.message[0] = 0;
    return s;
}

cg_status err_status(int code, const std::string& msg) {
    cg_status s;
    s.code = code;
    std::snprintf(s.message, sizeof(s.message), "%s", msg.c_str());
    return s;
}

template <class F>
cg_status guarded(F&& f) {
    try {
        f();
        return ok_status();
    } catch (const EngineError& e) {
        return err_status(e.code, e.what());
    } catch (const std::bad_alloc&) {
        return err_status(CG_ERR_CUDA, "host allocation failed");
    } catch (const std::exception& e) {
        return err_status(CG_ERR_CUDA, e.what());
    }
}

struct Timer {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    double ms() const {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
};

__global__ void k_iota_u64(unsigned long long* p, long long n) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) p[i] = (unsigned long long)i;
}

// Work list in sorted order: out[i] = in[perm[i]] (so a plan claim is one dependent load, not two).
__global__ void k_gather_recs(const unsigned long long* __restrict__ perm, long long n,
                              const ItemRec* __restrict__ in, ItemRec* __restrict__ out) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = in[perm[i]];
}


__global__ void k_fill_u64(unsigned long long* p, long long n, unsigned long long v) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

__global__ void k_score_keys(const double* __restrict__ s, long long n, unsigned long long* __restrict__ k) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) k[i] = dbl_to_key(s[i]);
}

// route_trace accept stage (routing.cpp:65-81), 1-based
__global__ void k_accept_stage(const double* __restrict__ scores, long long n, int C,
                               const double* __restrict__ h, int last, const int* __restrict__ deployed,
                               int* __restrict__ out) {
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= n) return;
    int acc = last;
    for (int i = 0; i < C; ++i) {
        if (!deployed[i]) continue;
        if (i == last) break;
        if (scores[(long long)i * n + r] >= h[i]) {
            acc = i;
            break;
        }
    }
    out[r] = acc + 1;
}

// Bound exchange: ub = min over the gathered ranks' bounds (bit patterns of
// non-negative doubles order like the values).
__global__ void k_min_ranks(const unsigned long long* __restrict__ gathered, int world, long long cells,
                            unsigned long long* __restrict__ ub) {
    const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (c >= cells) return;
    unsigned long long m = gathered[c];
    for (int r = 1; r < world; ++r) m = min(m, gathered[(long long)r * cells + c]);
    ub[c] = m;
}

unsigned long long shard_count(unsigned long long total, int rank, int world) {
    return total > (unsigned long long)rank ? (total - rank + world - 1) / world : 0ull;
}

// Cross-rank merge of per-budget bests: minimum latency; equal latency ->
// parts-lexicographic minimum plan (the reference's `better`, costmodel.cpp:347-352).
// Gathered layout: rank r occupies [r*2*cells, (r+1)*2*cells): lat bits, then plan.
__global__ void k_merge_ranks(const unsigned long long* __restrict__ gathered, int world, long long cells,
                              int N, const RowDesc* __restrict__ rows, const PlanSpace* __restrict__ spaces,
                              unsigned long long* __restrict__ lat_out, unsigned long long* __restrict__ plan_out) {
    const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (c >= cells) return;
    const int row = (int)(c / (N + 1));
    const PlanSpace& sp = spaces[rows[row].space];
    unsigned long long bl = kInfBits, bp = ~0ull;
    for (int r = 0; r < world; ++r) {
        const unsigned long long l = gathered[(long long)r * 2 * cells + c];
        const unsigned long long p = gathered[(long long)r * 2 * cells + cells + c];
        if (merge_take(sp, l, p, bl, bp)) {
            bl = l;
            bp = p;
        }
    }
    lat_out[c] = bl;
    plan_out[c] = bp;
}

}  // namespace

// ---------------------------------------------------------------------------

struct cg_engine {
    int device = 0;
    int sm_count = 148;
    cudaStream_t s = nullptr;
    cudaStream_t s2 = nullptr;  // second stream: the concurrent pilot launch
    cudaStream_t s3 = nullptr, s4 = nullptr;  // with s and s2: concurrent class lists of small waves
    int rank = 0, world = 1;
    cg_allgather_fn allgather = nullptr;
    void* ag_user = nullptr;
    // NCCL member (cg_engine_create_multi / cg_engine_set_nccl): the sharded
    // path runs even at world 1, so one device exercises the collective
    bool nccl_member = false;
    void* nccl_comm = nullptr;   // ncclComm_t owned by this engine
    struct MultiGroup* group = nullptr;  // a multi-device engine: its per-device members
    bool collective() const { return allgather && (world > 1 || nccl_member); }
    int prune = 1;
    int ub_oracle = 0;   // diagnostic: seed K4's bounds with the previous identical sweep's rows
    std::vector<unsigned long long> ub_saved;
    int fut_bound = 1;  // future-service bound in K4 (option fut_bound)
    int fut_block = 1;  // output-rank block of the future bound (option fut_block; 1 = exact counts)
    int fut_arrival_shift = 5;  // log2 arrival block of the future bound (option fut_arrival: 1, 2, 4, ..., 32)
    int lane_check = 32;  // k_lane request-steps between prune checks (option lane_check: 32, 64)
    int pilot = 1;      // pilot plans per (row, budget) cell before the lists (option pilot: 1 auto, 2 on, 0 off)
    int seeds = 1;      // homogeneous seed plans of the heavy rows first (option seeds)
    long long pilot_min_plans = 0;  // rows with fewer plans get no pilot (option pilot_min_plans)
    int pilot_merge = 1;            // pilot launches: see PilotArgs::merge (option pilot_merge)
    int pilot_sort = 1;             // pilot lists in ascending estimate order (option pilot_sort)
    int sort_key = 3;   // list/pilot order (option sort_key): 0 service bound, else an estimate (k_plan_filter)
    int class_order = 1;  // 0: lists by replica count descending, 1: ascending (option class_order)
    long long conc_lists_max = 1 << 16;  // waves with at most this many listed plans run classes concurrently
    int wave_plans = 256;  // plans per filter wave, in units of 2^20 (option wave_plans; <= 60% of free HBM)
    int k4_pack = 3;  // lane packing of the JSQ kernel classes (see class_shape; 3 = lane-major k_lane)
    int quality_form = 1;  // K2: 1 block-parallel exact (binade units), 0 one fp64 chain per tuple
    int quality_block = 0; // K2: minimum requests per block (diagnostic; 0 = automatic)
    int p95_tables = 1;    // K3: chunk tables for large traces (0: the direct column scan)
    long long max_waves = 0;   // rate sampling: stop after this many filter waves (0 = all; result partial)
    long long wave_stride = 1; // rate sampling: run every wave_stride-th wave only (result partial)
    int k1_form = 0;   // 0 auto (TMA ring), 1 tiled/u64 forms only, 2 u32 register form (3: 1 block/SM)
    int item_plans = 128;
    long long ovf_cap = 1 << 20;
    long long tie_cap = 1 << 22;
    cudaEvent_t ev[16];

    DevBuf d_scores, d_in, d_out;
    DevBuf d_gvals, d_ranks, d_hist, d_flags, d_lk0, d_lv0, d_lk1, d_lv1, d_rshist, d_orax;
    DevBuf d_p95tab;
    DevBuf d_wcount, d_wsin, d_wsout, d_wsinf, d_wsoutf, d_wp95i, d_wp95o, d_wstats, d_thr, d_qsum, d_qa, d_qe, d_qu, d_qseq;
    DevBuf d_rows, d_spaces, d_ways, d_models, d_ok, d_pre, d_dec, d_ms, d_ims, d_svck, d_T, d_O, d_crn;
    DevBuf d_latmin, d_ub, d_ties, d_tiecnt, d_ovf, d_ovfcnt, d_ovfcnt2, d_rowids, d_iprefix, d_ictr,
        d_scratch, d_ring, d_seeds, d_partials, d_lists, d_lkeys, d_lcount, d_tpart, d_ctrs, d_best, d_flat, d_fplan, d_gather, d_send;
    DevBuf d_wlrow, d_tfeas, d_tL, d_talloc, d_tplan, d_g2d, d_ctuple, d_cflag, d_pos, d_total, d_ecand,
        d_eL, d_eQ, d_skip, d_weights, d_sel, d_pk0, d_pk1, d_pv0, d_pv1, d_pkl, d_front, d_fsize, d_misc, d_dep, d_accept, d_acc, d_part32, d_hiacc, d_lrecs, d_grecs, d_qtab, d_pilot, d_plists, d_pkeys, d_pperm, d_cperm, d_ptk, d_ptv, d_prsh, d_pcount, d_lidx, d_probe, d_fut, d_pv;
    IngestBuffers ingest;
    JsonBuffers jsonbuf;
    SimRunBuffers simbuf;
    DriftBuffers driftbuf;
};

// A multi-device engine (cg_engine_create_multi): one member engine per
// device, rank r = members[r], each holding its communicator of one NCCL
// clique.  Sharded calls (cg_sweep, cg_stage_row) run every member on its
// own host thread; the rest go to members[0].
struct MultiGroup {
    std::vector<cg_engine*> members;
    std::atomic<bool> broken{false};  // a member failed inside a collective: communicators aborted
};

namespace {
cg_engine* primary(cg_engine* e) { return e && e->group ? e->group->members[0] : e; }
}  // namespace

namespace {

struct SweepCtx {
    cg_engine& E;
    cudaStream_t s;
    int launches = 0;
    cg_sweep_stats st{};
    explicit SweepCtx(cg_engine& e) : E(e), s(e.s) {}

    void d2h(void* dst, const void* src, size_t bytes) {
        if (!bytes) return;
        CG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
        st.d2h_bytes += (long long)bytes;
    }
    void h2d(void* dst, const void* src, size_t bytes) {
        if (!bytes) return;
        CG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        st.h2d_bytes += (long long)bytes;
    }
    void sync() { CG_CUDA(cudaStreamSynchronize(s)); }
    void fill(unsigned long long* p, long long n, unsigned long long v) {
        if (n <= 0) return;
        k_fill_u64<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, n, v);
        CG_LAUNCH_CHECK();
        ++launches;
    }
};

// Plan spaces of every model at budget N (host tables, uploaded).
std::vector<HostPlanSpace> build_spaces(SweepCtx& x, const cg_model* models, int C, const cg_hardware& hw,
                                        const cg_cost_params& q, int N) {
    std::vector<HostPlanSpace> hs(C);
    std::vector<PlanSpace> dsp(C);
    size_t ways_total = 0;
    for (int i = 0; i < C; ++i) {
        auto shapes = legal_shapes(models[i], hw, q);
        if ((int)shapes.size() > kMaxShapes) fail(CG_ERR_UNSUPPORTED, "too many replica shapes");
        hs[i].build(std::move(shapes), N);
        ways_total += hs[i].ways.size();
    }
    unsigned long long* dways = x.E.d_ways.as<unsigned long long>(ways_total);
    size_t off = 0;
    for (int i = 0; i < C; ++i) {
        PlanSpace& p = dsp[i];
        std::memset(&p, 0, sizeof(p));
        p.S = (int)hs[i].shapes.size();
        p.N = hs[i].N;
        for (int k = 0; k < p.S; ++k) p.shapes[k] = hs[i].shapes[k];
        p.ways = dways + off;
        p.num_plans = hs[i].num_plans;
        x.h2d(dways + off, hs[i].ways.data(), hs[i].ways.size() * sizeof(unsigned long long));
        off += hs[i].ways.size();
    }
    x.h2d(x.E.d_spaces.as<PlanSpace>(C), dsp.data(), sizeof(PlanSpace) * C);
    std::vector<ModelArgs> ma(C);
    for (int i = 0; i < C; ++i)
        ma[i] = {models[i].param_count, models[i].bytes_per_param, models[i].kv_bytes_per_token};
    x.h2d(x.E.d_models.as<ModelArgs>(C), ma.data(), sizeof(ModelArgs) * C);
    return hs;
}

int row_class(const HostPlanSpace& sp, int N) {
    if (sp.min_gpus <= 0 || N < 1) return 3;
    const int dpmax = N / sp.min_gpus;
    const int cls = class_for_dp(dpmax);
    if (cls < 0) fail(CG_ERR_UNSUPPORTED, "plans with more than 255 replicas are not supported");
    if (sp.num_plans > kItemPlanMask)  // work items pack (row << 44) | plan
        fail(CG_ERR_UNSUPPORTED, "plan space too large for 44-bit plan indices");
    return cls;
}

// K4-K5 for a set of unique rows.  Afterwards E.d_flat / E.d_fplan hold the
// final [row][N+1] latency / plan index (merged across ranks).
void evaluate_rows(SweepCtx& x, const std::vector<RowDesc>& rows, const std::vector<HostPlanSpace>& hs,
                   const cg_hardware& hw, const cg_cost_params& q, int N) {
    cg_engine& E = x.E;
    set_k4_pack(E.k4_pack >= 3 && q.queueing_sim_requests > 65535 ? 1 : E.k4_pack);  // k_lane rings hold u16 request indices
    const int nrows = (int)rows.size();
    if (rows.size() >= (1ull << (64 - kItemPlanBits)))
        fail(CG_ERR_UNSUPPORTED, "too many unique rows for the 20-bit row field of a work item");
    {
        std::vector<char> seen(hs.size(), 0);  // replica-count and plan-index limits of every live space
        for (const auto& rd : rows)
            if (!seen[rd.space]) {
                seen[rd.space] = 1;
                row_class(hs[rd.space], N);
            }
    }
    const long long cells = (long long)nrows * (N + 1);
    const int n_req = q.queueing_sim_requests;
    if (nrows == 0) return;
    x.h2d(E.d_rows.as<RowDesc>(nrows), rows.data(), sizeof(RowDesc) * nrows);

    RowTables tab;
    tab.shape_ok = E.d_ok.as<unsigned char>((size_t)nrows * kMaxShapes);
    tab.prefill = E.d_pre.as<double>((size_t)nrows * kMaxShapes);
    tab.decode = E.d_dec.as<double>((size_t)nrows * kMaxShapes);
    tab.mean_service = E.d_ms.as<double>((size_t)nrows * kMaxShapes);
    tab.inv_service = E.d_ims.as<double>((size_t)nrows * kMaxShapes);
    tab.svc_k = E.d_svck.as<double>((size_t)nrows * kMaxShapes);
    tab.ld = (n_req + 3) & ~3;
    const std::vector<double> L = crn_log1p_table(q.queueing_sim_seed, n_req);  // glibc log1p (H3), once
    {
        // future-service bound tables (RowTables): requests ranked by output,
        // largest first (outputs are monotone in -L[2k+1], ties by index)
        std::vector<int> desc(n_req), pos(n_req);
        for (int k = 0; k < n_req; ++k) desc[k] = k;
        std::stable_sort(desc.begin(), desc.end(), [&](int a, int b) { return L[2 * a + 1] < L[2 * b + 1]; });
        for (int k = 0; k < n_req; ++k) pos[desc[k]] = k;
        // output ranks in blocks of RB requests (option fut_block; 1 = exact
        // counts), arrivals in blocks of 32 (the prune checks' granularity)
        const int RB = E.fut_block;
        const int nc = (n_req + RB - 1) / RB;
        const int AB = 1 << E.fut_arrival_shift;  // arrival block (option fut_arrival: 1 = exact step)
        const int na = (n_req + AB - 1) / AB;
        std::vector<int> probe(nc);
        for (int i = 0; i < nc; ++i) probe[i] = desc[std::min(RB * i + RB - 1, n_req - 1)];
        // fut[c][i] = #requests j >= 32c whose output rank block pos[j]/RB <= i,
        // built backwards: fut[c] = fut[c+1] + the prefix histogram of block c
        std::vector<unsigned> fut;
        if (E.fut_bound) {
            fut.assign((size_t)(na + 1) * nc, 0u);
            std::vector<unsigned> h(nc);
            for (int c = na - 1; c >= 0; --c) {
                std::fill(h.begin(), h.end(), 0u);
                for (int j = AB * c; j < std::min(AB * c + AB, n_req); ++j) ++h[pos[j] / RB];
                unsigned run = 0;
                for (int i = 0; i < nc; ++i) {
                    run += h[i];
                    fut[(size_t)c * nc + i] = fut[(size_t)(c + 1) * nc + i] + run;
                }
            }
        } else {
            fut.assign(1, 0u);
        }
        int* dprobe = E.d_probe.as<int>((size_t)nc);
        unsigned* dfut = E.d_fut.as<unsigned>(fut.size());
        x.h2d(dprobe, probe.data(), probe.size() * sizeof(int));
        x.h2d(dfut, fut.data(), fut.size() * sizeof(unsigned));
        tab.nc = E.fut_bound ? nc : 0;
        tab.probe_req = dprobe;
        tab.fut_ab = AB;
        tab.fut_sh = E.fut_arrival_shift;
        tab.fut = dfut;
        tab.Pv = E.d_pv.as<double>((size_t)nrows * nc);
    }
    tab.T = E.d_T.as<double>((size_t)nrows * tab.ld);
    tab.O = E.d_O.as<double>((size_t)nrows * tab.ld);
    CG_CUDA(cudaMemsetAsync(tab.T, 0, (size_t)nrows * tab.ld * 8, x.s));
    CG_CUDA(cudaMemsetAsync(tab.O, 0, (size_t)nrows * tab.ld * 8, x.s));
    {
        double* dL = E.d_crn.as<double>(L.size());
        x.h2d(dL, L.data(), L.size() * sizeof(double));
        RowSetupArgs ra;
        ra.nrows = nrows;
        ra.n_req = n_req;
        ra.rows = static_cast<RowDesc*>(E.d_rows.p);
        ra.spaces = static_cast<PlanSpace*>(E.d_spaces.p);
        ra.models = static_cast<ModelArgs*>(E.d_models.p);
        ra.hw = {hw.flops_per_gpu, hw.mem_bandwidth_per_gpu, hw.mem_capacity_per_gpu};
        ra.p = {q.prefill_efficiency, q.decode_bw_efficiency, q.pipeline_bubble_factor,
                q.comm_overhead_per_stage, q.kv_memory_fraction};
        ra.tab = tab;
        launch_row_setup(ra, dL, x.s, &x.launches);
    }

    unsigned long long* latmin = E.d_latmin.as<unsigned long long>(cells);
    unsigned long long* ub = E.d_ub.as<unsigned long long>(cells);
    x.fill(latmin, cells, kInfBits);
    x.fill(ub, cells, kInfBits);
    if (E.ub_oracle && E.ub_saved.size() == (size_t)cells)
        x.h2d(ub, E.ub_saved.data(), (size_t)cells * 8);  // diagnostic: the exact final bounds
    TieEntry* ties = E.d_ties.as<TieEntry>(E.tie_cap);
    unsigned long long* tiecnt = E.d_tiecnt.as<unsigned long long>(1);
    unsigned long long* ovf = E.d_ovf.as<unsigned long long>(E.ovf_cap);
    // ring overflows are collected per replica-count class (slot 7: seeds,
    // whose overflows are dropped -- the lists re-visit them) over all waves
    // and re-run once at the end with global-memory rings
    const unsigned long long ovf_region = (unsigned long long)E.ovf_cap / 8;
    unsigned long long* ovfcnt = E.d_ovfcnt.as<unsigned long long>(8);
    CG_CUDA(cudaMemsetAsync(ovfcnt, 0, 8 * 8, x.s));
    unsigned long long* ovfcnt2 = E.d_ovfcnt2.as<unsigned long long>(1);
    unsigned long long* ctrs = E.d_ctrs.as<unsigned long long>(CTR_COUNT);
    unsigned long long* ictr = E.d_ictr.as<unsigned long long>(4);  // one per concurrent launch region
    CG_CUDA(cudaMemsetAsync(tiecnt, 0, 8, x.s));
    CG_CUDA(cudaMemsetAsync(ctrs, 0, 8 * CTR_COUNT, x.s));

    const int K = n_req - (int)p95_index(n_req);
    // index of the K-th largest CRN output: outputs are monotone in -L[2k+1]
    int kstar = 0;
    {
        std::vector<int> idx(n_req);
        for (int k = 0; k < n_req; ++k) idx[k] = k;
        std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return L[2 * a + 1] < L[2 * b + 1]; });
        kstar = idx[K - 1];
    }
    launch_row_svck(tab, nrows, kstar, x.s, &x.launches);
    // rows with a non-empty plan space
    std::vector<int> prow;
    std::vector<unsigned long long> chunk_prefix(1, 0);
    const int chunk = 64;
    for (int r = 0; r < nrows; ++r) {
        const auto& sp = hs[rows[r].space];
        x.st.plans_enumerated += (long long)sp.num_plans;
        if (sp.num_plans == 0 || N < 1) continue;
        prow.push_back(r);
        chunk_prefix.push_back(chunk_prefix.back() + (sp.num_plans + chunk - 1) / chunk);
    }
    long long max_slots = 1;
    for (int cls = 0; cls < 7; ++cls) {
        max_slots = std::max(max_slots, sim_geometry(cls, SIM_LIST, E.sm_count).slots);
        max_slots = std::max(max_slots, sim_geometry(cls, SIM_DEEP, E.sm_count).slots);
    }
    const int sld = (n_req + 3) & ~3;  // 32-byte scratch columns
    // scratch regions for concurrent launches: the pilot's two, or up to four
    // class lists of a small wave
    const int nregions = E.conc_lists_max > 0 ? 4 : 2;
    double* scratch = E.d_scratch.as<double>((size_t)nregions * max_slots * sld);
    int ring_cap = 1;
    while (ring_cap < n_req) ring_cap <<= 1;

    SimArgs base{};
    base.N = N;
    base.n_req = n_req;
    base.K = K;
    base.kstar = kstar;
    base.prune = E.prune;
    base.item_counter = ictr;
    base.rows = static_cast<RowDesc*>(E.d_rows.p);
    base.spaces = static_cast<PlanSpace*>(E.d_spaces.p);
    base.tab = tab;
    base.lat_min = latmin;
    base.ub = ub;
    base.ties = ties;
    base.tie_count = tiecnt;
    base.tie_cap = (unsigned long long)E.tie_cap;
    base.ovf = ovf;
    base.ovf_count = ovfcnt;
    base.ovf_cap = ovf_region;
    base.scratch = scratch;
    base.sld = sld;
    base.counters = ctrs;
    base.ring_cap = ring_cap;
    base.lane_check = (unsigned)std::max(0, E.lane_check / kLaneUnroll - 1);  // k_lane runs kLaneUnroll request-steps per trip

    // Runs one packed work list through the class kernel; ring overflows are
    // appended to the class's overflow region.
    // future-bound snapshot of the live bounds, refreshed before every list launch
    unsigned short* qtab = E.d_qtab.as<unsigned short>((size_t)cells * kMaxShapes);
    base.qtab = (E.prune && tab.nc > 0) ? qtab : nullptr;
    auto snapshot = [&](cudaStream_t st) {
        if (!base.qtab) return;
        FutSnapArgs fs{};
        fs.nrows = nrows;
        fs.N = N;
        fs.n_req = n_req;
        fs.rows = base.rows;
        fs.spaces = base.spaces;
        fs.tab = tab;
        fs.ub = ub;
        fs.qtab = qtab;
        launch_fut_snapshot(fs, st, &x.launches);
    };
    auto run_list_on = [&](const unsigned long long* items, const ItemRec* recs, unsigned long long nitems,
                           int cls, bool seeds, const unsigned long long* perm, cudaStream_t st, int region) {
        if (nitems == 0) return;
        CG_CUDA(cudaMemsetAsync(ictr + region, 0, 8, st));
        snapshot(st);
        SimArgs a = base;
        a.item_counter = ictr + region;
        a.scratch = scratch + (size_t)region * max_slots * sld;
        a.items = items;
        a.recs = recs;
        a.perm = perm;
        a.nitems = nitems;
        a.check_stable = seeds ? 1 : 0;
        a.seeds = seeds ? 1 : 0;
        const int slot = seeds ? 7 : cls;
        a.ovf = ovf + (size_t)slot * ovf_region;
        a.ovf_count = ovfcnt + slot;
        launch_sim(a, cls, SIM_LIST, E.sm_count, st, &x.launches, nullptr);
    };
    auto run_list = [&](const unsigned long long* items, const ItemRec* recs, unsigned long long nitems, int cls,
                        bool seeds, const unsigned long long* perm) {
        run_list_on(items, recs, nitems, cls, seeds, perm, x.s, 0);
    };
    // Deep-queue re-runs (rings in global memory, capacity >= n_req) of every
    // overflowed plan, one launch per class.
    auto run_overflows = [&]() {
        unsigned long long novf[8];
        x.d2h(novf, ovfcnt, sizeof(novf));
        x.sync();
        // one launch per class; the classes' launches are independent (own
        // item counter, scratch region and rings), so they run concurrently on
        // the engine's streams -- each is a few hundred plans with full request
        // chains, latency-bound on its own
        // each launch is sized to its overflow count (one plan per group of
        // W lanes): the global rings are 16 KB per lane-replica slot
        size_t ring_each = 0;
        int sms[7] = {0, 0, 0, 0, 0, 0, 0};
        for (int cls = 0; cls < 7; ++cls) {
            if (novf[cls] == 0) continue;
            if (novf[cls] > ovf_region) fail(CG_ERR_CUDA, "JSQ overflow list exhausted");
            x.st.plans_overflow += (long long)novf[cls];
            SimGeometry gd = sim_geometry(cls, SIM_DEEP, E.sm_count);
            const long long per_sm_groups = std::max<long long>(1, gd.warps * gd.G / E.sm_count);
            sms[cls] = (int)std::min<long long>(E.sm_count, ((long long)novf[cls] + per_sm_groups - 1) / per_sm_groups);
            const long long warps = gd.warps / E.sm_count * sms[cls];
            ring_each = std::max(ring_each, (size_t)warps * 32 * gd.R * ring_cap);
        }
        if (ring_each == 0) return;
        double* ring = E.d_ring.as<double>(ring_each * nregions);
        unsigned long long* oc2 = E.d_ovfcnt2.as<unsigned long long>((size_t)nregions);
        cudaStream_t streams[4] = {x.s, E.s2, E.s3, E.s4};
        CG_CUDA(cudaEventRecord(E.ev[12], x.s));
        int launched = 0;
        for (int cls = 0; cls < 7; ++cls) {
            if (novf[cls] == 0) continue;
            const int k = launched++ % nregions;
            cudaStream_t st = streams[k];
            if (k > 0 && launched <= nregions) CG_CUDA(cudaStreamWaitEvent(st, E.ev[12], 0));
            CG_CUDA(cudaMemsetAsync(ictr + k, 0, 8, st));
            CG_CUDA(cudaMemsetAsync(oc2 + k, 0, 8, st));
            SimArgs d = base;
            d.items = ovf + (size_t)cls * ovf_region;
            d.recs = nullptr;
            d.perm = nullptr;
            d.nitems = novf[cls];
            d.item_counter = ictr + k;
            d.scratch = scratch + (size_t)k * max_slots * sld;
            d.ring_global = ring + (size_t)k * ring_each;
            d.ovf = ovf + (size_t)7 * ovf_region;  // cannot overflow (capacity >= n_req)
            d.ovf_count = oc2 + k;
            launch_sim(d, cls, SIM_DEEP, sms[cls], st, &x.launches, nullptr);
        }
        for (int k = 1; k < nregions && k < launched; ++k) {
            CG_CUDA(cudaEventRecord(E.ev[12 + k], streams[k]));
            CG_CUDA(cudaStreamWaitEvent(x.s, E.ev[12 + k], 0));
        }
    };

    CG_CUDA(cudaEventRecord(E.ev[8], x.s));
    // Bound seeding: homogeneous plans (c replicas of one shape) of the heavy
    // rows first, so the exact bounds are tight from the start.  Seeds are
    // re-visited by the filtered lists (idempotent), so this only moves work.
    // With the pilot pass on, the seeds run in the pilot launch instead.
    std::vector<unsigned long long> seeds;
    // this rank's chunks: global chunk g belongs to rank g mod world (local
    // chunk l = global l*world + rank); every rank runs the same number of
    // waves (the largest share's), so the per-wave bound exchanges pair up
    const unsigned long long my_chunks = shard_count(chunk_prefix.back(), E.rank, E.world);
    const unsigned long long max_chunks = shard_count(chunk_prefix.back(), 0, E.world);
    // wave capacity: wave_plans, never more than this rank's plans, and the
    // class lists of a wave within 60% of the free device memory
    unsigned long long wave_chunks = std::max<unsigned long long>(
        1, std::min<unsigned long long>(((unsigned long long)E.wave_plans << 20) / chunk, max_chunks));
    // per-class list capacity: one wave, but never more plans than the sweep's
    // rows hold in that replica-count class (a host census of the plan spaces)
    unsigned long long class_total[7] = {0, 0, 0, 0, 0, 0, 0};
    {
        std::vector<std::array<unsigned long long, 7>> per_space(hs.size());
        std::vector<char> done(hs.size(), 0);
        for (int r : prow) {
            const int sp = rows[r].space;
            if (!done[sp]) {
                hs[sp].class_counts(per_space[sp].data());
                done[sp] = 1;
            }
            for (int c = 0; c < 7; ++c) class_total[c] += per_space[sp][c];
        }
    }
    unsigned long long ccap[7], coff[8], cmax = 1;
    auto size_lists = [&]() {
        coff[0] = 0;
        cmax = 1;
        for (int c = 0; c < 7; ++c) {
            ccap[c] = std::min<unsigned long long>(wave_chunks * chunk, class_total[c]);
            coff[c + 1] = coff[c] + ccap[c];
            cmax = std::max(cmax, ccap[c]);
        }
        // recs + keys per listed slot; sort / gather temporaries per class
        return (double)coff[7] * (sizeof(ItemRec) + 8) + (double)cmax * (sizeof(ItemRec) + 40);
    };
    {
        // the list buffers this engine already holds are reused, so they count
        // as available: the wave size does not depend on earlier sweeps
        size_t fr = 0, tot = 0;
        const double held = (double)(E.d_lrecs.bytes + E.d_lkeys.bytes + E.d_lidx.bytes + E.d_lk1.bytes +
                                     E.d_lv1.bytes + E.d_grecs.bytes);
        const double budget = cudaMemGetInfo(&fr, &tot) == cudaSuccess ? 0.6 * ((double)fr + held) : 64e9;
        while (size_lists() > budget && wave_chunks > 1) wave_chunks = (wave_chunks + 1) / 2;
    }
    const unsigned long long nwaves = (max_chunks + wave_chunks - 1) / wave_chunks;
    // pilot pass (option pilot): 1 = automatic -- single-wave sweeps only (a
    // multi-wave sweep's first sorted wave seeds the bounds as well, without a
    // second enumeration of every plan); 2 = always; 0 = never
    const bool use_pilot = E.prune && !prow.empty() && (E.pilot == 2 || (E.pilot == 1 && nwaves <= 1));
    const bool collective = E.collective();
    // Ranks share their bounds: one all-gather of ub and a min over ranks
    // (every rank's ub is realised by one of its own plans, so the min is a
    // valid bound for all of them), after the pilot pass and after every wave.
    auto exchange_ub = [&]() {
        if (!collective) return;
        CG_CUDA(cudaStreamWaitEvent(x.s, E.ev[11], 0));
        x.sync();
        unsigned long long* gathered = E.d_gather.as<unsigned long long>((size_t)cells * E.world);
        if (E.allgather(ub, gathered, (size_t)cells * 8, E.ag_user) != 0) fail(CG_ERR_CUDA, "all-gather callback failed");
        k_min_ranks<<<(unsigned)((cells + 255) / 256), 256, 0, x.s>>>(gathered, E.world, cells, ub);
        CG_LAUNCH_CHECK();
        ++x.launches;
        ++x.st.collectives;
    };
    if (E.prune && E.seeds) {
        int seed_no = 0;
        for (int r = 0; r < nrows; ++r) {
            const auto& sp = hs[rows[r].space];
            if (sp.num_plans < 4096 || N < 1) continue;
            const int S = (int)sp.shapes.size();
            for (int sidx = 0; sidx < S; ++sidx)
                for (int c = 1; c * sp.shapes[sidx].gpus <= N && c <= 32; ++c) {
                    unsigned long long q = 0;  // lexicographic rank of (0..0, c, 0..0)
                    for (int k = 0; k < c; ++k) q += sp.w(sidx + 1, N - k * sp.shapes[sidx].gpus);
                    if (seed_no++ % E.world == E.rank)  // seeds are dealt round-robin over the ranks
                        seeds.push_back(((unsigned long long)r << kItemPlanBits) | (q - 1));
                }
        }
        if (!seeds.empty() && !use_pilot) {
            unsigned long long* dseeds = E.d_seeds.as<unsigned long long>(seeds.size());
            x.h2d(dseeds, seeds.data(), seeds.size() * 8);
            run_list(dseeds, nullptr, seeds.size(), 3, true, nullptr);
        }
    }
    // Filter waves: enumerate every plan once, keep stable + not-bounded plans
    // in per-class lists, simulate each list with its lane width.
    if (!prow.empty()) {
        int* rowids = E.d_rowids.as<int>(prow.size());
        unsigned long long* cpre = E.d_iprefix.as<unsigned long long>(chunk_prefix.size());
        x.h2d(rowids, prow.data(), prow.size() * sizeof(int));
        x.h2d(cpre, chunk_prefix.data(), chunk_prefix.size() * 8);
        size_lists();
        ItemRec* lrecs = E.d_lrecs.as<ItemRec>((size_t)coff[7]);
        unsigned long long* tidx = E.d_lidx.as<unsigned long long>(cmax);
        unsigned long long* lkeys = E.d_lkeys.as<unsigned long long>((size_t)coff[7]);
        unsigned long long* tk = E.d_lk1.as<unsigned long long>(cmax);
        unsigned long long* tv = E.d_lv1.as<unsigned long long>(cmax);
        unsigned int* rsh = E.d_rshist.as<unsigned int>(radix_hist_entries((long long)cmax));
        unsigned long long* lcount = E.d_lcount.as<unsigned long long>(7);
        // pilot: the best-estimate stable plan of every (row, budget) cell
        const size_t pregion = (size_t)cells + seeds.size();  // per-class pilot list capacity
        unsigned long long* pilot = use_pilot ? E.d_pilot.as<unsigned long long>(cells) : nullptr;
        unsigned long long* plists = use_pilot ? E.d_plists.as<unsigned long long>(7 * pregion) : nullptr;
        unsigned long long* pkeys = use_pilot ? E.d_pkeys.as<unsigned long long>(7 * pregion) : nullptr;
        unsigned long long* ptk = use_pilot ? E.d_ptk.as<unsigned long long>(pregion) : nullptr;
        unsigned long long* ptv = use_pilot ? E.d_ptv.as<unsigned long long>(pregion) : nullptr;
        unsigned int* prsh = use_pilot ? E.d_prsh.as<unsigned int>(radix_hist_entries((long long)pregion)) : nullptr;
        unsigned long long* pcount = E.d_pcount.as<unsigned long long>(7);
        bool pilot_join = false;
        if (use_pilot) {
            // Pilot: one enumeration of this rank's plans finds, per (row,
            // budget) cell, the stable plan with the best heuristic estimate;
            // those are simulated first (one launch for dp <= 32) so the exact
            // bounds are tight before the bulk lists run.
            x.fill(pilot, cells, ~0ull);
            FilterArgs fp{};
            fp.N = N;
            fp.n_req = n_req;
            fp.kstar = kstar;
            fp.prune = E.prune;
            fp.nrows = (int)prow.size();
            fp.row_ids = rowids;
            fp.chunk_prefix = cpre;
            fp.chunk_base = 0;
            fp.nchunks = my_chunks;
            fp.shard_rank = E.rank;
            fp.shard_world = E.world;
            fp.chunk = chunk;
            fp.rows = base.rows;
            fp.spaces = base.spaces;
            fp.tab = tab;
            fp.ub = ub;
            fp.counters = ctrs;
            fp.pilot = pilot;
            fp.pilot_only = 1;
            fp.pilot_min_plans = (unsigned long long)E.pilot_min_plans;
            fp.sort_key = E.sort_key ? E.sort_key : 1;
            launch_plan_filter(fp, x.s, &x.launches);
            // the seeds lead the class-3 pilot list (dp <= 32)
            const unsigned long long pc0[7] = {0, 0, 0, (unsigned long long)seeds.size(), 0, 0, 0};
            x.h2d(pcount, pc0, sizeof(pc0));
            if (!seeds.empty()) {
                x.h2d(plists + 3 * pregion, seeds.data(), seeds.size() * 8);
                CG_CUDA(cudaMemsetAsync(pkeys + 3 * pregion, 0, seeds.size() * 8, x.s));
            }
            PilotArgs pa{};
            pa.cells = cells;
            pa.N = N;
            pa.pilot = pilot;
            pa.rows = base.rows;
            pa.spaces = base.spaces;
            for (int c = 0; c < 7; ++c) {
                pa.lists[c] = plists + (size_t)c * pregion;
                pa.keys[c] = pkeys + (size_t)c * pregion;
            }
            pa.list_count = pcount;
            pa.merge = E.pilot_merge;
            launch_pilot_lists(pa, x.s, &x.launches);
            unsigned long long pcounts[7];
            x.d2h(pcounts, pcount, sizeof(pcounts));
            x.sync();
            // each class list in ascending estimate order (seeds first): pilots of
            // a row then prune against the row's better cells already done
            const unsigned long long* pperm[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
            unsigned long long* permbuf = E.d_pperm.as<unsigned long long>(7 * pregion);
            for (int c = 0; c < 7; ++c) {
                if (pcounts[c] < 2 || !E.pilot_sort) continue;
                unsigned long long* pi = permbuf + (size_t)c * pregion;
                k_iota_u64<<<(unsigned)((pcounts[c] + 255) / 256), 256, 0, x.s>>>(pi, (long long)pcounts[c]);
                CG_LAUNCH_CHECK();
                ++x.launches;
                const int par = radix_sort_u64(pkeys + (size_t)c * pregion, pi, ptk, ptv, (long long)pcounts[c],
                                               (1ull << 21) - 1ull, prsh, x.s, &x.launches);
                if (par) CG_CUDA(cudaMemcpyAsync(pi, ptv, pcounts[c] * 8, cudaMemcpyDeviceToDevice, x.s));
                pperm[c] = pi;
            }
            // class 0 (dp <= 4) on the second stream, concurrently with the rest
            CG_CUDA(cudaEventRecord(E.ev[10], x.s));
            CG_CUDA(cudaStreamWaitEvent(E.s2, E.ev[10], 0));
            run_list_on(plists, nullptr, pcounts[0], 0, true, pperm[0], E.s2, 1);
            for (int c = 6; c >= 1; --c)
                run_list(plists + (size_t)c * pregion, nullptr, pcounts[c], c, true, pperm[c]);
            CG_CUDA(cudaEventRecord(E.ev[11], E.s2));
            pilot_join = true;  // joined before the first bulk list: it overlaps the wave filter
            if (collective) {
                exchange_ub();
                pilot_join = false;
            }
        }
        long long wave_no = -1, waves_run = 0;
        for (unsigned long long w0 = 0; w0 < max_chunks; w0 += wave_chunks) {
            const unsigned long long nch = w0 < my_chunks ? std::min<unsigned long long>(wave_chunks, my_chunks - w0) : 0;
            ++wave_no;
            ++x.st.waves_total;
            // rate sampling (diagnostic; the result is then partial): every
            // wave_stride-th wave, at most max_waves of them
            if (E.wave_stride > 1 && wave_no % E.wave_stride != 0) continue;
            if (E.max_waves > 0 && waves_run >= E.max_waves) continue;
            ++waves_run;
            ++x.st.waves_run;
            x.st.plans_in_waves += (long long)nch * chunk;
            CG_CUDA(cudaMemsetAsync(lcount, 0, 7 * 8, x.s));
            FilterArgs fa{};
            fa.N = N;
            fa.n_req = n_req;
            fa.kstar = kstar;
            fa.prune = E.prune;
            fa.nrows = (int)prow.size();
            fa.row_ids = rowids;
            fa.chunk_prefix = cpre;
            fa.chunk_base = w0;
            fa.nchunks = nch;
            fa.shard_rank = E.rank;
            fa.shard_world = E.world;
            fa.chunk = chunk;
            fa.rows = base.rows;
            fa.spaces = base.spaces;
            fa.tab = tab;
            fa.ub = ub;
            for (int c = 0; c < 7; ++c) {
                fa.recs[c] = lrecs + coff[c];
                fa.keys[c] = lkeys + coff[c];
                fa.list_caps[c] = ccap[c];
            }
            fa.list_count = lcount;
            fa.counters = ctrs;
            fa.sort_key = E.sort_key;
            launch_plan_filter(fa, x.s, &x.launches);
            unsigned long long counts[7];
            x.d2h(counts, lcount, sizeof(counts));
            x.sync();
            for (int c = 0; c < 7; ++c)  // the census bounds every class list: cannot happen
                if (counts[c] > ccap[c]) fail(CG_ERR_CUDA, "plan class list overflow");
            if (pilot_join) {
                CG_CUDA(cudaStreamWaitEvent(x.s, E.ev[11], 0));
                pilot_join = false;
            }
            // Small waves are latency-bound (each launch lasts at least one
            // plan's request chain): their class lists run concurrently, each on
            // its own stream, scratch region, item counter and perm slice.
            // Large waves run the classes in order so bounds tighten between them.
            unsigned long long total = 0;
            for (int c = 0; c < 7; ++c) total += counts[c];
            const bool conc = total <= (unsigned long long)E.conc_lists_max;
            unsigned long long* cperm = conc ? E.d_cperm.as<unsigned long long>(std::max<unsigned long long>(total, 1)) : nullptr;
            unsigned long long poff = 0;
            int nlaunched = 0;
            cudaStream_t streams[4] = {x.s, E.s2, E.s3, E.s4};
            if (conc) CG_CUDA(cudaEventRecord(E.ev[12], x.s));  // re-recorded after the sorts below
            for (int ci = 0; ci < 7; ++ci) {
                const int c = E.class_order ? ci : 6 - ci;
                const ItemRec* recs = lrecs + coff[c];
                const unsigned long long* perm = nullptr;
                if (E.prune && counts[c] > 1) {  // ascending order key (16 bits: 2 passes) of slot indices
                    k_iota_u64<<<(unsigned)((counts[c] + 255) / 256), 256, 0, x.s>>>(tidx, (long long)counts[c]);
                    CG_LAUNCH_CHECK();
                    ++x.launches;
                    const int par = radix_sort_u64(lkeys + coff[c], tidx, tk, tv, (long long)counts[c],
                                                   (1ull << kListKeyBits) - 1ull, rsh, x.s, &x.launches);
                    perm = par ? tv : tidx;
                    if (conc) {  // the shared sort buffers are reused by the next class
                        CG_CUDA(cudaMemcpyAsync(cperm + poff, perm, counts[c] * 8, cudaMemcpyDeviceToDevice, x.s));
                        perm = cperm + poff;
                        poff += counts[c];
                    }
                }
                if (!conc) {
                    const ItemRec* lr = recs;
                    if (perm) {  // gather into sorted order (the class lists run one after another)
                        ItemRec* gr = E.d_grecs.as<ItemRec>(cmax);
                        k_gather_recs<<<(unsigned)((counts[c] + 255) / 256), 256, 0, x.s>>>(
                            perm, (long long)counts[c], lr, gr);
                        CG_LAUNCH_CHECK();
                        ++x.launches;
                        lr = gr;
                        perm = nullptr;
                    }
                    run_list(nullptr, lr, counts[c], c, false, perm);
                    continue;
                }
                if (counts[c] == 0) continue;
                const int k = nlaunched++ % 4;
                if (k > 0) {
                    CG_CUDA(cudaEventRecord(E.ev[12], x.s));
                    CG_CUDA(cudaStreamWaitEvent(streams[k], E.ev[12], 0));
                }
                run_list_on(nullptr, recs, counts[c], c, false, perm, streams[k], k);
            }
            if (conc)
                for (int k = 1; k < 4 && k < nlaunched; ++k) {
                    CG_CUDA(cudaEventRecord(E.ev[12 + k], streams[k]));
                    CG_CUDA(cudaStreamWaitEvent(x.s, E.ev[12 + k], 0));
                }
            if (E.prune && w0 + wave_chunks < max_chunks) exchange_ub();
        }
    }
    CG_CUDA(cudaStreamWaitEvent(x.s, E.ev[11], 0));  // the pilot's second stream (no-op if unused)
    run_overflows();
    CG_CUDA(cudaEventRecord(E.ev[9], x.s));

    unsigned long long h_ctr[CTR_COUNT], h_ties = 0;
    x.d2h(h_ctr, ctrs, sizeof(h_ctr));
    x.d2h(&h_ties, tiecnt, 8);
    x.sync();
    float k4ms = 0;
    CG_CUDA(cudaEventElapsedTime(&k4ms, E.ev[8], E.ev[9]));
    x.st.ms_k4 += k4ms;
    if (h_ties > (unsigned long long)E.tie_cap) fail(CG_ERR_CUDA, "tie list exhausted");
    x.st.plans_stable += (long long)h_ctr[CTR_STABLE];
    x.st.plans_simulated_full += (long long)h_ctr[CTR_FULL];
    x.st.plans_pruned += (long long)h_ctr[CTR_PRUNED];
    x.st.plans_bound_skipped += (long long)h_ctr[CTR_BOUND];
    x.st.plans_seeded += (long long)h_ctr[CTR_SEED];
    x.st.request_steps += (long long)h_ctr[CTR_STEPS];

    unsigned long long* best = E.d_best.as<unsigned long long>(cells);
    x.fill(best, cells, ~0ull);
    ResolveArgs ra;
    ra.N = N;
    ra.nrows = nrows;
    ra.nties = h_ties;
    ra.ties = ties;
    ra.rows = static_cast<RowDesc*>(E.d_rows.p);
    ra.spaces = static_cast<PlanSpace*>(E.d_spaces.p);
    ra.lat_min = latmin;
    ra.best_plan = best;
    ra.final_lat = E.d_flat.as<double>(cells);
    ra.final_plan = E.d_fplan.as<long long>(cells);
    if (collective) {
        // resolve ties locally, exchange (lat_min, best) with one all-gather, merge
        ResolveArgs local = ra;
        local.nrows = 0;
        launch_resolve(local, x.s, &x.launches);
        unsigned long long* send = E.d_send.as<unsigned long long>((size_t)cells * 2);
        unsigned long long* gathered = E.d_gather.as<unsigned long long>((size_t)cells * 2 * E.world);
        CG_CUDA(cudaMemcpyAsync(send, latmin, cells * 8, cudaMemcpyDeviceToDevice, x.s));
        CG_CUDA(cudaMemcpyAsync(send + cells, best, cells * 8, cudaMemcpyDeviceToDevice, x.s));
        x.sync();
        if (!E.allgather || E.allgather(send, gathered, (size_t)cells * 16, E.ag_user) != 0)
            fail(CG_ERR_CUDA, "all-gather callback failed");
        k_merge_ranks<<<(unsigned)((cells + 127) / 128), 128, 0, x.s>>>(gathered, E.world, cells, N, ra.rows,
                                                                       ra.spaces, latmin, best);
        CG_LAUNCH_CHECK();
        ++x.launches;
        ra.nties = 0;
    }
    launch_resolve(ra, x.s, &x.launches);
    if (E.ub_oracle) {
        E.ub_saved.resize((size_t)cells);
        x.d2h(E.ub_saved.data(), ra.final_lat, (size_t)cells * 8);
        x.sync();
    }
}

// ParallelismPlan expansion of plan index p in space sp (canonical order).
void expand_plan(const HostPlanSpace& sp, long long p, std::vector<cg_replica>& reps, cg_plan& out) {
    std::vector<int> c;
    sp.unrank((unsigned long long)p, c);
    out.replica_offset = (int64_t)reps.size();
    out.gpus_used = 0;
    out.dp = 0;
    for (size_t s = 0; s < c.size(); ++s)
        for (int k = 0; k < c[s]; ++k) {
            reps.push_back({sp.shapes[s].tp, sp.shapes[s].pp});
            out.gpus_used += sp.shapes[s].gpus;
            out.dp += 1;
        }
}

template <class T>
T* hcopy(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.empty() ? 1 : v.size())));
    if (!p) throw std::bad_alloc();
    if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
    return p;
}

struct WlKey {
    int stage;
    unsigned long long b[5];
    bool operator==(const WlKey& o) const {
        return stage == o.stage && std::memcmp(b, o.b, sizeof(b)) == 0;
    }
};
struct WlKeyHash {
    size_t operator()(const WlKey& k) const {
        unsigned long long h = 1469598103934665603ull ^ (unsigned long long)k.stage;
        for (auto v : k.b) {
            h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
            h *= 1099511628211ull;
        }
        return (size_t)h;
    }
};

// Trace columns in HBM (copied when the caller passed host pointers).
struct TraceDev {
    long long n;
    int C;
    const double *scores, *in, *out;
    double first_arrival, last_arrival;
};

TraceDev trace_to_device(SweepCtx& x, const cg_trace& tr) {
    TraceDev t{};
    t.n = tr.n;
    t.C = tr.stages;
    const size_t n = (size_t)tr.n;
    if (tr.on_device) {
        t.scores = tr.scores;
        t.in = tr.input_tokens;
        t.out = tr.output_tokens;
        if (n >= 1) {
            x.d2h(&t.first_arrival, tr.arrival_s, 8);
            x.d2h(&t.last_arrival, tr.arrival_s + n - 1, 8);
            x.sync();
        }
    } else {
        double* s = x.E.d_scores.as<double>(n * tr.stages);
        double* in = x.E.d_in.as<double>(n);
        double* out = x.E.d_out.as<double>(n * tr.stages);
        x.h2d(s, tr.scores, n * tr.stages * sizeof(double));
        x.h2d(in, tr.input_tokens, n * sizeof(double));
        x.h2d(out, tr.output_tokens, n * tr.stages * sizeof(double));
        t.scores = s;
        t.in = in;
        t.out = out;
        if (n >= 1) {
            t.first_arrival = tr.arrival_s[0];
            t.last_arrival = tr.arrival_s[n - 1];
        }
    }
    return t;
}

// overall_arrival_rate (domain.cpp:396-401)
double overall_rate(const TraceDev& t) {
    if (t.n < 2) return 0.0;
    const double span = t.last_arrival - t.first_arrival;
    if (span <= 0.0) return 0.0;
    return static_cast<double>(t.n) / span;
}

// default_threshold_grid (outerplan.cpp:114-132) with GPU-sorted scores.
std::vector<std::vector<double>> default_grid(SweepCtx& x, const TraceDev& t) {
    std::vector<std::vector<double>> grid;
    const long long n = t.n;
    cg_engine& E = x.E;
    for (int d = 0; d + 1 < t.C; ++d) {
        unsigned long long* k0 = E.d_lk0.as<unsigned long long>(n);
        unsigned long long* k1 = E.d_lk1.as<unsigned long long>(n);
        unsigned int* hist = E.d_rshist.as<unsigned int>(radix_hist_entries(n));
        unsigned long long* orax = E.d_orax.as<unsigned long long>(2);
        k_score_keys<<<(unsigned)((n + 255) / 256), 256, 0, x.s>>>(t.scores + (long long)d * n, n, k0);
        CG_LAUNCH_CHECK();
        ++x.launches;
        launch_or_and(k0, n, orax, x.s, &x.launches);
        unsigned long long h[2];
        x.d2h(h, orax, sizeof(h));
        x.sync();
        const int par = radix_sort_u64(k0, nullptr, k1, nullptr, n, h[0] ^ h[1], hist, x.s, &x.launches);
        const unsigned long long* sorted = par ? k1 : k0;
        std::vector<double> values{0.0, kThresholdSentinel};
        std::vector<unsigned long long> keys(9);
        for (int q = 1; q <= 9; ++q) {
            const double qq = q / 10.0;
            auto rank = static_cast<long long>(std::ceil(qq * static_cast<double>(n)));
            rank = std::clamp<long long>(rank, 1, n);
            x.d2h(&keys[q - 1], sorted + (rank - 1), 8);
        }
        x.sync();
        for (auto k : keys) values.push_back(key_to_dbl(k));
        std::sort(values.begin(), values.end());
        values.erase(std::unique(values.begin(), values.end()), values.end());
        grid.push_back(std::move(values));
    }
    return grid;
}

struct RoutingOut {
    int C = 0, D = 0;
    long long n = 0;
    std::vector<int> G;                  // distinct per dim
    std::vector<long long> P;            // workloads per stage
    std::vector<long long> off;          // workload offsets per stage (C+1)
    long long total = 0;
    long long ntuples = 0;
    std::vector<double> stats;           // [total][5]
    std::vector<unsigned long long> count;
    double z2_qsum = 0;                  // all-forward score sum
    bool integral = true;
};

// K1-K3 + K2 for distinct sorted grids (one value list per dim).
RoutingOut route_all(SweepCtx& x, const TraceDev& t, const std::vector<std::vector<double>>& distinct,
                     double rate, const std::vector<double>* extra_thresholds) {
    cg_engine& E = x.E;
    RoutingOut R;
    R.C = t.C;
    R.D = t.C - 1;
    R.n = t.n;
    const long long n = t.n;
    const int C = t.C, D = R.D;
    const int Q = 2 + C;
    RouteArgs ra{};
    ra.n = n;
    ra.scores = t.scores;
    ra.in = t.in;
    ra.out = t.out;
    std::vector<double> gv;
    long long cells = 1;
    for (int d = 0; d < D; ++d) {
        const int g = (int)distinct[d].size();
        if (g > 65534) fail(CG_ERR_UNSUPPORTED, "more than 65534 distinct thresholds in a grid dimension");
        R.G.push_back(g);
        ra.goff[d] = (int)gv.size();
        ra.G[d] = g;
        ra.stride[d] = cells;
        cells *= (g + 1);
        if (cells > (1LL << 31)) fail(CG_ERR_UNSUPPORTED, "threshold grid too large for the rank histogram");
        gv.insert(gv.end(), distinct[d].begin(), distinct[d].end());
    }
    ra.gtotal = (int)gv.size();
    ra.grid_in_smem = ra.gtotal <= 6144 ? 1 : 0;
    double* dgv = E.d_gvals.as<double>(std::max<size_t>(1, gv.size()));
    x.h2d(dgv, gv.data(), gv.size() * sizeof(double));
    ra.gvals = dgv;
    ra.ranks = E.d_ranks.as<unsigned long long>(n);
    ra.hist = E.d_hist.as<unsigned long long>((size_t)cells * Q);
    ra.flags = E.d_flags.as<unsigned int>(1);
    ra.cells = cells;
    {
        long long words = 3 * cells;
        for (int i = 0; i < D; ++i) {  // marginal of stage-i output sums over dims < i
            ra.marg_off[i] = words;
            words += (i == 0) ? 1 : ra.stride[i];
        }
        ra.priv_words = words;
        for (int d = 0; d < D; ++d) {
            int top = 1;
            while (top * 2 <= ra.G[d]) top *= 2;
            ra.gtop[d] = ra.G[d] > 0 ? top : 0;
        }
    }
    ra.max_partials = (long long)E.sm_count * 8;
    ra.partials = (size_t)ra.priv_words * 8 <= 96 * 1024
                      ? E.d_partials.as<unsigned long long>((size_t)ra.max_partials * ra.priv_words)
                      : nullptr;
    ra.acc = E.d_acc.as<unsigned long long>((size_t)ra.priv_words);
    ra.tile_partials = tile_smem_bytes(cells, D, ra.gtotal) <= 200 * 1024
                           ? E.d_tpart.as<unsigned long long>((size_t)ra.max_partials * cells * Q)
                           : nullptr;
    {
        // u32 form of K1: one u32 [cells][Q] slice per block (blocks handle <= 2^16 requests each)
        bool nan = false;
        for (double v : gv) nan |= (v != v);
        ra.bin_ok = nan ? 0 : 1;
        const long long blocks = std::max<long long>((long long)E.sm_count * 4, (n + 65535) / 65536 + E.sm_count);
        ra.k1_form = E.k1_form;
        if ((size_t)cells * Q * 4 <= 96 * 1024 && E.k1_form != 1) {
            ra.part32_words = blocks * cells * Q;
            ra.part32 = E.d_part32.as<unsigned int>((size_t)ra.part32_words);
            ra.hi_acc = E.d_hiacc.as<unsigned long long>((size_t)cells * Q);
        }
    }
    CG_CUDA(cudaMemsetAsync(ra.flags, 0, 4, x.s));
    if (ra.hi_acc) CG_CUDA(cudaMemsetAsync(ra.hi_acc, 0, (size_t)cells * Q * 8, x.s));
    CG_CUDA(cudaEventRecord(E.ev[0], x.s));
    int k1_blocks = 0;
    launch_route_aggregate(ra, D, E.sm_count, x.s, &x.launches, &k1_blocks);
    CG_CUDA(cudaEventRecord(E.ev[1], x.s));
    launch_hist_expand(ra, C, k1_blocks, x.s, &x.launches);
    launch_hist_scan(ra.hist, cells, Q, ra.stride, ra.G, D, x.s, &x.launches);

    // workloads per (stage, prefix)
    R.P.assign(C, 1);
    R.off.assign(C + 1, 0);
    for (int i = 0; i < C; ++i) {
        long long p = 1;
        for (int d = 0; d < i; ++d) p *= R.G[d];
        R.P[i] = p;
        R.off[i + 1] = R.off[i] + p;
    }
    R.total = R.off[C];
    R.ntuples = R.P[C - 1];
    WorkloadArgs wa{};
    wa.C = C;
    wa.total = R.total;
    for (int i = 0; i <= C; ++i) wa.wl_off[i] = R.off[i];
    for (int d = 0; d < D; ++d) {
        wa.G[d] = R.G[d];
        wa.stride[d] = ra.stride[d];
    }
    wa.hist = ra.hist;
    wa.count = E.d_wcount.as<unsigned long long>(R.total);
    wa.sum_in = E.d_wsin.as<unsigned long long>(R.total);
    wa.sum_out = E.d_wsout.as<unsigned long long>(R.total);
    launch_workload_counts(wa, x.s, &x.launches);

    // sorted token columns for the p95 scans
    const int L = C + 1;
    unsigned long long* lk0 = E.d_lk0.as<unsigned long long>((size_t)L * n);
    unsigned long long* lv0 = E.d_lv0.as<unsigned long long>((size_t)L * n);
    unsigned long long* lk1 = E.d_lk1.as<unsigned long long>((size_t)L * n);
    unsigned long long* lv1 = E.d_lv1.as<unsigned long long>((size_t)L * n);
    unsigned int* rshist = E.d_rshist.as<unsigned int>(radix_hist_entries(n));
    unsigned long long* orax = E.d_orax.as<unsigned long long>(2 * L + Q);
    launch_make_lists(t.in, t.out, ra.ranks, n, C, lk0, lv0, E.sm_count, x.s, &x.launches);
    for (int l = 0; l < L; ++l) launch_or_and(lk0 + (long long)l * n, n, orax + 2 * l, x.s, &x.launches);
    // totals of the full histogram cell (sums over the whole trace)
    CG_CUDA(cudaMemcpyAsync(orax + 2 * L, ra.hist + (cells - 1) * Q, Q * 8, cudaMemcpyDeviceToDevice, x.s));
    std::vector<unsigned long long> h_orax(2 * L + Q);
    unsigned int h_flags = 0;
    x.d2h(h_orax.data(), orax, h_orax.size() * 8);
    x.d2h(&h_flags, ra.flags, 4);
    x.sync();
    unsigned long long varying = 0;
    for (int l = 0; l < L; ++l) varying |= h_orax[2 * l] ^ h_orax[2 * l + 1];
    R.integral = (h_flags & 1u) == 0;
    for (int q = 1; q < Q; ++q)
        if (h_orax[2 * L + q] >= (1ull << 53)) R.integral = false;
    int par = 0;
    for (int l = 0; l < L; ++l)
        par = radix_sort_u64(lk0 + (long long)l * n, lv0 + (long long)l * n, lk1 + (long long)l * n,
                             lv1 + (long long)l * n, n, varying, rshist, x.s, &x.launches);
    const unsigned long long* sk = par ? lk1 : lk0;
    const unsigned long long* sv = par ? lv1 : lv0;
    double* p95i = E.d_wp95i.as<double>(R.total);
    double* p95o = E.d_wp95o.as<double>(R.total);
    const long long p95_tab = E.p95_tables ? p95_table_entries(wa, n) : 0;
    launch_p95_scan(wa, sk, sv, n, p95i, p95o,
                    p95_tab > 0 ? E.d_p95tab.as<unsigned short>((size_t)p95_tab) : nullptr, x.s, &x.launches);
    double* sinf = E.d_wsinf.as<double>(R.total);
    double* soutf = E.d_wsoutf.as<double>(R.total);
    if (!R.integral)
        launch_workload_seq_sums(wa, ra.ranks, t.in, t.out, n, sinf, soutf, x.s, &x.launches);
    double* stats = E.d_wstats.as<double>((size_t)R.total * 5);
    launch_workload_stats(wa, n, rate, R.integral ? 1 : 0, sinf, soutf, p95i, p95o, stats, x.s, &x.launches);
    CG_CUDA(cudaEventRecord(E.ev[2], x.s));

    // K2: quality for every distinct tuple (+ optional extra threshold rows)
    const long long extra = extra_thresholds ? (long long)(extra_thresholds->size() / std::max(1, D)) : 0;
    const long long nq = R.ntuples + (extra_thresholds ? (D > 0 ? extra : 1) : 0);
    std::vector<double> thr((size_t)std::max(1LL, nq * D));
    for (long long tu = 0; tu < R.ntuples; ++tu) {
        long long w = tu;
        for (int d = 0; d < D; ++d) {
            thr[(size_t)tu * D + d] = distinct[d][w % R.G[d]];
            w /= R.G[d];
        }
    }
    if (extra_thresholds && D > 0)
        std::copy(extra_thresholds->begin(), extra_thresholds->end(), thr.begin() + (size_t)R.ntuples * D);
    double* dthr = E.d_thr.as<double>(thr.size());
    x.h2d(dthr, thr.data(), (size_t)nq * D * sizeof(double));
    double* qsum = E.d_qsum.as<double>(nq);
    QualityScratch qs{};
    if (E.quality_form == 1) {
        qs.B = std::max(quality_block(n, nq), E.quality_block);  // option: larger blocks (multi-tile path)
        const size_t ent = (size_t)nq * (size_t)((n + qs.B - 1) / qs.B);
        qs.A = E.d_qa.as<double>(ent);
        qs.E = E.d_qe.as<short>(ent);
        qs.U = E.d_qu.as<unsigned long long>(ent);
        qs.seq_blocks = E.d_qseq.as<unsigned long long>(1);
        CG_CUDA(cudaMemsetAsync(qs.seq_blocks, 0, 8, x.s));
    }
    launch_quality(t.scores, n, D, dthr, nq, qsum, E.quality_form == 1 ? &qs : nullptr, x.s, &x.launches);
    CG_CUDA(cudaEventRecord(E.ev[3], x.s));

    R.stats.resize((size_t)R.total * 5);
    R.count.resize(R.total);
    x.d2h(R.stats.data(), stats, R.stats.size() * 8);
    x.d2h(R.count.data(), wa.count, R.count.size() * 8);
    if (extra_thresholds) x.d2h(&R.z2_qsum, qsum + R.ntuples, 8);
    unsigned long long qseq = 0;
    if (qs.seq_blocks) x.d2h(&qseq, qs.seq_blocks, 8);
    x.sync();
    if (qs.seq_blocks) {
        x.st.quality_blocks += nq * ((n + qs.B - 1) / qs.B);
        x.st.quality_blocks_seq += (long long)qseq;
    }
    float m_k1 = 0, m_route = 0, m_q = 0;
    CG_CUDA(cudaEventElapsedTime(&m_k1, E.ev[0], E.ev[1]));
    CG_CUDA(cudaEventElapsedTime(&m_route, E.ev[0], E.ev[2]));
    CG_CUDA(cudaEventElapsedTime(&m_q, E.ev[2], E.ev[3]));
    x.st.ms_k1 += m_k1;
    x.st.k1_bytes += (double)n * (8.0 * (D + 1 + C) + 8.0);
    x.st.ms_route += m_route;
    x.st.ms_quality += m_q;
    x.st.stage_workloads += R.total;
    return R;
}

void free_result(cg_sweep_result* r) {
    if (!r) return;
    std::free(r->eval_candidate);
    std::free(r->eval_thresholds);
    std::free(r->eval_latency);
    std::free(r->eval_quality);
    std::free(r->eval_ratios);
    std::free(r->eval_allocations);
    std::free(r->eval_plan);
    std::free(r->plans);
    std::free(r->replicas);
    std::free(r->weights);
    std::free(r->weight_selection);
    std::free(r->front);
    std::free(r->skipped_candidate);
    std::free(r->skipped_thresholds);
    std::free(r);
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI

// ---------------------------------------------------------------------------
// NCCL inside the library.  libnccl is bound at first use (dlopen), so the
// library carries no link-time NCCL dependency and, inside a process that
// already loaded NCCL (e.g. torch's), reuses that copy instead of mapping a
// second one.  CG_NCCL_LIBRARY overrides the soname.
namespace {
struct NcclApi {
    bool ok = false;
    std::string error;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* env = std::getenv("CG_NCCL_LIBRARY");
        const char* name = env && *env ? env : "libnccl.so.2";
        void* h = dlopen(name, RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            api.error = std::string("cannot load NCCL (") + name + "): " + (e ? e : "unknown error");
            return;
        }
        auto sym = [&](auto& fn, const char* n) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, n));
            if (!fn && api.error.empty()) api.error = std::string("NCCL symbol missing: ") + n;
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommInitAll, "ncclCommInitAll");
        sym(api.AllGather, "ncclAllGather");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.CommAbort, "ncclCommAbort");
        sym(api.GetErrorString, "ncclGetErrorString");
        sym(api.GetVersion, "ncclGetVersion");
        api.ok = api.error.empty();
    });
    return api;
}

const NcclApi& nccl_checked() {
    const NcclApi& n = nccl();
    if (!n.ok) fail(CG_ERR_CUDA, n.error);
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(CG_ERR_CUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}

// The engine's all-gather over its own communicator, enqueued on its stream
// (the kernels that consume the gathered buffer follow on the same stream).
int nccl_allgather(const void* send, void* recv, size_t bytes, void* user) {
    auto* e = static_cast<cg_engine*>(user);
    const NcclApi& n = nccl();
    if (!n.ok || !e->nccl_comm) return 1;
    return n.AllGather(send, recv, bytes, ncclUint8, static_cast<ncclComm_t>(e->nccl_comm), e->s) == ncclSuccess
               ? 0 : 1;
}

void join_nccl(cg_engine* e, ncclComm_t comm, int rank, int world) {
    e->rank = rank;
    e->world = world;
    e->allgather = nccl_allgather;
    e->ag_user = e;
    e->nccl_member = true;
    e->nccl_comm = comm;
}

void release_nccl(cg_engine* e, bool abort) {
    if (!e->nccl_comm) return;
    const NcclApi& n = nccl();
    if (n.ok) (abort ? n.CommAbort : n.CommDestroy)(static_cast<ncclComm_t>(e->nccl_comm));
    e->nccl_comm = nullptr;
    e->nccl_member = false;
    e->allgather = nullptr;
    e->rank = 0;
    e->world = 1;
}

// Runs `call(member, &result)` on every member of a multi-device engine, one
// host thread per device, and returns rank 0's result.  Counters that are
// per-rank shares are summed; device times are the maximum over ranks.  A
// member that fails while the others are still running (they may be waiting
// in a collective) aborts every communicator after a grace period, so no
// call can hang; the group then refuses further sharded calls.
template <class R, class Call, class Free>
cg_status run_group(cg_engine* E, R** out, Call&& call, Free&& free_fn) {
    MultiGroup& g = *E->group;
    if (g.broken) return err_status(CG_ERR_CUDA, "multi-device engine unusable: its NCCL communicators were aborted");
    const int n = (int)g.members.size();
    std::vector<R*> res(n, nullptr);
    std::vector<cg_status> st(n);
    std::vector<std::future<void>> fut;
    for (int r = 0; r < n; ++r)
        fut.push_back(std::async(std::launch::async, [&, r] { st[r] = call(g.members[r], &res[r]); }));
    bool failed_early = false;
    for (;;) {
        int done = 0, failed = 0;
        for (int r = 0; r < n; ++r)
            if (fut[r].wait_for(std::chrono::milliseconds(0)) == std::future_status::ready) {
                ++done;
                failed += st[r].code != CG_OK;
            }
        if (done == n) break;
        if (failed && !failed_early) {
            failed_early = true;
            // deterministic errors (validation) reach every rank within
            // moments; a lone failure leaves the others in a collective
            bool all_done = false;
            for (int t = 0; t < 200 && !all_done; ++t) {
                std::this_thread::sleep_for(std::chrono::milliseconds(50));
                all_done = true;
                for (int r = 0; r < n; ++r)
                    all_done &= fut[r].wait_for(std::chrono::milliseconds(0)) == std::future_status::ready;
            }
            if (!all_done) {
                g.broken = true;
                for (cg_engine* m : g.members)
                    if (m->nccl_comm) nccl().CommAbort(static_cast<ncclComm_t>(m->nccl_comm));
            }
            continue;
        }
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    if (g.broken)
        for (cg_engine* m : g.members) m->nccl_comm = nullptr;  // aborted above
    for (int r = 0; r < n; ++r)
        if (st[r].code != CG_OK) {
            for (R* p : res)
                if (p) free_fn(p);
            return st[r];
        }
    cg_sweep_stats& s0 = res[0]->stats;
    for (int r = 1; r < n; ++r) {
        const cg_sweep_stats& s = res[r]->stats;
        s0.plans_stable += s.plans_stable;
        s0.plans_simulated_full += s.plans_simulated_full;
        s0.plans_pruned += s.plans_pruned;
        s0.plans_bound_skipped += s.plans_bound_skipped;
        s0.plans_seeded += s.plans_seeded;
        s0.plans_overflow += s.plans_overflow;
        s0.request_steps += s.request_steps;
        s0.h2d_bytes += s.h2d_bytes;
        s0.d2h_bytes += s.d2h_bytes;
        s0.gpu_launches += s.gpu_launches;
        s0.ms_rows = std::max(s0.ms_rows, s.ms_rows);
        s0.ms_k4 = std::max(s0.ms_k4, s.ms_k4);
        s0.ms_total = std::max(s0.ms_total, s.ms_total);
        free_fn(res[r]);
    }
    *out = res[0];
    return ok_status();
}
}  // namespace

extern "C" {

const char* cg_version(void) { return "cascade-gpu 0.1 (sm_100a)"; }

cg_status cg_sweep_result_json(cg_engine* E, const cg_sweep_result* r, int32_t indent, int32_t what,
                               int32_t flags, char** text, int64_t* len) {
    E = primary(E);
    return guarded([&] {
        if (!E || !r || !text || !len) fail(CG_ERR_INVALID_INPUT, "null engine/result/output");
        if (indent < 0) fail(CG_ERR_UNSUPPORTED, "compact JSON (indent < 0) is not produced by the planner");
        if (what != 0 && what != 1) fail(CG_ERR_INVALID_INPUT, "what must be 0 (sweep) or 1 (front)");
        *text = nullptr;
        *len = 0;
        int launches = 0;
        const std::string s = result_json(E->jsonbuf, E->s, *r, indent, what, flags, &launches);
        char* p = static_cast<char*>(std::malloc(s.size() + 1));
        if (!p) throw std::bad_alloc();
        std::memcpy(p, s.data(), s.size());
        p[s.size()] = 0;
        *text = p;
        *len = (int64_t)s.size();
    });
}

void cg_text_free(char* text) { std::free(text); }

static DriftArgs drift_args(cg_engine* E, const cg_trace* tr) {
    DriftBuffers& B = E->driftbuf;
    const long long n = tr->n;
    auto dev = [&](DevBuf& b, const double* src) -> const double* {
        if (tr->on_device) return src;
        double* d = b.as<double>((size_t)std::max<long long>(1, n));
        CG_CUDA(cudaMemcpyAsync(d, src, (size_t)n * 8, cudaMemcpyHostToDevice, E->s));
        return d;
    };
    DriftArgs a{};
    a.n = n;
    a.arrival = dev(B.arr, tr->arrival_s);
    a.in = dev(B.in, tr->input_tokens);
    a.out0 = dev(B.out0, tr->output_tokens);  // stage 1 = rows [0, n)
    a.score0 = dev(B.sc0, tr->scores);
    return a;
}

static double host_at(cg_engine* E, const cg_trace* tr, const double* col, long long i) {
    if (!tr->on_device) return col[i];
    double v = 0;
    CG_CUDA(cudaMemcpyAsync(&v, col + i, 8, cudaMemcpyDeviceToHost, E->s));
    CG_CUDA(cudaStreamSynchronize(E->s));
    return v;
}

cg_status cg_drift_windows(cg_engine* E, const cg_trace* tr, const cg_drift_stats* base, const cg_drift_policy* pol,
                           cg_drift_result** out) {
    E = primary(E);
    return guarded([&] {
        if (!E || !tr || !base || !pol || !out) fail(CG_ERR_INVALID_INPUT, "null argument");
        *out = nullptr;
        if (tr->n <= 0) fail(CG_ERR_EMPTY_TRACE, "drift stream is empty");
        if (tr->stages < 1) fail(CG_ERR_INVALID_INPUT, "drift stream has no stages");
        DriftArgs a = drift_args(E, tr);
        a.t0 = host_at(E, tr, tr->arrival_s, 0);
        a.stream_end = host_at(E, tr, tr->arrival_s, tr->n - 1);
        a.interval = pol->window_interval_s;
        a.window_requests = pol->window_requests;
        a.has_h1 = base->has_h1;
        a.h1 = base->h1;
        int launches = 0;
        std::vector<DriftWindowOut> w;
        drift_windows(E->driftbuf, E->s, a, w, &launches);
        auto* res = new cg_drift_result{};
        std::vector<cg_drift_window> keep;
        for (const auto& x : w) {
            if (!x.valid) continue;  // window.empty() || span <= 0 (cli.cpp:238)
            cg_drift_window o{};
            o.start_s = x.start;
            o.span_s = x.span;
            o.requests = (int32_t)x.requests;
            o.first_record = x.first;
            o.sampled = (int32_t)x.sampled;
            o.stats = cg_drift_stats{x.rate, x.mean_in, x.mean_out, x.accept, base->has_h1, base->h1};
            const double b4[4] = {base->arrival_rate, base->mean_input_tokens, base->mean_output_tokens,
                                  base->stage1_accept_rate};
            const double c4[4] = {x.rate, x.mean_in, x.mean_out, x.accept};
            for (int q = 0; q < 4; ++q) {  // check() (cli.cpp:252-266)
                if (b4[q] != 0.0) {
                    const double d = std::abs(c4[q] - b4[q]) / std::abs(b4[q]);
                    o.deviation[q] = d;
                    o.drifted[q] = d > pol->rel_tolerance ? 1 : 0;
                } else {
                    o.deviation_is_null[q] = 1;
                    o.drifted[q] = c4[q] != 0.0 ? 1 : 0;
                }
                o.any_drift |= o.drifted[q];
            }
            res->drift_detected |= o.any_drift;
            keep.push_back(o);
        }
        res->num_windows = (int64_t)keep.size();
        res->windows = static_cast<cg_drift_window*>(std::malloc(sizeof(cg_drift_window) * std::max<size_t>(1, keep.size())));
        for (size_t i = 0; i < keep.size(); ++i) res->windows[i] = keep[i];
        *out = res;
    });
}

void cg_drift_result_free(cg_drift_result* r) {
    if (!r) return;
    std::free(r->windows);
    delete r;
}

cg_status cg_trace_baseline(cg_engine* E, const cg_trace* tr, int32_t has_h1, double h1, cg_drift_stats* out) {
    E = primary(E);
    return guarded([&] {
        if (!E || !tr || !out) fail(CG_ERR_INVALID_INPUT, "null argument");
        *out = cg_drift_stats{0, 0, 0, 1, has_h1, h1};
        // overall_arrival_rate (domain.cpp:396-401)
        double rate = 0.0;
        if (tr->n >= 2) {
            const double span = host_at(E, tr, tr->arrival_s, tr->n - 1) - host_at(E, tr, tr->arrival_s, 0);
            rate = span <= 0.0 ? 0.0 : static_cast<double>(tr->n) / span;
        }
        out->arrival_rate = rate;
        if (tr->n <= 0 || tr->stages < 1) return;  // stats_of_records of an empty trace
        DriftArgs a = drift_args(E, tr);
        a.has_h1 = has_h1;
        a.h1 = h1;
        double r3[3];
        int launches = 0;
        trace_baseline(E->driftbuf, E->s, a, r3, &launches);
        out->mean_input_tokens = r3[0];
        out->mean_output_tokens = r3[1];
        out->stage1_accept_rate = r3[2];
    });
}

void cg_sim_result_free(cg_sim_result* r) {
    if (!r) return;
    for (int i = 0; i < r->num_reports; ++i) {
        std::free(r->reports[i].end_to_end_s);
        std::free(r->reports[i].accept_stage);
        std::free(r->reports[i].attainment_scale);
        std::free(r->reports[i].attainment_fraction);
    }
    std::free(r->reports);
    delete r;
}

cg_status cg_simulate(cg_engine* E, const cg_trace* tr, const cg_model* models, int32_t C, const cg_hardware* hw,
                      const cg_cost_params* q, const cg_sim_config* cfg, const cg_cascade_plan* plans,
                      int32_t P, int32_t compare, cg_sim_result** out) {
    E = primary(E);
    return guarded([&] {
        if (!E || !tr || !models || !hw || !q || !cfg || (P > 0 && !plans) || !out)
            fail(CG_ERR_INVALID_INPUT, "null argument");
        *out = nullptr;
        Timer tm;
        if (compare && P < 2) fail(CG_ERR_INVALID_INPUT, "compare requires >= 2 plans");
        if (C < 1 || C > kSimMaxStages) fail(CG_ERR_UNSUPPORTED, "simulator supports 1..8 cascade stages");
        if (cfg->num_scales < 0 || cfg->num_scales > 32) fail(CG_ERR_UNSUPPORTED, "at most 32 SLO scales");
        const long long n = tr->n;
        // run() preconditions per plan, in plan order (simulator.cpp:180-206)
        std::vector<SimPlanDesc> desc(P);
        std::vector<double> ppt, pfix, dpt;
        for (int pi = 0; pi < P; ++pi) {
            const cg_cascade_plan& p = plans[pi];
            if (n <= 0) fail(CG_ERR_EMPTY_TRACE, "run: empty trace");
            const auto probs = validate_cascade_plan(p, *hw, models, C);
            if (!probs.empty()) {
                std::string m = "run: invalid plan:";
                for (const auto& x : probs) m += " " + x + ";";
                fail(CG_ERR_INVALID_INPUT, m);
            }
            if (!(cfg->warmup_fraction >= 0.0 && cfg->warmup_fraction < 1.0))
                fail(CG_ERR_INVALID_INPUT, "warmup_fraction outside [0,1)");
            for (int k = 1; k < cfg->num_scales; ++k)
                if (cfg->slo_scales[k] <= cfg->slo_scales[k - 1])
                    fail(CG_ERR_INVALID_INPUT, "slo_scales must be sorted ascending");
            for (int k = 0; k < cfg->num_scales; ++k)
                if (cfg->slo_scales[k] <= 0) fail(CG_ERR_INVALID_INPUT, "slo_scales must be positive");
            if (tr->stages != C) fail(CG_ERR_INVALID_INPUT, "trace record stage count != C");
            SimPlanDesc& d = desc[pi];
            d = SimPlanDesc{};
            d.C = C;
            d.entry = -1;
            d.last = -1;
            long long off = 0;
            int nchain = 0;
            for (int i = 0; i < kSimMaxStages; ++i) {
                d.next[i] = -1;
                d.chain[i] = -1;
            }
            for (int i = 0; i < C; ++i) {
                const int dp = p.has_plan[i] ? p.dp[i] : 0;
                d.dp[i] = dp;
                d.roff[i] = (int)ppt.size();
                d.thr[i] = i + 1 < C ? p.thresholds[i] : 0.0;
                if (dp > 256) fail(CG_ERR_UNSUPPORTED, "simulator supports up to 256 replicas per stage");
                for (int k = 0; k < dp; ++k) {  // build_context (simulator.cpp:123-143)
                    const cg_replica& r = p.replicas[off + k];
                    const double bubble = 1.0 + q->pipeline_bubble_factor * (r.pp - 1);
                    ppt.push_back(2.0 * models[i].param_count /
                                  (r.tp * r.pp * hw->flops_per_gpu * q->prefill_efficiency) * bubble);
                    pfix.push_back(r.pp * q->comm_overhead_per_stage * bubble);
                    dpt.push_back(models[i].param_count * models[i].bytes_per_param /
                                      (r.tp * hw->mem_bandwidth_per_gpu * q->decode_bw_efficiency) +
                                  r.pp * q->comm_overhead_per_stage);
                }
                off += dp;
                if (dp > 0) {
                    if (d.entry < 0) d.entry = i;
                    d.last = i;
                    d.chain[nchain++] = i;
                }
            }
            for (int k = 0; k + 1 < nchain; ++k) d.next[d.chain[k]] = d.chain[k + 1];
            if (d.entry < 0) fail(CG_ERR_NO_DEPLOYED_STAGE, "plan deploys no stage");
        }
        auto* res = new cg_sim_result{};
        res->n = n;
        *out = res;
        if (P == 0) return;
        SimRunBuffers& B = E->simbuf;
        cudaStream_t s = E->s;
        auto dev = [&](DevBuf& b, const double* src, size_t count) -> const double* {
            if (tr->on_device) return src;
            double* d = b.as<double>(std::max<size_t>(1, count));
            CG_CUDA(cudaMemcpyAsync(d, src, count * 8, cudaMemcpyHostToDevice, s));
            return d;
        };
        SimRunArgs a{};
        a.n = n;
        a.arrival = dev(B.arr, tr->arrival_s, (size_t)n);
        a.in = dev(B.in, tr->input_tokens, (size_t)n);
        a.out = dev(B.out, tr->output_tokens, (size_t)C * n);
        a.scores = dev(B.sc, tr->scores, (size_t)C * n);
        auto up = [&](DevBuf& b, const std::vector<double>& v) {
            double* d = b.as<double>(std::max<size_t>(1, v.size()));
            if (!v.empty()) CG_CUDA(cudaMemcpyAsync(d, v.data(), v.size() * 8, cudaMemcpyHostToDevice, s));
            return d;
        };
        a.ppt = up(B.ppt, ppt);
        a.pf = up(B.pf, pfix);
        a.dpt = up(B.dpt, dpt);
        std::vector<double> scales(cfg->slo_scales, cfg->slo_scales + cfg->num_scales);
        a.scales = up(B.scales, scales);
        a.nscales = cfg->num_scales;
        const long long warmup = (long long)(size_t)(cfg->warmup_fraction * (double)n);
        a.warmup = warmup;
        const int base_mode = cfg->slo_base_s > 0 ? 0 : (compare ? 2 : 1);
        int launches = 0;
        std::vector<SimPlanOut> o;
        sim_run_batch(B, s, a, desc, C, base_mode, cfg->slo_base_s, &launches, o);
        double arr_w = 0.0;
        if (warmup < n) {
            if (tr->on_device) {
                CG_CUDA(cudaMemcpyAsync(&arr_w, tr->arrival_s + warmup, 8, cudaMemcpyDeviceToHost, s));
                CG_CUDA(cudaStreamSynchronize(s));
            } else {
                arr_w = tr->arrival_s[warmup];
            }
        }
        res->reports = static_cast<cg_sim_report*>(std::calloc((size_t)P, sizeof(cg_sim_report)));
        res->num_reports = P;
        const long long m = n - warmup;
        for (int pi = 0; pi < P; ++pi) {
            cg_sim_report& r = res->reports[pi];
            SimPlanOut& x = o[pi];
            r.end_to_end_s = static_cast<double*>(std::malloc(sizeof(double) * n));
            r.accept_stage = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * n));
            std::memcpy(r.end_to_end_s, x.e2e.data(), sizeof(double) * n);
            std::memcpy(r.accept_stage, x.stage.data(), sizeof(int32_t) * n);
            r.slo_base_s = x.base;
            if (m > 0) {  // simulator.cpp:259-274
                r.p95_s = x.p95;
                const double span = x.last_completion - arr_w;
                r.throughput_rps = span > 0 ? static_cast<double>(m) / span : 0.0;
            }
            r.num_scales = cfg->num_scales;
            r.attainment_scale = static_cast<double*>(std::malloc(sizeof(double) * std::max(1, cfg->num_scales)));
            r.attainment_fraction = static_cast<double*>(std::malloc(sizeof(double) * std::max(1, cfg->num_scales)));
            const double considered = static_cast<double>(n - warmup);
            for (int k = 0; k < cfg->num_scales; ++k) {  // attainment_curve (simulator.cpp:301-316)
                r.attainment_scale[k] = cfg->slo_scales[k];
                r.attainment_fraction[k] = considered > 0 ? (double)x.ok[k] / considered : 1.0;
                if (!r.has_min_scale_95 && r.attainment_fraction[k] >= 0.95) {
                    r.has_min_scale_95 = 1;
                    r.min_scale_95 = cfg->slo_scales[k];
                }
            }
            for (int st = 0; st < C; ++st) {  // queue-growth warning (simulator.cpp:280-296)
                const long long size = x.served[st];
                if (desc[pi].dp[st] == 0 || size < 8) continue;
                const long long half = size / 2;
                const double w1 = x.w1[st] / static_cast<double>(half);
                const double w2 = x.w2[st] / static_cast<double>(size - half);
                const double mean_service = x.service_sum[st] / static_cast<double>(size);
                if (w2 > 2.0 * w1 && w2 > mean_service && r.num_unstable < 8) r.unstable_stages[r.num_unstable++] = st + 1;
            }
        }
        res->gpu_launches = launches;
        res->ms_total = tm.ms();
    });
}

void cg_trace_buffer_free(cg_trace_buffer* b) {
    if (!b) return;
    std::free(const_cast<double*>(b->host.arrival_s));
    std::free(const_cast<double*>(b->host.input_tokens));
    std::free(const_cast<double*>(b->host.output_tokens));
    std::free(const_cast<double*>(b->host.scores));
    delete b;
}

static cg_status ingest_common(cg_engine* E, const char* bytes, int64_t len, const std::string& path,
                               double ms_read, cg_trace_buffer** out) {
    return guarded([&] {
        if (!E || !out || (len > 0 && !bytes)) fail(CG_ERR_INVALID_INPUT, "null engine/buffer");
        *out = nullptr;
        Timer tm;
        IngestOut io;
        ingest_jsonl(E->ingest, E->s, bytes, len, path, io);
        auto* b = new cg_trace_buffer{};
        const long long n = io.n;
        const int C = io.stages;
        auto alloc = [](size_t count) {
            double* p = static_cast<double*>(std::malloc(std::max<size_t>(1, count) * sizeof(double)));
            if (!p) throw std::bad_alloc();
            return p;
        };
        double* ha = alloc(n);
        double* hi = alloc(n);
        double* ho = alloc((size_t)C * n);
        double* hs = alloc((size_t)C * n);
        b->host = cg_trace{n, C, 0, ha, hi, ho, hs};
        b->device = cg_trace{n, C, 1, io.d_arrival, io.d_in, io.d_out, io.d_scores};
        if (n > 0) {
            CG_CUDA(cudaMemcpyAsync(ha, io.d_arrival, n * 8, cudaMemcpyDeviceToHost, E->s));
            CG_CUDA(cudaMemcpyAsync(hi, io.d_in, n * 8, cudaMemcpyDeviceToHost, E->s));
            if (C > 0) {
                CG_CUDA(cudaMemcpyAsync(ho, io.d_out, (size_t)C * n * 8, cudaMemcpyDeviceToHost, E->s));
                CG_CUDA(cudaMemcpyAsync(hs, io.d_scores, (size_t)C * n * 8, cudaMemcpyDeviceToHost, E->s));
            }
            CG_CUDA(cudaStreamSynchronize(E->s));
        }
        b->stats.bytes = len;
        b->stats.lines = io.lines;
        b->stats.records = n;
        b->stats.host_lines = io.host_lines;
        b->stats.gpu_launches = io.launches;
        b->stats.ms_total = tm.ms();
        b->stats.ms_read = ms_read;
        *out = b;
    });
}

cg_status cg_parse_trace_jsonl(cg_engine* E, const char* bytes, int64_t len, const char* path,
                               cg_trace_buffer** out) {
    E = primary(E);
    return ingest_common(E, bytes, len, path ? path : "<memory>", 0.0, out);
}

cg_status cg_read_trace_jsonl(cg_engine* E, const char* path, cg_trace_buffer** out) {
    E = primary(E);
    if (!E || !path || !out) return err_status(CG_ERR_INVALID_INPUT, "null engine/path");
    Timer tm;
    FILE* f = std::fopen(path, "rb");
    if (!f) return err_status(CG_ERR_IO, std::string("cannot open trace file: ") + path);
    long long len = 0;
    char* buf = nullptr;
    cg_status st = guarded([&] {
        if (std::fseek(f, 0, SEEK_END) != 0) fail(CG_ERR_IO, std::string("cannot open trace file: ") + path);
        len = std::ftell(f);
        std::fseek(f, 0, SEEK_SET);
        if (len < 0) fail(CG_ERR_IO, std::string("cannot open trace file: ") + path);
        buf = static_cast<char*>(E->ingest.pinned.reserve((size_t)len + 1));
        if (len > 0 && std::fread(buf, 1, (size_t)len, f) != (size_t)len)
            fail(CG_ERR_IO, std::string("cannot open trace file: ") + path);
    });
    std::fclose(f);
    if (st.code != CG_OK) return st;
    return ingest_common(E, buf, len, path, tm.ms(), out);
}

cg_status cg_engine_create(int32_t device, cg_engine** out) {
    return guarded([&] {
        *out = nullptr;
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
            fail(CG_ERR_CUDA, "no CUDA device available (the engine has no CPU fallback)");
        if (device < 0 || device >= n) fail(CG_ERR_CUDA, "invalid CUDA device ordinal");
        CG_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop;
        CG_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10) fail(CG_ERR_CUDA, std::string("device ") + prop.name + " is not sm_100 class");
        auto* e = new cg_engine();
        e->device = device;
        e->sm_count = prop.multiProcessorCount;
        CG_CUDA(cudaStreamCreateWithFlags(&e->s, cudaStreamNonBlocking));
        CG_CUDA(cudaStreamCreateWithFlags(&e->s2, cudaStreamNonBlocking));
        CG_CUDA(cudaStreamCreateWithFlags(&e->s3, cudaStreamNonBlocking));
        CG_CUDA(cudaStreamCreateWithFlags(&e->s4, cudaStreamNonBlocking));
        for (auto& ev : e->ev) CG_CUDA(cudaEventCreate(&ev));
        *out = e;
    });
}

void* cg_engine_stream(cg_engine* e) {
    e = primary(e);
    return e ? static_cast<void*>(e->s) : nullptr;
}

void cg_engine_destroy(cg_engine* e) {
    if (!e) return;
    if (e->group) {
        for (cg_engine* m : e->group->members) cg_engine_destroy(m);
        delete e->group;
        delete e;
        return;
    }
    cudaSetDevice(e->device);
    release_nccl(e, false);
    for (auto& ev : e->ev) cudaEventDestroy(ev);
    if (e->s) cudaStreamDestroy(e->s);
    if (e->s2) cudaStreamDestroy(e->s2);
    if (e->s3) cudaStreamDestroy(e->s3);
    if (e->s4) cudaStreamDestroy(e->s4);
    delete e;
}

cg_status cg_engine_set_collective(cg_engine* e, int32_t rank, int32_t world, cg_allgather_fn fn, void* user) {
    return guarded([&] {
        if (!e) fail(CG_ERR_INVALID_INPUT, "null engine");
        if (e->group || e->nccl_member) fail(CG_ERR_INVALID_INPUT, "engine already bound to NCCL communicators");
        if (world < 1 || rank < 0 || rank >= world) fail(CG_ERR_INVALID_INPUT, "invalid rank/world");
        if (world > 1 && !fn) fail(CG_ERR_INVALID_INPUT, "multi-rank engine needs an all-gather callback");
        e->rank = rank;
        e->world = world;
        e->allgather = fn;
        e->ag_user = user;
    });
}

cg_status cg_nccl_unique_id(void* out, int32_t capacity) {
    return guarded([&] {
        if (!out || capacity < (int32_t)sizeof(ncclUniqueId)) fail(CG_ERR_INVALID_INPUT, "unique id buffer too small");
        ncclUniqueId id;
        nccl_check(nccl_checked().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out, &id, sizeof(id));
    });
}

int32_t cg_nccl_unique_id_bytes(void) { return (int32_t)sizeof(ncclUniqueId); }

cg_status cg_engine_set_nccl(cg_engine* e, const void* unique_id, int32_t rank, int32_t world) {
    return guarded([&] {
        if (!e || !unique_id) fail(CG_ERR_INVALID_INPUT, "null engine/unique id");
        if (e->group) fail(CG_ERR_INVALID_INPUT, "a multi-device engine already owns its communicators");
        if (world < 1 || rank < 0 || rank >= world) fail(CG_ERR_INVALID_INPUT, "invalid rank/world");
        const NcclApi& n = nccl_checked();
        CG_CUDA(cudaSetDevice(e->device));
        release_nccl(e, false);
        ncclUniqueId id;
        std::memcpy(&id, unique_id, sizeof(id));
        ncclComm_t comm = nullptr;
        nccl_check(n.CommInitRank(&comm, world, id, rank), "ncclCommInitRank");
        join_nccl(e, comm, rank, world);
    });
}

cg_status cg_engine_create_multi(const int32_t* devices, int32_t ndev, cg_engine** out) {
    std::vector<cg_engine*> made;
    cg_status st = guarded([&] {
        if (!out) fail(CG_ERR_INVALID_INPUT, "null output");
        *out = nullptr;
        std::vector<int32_t> all;
        if (!devices && ndev == 0) {  // every visible device
            int n = 0;
            if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
                fail(CG_ERR_CUDA, "no CUDA device available (the engine has no CPU fallback)");
            for (int i = 0; i < n; ++i) all.push_back(i);
            devices = all.data();
            ndev = n;
        }
        if (!devices || ndev < 1) fail(CG_ERR_INVALID_INPUT, "multi-device engine needs at least one device");
        for (int i = 0; i < ndev; ++i)
            for (int j = 0; j < i; ++j)
                if (devices[i] == devices[j]) fail(CG_ERR_INVALID_INPUT, "duplicate device in the multi-device engine");
        const NcclApi& n = nccl_checked();
        for (int i = 0; i < ndev; ++i) {
            cg_engine* m = nullptr;
            cg_status cs = cg_engine_create(devices[i], &m);
            if (cs.code != CG_OK) fail(cs.code, cs.message);
            made.push_back(m);
        }
        std::vector<ncclComm_t> comms(ndev, nullptr);
        nccl_check(n.CommInitAll(comms.data(), ndev, devices), "ncclCommInitAll");
        for (int i = 0; i < ndev; ++i) join_nccl(made[i], comms[i], i, ndev);
        auto* parent = new cg_engine();
        parent->device = devices[0];
        parent->sm_count = made[0]->sm_count;
        parent->group = new MultiGroup();
        parent->group->members = made;
        *out = parent;
    });
    if (st.code != CG_OK)
        for (cg_engine* m : made) cg_engine_destroy(m);
    return st;
}

int32_t cg_engine_device_count(cg_engine* e) {
    if (!e) return 0;
    return e->group ? (int32_t)e->group->members.size() : 1;
}

cg_status cg_engine_set_option(cg_engine* e, const char* key, int64_t value) {
    return guarded([&] {
        if (!e || !key) fail(CG_ERR_INVALID_INPUT, "null engine/key");
        if (e->group) {
            for (cg_engine* m : e->group->members) {
                cg_status ms = cg_engine_set_option(m, key, value);
                if (ms.code != CG_OK) fail(ms.code, ms.message);
            }
            return;
        }
        const std::string k(key);
        if (k == "prune") e->prune = value ? 1 : 0;
        else if (k == "k1_form") e->k1_form = (int)value;
        else if (k == "quality_form") e->quality_form = value ? 1 : 0;
        else if (k == "p95_tables") e->p95_tables = value ? 1 : 0;
        else if (k == "max_waves") e->max_waves = std::max<int64_t>(0, value);
        else if (k == "wave_stride") e->wave_stride = std::max<int64_t>(1, value);
        else if (k == "quality_block") e->quality_block = (int)std::min<int64_t>(1 << 30, std::max<int64_t>(0, value));
        else if (k == "ub_oracle") e->ub_oracle = (int)value;
        else if (k == "k4_pack") e->k4_pack = (int)value;
        else if (k == "fut_bound") e->fut_bound = (int)value;
        else if (k == "fut_block") e->fut_block = (int)std::min<int64_t>(1024, std::max<int64_t>(1, value));
        else if (k == "fut_arrival") {
            int sh = 0;
            while ((1 << sh) < value && sh < 5) ++sh;
            if (value < 1 || (1 << sh) != value) fail(CG_ERR_INVALID_INPUT, "fut_arrival must be 1, 2, 4, 8, 16 or 32");
            e->fut_arrival_shift = sh;
        }
        else if (k == "lane_check") {
            if (value != 32 && value != 64) fail(CG_ERR_INVALID_INPUT, "lane_check must be 32 or 64");
            e->lane_check = (int)value;
        }
        else if (k == "pilot") e->pilot = (int)std::min<int64_t>(2, std::max<int64_t>(0, value));
        else if (k == "seeds") e->seeds = value ? 1 : 0;
        else if (k == "sort_key") e->sort_key = (int)value;
        else if (k == "class_order") e->class_order = (int)value;
        else if (k == "pilot_min_plans") e->pilot_min_plans = std::max<int64_t>(0, value);
        else if (k == "pilot_sort") e->pilot_sort = (int)value;
        else if (k == "conc_lists_max") e->conc_lists_max = std::max<int64_t>(0, value);
        else if (k == "pilot_merge") e->pilot_merge = (int)std::min<int64_t>(2, std::max<int64_t>(0, value));
        else if (k == "wave_plans") e->wave_plans = (int)std::min<int64_t>(1024, std::max<int64_t>(1, value));
        else if (k == "item_plans") e->item_plans = (int)std::max<int64_t>(1, value);
        else if (k == "overflow_capacity") e->ovf_cap = std::max<int64_t>(16, value);
        else if (k == "tie_capacity") e->tie_cap = std::max<int64_t>(16, value);
        else fail(CG_ERR_INVALID_INPUT, "unknown option " + k);
    });
}

cg_status cg_sweep(cg_engine* E, const cg_trace* tr, const cg_model* models, int32_t C, const cg_hardware* hw,
                   const cg_cost_params* q, int32_t total_gpus, const cg_sweep_config* cfg,
                   cg_sweep_result** out) {
    if (E && E->group) {
        if (!out) return err_status(CG_ERR_INVALID_INPUT, "null argument");
        return run_group(E, out, [&](cg_engine* m, cg_sweep_result** o) {
            return cg_sweep(m, tr, models, C, hw, q, total_gpus, cfg, o);
        }, cg_sweep_result_free);
    }
    return guarded([&] {
        Timer timer;
        if (out) *out = nullptr;
        if (!E || !tr || !hw || !q || !cfg || !out) fail(CG_ERR_INVALID_INPUT, "null argument");
        CG_CUDA(cudaSetDevice(E->device));
        SweepCtx x(*E);

        // ---- validation in the reference order (outerplan.cpp:170-189)
        if (tr->n <= 0) fail(CG_ERR_EMPTY_TRACE, "sweep: empty trace");
        validate_models(models, C);
        if (C > kMaxStages) fail(CG_ERR_UNSUPPORTED, "GPU engine supports up to 5 cascade stages");
        TraceDev t = trace_to_device(x, *tr);
        const double rate = overall_rate(t);
        if (rate <= 0.0) fail(CG_ERR_INVALID_INPUT, "sweep: trace has no positive arrival-rate span");
        if (tr->stages != C) fail(CG_ERR_INVALID_INPUT, "sweep: trace record stage count != C");
        const int D = C - 1;

        std::vector<std::vector<double>> given;
        if (cfg->grid_dims == 0) {
            given = default_grid(x, t);
        } else {
            long long off = 0;
            for (int d = 0; d < cfg->grid_dims; ++d) {
                given.emplace_back(cfg->grid_values + off, cfg->grid_values + off + cfg->grid_sizes[d]);
                off += cfg->grid_sizes[d];
            }
        }
        if ((int)given.size() != D) fail(CG_ERR_INVALID_INPUT, "sweep: threshold grid must have C-1 dimensions");
        for (const auto& dim : given)
            if (dim.empty()) fail(CG_ERR_INVALID_INPUT, "sweep: empty threshold grid dimension");
        // StageEvaluator constructor (costmodel.cpp:199-203)
        validate_hw(*hw);
        validate_params(*q);

        std::vector<std::vector<double>> distinct(D);
        std::vector<std::vector<int>> g2d(D);
        for (int d = 0; d < D; ++d) {
            distinct[d] = given[d];
            std::sort(distinct[d].begin(), distinct[d].end());
            distinct[d].erase(std::unique(distinct[d].begin(), distinct[d].end()), distinct[d].end());
            for (double v : given[d])
                g2d[d].push_back(
                    (int)(std::lower_bound(distinct[d].begin(), distinct[d].end(), v) - distinct[d].begin()));
        }
        long long ncand = 1;
        for (int d = 0; d < D; ++d) ncand *= (long long)given[d].size();
        x.st.candidates = ncand;

        // ---- routing of every workload + quality of every tuple (+ all-forward for z2*)
        std::vector<double> allfwd((size_t)std::max(1, D), kThresholdSentinel);
        RoutingOut R = route_all(x, t, distinct, rate, &allfwd);
        x.st.distinct_candidates = R.ntuples;

        // ---- row cache: validation in candidate order, exact-bit dedup
        const int N = total_gpus;
        if (N < 0) fail(CG_ERR_INVALID_INPUT, "sweep: total_gpus must be >= 0");
        std::string w0 = workload_problems(&R.stats[0]);
        if (!w0.empty()) fail(CG_ERR_INVALID_INPUT, w0);
        std::vector<char> invalid(R.total, 0);
        bool any_invalid = false;
        for (long long w = 0; w < R.total; ++w)
            if (R.count[w] > 0 && !workload_problems(&R.stats[(size_t)w * 5]).empty()) {
                invalid[w] = 1;
                any_invalid = true;
            }
        auto hs = build_spaces(x, models, C, *hw, *q, N);
        std::vector<int> wl_row(R.total, -1);
        std::vector<RowDesc> rows;
        std::unordered_map<WlKey, int, WlKeyHash> cache;
        for (int i = 0; i < C; ++i) {
            for (long long w = R.off[i]; w < R.off[i + 1]; ++w) {
                if (R.count[w] == 0 || invalid[w]) continue;
                if (any_invalid && w != 0) continue;  // only the utopia row is evaluated
                WlKey key{};
                key.stage = i;
                std::memcpy(key.b, &R.stats[(size_t)w * 5], 40);
                auto it = cache.find(key);
                if (it != cache.end()) {
                    wl_row[w] = it->second;
                    continue;
                }
                RowDesc rd{};
                rd.stage = i;
                rd.space = i;
                rd.cls = 0;
                rd.dpmax = hs[i].min_gpus > 0 ? N / hs[i].min_gpus : 0;
                rd.rate = R.stats[(size_t)w * 5 + 0];
                rd.mean_in = R.stats[(size_t)w * 5 + 1];
                rd.mean_out = R.stats[(size_t)w * 5 + 2];
                rd.p95_in = R.stats[(size_t)w * 5 + 3];
                rd.p95_out = R.stats[(size_t)w * 5 + 4];
                const int id = (int)rows.size();
                rows.push_back(rd);
                cache.emplace(key, id);
                wl_row[w] = id;
            }
        }
        x.st.unique_rows = (long long)rows.size();

        CG_CUDA(cudaEventRecord(E->ev[4], x.s));
        evaluate_rows(x, rows, hs, *hw, *q, N);
        CG_CUDA(cudaEventRecord(E->ev[5], x.s));

        // utopia (outerplan.cpp:206-219)
        double z1 = dinf();
        x.d2h(&z1, static_cast<double*>(E->d_flat.p) + (size_t)wl_row[0] * (N + 1) + N, 8);
        x.sync();
        if (std::isinf(z1)) fail(CG_ERR_INFEASIBLE, "smallest model cannot be served within the budget");
        const double z2 = R.z2_qsum / static_cast<double>(t.n);
        if (any_invalid) {
            // first live invalid workload in candidate order (the reference's throw point)
            for (long long c = 0; c < ncand; ++c) {
                long long rem = c, tuple = 0, ts = 1;
                std::vector<int> gi(D);
                for (int d = D - 1; d >= 0; --d) {
                    gi[d] = (int)(rem % (long long)given[d].size());
                    rem /= (long long)given[d].size();
                }
                for (int d = 0; d < D; ++d) {
                    tuple += (long long)g2d[d][gi[d]] * ts;
                    ts *= R.G[d];
                }
                for (int i = 0; i < C; ++i) {
                    const long long w = R.off[i] + (i == 0 ? 0 : tuple % R.P[i]);
                    if (R.count[w] > 0 && invalid[w]) fail(CG_ERR_INVALID_INPUT, workload_problems(&R.stats[(size_t)w * 5]));
                }
            }
        }

        // ---- K6: min-max solve per distinct tuple
        int* dwlrow = E->d_wlrow.as<int>(R.total);
        x.h2d(dwlrow, wl_row.data(), wl_row.size() * sizeof(int));
        SolveArgs sa{};
        sa.C = C;
        sa.N = N;
        sa.total_gpus = N;
        sa.raw_f0 = 0;
        sa.ntuples = R.ntuples;
        for (int i = 0; i <= C; ++i) sa.wl_off[i] = R.off[i];
        for (int i = 0; i < C; ++i) sa.wl_P[i] = R.P[i];
        sa.wl_count = static_cast<unsigned long long*>(E->d_wcount.p);
        sa.wl_row = dwlrow;
        sa.final_lat = static_cast<double*>(E->d_flat.p);
        sa.final_plan = static_cast<long long*>(E->d_fplan.p);
        sa.feasible = E->d_tfeas.as<unsigned char>(R.ntuples);
        sa.L = E->d_tL.as<double>(R.ntuples);
        sa.alloc = E->d_talloc.as<int>((size_t)R.ntuples * C);
        sa.plan = E->d_tplan.as<long long>((size_t)R.ntuples * C);
        launch_solve(sa, x.s, &x.launches);

        // ---- grid-order expansion, compaction into evaluations / skipped
        ExpandArgs ea{};
        ea.D = D;
        ea.ncand = ncand;
        std::vector<int> g2d_flat;
        for (int d = 0; d < D; ++d) {
            ea.Gg[d] = (int)given[d].size();
            ea.Gd[d] = R.G[d];
            ea.goff[d] = (int)g2d_flat.size();
            g2d_flat.insert(g2d_flat.end(), g2d[d].begin(), g2d[d].end());
        }
        int* dg2d = E->d_g2d.as<int>(std::max<size_t>(1, g2d_flat.size()));
        x.h2d(dg2d, g2d_flat.data(), g2d_flat.size() * sizeof(int));
        ea.g2d = dg2d;
        ea.tuple_feasible = sa.feasible;
        ea.cand_tuple = E->d_ctuple.as<long long>(ncand);
        ea.flag = E->d_cflag.as<unsigned>(ncand);
        unsigned* pos = E->d_pos.as<unsigned>(ncand);
        unsigned long long* total = E->d_total.as<unsigned long long>(1);
        long long* ecand = E->d_ecand.as<long long>(ncand);
        double* eL = E->d_eL.as<double>(ncand);
        double* eQ = E->d_eQ.as<double>(ncand);
        long long* skip = E->d_skip.as<long long>(ncand);
        double* qsum = static_cast<double*>(E->d_qsum.p);
        launch_expand(ea, pos, total, sa.L, qsum, static_cast<double>(t.n), ecand, eL, eQ, skip, x.s, &x.launches);
        unsigned long long h_total = 0;
        x.d2h(&h_total, total, 8);
        x.sync();
        const long long nE = (long long)h_total;
        if (nE == 0) fail(CG_ERR_INFEASIBLE_PROBLEM, "sweep: every threshold candidate is infeasible");
        auto weights = weight_ladder(cfg->weight_ratio_min, cfg->weight_ratio_max, cfg->weight_count);
        const int nw = (int)weights.size() / 2;

        // ---- K7: Tchebycheff per weight + Pareto front
        double* dw = E->d_weights.as<double>(weights.size());
        x.h2d(dw, weights.data(), weights.size() * sizeof(double));
        int* sel = E->d_sel.as<int>(nw);
        launch_tchebycheff(eL, eQ, nE, dw, nw, z1, z2, sel, x.s, &x.launches);
        long long* front = E->d_front.as<long long>(nE);
        long long* fsize = E->d_fsize.as<long long>(1);
        launch_pareto(eL, eQ, nE, E->d_pk0.as<unsigned long long>(nE), E->d_pk1.as<unsigned long long>(nE),
                      E->d_pv0.as<unsigned long long>(nE), E->d_pv1.as<unsigned long long>(nE),
                      E->d_pkl.as<unsigned long long>(nE), E->d_orax.as<unsigned long long>(2),
                      E->d_rshist.as<unsigned int>(radix_hist_entries(nE)), front, fsize, x.s, &x.launches);
        CG_CUDA(cudaEventRecord(E->ev[6], x.s));

        // ---- results to host
        std::vector<long long> h_ecand(nE), h_ctuple(ncand), h_front, h_skip(ncand - nE);
        std::vector<double> h_eL(nE), h_eQ(nE);
        std::vector<int> h_sel(nw), h_alloc((size_t)R.ntuples * C);
        std::vector<long long> h_plan((size_t)R.ntuples * C);
        long long h_fsize = 0;
        x.d2h(h_ecand.data(), ecand, nE * 8);
        x.d2h(h_eL.data(), eL, nE * 8);
        x.d2h(h_eQ.data(), eQ, nE * 8);
        x.d2h(h_ctuple.data(), ea.cand_tuple, ncand * 8);
        x.d2h(h_skip.data(), skip, (ncand - nE) * 8);
        x.d2h(h_sel.data(), sel, nw * 4);
        x.d2h(h_alloc.data(), sa.alloc, h_alloc.size() * 4);
        x.d2h(h_plan.data(), sa.plan, h_plan.size() * 8);
        x.d2h(&h_fsize, fsize, 8);
        x.sync();
        h_front.resize(h_fsize);
        x.d2h(h_front.data(), front, h_fsize * 8);
        x.sync();
        float m_rows = 0, m_solve = 0;
        CG_CUDA(cudaEventElapsedTime(&m_rows, E->ev[4], E->ev[5]));
        CG_CUDA(cudaEventElapsedTime(&m_solve, E->ev[5], E->ev[6]));
        x.st.ms_rows += m_rows;
        x.st.ms_solve += m_solve;

        // ---- assemble SweepResult
        auto* r = static_cast<cg_sweep_result*>(std::calloc(1, sizeof(cg_sweep_result)));
        if (!r) throw std::bad_alloc();
        try {
            r->stages = C;
            r->z1_star = z1;
            r->z2_star = z2;
            r->num_evaluations = nE;
            std::vector<double> thr((size_t)nE * D), ratios((size_t)nE * C);
            std::vector<int32_t> alloc((size_t)nE * C);
            std::vector<int64_t> eplan((size_t)nE * C, -1);
            std::vector<cg_plan> plans;
            std::vector<cg_replica> reps;
            std::map<std::pair<int, long long>, int64_t> plan_ids;
            auto decode_thresholds = [&](long long c, double* dst) {
                long long rem = c;
                for (int d = D - 1; d >= 0; --d) {
                    const long long gi = rem % (long long)given[d].size();
                    rem /= (long long)given[d].size();
                    dst[d] = given[d][gi];
                }
            };
            for (long long e = 0; e < nE; ++e) {
                const long long c = h_ecand[e];
                const long long tu = h_ctuple[c];
                decode_thresholds(c, thr.data() + (size_t)e * D);
                for (int i = 0; i < C; ++i) {
                    const long long w = R.off[i] + (i == 0 ? 0 : tu % R.P[i]);
                    ratios[(size_t)e * C + i] = static_cast<double>(R.count[w]) / static_cast<double>(t.n);
                    alloc[(size_t)e * C + i] = h_alloc[(size_t)tu * C + i];
                    const long long p = h_plan[(size_t)tu * C + i];
                    if (p >= 0) {
                        auto key = std::make_pair(i, p);
                        auto it = plan_ids.find(key);
                        if (it == plan_ids.end()) {
                            cg_plan cp;
                            expand_plan(hs[i], p, reps, cp);
                            it = plan_ids.emplace(key, (int64_t)plans.size()).first;
                            plans.push_back(cp);
                        }
                        eplan[(size_t)e * C + i] = it->second;
                    }
                }
            }
            std::vector<int64_t> ec(h_ecand.begin(), h_ecand.end());
            r->eval_candidate = hcopy(ec);
            r->eval_thresholds = hcopy(thr);
            r->eval_latency = hcopy(h_eL);
            r->eval_quality = hcopy(h_eQ);
            r->eval_ratios = hcopy(ratios);
            r->eval_allocations = hcopy(alloc);
            r->eval_plan = hcopy(eplan);
            r->num_plans = (int64_t)plans.size();
            r->plans = hcopy(plans);
            r->num_replicas = (int64_t)reps.size();
            r->replicas = hcopy(reps);
            r->num_weights = nw;
            r->weights = hcopy(weights);
            std::vector<int32_t> selv(h_sel.begin(), h_sel.end());
            r->weight_selection = hcopy(selv);
            r->front_size = h_fsize;
            std::vector<int64_t> fr(h_front.begin(), h_front.end());
            r->front = hcopy(fr);
            r->num_skipped = ncand - nE;
            std::vector<int64_t> sk(h_skip.begin(), h_skip.end());
            std::vector<double> skt((size_t)sk.size() * D);
            for (size_t i = 0; i < sk.size(); ++i) decode_thresholds(sk[i], skt.data() + i * D);
            r->skipped_candidate = hcopy(sk);
            r->skipped_thresholds = hcopy(skt);
            x.st.num_ranks = E->world;
            x.st.gpu_launches = x.launches;
            x.st.ms_total = timer.ms();
            r->stats = x.st;
        } catch (...) {
            free_result(r);
            throw;
        }
        *out = r;
    });
}

void cg_sweep_result_free(cg_sweep_result* r) { free_result(r); }

cg_status cg_route(cg_engine* E, const cg_trace* tr, const double* thresholds, const int32_t* deployed,
                   cg_route_result* out, int32_t* accept_stage) {
    E = primary(E);
    return guarded([&] {
        if (!E || !tr || !out) fail(CG_ERR_INVALID_INPUT, "null argument");
        CG_CUDA(cudaSetDevice(E->device));
        SweepCtx x(*E);
        const int C = tr->stages;
        if (tr->n <= 0) fail(CG_ERR_EMPTY_TRACE, "route_trace: empty trace");
        int last = -1;
        for (int i = C - 1; i >= 0; --i)
            if (deployed[i]) {
                last = i;
                break;
            }
        if (last < 0) fail(CG_ERR_NO_DEPLOYED_STAGE, "route_trace: no deployed stage");
        if (C <= 0) fail(CG_ERR_INVALID_INPUT, "route_trace: thresholds length != C-1");
        if (C > kMaxStages) fail(CG_ERR_UNSUPPORTED, "GPU engine supports up to 5 cascade stages");
        TraceDev t = trace_to_device(x, *tr);
        const double rate = overall_rate(t);
        const int D = C - 1;
        // Deployment mask folded into one threshold per dimension: undeployed
        // stages never accept (+inf), the last deployed stage accepts all (-inf).
        std::vector<std::vector<double>> one(D);
        std::vector<double> eff(std::max(1, D));
        for (int d = 0; d < D; ++d) {
            double h = thresholds[d];
            if (!deployed[d]) h = dinf();
            if (d == last) h = -dinf();
            if (d > last) h = -dinf();
            eff[d] = h;
            one[d] = {h};
        }
        RoutingOut R = route_all(x, t, one, rate, nullptr);
        out->stages = C;
        for (int i = 0; i < C && i < 8; ++i) {
            const long long w = R.off[i];  // single prefix (all m_d = 0)
            const bool reached = deployed[i] && i <= last;
            out->ratios[i] = reached ? static_cast<double>(R.count[w]) / static_cast<double>(t.n) : 0.0;
            if (reached) {
                out->stage_workloads[i] = {R.stats[(size_t)w * 5 + 0], R.stats[(size_t)w * 5 + 1],
                                           R.stats[(size_t)w * 5 + 2], R.stats[(size_t)w * 5 + 3],
                                           R.stats[(size_t)w * 5 + 4]};
            } else {
                out->stage_workloads[i] = {rate * 0.0, 0, 0, 0, 0};
            }
        }
        // quality of the single tuple
        double qs = 0;
        x.d2h(&qs, E->d_qsum.p, 8);
        x.sync();
        out->quality = qs / static_cast<double>(t.n);
        if (accept_stage) {
            double* dh = E->d_misc.as<double>(std::max(1, C));
            int* ddep = E->d_dep.as<int>(std::max(1, C));
            int* dout = E->d_accept.as<int>((size_t)t.n);
            std::vector<double> hh(thresholds, thresholds + D);
            hh.resize(std::max(1, C), 0.0);
            std::vector<int> dep(deployed, deployed + C);
            x.h2d(dh, hh.data(), hh.size() * 8);
            x.h2d(ddep, dep.data(), dep.size() * 4);
            k_accept_stage<<<(unsigned)((t.n + 255) / 256), 256, 0, x.s>>>(t.scores, t.n, C, dh, last, ddep, dout);
            CG_LAUNCH_CHECK();
            x.d2h(accept_stage, dout, (size_t)t.n * 4);
            x.sync();
        }
    });
}

cg_status cg_route_grid(cg_engine* E, const cg_trace* tr, const cg_sweep_config* cfg, cg_route_grid_result** out) {
    E = primary(E);
    return guarded([&] {
        Timer timer;
        if (out) *out = nullptr;
        if (!E || !tr || !cfg || !out) fail(CG_ERR_INVALID_INPUT, "null argument");
        CG_CUDA(cudaSetDevice(E->device));
        SweepCtx x(*E);
        if (tr->n <= 0) fail(CG_ERR_EMPTY_TRACE, "route_trace: empty trace");
        const int C = tr->stages;
        if (C < 1 || C > kMaxStages) fail(CG_ERR_UNSUPPORTED, "GPU engine supports up to 5 cascade stages");
        TraceDev t = trace_to_device(x, *tr);
        const double rate = overall_rate(t);
        const int D = C - 1;
        std::vector<std::vector<double>> given;
        if (cfg->grid_dims == 0) {
            given = default_grid(x, t);
        } else {
            long long off = 0;
            for (int d = 0; d < cfg->grid_dims; ++d) {
                given.emplace_back(cfg->grid_values + off, cfg->grid_values + off + cfg->grid_sizes[d]);
                off += cfg->grid_sizes[d];
            }
        }
        if ((int)given.size() != D) fail(CG_ERR_INVALID_INPUT, "route_trace: thresholds length != C-1");
        for (const auto& dim : given)
            if (dim.empty()) fail(CG_ERR_INVALID_INPUT, "sweep: empty threshold grid dimension");
        std::vector<std::vector<double>> distinct(D);
        std::vector<std::vector<int>> g2d(D);
        for (int d = 0; d < D; ++d) {
            distinct[d] = given[d];
            std::sort(distinct[d].begin(), distinct[d].end());
            distinct[d].erase(std::unique(distinct[d].begin(), distinct[d].end()), distinct[d].end());
            for (double v : given[d])
                g2d[d].push_back(
                    (int)(std::lower_bound(distinct[d].begin(), distinct[d].end(), v) - distinct[d].begin()));
        }
        RoutingOut R = route_all(x, t, distinct, rate, nullptr);
        std::vector<double> qsum(R.ntuples);
        x.d2h(qsum.data(), E->d_qsum.p, qsum.size() * 8);
        x.sync();
        long long ncand = 1;
        for (int d = 0; d < D; ++d) ncand *= (long long)given[d].size();
        auto* r = static_cast<cg_route_grid_result*>(std::calloc(1, sizeof(cg_route_grid_result)));
        r->stages = C;
        r->num_candidates = ncand;
        std::vector<double> thr((size_t)ncand * D), ratios((size_t)ncand * C), q(ncand);
        std::vector<cg_workload> wl((size_t)ncand * C);
        for (long long c = 0; c < ncand; ++c) {
            long long rem = c, tuple = 0, ts = 1;
            std::vector<int> gi(D);
            for (int d = D - 1; d >= 0; --d) {
                gi[d] = (int)(rem % (long long)given[d].size());
                rem /= (long long)given[d].size();
            }
            for (int d = 0; d < D; ++d) {
                thr[(size_t)c * D + d] = given[d][gi[d]];
                tuple += (long long)g2d[d][gi[d]] * ts;
                ts *= R.G[d];
            }
            for (int i = 0; i < C; ++i) {
                const long long w = R.off[i] + (i == 0 ? 0 : tuple % R.P[i]);
                ratios[(size_t)c * C + i] = static_cast<double>(R.count[w]) / static_cast<double>(t.n);
                const double* s = &R.stats[(size_t)w * 5];
                wl[(size_t)c * C + i] = {s[0], s[1], s[2], s[3], s[4]};
            }
            q[c] = qsum[tuple] / static_cast<double>(t.n);
        }
        r->thresholds = hcopy(thr);
        r->ratios = hcopy(ratios);
        r->workloads = hcopy(wl);
        r->quality = hcopy(q);
        x.st.candidates = ncand;
        x.st.distinct_candidates = R.ntuples;
        x.st.gpu_launches = x.launches;
        x.st.ms_total = timer.ms();
        r->stats = x.st;
        *out = r;
    });
}

void cg_route_grid_result_free(cg_route_grid_result* r) {
    if (!r) return;
    std::free(r->thresholds);
    std::free(r->ratios);
    std::free(r->workloads);
    std::free(r->quality);
    std::free(r);
}

// Host-side shard merge with the device merge's rule (merge_take): per budget
// the best (latency, plan) over all shards, then the reference's prefix
// minimum.  No GPU needed; used by the multi-rank CPU tests.
cg_status cg_merge_row_shards(const cg_model* model, const cg_hardware* hw, const cg_cost_params* q,
                              int32_t max_budget, int32_t shards, const uint64_t* lat_bits,
                              const uint64_t* plan_index, cg_row_result** out) {
    return guarded([&] {
        if (out) *out = nullptr;
        if (!model || !hw || !q || !lat_bits || !plan_index || !out || shards < 1 || max_budget < 0)
            fail(CG_ERR_INVALID_INPUT, "invalid merge arguments");
        const int N = max_budget;
        HostPlanSpace hs;
        hs.build(legal_shapes(*model, *hw, *q), N);
        PlanSpace sp;
        std::memset(&sp, 0, sizeof(sp));
        sp.S = (int)hs.shapes.size();
        sp.N = N;
        for (int k = 0; k < sp.S; ++k) sp.shapes[k] = hs.shapes[k];
        sp.ways = hs.ways.data();
        sp.num_plans = hs.num_plans;
        auto* r = static_cast<cg_row_result*>(std::calloc(1, sizeof(cg_row_result)));
        r->max_budget = N;
        r->latency = static_cast<double*>(std::malloc(sizeof(double) * (N + 1)));
        r->plan_index = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (N + 1)));
        std::vector<cg_plan> plans;
        std::vector<cg_replica> reps;
        std::map<unsigned long long, int64_t> ids;
        double running = dinf();
        unsigned long long run_plan = ~0ull;
        r->latency[0] = dinf();
        r->plan_index[0] = -1;
        for (int g = 1; g <= N; ++g) {
            unsigned long long bl = kInfBits, bp = ~0ull;
            for (int s = 0; s < shards; ++s) {
                const unsigned long long l = lat_bits[(size_t)s * (N + 1) + g];
                const unsigned long long p = plan_index[(size_t)s * (N + 1) + g];
                if (merge_take(sp, l, p, bl, bp)) {
                    bl = l;
                    bp = p;
                }
            }
            if (bp != ~0ull) {
                double l;
                std::memcpy(&l, &bl, 8);
                if (l < running) {
                    running = l;
                    run_plan = bp;
                }
            }
            r->latency[g] = running;
            r->plan_index[g] = -1;
            if (run_plan != ~0ull) {
                auto it = ids.find(run_plan);
                if (it == ids.end()) {
                    cg_plan cp;
                    expand_plan(hs, (long long)run_plan, reps, cp);
                    it = ids.emplace(run_plan, (int64_t)plans.size()).first;
                    plans.push_back(cp);
                }
                r->plan_index[g] = it->second;
            }
        }
        r->num_plans = (int64_t)plans.size();
        r->plans = hcopy(plans);
        r->num_replicas = (int64_t)reps.size();
        r->replicas = hcopy(reps);
        *out = r;
    });
}

/* Plan ranges a rank evaluates: the host restatement of k_plan_filter's chunk
 * mapping (shard_global_chunk, shared with the kernel) over the same chunk
 * list evaluate_rows builds (rows with plans, 64-plan chunks, reversed). */
int64_t cg_shard_row_plans(const uint64_t* num_plans, int32_t nrows, int32_t row, int32_t rank, int32_t world,
                           uint64_t* ranges, int64_t cap) {
    if (!num_plans || nrows < 1 || row < 0 || row >= nrows || world < 1 || rank < 0 || rank >= world) return -1;
    const unsigned long long chunk = 64;
    unsigned long long first = 0;  // chunk_prefix of `row`
    for (int r = 0; r < row; ++r) first += (num_plans[r] + chunk - 1) / chunk;
    const unsigned long long P = num_plans[row], nrc = (P + chunk - 1) / chunk;
    unsigned long long total = first + nrc;
    for (int r = row + 1; r < nrows; ++r) total += (num_plans[r] + chunk - 1) / chunk;
    const unsigned long long mine = shard_count(total, rank, world);
    std::vector<std::pair<unsigned long long, unsigned long long>> out;
    // local chunks whose global chunk lies in [first, first + nrc)
    unsigned long long l0 = first > (unsigned long long)rank ? (first - rank + world - 1) / world : 0;
    for (unsigned long long l = l0; l < mine; ++l) {
        const unsigned long long g = shard_global_chunk(l, rank, world);
        if (g >= first + nrc) break;
        const unsigned long long j = nrc - 1 - (g - first);
        out.emplace_back(j * chunk, std::min(j * chunk + chunk, P));
    }
    std::sort(out.begin(), out.end());
    for (size_t i = 0; i < out.size() && (int64_t)i < cap; ++i) {
        ranges[2 * i] = out[i].first;
        ranges[2 * i + 1] = out[i].second;
    }
    return (int64_t)out.size();
}

/* Per-budget reduction of shard bests with merge_take (the rule of the
 * device's atomicMin + tie resolve and of k_merge_ranks), no prefix minimum. */
cg_status cg_merge_budget_bests(const cg_model* model, const cg_hardware* hw, const cg_cost_params* q,
                                int32_t max_budget, int32_t shards, const uint64_t* lat_bits,
                                const uint64_t* plan_index, uint64_t* lat_out, uint64_t* plan_out) {
    return guarded([&] {
        if (!model || !hw || !q || !lat_bits || !plan_index || !lat_out || !plan_out || shards < 1 || max_budget < 0)
            fail(CG_ERR_INVALID_INPUT, "invalid merge arguments");
        const int N = max_budget;
        HostPlanSpace hs;
        hs.build(legal_shapes(*model, *hw, *q), N);
        PlanSpace sp;
        std::memset(&sp, 0, sizeof(sp));
        sp.S = (int)hs.shapes.size();
        sp.N = N;
        for (int k = 0; k < sp.S; ++k) sp.shapes[k] = hs.shapes[k];
        sp.ways = hs.ways.data();
        sp.num_plans = hs.num_plans;
        for (int g = 0; g <= N; ++g) {
            unsigned long long bl = kInfBits, bp = ~0ull;
            for (int s = 0; s < shards; ++s) {
                const unsigned long long l = lat_bits[(size_t)s * (N + 1) + g];
                const unsigned long long p = plan_index[(size_t)s * (N + 1) + g];
                if (merge_take(sp, l, p, bl, bp)) {
                    bl = l;
                    bp = p;
                }
            }
            lat_out[g] = bl;
            plan_out[g] = bp;
        }
    });
}

cg_status cg_stage_row(cg_engine* E, const cg_model* model, const cg_workload* w, const cg_hardware* hw,
                       const cg_cost_params* q, int32_t max_budget, cg_row_result** out) {
    if (E && E->group) {
        if (!out) return err_status(CG_ERR_INVALID_INPUT, "null argument");
        return run_group(E, out, [&](cg_engine* m, cg_row_result** o) {
            return cg_stage_row(m, model, w, hw, q, max_budget, o);
        }, cg_row_result_free);
    }
    return guarded([&] {
        if (out) *out = nullptr;
        if (!E || !model || !w || !hw || !q || !out) fail(CG_ERR_INVALID_INPUT, "null argument");
        CG_CUDA(cudaSetDevice(E->device));
        Timer timer;
        SweepCtx x(*E);
        validate_hw(*hw);
        validate_params(*q);
        const double ws[5] = {w->arrival_rate, w->mean_input_tokens, w->mean_output_tokens, w->p95_input_tokens,
                              w->p95_output_tokens};
        const std::string prob = workload_problems(ws);
        if (!prob.empty()) fail(CG_ERR_INVALID_INPUT, prob);
        if (max_budget < 0) fail(CG_ERR_INVALID_INPUT, "row: max_budget must be >= 0");
        const int N = max_budget;
        auto* r = static_cast<cg_row_result*>(std::calloc(1, sizeof(cg_row_result)));
        r->max_budget = N;
        r->latency = static_cast<double*>(std::malloc(sizeof(double) * (N + 1)));
        r->plan_index = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (N + 1)));
        std::vector<cg_plan> plans;
        std::vector<cg_replica> reps;
        for (int f = 0; f <= N; ++f) {
            r->latency[f] = w->arrival_rate == 0.0 ? 0.0 : dinf();
            r->plan_index[f] = -1;
        }
        if (w->arrival_rate != 0.0 && N >= 1) {
            cg_model m = *model;
            auto hs = build_spaces(x, &m, 1, *hw, *q, N);
            std::vector<RowDesc> rows(1);
            rows[0] = RowDesc{0, 0, 0, hs[0].min_gpus > 0 ? N / hs[0].min_gpus : 0,
                              ws[0], ws[1], ws[2], ws[3], ws[4]};
            evaluate_rows(x, rows, hs, *hw, *q, N);
            std::vector<double> lat(N + 1);
            std::vector<long long> pl(N + 1);
            x.d2h(lat.data(), E->d_flat.p, (N + 1) * 8);
            x.d2h(pl.data(), E->d_fplan.p, (N + 1) * 8);
            x.sync();
            std::map<long long, int64_t> ids;
            for (int f = 0; f <= N; ++f) {
                r->latency[f] = lat[f];
                if (pl[f] >= 0) {
                    auto it = ids.find(pl[f]);
                    if (it == ids.end()) {
                        cg_plan cp;
                        expand_plan(hs[0], pl[f], reps, cp);
                        it = ids.emplace(pl[f], (int64_t)plans.size()).first;
                        plans.push_back(cp);
                    }
                    r->plan_index[f] = it->second;
                }
            }
        }
        r->num_plans = (int64_t)plans.size();
        r->plans = hcopy(plans);
        r->num_replicas = (int64_t)reps.size();
        r->replicas = hcopy(reps);
        x.st.gpu_launches = x.launches;
        x.st.unique_rows = 1;
        x.st.ms_total = timer.ms();
        r->stats = x.st;
        *out = r;
    });
}

void cg_row_result_free(cg_row_result* r) {
    if (!r) return;
    std::free(r->latency);
    std::free(r->plan_index);
    std::free(r->plans);
    std::free(r->replicas);
    std::free(r);
}

cg_status cg_solve_min_max(cg_engine* E, const double* entries, int32_t stages, int32_t gpu_budget,
                           int32_t total_gpus, int32_t* allocations, double* per_stage_latency,
                           double* objective_L) {
    E = primary(E);
    return guarded([&] {
        if (!E || !entries) fail(CG_ERR_INVALID_INPUT, "null argument");
        CG_CUDA(cudaSetDevice(E->device));
        SweepCtx x(*E);
        // validate_table (innerplan.cpp:58-93)
        const int n = gpu_budget;
        if (n < 0) fail(CG_ERR_INVALID_INPUT, "latency table: negative budget");
        if (stages <= 0) fail(CG_ERR_INVALID_INPUT, "latency table: no stages");
        for (int i = 0; i < stages; ++i) {
            bool seen = false;
            double prev = dinf();
            for (int f = 0; f <= n; ++f) {
                const double cell = entries[(size_t)i * (n + 1) + f];
                if (std::isinf(cell)) {
                    if (seen && f > 0) fail(CG_ERR_INVALID_INPUT, "latency table: feasibility not upward-closed");
                    continue;
                }
                if (cell < 0.0) fail(CG_ERR_INVALID_INPUT, "latency table: negative latency");
                if (seen && cell > prev) fail(CG_ERR_INVALID_INPUT, "latency table: row not non-increasing");
                seen = true;
                prev = cell;
            }
        }
        if (total_gpus < 0 || total_gpus > gpu_budget)
            fail(CG_ERR_INVALID_INPUT, "solve_min_max: budget outside table range");
        if (stages > kMaxStages) fail(CG_ERR_UNSUPPORTED, "GPU engine supports up to 5 cascade stages");
        const size_t cells = (size_t)stages * (n + 1);
        double* dlat = E->d_flat.as<double>(cells);
        long long* dplan = E->d_fplan.as<long long>(cells);
        x.h2d(dlat, entries, cells * 8);
        CG_CUDA(cudaMemsetAsync(dplan, 0xff, cells * 8, x.s));
        std::vector<unsigned long long> cnt(stages, 1);
        std::vector<int> rowid(stages);
        for (int i = 0; i < stages; ++i) rowid[i] = i;
        unsigned long long* dcnt = E->d_wcount.as<unsigned long long>(stages);
        int* drow = E->d_wlrow.as<int>(stages);
        x.h2d(dcnt, cnt.data(), stages * 8);
        x.h2d(drow, rowid.data(), stages * 4);
        SolveArgs sa{};
        sa.C = stages;
        sa.N = n;
        sa.total_gpus = total_gpus;
        sa.raw_f0 = 1;
        sa.ntuples = 1;
        for (int i = 0; i <= stages; ++i) sa.wl_off[i] = i;
        for (int i = 0; i < stages; ++i) sa.wl_P[i] = 1;
        sa.wl_count = dcnt;
        sa.wl_row = drow;
        sa.final_lat = dlat;
        sa.final_plan = dplan;
        sa.feasible = E->d_tfeas.as<unsigned char>(1);
        sa.L = E->d_tL.as<double>(1);
        sa.alloc = E->d_talloc.as<int>(stages);
        sa.plan = E->d_tplan.as<long long>(stages);
        launch_solve(sa, x.s, &x.launches);
        unsigned char feas = 0;
        double L = 0;
        std::vector<int> al(stages);
        x.d2h(&feas, sa.feasible, 1);
        x.d2h(&L, sa.L, 8);
        x.d2h(al.data(), sa.alloc, stages * 4);
        x.sync();
        if (!feas) fail(CG_ERR_INFEASIBLE_PROBLEM, "no allocation satisfies the GPU budget");
        for (int i = 0; i < stages; ++i) {
            if (allocations) allocations[i] = al[i];
            if (per_stage_latency) per_stage_latency[i] = entries[(size_t)i * (n + 1) + al[i]];
        }
        if (objective_L) *objective_L = L;
    });
}

}  // extern "C"
