// Kernel argument blocks and host-side launchers (implemented in k_*.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

#include "cg_internal.h"

namespace cg {

// ---------------- routing (k_route.cu)
struct RouteArgs {
    long long n;
    const double* scores;  // [C][n]
    const double* in;      // [n]
    const double* out;     // [C][n]
    const double* gvals;   // distinct sorted grid values, concatenated
    int goff[4];
    int G[4];
    int gtotal;
    int grid_in_smem;
    long long stride[4];   // histogram strides (dim 0 fastest, extent G+1)
    unsigned long long* ranks;  // [n] packed 16-bit ranks
    unsigned long long* hist;   // [cells][2+C]
    unsigned int* flags;        // bit0: a token is not an integer in [0, 2^32)
    long long cells;
    int gtop[4];                   // highest power of two <= G (branch-free rank search)
    long long marg_off[4];         // word offset of the stage-i output-sum marginal (i < C-1)
    long long priv_words;          // 3*cells + sum of marginal sizes
    unsigned long long* partials;  // [blocks][priv_words] block-private histograms (or null)
    long long max_partials;        // capacity of `partials` in blocks
    unsigned long long* acc;       // [priv_words] global accumulator (non-private path)
    unsigned long long* tile_partials;  // [blocks][cells][2+C] for the tiled form (or null)
    // u32 form (k_route_hist): block-private u32 [cells][2+C] partials, the
    // high 16 bits of tokens >= 2^16 accumulated in hi_acc (u64 [cells][2+C])
    unsigned int* part32;
    long long part32_words;        // capacity of part32
    unsigned long long* hi_acc;
    int bin_ok;                    // grid has no NaN: binned exact rank search allowed
    int k1_form;                   // variant selector (engine option k1_form)
};
size_t tile_smem_bytes(long long cells, int D, int gtotal);

struct WorkloadArgs {
    int C;
    long long total;        // sum over stages of P_i
    long long wl_off[kMaxStages + 1];
    int G[4];
    long long stride[4];
    const unsigned long long* hist;
    unsigned long long* count;
    unsigned long long* sum_in;
    unsigned long long* sum_out;
};

void launch_route_aggregate(const RouteArgs& a, int D, int sm_count, cudaStream_t s, int* launches,
                            int* nblocks_out);
void launch_hist_expand(const RouteArgs& a, int C, int nblocks, cudaStream_t s, int* launches);
void launch_hist_scan(unsigned long long* hist, long long cells, int Q, const long long* stride,
                      const int* G, int D, cudaStream_t s, int* launches);
void launch_workload_counts(const WorkloadArgs& a, cudaStream_t s, int* launches);
void launch_workload_seq_sums(const WorkloadArgs& a, const unsigned long long* ranks, const double* in,
                              const double* out, long long n, double* sum_in_f, double* sum_out_f,
                              cudaStream_t s, int* launches);
void launch_make_lists(const double* in, const double* out, const unsigned long long* ranks, long long n,
                       int C, unsigned long long* keys, unsigned long long* vals, int sm_count,
                       cudaStream_t s, int* launches);
// tables: u16 chunk tables (p95_table_entries entries; 0 = the direct scan)
long long p95_table_entries(const WorkloadArgs& a, long long n);
void launch_p95_scan(const WorkloadArgs& a, const unsigned long long* keys, const unsigned long long* vals,
                     long long n, double* p95_in, double* p95_out, unsigned short* tables, cudaStream_t s,
                     int* launches);
void launch_workload_stats(const WorkloadArgs& a, long long n, double rate, int integral,
                           const double* sum_in_f, const double* sum_out_f, const double* p95_in,
                           const double* p95_out, double* stats, cudaStream_t s, int* launches);
// K2 scratch for the block-parallel exact quality sums (entries = tuples x blocks)
struct QualityScratch {
    int B;                          // requests per block (quality_block)
    double* A;                      // approximate block sums
    short* E;                       // binade per block, -1 = sequential
    unsigned long long* U;          // units of 2^(e-52) per block
    unsigned long long* seq_blocks; // optional counter of sequentially folded blocks
};
int quality_block(long long n, long long ncand);
void launch_quality(const double* scores, long long n, int D, const double* thr, long long ncand,
                    double* qsum, const QualityScratch* q, cudaStream_t s, int* launches);

// ---------------- sort (k_sort.cu)
void launch_or_and(const unsigned long long* keys, long long n, unsigned long long* out2, cudaStream_t s,
                   int* launches);
// Returns 1 when the sorted data ended in the *_tmp buffers.
int radix_sort_u64(unsigned long long* keys, unsigned long long* vals, unsigned long long* keys_tmp,
                   unsigned long long* vals_tmp, long long n, unsigned long long varying_bits,
                   unsigned int* hist_scratch, cudaStream_t s, int* launches);
size_t radix_hist_entries(long long n);

// ---------------- cost model (k_cost.cu)
struct ModelArgs {
    double param_count, bytes_per_param, kv_bytes_per_token;
};
struct HwArgs {
    double flops, mem_bandwidth, mem_capacity;
};
struct ParamArgs {
    double prefill_efficiency, decode_bw_efficiency, pipeline_bubble_factor, comm_overhead_per_stage,
        kv_memory_fraction;
};

struct RowSetupArgs {
    int nrows;
    int n_req;
    const RowDesc* rows;
    const PlanSpace* spaces;
    const ModelArgs* models;
    HwArgs hw;
    ParamArgs p;
    RowTables tab;
};

enum : int { CTR_STABLE = 0, CTR_FULL = 1, CTR_PRUNED = 2, CTR_STEPS = 3, CTR_BOUND = 4, CTR_SEED = 5,
             CTR_COUNT = 8 };
enum : int { SIM_RANGE = 0, SIM_LIST = 1, SIM_DEEP = 2 };

// Bits of the filter's order key (top bits of the sortable estimate) the lists are sorted by.
constexpr int kListKeyBits = 16;

// Work items: (row << 44) | plan index.
constexpr int kItemPlanBits = 44;
constexpr unsigned long long kItemPlanMask = (1ull << kItemPlanBits) - 1ull;

// A filtered work item: the plan and everything a JSQ kernel needs to start
// it without unranking or table walks (k_plan_filter writes, k_lane/k_sim read).
//   w[0..2]: a 192-bit little-endian bit stream -- bits 0-3 the number of
//            parts np (0: more than kRecMaxParts parts, unrank instead), bits
//            4-12 the GPUs used, then np fields of 13 bits (5-bit shape index
//            | 8-bit replica count << 5) in ascending shape order;
//   lb:      the exact service-time lower bound of the plan's K-th largest
//            sojourn (k_plan_filter's header comment), already with its
//            1e-12 margins: sojourns below it never reach the p95.
constexpr int kRecMaxParts = 13;
// request-steps per k_lane trip (prune checks every SimArgs::lane_check + 1
// trips).  One trip per 32-step check interval: the per-trip bookkeeping
// (claim/finish votes, the bound broadcast, check set-up) is paid once per
// check (C3 K4: 4-step trips 265 ms, 8: 250, 16: 242, 32: 238)
#ifndef CG_UNROLL
#define CG_UNROLL 32
#endif
constexpr int kLaneUnroll = CG_UNROLL;
struct ItemRec {
    unsigned long long item;   // (row << 44) | plan index
    unsigned long long w[3];
    double lb;
};

struct SimArgs {
    int N, n_req, K, prune;
    int kstar;                                 // index of the K-th largest CRN output
    int check_stable;                          // 1: items are not pre-filtered (seeds)
    unsigned lane_check;                       // k_lane: prune checks every 4(lane_check+1) request-steps
    int seeds;                                 // 1: count completions as seeding work
    const unsigned long long* items;           // packed (row, plan) work items (when recs == nullptr)
    const ItemRec* recs;                       // filtered items with parts and bound (else nullptr)
    const unsigned long long* perm;            // optional: item i is items/recs[perm[i]] (sorted lists)
    unsigned long long nitems;
    unsigned long long* item_counter;
    const RowDesc* rows;
    const PlanSpace* spaces;
    RowTables tab;
    unsigned long long* lat_min;               // [row][N+1] latency bits, exact per-budget min
    unsigned long long* ub;                    // [row][N+1] prefix-min bound for pruning
    TieEntry* ties;
    unsigned long long* tie_count;
    unsigned long long tie_cap;
    unsigned long long* ovf;                   // packed items whose smem ring overflowed
    unsigned long long* ovf_count;
    unsigned long long ovf_cap;
    double* scratch;                           // [slots][sld]
    int sld;                                   // scratch column stride: n_req rounded up to 4
    double* ring_global;                       // DEEP: [warps][32*R*ring_cap]
    int ring_cap;
    unsigned long long* counters;
    // future-service bound snapshot: qtab[(row*(N+1) + g)*32 + s] = number of
    // leading output-ranked request blocks whose every request's service on
    // shape s exceeds ub[row][g] as it was when the table was built
    // (k_fut_snapshot); a plan's count is the minimum over its shapes
    const unsigned short* qtab;
};

// Future-bound snapshot (see SimArgs::qtab).
struct FutSnapArgs {
    int nrows, N, n_req;
    const RowDesc* rows;
    const PlanSpace* spaces;
    RowTables tab;
    const unsigned long long* ub;
    unsigned short* qtab;
};
void launch_fut_snapshot(const FutSnapArgs& a, cudaStream_t s, int* launches);

struct FilterArgs {
    int N, n_req, kstar, prune;
    int nrows;                                 // rows with plans
    const int* row_ids;
    const unsigned long long* chunk_prefix;    // [nrows+1] cumulative chunk counts per row
    unsigned long long chunk_base;             // first chunk of this launch (waves / rank shard)
    unsigned long long nchunks;                // chunks in this launch
    int shard_rank, shard_world;               // local chunk l is global chunk l*world + rank (0, 1: unsharded)
    int chunk;                                 // plans per chunk
    const RowDesc* rows;
    const PlanSpace* spaces;
    RowTables tab;
    const unsigned long long* ub;
    ItemRec* recs[7];                          // listed plans (ItemRec)
    unsigned long long* keys[7];               // coarse service-bound order keys
    unsigned long long* list_count;            // [7]
    unsigned long long list_caps[7];           // per class
    unsigned long long* counters;
    unsigned long long* pilot;                 // optional [row][N+1]: (estimate20 << 44 | plan) minimum
    int pilot_only;                            // 1: only the pilot minima (no lists, no counters)
    unsigned long long pilot_min_plans;        // rows with fewer plans get no pilot
    int sort_key;                              // list order: 0 service bound, 1 estimate
};

// Pilot lists: the best-estimate plan of every (row, budget) cell, by class.
struct PilotArgs {
    long long cells;
    int N;
    const unsigned long long* pilot;
    const RowDesc* rows;
    const PlanSpace* spaces;
    unsigned long long* lists[7];
    unsigned long long* keys[7];               // the items' estimate (order key)
    unsigned long long* list_count;            // [7]
    int merge;                                 // 0: native classes, 1: class 0 + {1,2,3} -> 3, 2: {0..3} -> 3
};
void launch_pilot_lists(const PilotArgs& a, cudaStream_t s, int* launches);

struct SimGeometry {
    int W, R, G, grid;
    long long slots, warps;
};

int class_for_dp(int dpmax);
void set_k4_pack(int p);
void class_shape(int cls, int* W, int* R);
void class_dp_range(int cls, int* lo, int* hi);
SimGeometry sim_geometry(int cls, int mode, int sm_count);
void launch_row_setup(const RowSetupArgs& a, const double* L, cudaStream_t s, int* launches);
void launch_row_svck(const RowTables& tab, int nrows, int kstar, cudaStream_t s, int* launches);
void launch_plan_filter(const FilterArgs& a, cudaStream_t s, int* launches);
void launch_sim(const SimArgs& a, int cls, int mode, int sm_count, cudaStream_t s, int* launches,
                int* grid_out);

struct ResolveArgs {
    int N, nrows;
    unsigned long long nties;
    const TieEntry* ties;
    const RowDesc* rows;
    const PlanSpace* spaces;
    const unsigned long long* lat_min;
    unsigned long long* best_plan;   // [row][N+1], ~0 = empty
    double* final_lat;               // [row][N+1]
    long long* final_plan;           // [row][N+1]
};
void launch_resolve(const ResolveArgs& a, cudaStream_t s, int* launches);

// ---------------- solve (k_solve.cu)
struct SolveArgs {
    int C, N, total_gpus;
    int raw_f0;              // 1: use cell f=0 as given (standalone solve)
    long long ntuples;
    long long wl_off[kMaxStages + 1];
    long long wl_P[kMaxStages];
    const unsigned long long* wl_count;
    const int* wl_row;
    const double* final_lat;
    const long long* final_plan;
    unsigned char* feasible;
    double* L;
    int* alloc;        // [t][C]
    long long* plan;   // [t][C]
};
void launch_solve(const SolveArgs& a, cudaStream_t s, int* launches);

struct ExpandArgs {
    int D;
    long long ncand;
    int Gg[4];               // given grid sizes
    int Gd[4];               // distinct sizes
    int goff[4];             // offsets into g2d
    const int* g2d;          // given index -> distinct index
    const unsigned char* tuple_feasible;
    long long* cand_tuple;
    unsigned* flag;
};
void launch_expand(const ExpandArgs& a, unsigned* pos, unsigned long long* total, const double* tuple_L,
                   const double* tuple_qsum, double n, long long* eval_cand, double* eval_L,
                   double* eval_Q, long long* skip_cand, cudaStream_t s, int* launches);
void launch_tchebycheff(const double* L, const double* Q, long long E, const double* weights, int nw,
                        double z1, double z2, int* sel, cudaStream_t s, int* launches);
void launch_pareto(const double* L, const double* Q, long long E, unsigned long long* k0,
                   unsigned long long* k1, unsigned long long* v0, unsigned long long* v1,
                   unsigned long long* kl, unsigned long long* orax, unsigned int* hist, long long* front,
                   long long* front_size, cudaStream_t s, int* launches);

}  // namespace cg
