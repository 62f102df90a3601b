/*
 * cascade_gpu.h -- C ABI of the B200-native plan-search engine.
 *
 * This is the drop-in boundary for the hot path of the Cascade Planner's
 * bi-level scheduler: batched evaluation of candidate plans, i.e. the body
 * of cascade::outerplan::sweep and the three entry points it calls.  Every
 * entry point below replaces exactly one reference C++ interface
 * (paths relative to the reference tree proj/):
 *
 *   cg_sweep              <- cascade::outerplan::sweep
 *                            include/cascade/outerplan.hpp:89-92, src/outerplan.cpp:166-319
 *   cg_route              <- cascade::routing::route_trace
 *                            include/cascade/routing.hpp:26-28, src/routing.cpp:42-93
 *   cg_stage_row          <- cascade::costmodel::StageEvaluator::row
 *                            include/cascade/costmodel.hpp:110-111, src/costmodel.cpp:296-414
 *   cg_solve_min_max      <- cascade::innerplan::solve_min_max
 *                            include/cascade/innerplan.hpp:63, src/innerplan.cpp:131-194
 *   cg_generate_trace     <- cascade::cli::generate_trace (synthetic input only)
 *                            include/cascade/cli.hpp:171-172, src/cli.cpp:428-460
 *   cg_read_trace_jsonl   <- cascade::read_trace_jsonl (trace ingest)
 *                            include/cascade/domain.hpp:162, src/domain.cpp:361-387
 *   cg_simulate           <- cascade::sim::run / sim::compare (validation simulator)
 *                            include/cascade/simulator.hpp:69-88, src/simulator.cpp:177-334
 *   cg_drift_windows      <- the windowing / statistics of cli::cmd_drift
 *                            src/cli.cpp:101-131 (stats_of_records, compute_baseline), 216-300
 *   cg_sweep_result_json  <- nlohmann::json(SweepResult).dump(indent) / json(front).dump(indent)
 *                            (sweep.json / front.json, src/cli.cpp:121,165-172,
 *                            src/outerplan.cpp:20-59, src/domain.cpp:270-356)
 *
 * Conventions
 *   - Plain pointers and sizes only; no exceptions cross the ABI.  Every call
 *     returns a cg_status whose code is CG_OK (-1) on success or the
 *     reference's cascade::Errc value (include/cascade/errors.hpp:10-18) with
 *     the reference's own message text.  CG_ERR_CUDA / CG_ERR_UNSUPPORTED are
 *     engine-only codes.
 *   - Traces are SoA, stage-major: output_tokens[i*n + r], scores[i*n + r].
 *     With cg_trace.on_device != 0 all four pointers are device pointers
 *     (HBM-resident input); otherwise they are host pointers and the engine
 *     copies them to the GPU inside the call.
 *   - Output buffers are owned by the library until the matching *_free.
 *   - One engine per GPU; calls on one engine must not overlap.
 *   - There is no CPU fallback: if no sm_100 device is present every compute
 *     entry point fails with CG_ERR_CUDA.
 */
#ifndef CASCADE_GPU_H
#define CASCADE_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CG_OK (-1)
/* cascade::Errc values (errors.hpp:10-18) */
#define CG_ERR_INVALID_INPUT 0
#define CG_ERR_IO 1
#define CG_ERR_EMPTY_TRACE 2
#define CG_ERR_NO_DEPLOYED_STAGE 3
#define CG_ERR_INFEASIBLE 4
#define CG_ERR_INFEASIBLE_PROBLEM 5
#define CG_ERR_NO_FEASIBLE_POINT 6
/* engine-only */
#define CG_ERR_CUDA 100
#define CG_ERR_UNSUPPORTED 101

typedef struct cg_status {
    int32_t code;
    char message[512];
} cg_status;

/* cascade::HardwareSpec (domain.hpp:23-33) */
typedef struct cg_hardware {
    int32_t gpu_count;
    double flops_per_gpu;
    double mem_bandwidth_per_gpu;
    double mem_capacity_per_gpu;
    double intra_node_bw;
    double inter_node_bw;
    int32_t gpus_per_node;
} cg_hardware;

/* cascade::ModelSpec (domain.hpp:35-46) */
typedef struct cg_model {
    const char* id;
    double param_count;
    double bytes_per_param;
    double kv_bytes_per_token;
    int32_t min_gpus;
    int32_t stage_index;
} cg_model;

/* cascade::costmodel::CostModelParams (costmodel.hpp:27-35) */
typedef struct cg_cost_params {
    double prefill_efficiency;
    double decode_bw_efficiency;
    double pipeline_bubble_factor;
    double comm_overhead_per_stage;
    double kv_memory_fraction;
    int32_t queueing_sim_requests;
    uint64_t queueing_sim_seed;
} cg_cost_params;

/* cascade::WorkloadStats (domain.hpp:48-56) */
typedef struct cg_workload {
    double arrival_rate;
    double mean_input_tokens;
    double mean_output_tokens;
    double p95_input_tokens;
    double p95_output_tokens;
} cg_workload;

/* std::vector<TraceRecord> (domain.hpp:90-103) as SoA columns. */
typedef struct cg_trace {
    int64_t n;
    int32_t stages;
    int32_t on_device;            /* 0: host pointers, 1: device pointers */
    const double* arrival_s;      /* [n] */
    const double* input_tokens;   /* [n] */
    const double* output_tokens;  /* [stages][n] */
    const double* scores;         /* [stages][n] */
} cg_trace;

/* cascade::outerplan::SweepConfig (outerplan.hpp:56-63).  grid_dims == 0
 * means "empty threshold_grid" (the reference's default decile grid). */
typedef struct cg_sweep_config {
    int32_t grid_dims;
    const int64_t* grid_sizes;    /* [grid_dims] */
    const double* grid_values;    /* concatenated, given order kept */
    double weight_ratio_min;
    double weight_ratio_max;
    int32_t weight_count;
} cg_sweep_config;

typedef struct cg_replica {
    int32_t tp;
    int32_t pp;
} cg_replica;

/* cascade::ParallelismPlan (domain.hpp:67-72): replicas[offset .. offset+dp) */
typedef struct cg_plan {
    int32_t gpus_used;
    int32_t dp;
    int64_t replica_offset;
} cg_plan;

/* Engine-side counters and per-phase device times of the last sweep. */
typedef struct cg_sweep_stats {
    int64_t candidates;           /* threshold vectors in the grid */
    int64_t distinct_candidates;  /* after collapsing duplicate grid values */
    int64_t stage_workloads;      /* (stage, threshold-prefix) workloads routed */
    int64_t unique_rows;          /* latency rows evaluated (reference row cache) */
    int64_t plans_enumerated;     /* sum over rows of |plan set| */
    int64_t plans_stable;         /* plans passing the stability filter */
    int64_t plans_simulated_full; /* 2000-request simulations run to completion */
    int64_t plans_pruned;         /* simulations stopped by the exact p95 bound */
    int64_t plans_bound_skipped;  /* excluded by the exact service-time bound, unsimulated */
    int64_t plans_seeded;         /* bound-seeding simulations (re-visited by the sweep) */
    int64_t plans_overflow;       /* re-run by the deep-queue kernel */
    int64_t request_steps;        /* JSQ dispatch steps executed */
    int64_t h2d_bytes;
    int64_t d2h_bytes;
    int32_t num_ranks;
    int32_t gpu_launches;         /* engine kernels launched by this call */
    double ms_total;              /* host wall time of the call */
    double ms_route;              /* K1-K3: routing / aggregation / p95 */
    double ms_quality;            /* K2: trace-order quality sums */
    double ms_rows;               /* K4-K5: cost-model rows */
    double ms_solve;              /* K6-K7: min-max solve, Tchebycheff, Pareto */
    double ms_k1;                 /* the routing/aggregation pass alone */
    double k1_bytes;              /* algorithmic bytes moved by that pass */
    double ms_k4;                 /* the queueing-simulation kernels alone */
    int64_t collectives;          /* bound exchanges (all-gathers) of a sharded call, final merge excluded */
    int64_t quality_blocks;       /* K2 (tuple, request block) pairs */
    int64_t quality_blocks_seq;   /* of those, folded request by request (binade crossings, ties, s = 0) */
    int64_t waves_total;          /* K4 filter waves of the plan lists */
    int64_t waves_run;            /* of those, run (< waves_total only under max_waves / wave_stride) */
    int64_t plans_in_waves;       /* plan indices covered by the waves run (64-plan chunks) */
} cg_sweep_stats;

/* cascade::outerplan::SweepResult (outerplan.hpp:73-80), flattened. */
typedef struct cg_sweep_result {
    int32_t stages;                 /* C */
    double z1_star;                 /* UtopiaPoint */
    double z2_star;
    int64_t num_evaluations;        /* E, grid order */
    int64_t* eval_candidate;        /* [E] cartesian index, first dim outermost */
    double* eval_thresholds;        /* [E][C-1] */
    double* eval_latency;           /* [E] L */
    double* eval_quality;           /* [E] Q */
    double* eval_ratios;            /* [E][C] processing_ratios */
    int32_t* eval_allocations;      /* [E][C] */
    int64_t* eval_plan;             /* [E][C] index into plans, -1 = nullopt */
    int64_t num_plans;
    cg_plan* plans;
    int64_t num_replicas;
    cg_replica* replicas;
    int32_t num_weights;
    double* weights;                /* [W][2] lambda1, lambda2 */
    int32_t* weight_selection;      /* [W] index into evaluations */
    int64_t front_size;
    int64_t* front;                 /* [F] index into evaluations, latency asc */
    int64_t num_skipped;
    int64_t* skipped_candidate;     /* [S] cartesian index */
    double* skipped_thresholds;     /* [S][C-1] */
    cg_sweep_stats stats;
} cg_sweep_result;

/* Host-side all-gather over device buffers, used by multi-GPU sweeps: must
 * gather `bytes_per_rank` bytes from every rank into recv (rank-major) and
 * return 0 on success.  Called on the engine's stream, which is synchronised
 * before the call. */
typedef int (*cg_allgather_fn)(const void* send_dev, void* recv_dev, size_t bytes_per_rank,
                               void* user);

typedef struct cg_engine cg_engine;

cg_status cg_engine_create(int32_t device, cg_engine** out);
void cg_engine_destroy(cg_engine* engine);
/* Shard the cost-model work over `world` ranks (this engine is `rank`). */
cg_status cg_engine_set_collective(cg_engine* engine, int32_t rank, int32_t world,
                                   cg_allgather_fn allgather, void* user);
/* Multi-GPU inside the library (the CASCADE_PLANNER_THREADS
 * analogue of util.cpp:31-38).  Sharded calls -- cg_sweep and cg_stage_row --
 * split every row's plan chunks over the ranks (chunk g -> rank g mod world),
 * exchange their p95 bounds after the pilot pass and after every filter wave,
 * and merge the per-budget bests with one all-gather; the result is the
 * single-GPU result bit for bit.  NCCL is bound at first use (dlopen of
 * libnccl.so.2, or CG_NCCL_LIBRARY); no torch dependency.
 *
 * One process, several GPUs: one member engine per device, one NCCL clique
 * (ncclCommInitAll), one host thread per device inside each sharded call;
 * every other call runs on devices[0].  devices = NULL with ndev = 0 takes every
 * visible device.  cg_engine_destroy releases it all. */
cg_status cg_engine_create_multi(const int32_t* devices, int32_t ndev, cg_engine** out);
int32_t cg_engine_device_count(cg_engine* engine);
/* One process per GPU: rank 0 makes the unique id (cg_nccl_unique_id_bytes()
 * bytes), the caller's launcher broadcasts it, every rank joins.  Replaces a
 * cg_engine_set_collective callback; the all-gathers then run in the library
 * on the engine's stream. */
int32_t cg_nccl_unique_id_bytes(void);
cg_status cg_nccl_unique_id(void* out, int32_t capacity);
cg_status cg_engine_set_nccl(cg_engine* engine, const void* unique_id, int32_t rank, int32_t world);
/* The engine's CUDA stream (cudaStream_t): every kernel and copy of a call runs
 * on it, so callers can bracket calls with their own CUDA events. */
void* cg_engine_stream(cg_engine* engine);
/* Engine options.  None changes any result (tests/test_gpu_parity.py checks
 * each); they select work order and kernel forms:
 *   "prune"            1 (default) exact p95-bound elimination in K4; 0 simulates every stable plan
 *   "k4_pack"          3 (default) lane-major k_lane for dp <= 32, one lane per plan (R = 4/8/16/32
 *                      replicas per lane); 4: W = 1/1/2/1 lanes per plan, R = 4/8/8/32; 5: W = 1/1/2/4,
 *                      R = 4/8/8/8; 0-2 group-per-plan k_sim forms
 *   "pilot"            best-estimate plan per (row, budget) simulated first: 1 (default) when the
 *                      sweep's plan lists fit one filter wave, 2 always, 0 never
 *   "pilot_merge"      1 (default) pilot launch grouping (0 per class, 2 one launch)
 *   "pilot_min_plans"  0 (default) rows with fewer plans get no pilot
 *   "pilot_sort"       1 (default) pilot lists in ascending estimate order
 *   "sort_key"         3 (default) work-list order estimate (0 raw service bound)
 *   "class_order"      1 (default) replica-count classes ascending (0 descending)
 *   "wave_plans"       256 (default) plans per filter wave in units of 2^20; class lists sized by a
 *                      census of the plan spaces, the wave shrunk to fit 60% of the free HBM
 *   "conc_lists_max"   65536 (default) waves with at most this many listed plans run their
 *                      replica-count classes concurrently on four streams (0: never)
 *   "quality_form"     1 (default) block-parallel exact K2 quality sums; 0 one fp64 add chain per tuple
 *   "p95_tables"       1 (default) K3 chunk tables for traces >= 65536 requests; 0 direct column scans
 *   "max_waves", "wave_stride"  rate sampling only: run at most max_waves filter waves, every
 *                      wave_stride-th one; the result is then PARTIAL (stats.waves_run < waves_total)
 *   "fut_block"        1 (default) output-rank granularity of K4's future-service bound (exact counts)
 *   "lane_check"       32 (default) request-steps between K4's prune checks (32 or 64)
 *   "seeds"            1 (default) homogeneous plans of the heavy rows simulated first; 0 off
 *   "fut_bound", "item_plans", "k1_form", "overflow_capacity", "tie_capacity", "ub_oracle",
 *   "quality_block" (diagnostic)
 * Unknown keys return CG_ERR_INVALID_INPUT. */
cg_status cg_engine_set_option(cg_engine* engine, const char* key, int64_t value);

cg_status cg_sweep(cg_engine* engine, const cg_trace* trace, const cg_model* models,
                   int32_t num_models, const cg_hardware* hw, const cg_cost_params* params,
                   int32_t total_gpus, const cg_sweep_config* cfg, cg_sweep_result** out);
void cg_sweep_result_free(cg_sweep_result* result);

/* cascade::routing::RoutingOutcome (routing.hpp:15-20). */
typedef struct cg_route_result {
    int32_t stages;
    double ratios[8];
    cg_workload stage_workloads[8];
    double quality;
} cg_route_result;

/* route_trace with a deployment mask (deployed[i] != 0).  accept_stage, if
 * non-NULL, receives the 1-based accept stage of every request (host). */
cg_status cg_route(cg_engine* engine, const cg_trace* trace, const double* thresholds,
                   const int32_t* deployed, cg_route_result* out, int32_t* accept_stage);

/* Batched route_trace over every threshold candidate of a grid (all stages
 * deployed), i.e. the routing phase of sweep on its own (outerplan.cpp:229-234):
 * per candidate (cartesian order, first dimension outermost) the
 * RoutingOutcome ratios, stage workloads and quality. */
typedef struct cg_route_grid_result {
    int32_t stages;
    int64_t num_candidates;
    double* thresholds;   /* [K][C-1] */
    double* ratios;       /* [K][C] */
    cg_workload* workloads; /* [K][C] */
    double* quality;      /* [K] */
    cg_sweep_stats stats;
} cg_route_grid_result;

cg_status cg_route_grid(cg_engine* engine, const cg_trace* trace, const cg_sweep_config* cfg,
                        cg_route_grid_result** out);
void cg_route_grid_result_free(cg_route_grid_result* result);

/* StageEvaluator::row: latency[f] for f in 0..max_budget (INFINITY when
 * infeasible) and plan_index[f] (-1 = nullopt) into *plans / *replicas. */
typedef struct cg_row_result {
    int32_t max_budget;
    double* latency;                /* [max_budget+1] */
    int64_t* plan_index;            /* [max_budget+1] */
    int64_t num_plans;
    cg_plan* plans;
    int64_t num_replicas;
    cg_replica* replicas;
    cg_sweep_stats stats;
} cg_row_result;

cg_status cg_stage_row(cg_engine* engine, const cg_model* model, const cg_workload* w,
                       const cg_hardware* hw, const cg_cost_params* params,
                       int32_t max_budget, cg_row_result** out);
void cg_row_result_free(cg_row_result* result);

/* Host-only (no GPU): merge per-budget bests of `shards` disjoint plan-index
 * shards of one row -- lat_bits/plan_index[s*(max_budget+1) + g], ~0 = none --
 * with the same rule the multi-GPU device merge applies after its all-gather,
 * then the reference's prefix minimum (costmodel.cpp:347-352, 398-412). */
cg_status cg_merge_row_shards(const cg_model* model, const cg_hardware* hw, const cg_cost_params* params,
                              int32_t max_budget, int32_t shards, const uint64_t* lat_bits,
                              const uint64_t* plan_index, cg_row_result** out);
/* The plan-index ranges [lo, hi) of row `row` that `rank` of `world`
 * evaluates in a sharded call whose work list holds rows with num_plans[0..nrows)
 * plans (rows with 0 plans take no chunks): 64-plan chunks, global chunk g ->
 * rank g mod world (the device filter's mapping).  Writes up to `cap` pairs,
 * ascending; returns the number of ranges (-1 on invalid arguments). */
int64_t cg_shard_row_plans(const uint64_t* num_plans, int32_t nrows, int32_t row, int32_t rank, int32_t world,
                           uint64_t* ranges, int64_t cap);
/* Host-only: per-budget best over `shards` partial results with the merge rule
 * alone (no prefix minimum) -- what one rank holds after its own plans. */
cg_status cg_merge_budget_bests(const cg_model* model, const cg_hardware* hw, const cg_cost_params* params,
                                int32_t max_budget, int32_t shards, const uint64_t* lat_bits,
                                const uint64_t* plan_index, uint64_t* lat_out, uint64_t* plan_out);

/* solve_min_max on a latency table entries[i*(gpu_budget+1) + f]
 * (INFINITY = masked cell).  Writes allocations[stages], per_stage[stages]
 * and *objective_L. */
cg_status cg_solve_min_max(cg_engine* engine, const double* entries, int32_t stages,
                           int32_t gpu_budget, int32_t total_gpus, int32_t* allocations,
                           double* per_stage_latency, double* objective_L);

/* Synthetic trace generation with the reference generator's semantics and
 * bit-identical output.  spec_json is the TraceGenSpec JSON
 * (cli.hpp:141-169).  Host buffers of capacity >= count (and
 * stages*count for the per-stage columns); *n_out = count. */
cg_status cg_generate_trace(const char* spec_json, uint64_t seed, double* arrival_s,
                            double* input_tokens, double* output_tokens, double* scores,
                            int64_t capacity, int64_t* n_out, int32_t* stages_out);

/* Trace ingest: cascade::read_trace_jsonl (domain.cpp:361-387) on the GPU.
 * The JSONL bytes are split, parsed, validated (require_valid per record,
 * non-decreasing arrivals) and decoded into SoA columns in HBM.  Errors carry
 * the reference's Errc and exact message (io_error "cannot open trace file:
 * <path>", invalid_input "<path>:<line>: bad trace record: <json what()>",
 * "invalid TraceRecord: ...;", "<path>:<line>: arrival times must be
 * non-decreasing").  An empty file (or only empty lines) yields n = 0. */
typedef struct cg_ingest_stats {
    int64_t bytes;
    int64_t lines;
    int64_t records;
    int64_t host_lines;      /* lines the device parser left to the host JSON decoder */
    int32_t gpu_launches;
    double ms_total;         /* host wall time of the call (file read excluded) */
    double ms_read;          /* file read into pinned memory (cg_read_trace_jsonl) */
} cg_ingest_stats;

typedef struct cg_trace_buffer {
    cg_trace host;           /* host SoA columns, owned by this buffer */
    cg_trace device;         /* the same columns in HBM (on_device = 1), owned by the
                                engine: valid until its next ingest call or destroy */
    cg_ingest_stats stats;
} cg_trace_buffer;

cg_status cg_read_trace_jsonl(cg_engine* engine, const char* path, cg_trace_buffer** out);
/* Same on an in-memory file image; `path` is used in error messages only. */
cg_status cg_parse_trace_jsonl(cg_engine* engine, const char* bytes, int64_t len, const char* path,
                               cg_trace_buffer** out);
void cg_trace_buffer_free(cg_trace_buffer* buffer);

/* Output serialisation: the exact bytes nlohmann's dump(indent) writes for
 * json(SweepResult) (what = 0, sweep.json without its trailing "\n") or
 * json(SweepResult::front) (what = 1, front.json), formatted on the GPU.
 * flags: CG_JSON_COMPACT_INT_ARRAYS reproduces nlohmann builds that print
 * integer arrays on one line (the cudnn-frontend copy of 3.11.3 in this image
 * does; upstream 3.11.3 does not -- bindings probe their own nlohmann once).
 * *text is NUL-terminated, owned by the caller (cg_text_free). */
#define CG_JSON_COMPACT_INT_ARRAYS 1
cg_status cg_sweep_result_json(cg_engine* engine, const cg_sweep_result* result, int32_t indent, int32_t what,
                               int32_t flags, char** text, int64_t* len);
void cg_text_free(char* text);

/* Validation simulator: sim::run (simulator.cpp:177-299) of every plan, or
 * sim::compare (simulator.cpp:318-334, >= 2 plans, the first plan's dry-run
 * SLO base shared) when compare != 0.  Same preconditions, Errc and messages
 * as the reference ("run: invalid plan: ...;" from validate_plan, ...). */
typedef struct cg_sim_config {      /* sim::SimConfig (simulator.hpp:20-28) */
    uint64_t seed;
    double slo_base_s;              /* <= 0: no-contention dry-run base */
    const double* slo_scales;
    int32_t num_scales;             /* <= 32 */
    double warmup_fraction;
} cg_sim_config;

typedef struct cg_cascade_plan {    /* cascade::CascadePlan (domain.hpp:105-114) */
    const int32_t* allocations;     /* [C] */
    const double* processing_ratios;/* [C] */
    const double* thresholds;       /* [C-1] */
    const int32_t* has_plan;        /* [C] */
    const int32_t* gpus_used;       /* [C] */
    const int32_t* dp;              /* [C] replicas of each deployed stage */
    const cg_replica* replicas;     /* concatenated, stage order */
} cg_cascade_plan;

typedef struct cg_sim_report {      /* sim::SimReport (simulator.hpp:40-48) */
    double* end_to_end_s;           /* [n] trace order */
    int32_t* accept_stage;          /* [n] 1-based */
    double p95_s;
    double throughput_rps;
    int32_t num_scales;
    double* attainment_scale;       /* [num_scales] */
    double* attainment_fraction;    /* [num_scales] */
    int32_t has_min_scale_95;
    double min_scale_95;
    double slo_base_s;
    int32_t num_unstable;
    int32_t unstable_stages[8];     /* 1-based */
} cg_sim_report;

typedef struct cg_sim_result {
    int64_t n;
    int32_t num_reports;
    cg_sim_report* reports;
    int32_t gpu_launches;
    double ms_total;
} cg_sim_result;

cg_status cg_simulate(cg_engine* engine, const cg_trace* trace, const cg_model* models, int32_t num_models,
                      const cg_hardware* hw, const cg_cost_params* params, const cg_sim_config* cfg,
                      const cg_cascade_plan* plans, int32_t num_plans, int32_t compare, cg_sim_result** out);
void cg_sim_result_free(cg_sim_result* result);

/* Drift detection (cli.cpp:216-300): windows [t0 + k*I, t0 + k*I + I) over a
 * non-decreasing stream, per-window statistics of the first window_requests
 * records, relative deviations against the baseline (null when the baseline
 * value is 0).  Windows with no records or span <= 0 are omitted, as in the
 * reference.  Errc empty_trace "drift stream is empty" for n = 0. */
typedef struct cg_drift_policy {    /* cli::DriftPolicy (cli.hpp:23-27) */
    int32_t window_requests;
    double window_interval_s;
    double rel_tolerance;
} cg_drift_policy;

typedef struct cg_drift_stats {     /* cli::DriftBaseline (cli.hpp:50-56) */
    double arrival_rate;
    double mean_input_tokens;
    double mean_output_tokens;
    double stage1_accept_rate;
    int32_t has_h1;
    double h1;
} cg_drift_stats;

typedef struct cg_drift_window {    /* cli::DriftWindowReport (cli.hpp:118-127) */
    double start_s;
    double span_s;
    int32_t requests;
    int32_t sampled;
    int64_t first_record;           /* trace index of the window's first record */
    cg_drift_stats stats;
    double deviation[4];            /* arrival_rate, mean_input_tokens, mean_output_tokens, stage1_accept_rate */
    int32_t deviation_is_null[4];
    int32_t drifted[4];
    int32_t any_drift;
} cg_drift_window;

typedef struct cg_drift_result {
    int64_t num_windows;
    cg_drift_window* windows;
    int32_t drift_detected;
} cg_drift_result;

cg_status cg_drift_windows(cg_engine* engine, const cg_trace* stream, const cg_drift_stats* baseline,
                           const cg_drift_policy* policy, cg_drift_result** out);
void cg_drift_result_free(cg_drift_result* result);
/* compute_baseline (cli.cpp:125-131): whole-trace statistics, h1 = the plan's
 * first threshold when it has one, arrival rate = overall_arrival_rate. */
cg_status cg_trace_baseline(cg_engine* engine, const cg_trace* trace, int32_t has_h1, double h1,
                            cg_drift_stats* out);

const char* cg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CASCADE_GPU_H */
