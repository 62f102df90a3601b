/*
 * TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference planner's
 * plan-search hot path (oracle/cascade_oracle.c).  Used by tests/ and by
 * __graft_entry__.smoke() as a checker; never linked into the product.
 * Parity of this restatement is pinned against the compiled, unmodified
 * reference (oracle/_ref/libcascade_ref.so) in tests/test_oracle.py.
 */
#ifndef CASCADE_ORACLE_H
#define CASCADE_ORACLE_H

#include <stdint.h>

typedef struct {
    int gpu_count;
    double flops, mem_bw, mem_cap, intra_bw, inter_bw;
    int gpus_per_node;
} co_hw;

typedef struct {
    double param_count, bytes_per_param, kv_bytes_per_token;
    int min_gpus, stage_index;
} co_model;

typedef struct {
    double prefill_eff, decode_eff, bubble, comm, kv_frac;
    int n_req;
    uint64_t seed;
} co_params;

/* routing::route_trace; workloads[i*5 + {rate, mean_in, mean_out, p95_in, p95_out}] */
int co_route(const double* arrival, const double* in_tok, const double* out_tok, const double* scores,
             int64_t n, int c, const double* h, const int* deployed, double* ratios, double* workloads,
             double* quality, int* accept_stage);

/* StageEvaluator::row: latency[N+1] (INFINITY = infeasible), plan_counts[(N+1)*32]
 * (shape counts of the chosen plan, all zero = nullopt); shapes[2*32] = (tp, pp) */
int co_row(const co_model* m, const double* w, const co_hw* hw, const co_params* p, int max_budget,
           double* latency, int* plan_counts, int* num_shapes, int* shapes);

/* Per-budget best over the plan-index shard [plan_lo, plan_hi) of a row (no
 * prefix minimum): best_lat[g] (INFINITY = none), best_idx[g] (-1 = none). */
int co_row_shard(const co_model* m, const double* w, const co_hw* hw, const co_params* p, int max_budget,
                 int64_t plan_lo, int64_t plan_hi, double* best_lat, int64_t* best_idx, int64_t* total_plans);

/* innerplan::solve_min_max on entries[i*(gpu_budget+1)+f].
 * All functions return -1 on success, else the cascade::Errc value. */
int co_solve(const double* entries, int stages, int gpu_budget, int total_gpus, int* alloc, double* objective);

/* outerplan::sweep.  grid given as (dims, sizes, values) or dims = 0 for the
 * default grid.  Outputs (caller-allocated, capacity = number of candidates):
 *   eval_cand[E], eval_L[E], eval_Q[E], eval_alloc[E*C], eval_plan_counts[E*C*32]
 *   weights[2*W], sel[W], front[F] (indices into evaluations), skipped[S] (candidate idx)
 * counts[0..3] = E, F, S, W;  z[0..1] = utopia. */
int co_sweep(const double* arrival, const double* in_tok, const double* out_tok, const double* scores,
             int64_t n, int c, const co_model* models, const co_hw* hw, const co_params* p, int total_gpus,
             int grid_dims, const int64_t* grid_sizes, const double* grid_values, double wmin, double wmax,
             int wcount, int64_t* eval_cand, double* eval_L, double* eval_Q, int* eval_alloc,
             int* eval_plan_counts, double* weights, int* sel, int64_t* front, int64_t* skipped,
             int64_t* counts, double* z);

/* Plan census of one row for the CPU-baseline extrapolation (no simulation):
 * out[0] = plans enumerated, out[1] = stable plans (= queueing simulations the
 * reference runs), out[2+b] / out[10+b] = stable plans / sum of dp in replica
 * bins b (dp <= 4, 8, 16, 32, 64, 128, 256, > 256).  threads = pthreads used. */
int co_row_census(const co_model* m, const double* w, const co_hw* hw, const co_params* p, int max_budget,
                  int threads, int64_t* out);

#endif
