// Validation simulator (k_simrun.cu): internal interface.
#pragma once

#include <string>
#include <vector>

#include "cascade_gpu.h"
#include "cg_cuda.h"

namespace cg {

constexpr int kSimMaxStages = 8;

// One plan of the batch: deployed stages, escalation chain, replica profiles.
struct SimPlanDesc {
    int C;
    int entry, last;
    int next[kSimMaxStages];    // next deployed stage or -1
    int chain[kSimMaxStages];   // deployed stages in order, -1 padded
    int dp[kSimMaxStages];      // replicas per stage (0 = not deployed)
    int roff[kSimMaxStages];    // offset of the stage's replicas in the profile arrays
    double thr[kSimMaxStages];
};

struct SimRunArgs {
    long long n;
    int nplans;
    const double* arrival;
    const double* in;
    const double* out;      // [C][n]
    const double* scores;   // [C][n]
    const double* ppt;      // per replica: prefill per input token (bubble-scaled)
    const double* pf;       // prefill fixed
    const double* dpt;      // decode per output token
    const SimPlanDesc* plans;
    const double* base;     // [P] slo base per plan
    const double* scales;   // [nscales]
    int nscales;
    long long warmup;
    unsigned long long *ev_keys, *ev_vals, *nx_keys, *nx_vals;  // [P][n]
    long long *ev_count, *nx_count;
    double* e2e;            // [P][n]
    int* astage;            // [P][n]
    double* stage_stats;    // [P][kSimMaxStages][4]: wait sum 1st half, 2nd half, service sum, served
    double* p95;
    double* last_completion;
    unsigned long long* attain_ok;  // [P][32]
};

struct SimRunBuffers {
    DevBuf plans, base, lat, k0, v0, k1, v1, rsh, ek, ev, nk, nv, ec, nc, e2e, ast, stats, p95, lastc, ok;
    DevBuf arr, in, out, sc, ppt, pf, dpt, scales;
};

struct SimPlanOut {
    std::vector<double> e2e;
    std::vector<int> stage;
    double base = 0, p95 = 0, last_completion = 0;
    std::vector<unsigned long long> ok;
    double w1[kSimMaxStages] = {}, w2[kSimMaxStages] = {}, service_sum[kSimMaxStages] = {};
    long long served[kSimMaxStages] = {};
};

// base_mode: 0 = cfg_base for every plan, 1 = each plan's own dry run,
// 2 = the first plan's dry run shared (sim::compare).
void sim_run_batch(SimRunBuffers& B, cudaStream_t s, SimRunArgs a, std::vector<SimPlanDesc>& plans,
                   int max_steps, int base_mode, double cfg_base, int* launches, std::vector<SimPlanOut>& out);

// validate_plan (domain.cpp:73-148): the reference's problem list.
std::vector<std::string> validate_cascade_plan(const cg_cascade_plan& p, const cg_hardware& hw, const cg_model* models,
                                               int C);

}  // namespace cg
