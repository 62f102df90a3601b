// Reference-side binding: cascade::outerplan::sweep implemented on the
// B200 engine's C ABI (include/cascade_gpu.h).
//
// This is the file a Cascade Planner maintainer adds to proj/src/ to make the
// GPU engine the plan-search path: it defines exactly the reference's entry
// point (proj/include/cascade/outerplan.hpp:89-92) with the reference's
// types, so cli::cmd_plan (proj/src/cli.cpp:160-162), cmd_drift --replan and
// the tests call it unchanged, and to_json(SweepResult) (outerplan.cpp:52-59)
// emits byte-identical sweep.json / front.json / plan.json.  The reference's
// own CPU body is compiled alongside under another name.
//
// Conventions: AoS TraceRecord -> SoA columns (host), one process-wide engine
// on CASCADE_PLANNER_GPU (default 0), cg_status -> CascadeError with the same
// Errc and message the reference throws.
#include <cstdlib>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "cascade/outerplan.hpp"
#include "cascade_gpu.h"
#include "gpu_engine.hpp"

namespace cascade::outerplan {

using gpu_binding::engine;
using gpu_binding::raise;

SweepResult sweep(const std::vector<TraceRecord>& trace, const std::vector<ModelSpec>& models,
                  const HardwareSpec& hw, const costmodel::CostModelParams& params, int total_gpus,
                  const SweepConfig& cfg) {
    // Cheap checks whose error must not depend on GPU availability.
    if (trace.empty()) throw CascadeError(Errc::empty_trace, "sweep: empty trace");
    const std::size_t n = trace.size();
    const int c = static_cast<int>(models.size());
    // The reference validates the per-record stage count before reading the
    // columns (outerplan.cpp:175-178); a ragged trace cannot be laid out SoA.
    for (const auto& rec : trace)
        if (rec.per_stage.size() != static_cast<std::size_t>(c)) {
            require_valid(models);
            if (overall_arrival_rate(trace) <= 0.0)
                throw CascadeError(Errc::invalid_input, "sweep: trace has no positive arrival-rate span");
            throw CascadeError(Errc::invalid_input, "sweep: trace record stage count != C");
        }

    std::vector<double> arrival(n), in(n), out(n * c), sc(n * c);
    for (std::size_t r = 0; r < n; ++r) {
        arrival[r] = trace[r].arrival_s;
        in[r] = trace[r].input_tokens;
        for (int i = 0; i < c; ++i) {
            out[i * n + r] = trace[r].per_stage[i].output_tokens;
            sc[i * n + r] = trace[r].per_stage[i].score;
        }
    }
    cg_trace tr{static_cast<int64_t>(n), c, 0, arrival.data(), in.data(), out.data(), sc.data()};
    std::vector<cg_model> cm(models.size());
    for (std::size_t i = 0; i < models.size(); ++i)
        cm[i] = cg_model{models[i].id.c_str(), models[i].param_count, models[i].bytes_per_param,
                         models[i].kv_bytes_per_token, models[i].min_gpus, models[i].stage_index};
    cg_hardware ch{hw.gpu_count, hw.flops_per_gpu, hw.mem_bandwidth_per_gpu, hw.mem_capacity_per_gpu,
                   hw.intra_node_bw, hw.inter_node_bw, hw.gpus_per_node};
    cg_cost_params cp{params.prefill_efficiency, params.decode_bw_efficiency, params.pipeline_bubble_factor,
                      params.comm_overhead_per_stage, params.kv_memory_fraction, params.queueing_sim_requests,
                      params.queueing_sim_seed};
    std::vector<int64_t> sizes;
    std::vector<double> values;
    for (const auto& dim : cfg.threshold_grid) {
        sizes.push_back(static_cast<int64_t>(dim.size()));
        values.insert(values.end(), dim.begin(), dim.end());
    }
    cg_sweep_config cc{static_cast<int32_t>(sizes.size()), sizes.data(), values.data(), cfg.weight_ratio_min,
                       cfg.weight_ratio_max, cfg.weight_count};

    cg_sweep_result* res = nullptr;
    cg_status st = cg_sweep(engine(), &tr, cm.data(), c, &ch, &cp, total_gpus, &cc, &res);
    if (st.code != CG_OK) raise(st);
    std::unique_ptr<cg_sweep_result, void (*)(cg_sweep_result*)> guard(res, cg_sweep_result_free);

    const int D = c - 1;
    auto plan_of = [&](int64_t idx) -> std::optional<ParallelismPlan> {
        if (idx < 0) return std::nullopt;
        const cg_plan& p = res->plans[idx];
        ParallelismPlan pp;
        pp.gpus_used = p.gpus_used;
        for (int k = 0; k < p.dp; ++k)
            pp.replicas.push_back({res->replicas[p.replica_offset + k].tp, res->replicas[p.replica_offset + k].pp});
        return pp;
    };
    SweepResult out_res;
    out_res.utopia = {res->z1_star, res->z2_star};
    out_res.evaluations.reserve(static_cast<std::size_t>(res->num_evaluations));
    for (int64_t e = 0; e < res->num_evaluations; ++e) {
        ObjectivePoint pt;
        pt.latency_s = res->eval_latency[e];
        pt.quality = res->eval_quality[e];
        pt.thresholds.thresholds.assign(res->eval_thresholds + e * D, res->eval_thresholds + (e + 1) * D);
        CascadePlan& plan = pt.plan_ref;
        plan.thresholds = pt.thresholds;
        plan.predicted_max_p95_s = pt.latency_s;
        plan.predicted_quality = pt.quality;
        for (int i = 0; i < c; ++i) {
            plan.allocations.push_back(res->eval_allocations[e * c + i]);
            plan.plans.push_back(plan_of(res->eval_plan[e * c + i]));
            plan.processing_ratios.push_back(res->eval_ratios[e * c + i]);
        }
        out_res.evaluations.push_back(std::move(pt));
    }
    for (int64_t k = 0; k < res->front_size; ++k) out_res.front.points.push_back(out_res.evaluations[res->front[k]]);
    for (int k = 0; k < res->num_weights; ++k) {
        out_res.weights.push_back({res->weights[2 * k], res->weights[2 * k + 1]});
        out_res.weight_selection.push_back(res->weight_selection[k]);
    }
    for (int64_t s = 0; s < res->num_skipped; ++s) {
        RoutingThresholds h;
        h.thresholds.assign(res->skipped_thresholds + s * D, res->skipped_thresholds + (s + 1) * D);
        out_res.skipped.push_back(std::move(h));
    }
    return out_res;
}

}  // namespace cascade::outerplan
