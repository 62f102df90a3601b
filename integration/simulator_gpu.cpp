// Reference-side binding: cascade::sim::run and sim::compare
// (proj/include/cascade/simulator.hpp:69-88, proj/src/simulator.cpp:177-334)
// on the B200 engine's batched validation simulator (cg_simulate).  Same
// SimReport / CompareResult values (bit-identical), same CascadeError codes
// and messages.  The reference's bodies are compiled alongside as
// cpu_run / cpu_compare (oracle/Makefile `dropin`).
#include <vector>

#include "cascade/simulator.hpp"
#include "gpu_engine.hpp"

namespace cascade::sim {

namespace {

std::vector<SimReport> simulate(const std::vector<CascadePlan>& plans, const std::vector<TraceRecord>& trace,
                                const std::vector<ModelSpec>& models, const HardwareSpec& hw,
                                const costmodel::CostModelParams& params, const SimConfig& cfg, bool cmp) {
    const std::size_t n = trace.size();
    const int c = static_cast<int>(models.size());
    bool ragged = false;
    for (const auto& rec : trace) ragged |= rec.per_stage.size() != models.size();
    std::vector<double> arrival(n), in(n), out(ragged ? 0 : n * c), sc(ragged ? 0 : n * c);
    for (std::size_t r = 0; r < n; ++r) {
        arrival[r] = trace[r].arrival_s;
        in[r] = trace[r].input_tokens;
        if (ragged) continue;
        for (int i = 0; i < c; ++i) {
            out[i * n + r] = trace[r].per_stage[i].output_tokens;
            sc[i * n + r] = trace[r].per_stage[i].score;
        }
    }
    // a ragged trace fails run()'s stage-count check (after the plan checks)
    cg_trace tr{static_cast<int64_t>(n), ragged ? c + 1 : c, 0, arrival.data(), in.data(), out.data(), sc.data()};
    std::vector<cg_model> cm(models.size());
    for (std::size_t i = 0; i < models.size(); ++i)
        cm[i] = cg_model{models[i].id.c_str(), models[i].param_count, models[i].bytes_per_param,
                         models[i].kv_bytes_per_token, models[i].min_gpus, models[i].stage_index};
    cg_hardware ch{hw.gpu_count, hw.flops_per_gpu, hw.mem_bandwidth_per_gpu, hw.mem_capacity_per_gpu,
                   hw.intra_node_bw, hw.inter_node_bw, hw.gpus_per_node};
    cg_cost_params cp{params.prefill_efficiency, params.decode_bw_efficiency, params.pipeline_bubble_factor,
                      params.comm_overhead_per_stage, params.kv_memory_fraction, params.queueing_sim_requests,
                      params.queueing_sim_seed};
    cg_sim_config scfg{cfg.seed, cfg.slo_base_s, cfg.slo_scales.data(), static_cast<int32_t>(cfg.slo_scales.size()),
                       cfg.warmup_fraction};
    // CascadePlan -> cg_cascade_plan (C entries per stage, replicas concatenated)
    struct Flat {
        std::vector<int32_t> alloc, has, used, dp;
        std::vector<double> ratios, thr;
        std::vector<cg_replica> reps;
    };
    std::vector<Flat> flat(plans.size());
    std::vector<cg_cascade_plan> cps(plans.size());
    for (std::size_t p = 0; p < plans.size(); ++p) {
        const CascadePlan& pl = plans[p];
        Flat& f = flat[p];
        for (int i = 0; i < c; ++i) {
            f.alloc.push_back(i < static_cast<int>(pl.allocations.size()) ? pl.allocations[i] : 0);
            f.ratios.push_back(i < static_cast<int>(pl.processing_ratios.size()) ? pl.processing_ratios[i] : 0.0);
            const bool has = i < static_cast<int>(pl.plans.size()) && pl.plans[i].has_value();
            f.has.push_back(has ? 1 : 0);
            f.used.push_back(has ? pl.plans[i]->gpus_used : 0);
            f.dp.push_back(has ? static_cast<int32_t>(pl.plans[i]->replicas.size()) : 0);
            if (has)
                for (const auto& r : pl.plans[i]->replicas) f.reps.push_back(cg_replica{r.tp, r.pp});
        }
        f.thr = pl.thresholds.thresholds;
        f.thr.resize(c > 1 ? c - 1 : 1, 0.0);
        if (f.reps.empty()) f.reps.push_back(cg_replica{1, 1});
        cps[p] = cg_cascade_plan{f.alloc.data(), f.ratios.data(), f.thr.data(), f.has.data(), f.used.data(),
                                 f.dp.data(), f.reps.data()};
    }
    cg_sim_result* res = nullptr;
    const cg_status st = cg_simulate(gpu_binding::engine(), &tr, cm.data(), c, &ch, &cp, &scfg, cps.data(),
                                     static_cast<int32_t>(cps.size()), cmp ? 1 : 0, &res);
    if (st.code != CG_OK) gpu_binding::raise(st);
    std::vector<SimReport> reps(static_cast<std::size_t>(res->num_reports));
    for (int p = 0; p < res->num_reports; ++p) {
        const cg_sim_report& r = res->reports[p];
        SimReport& o = reps[p];
        o.per_request.resize(n);
        for (std::size_t k = 0; k < n; ++k) o.per_request[k] = {r.end_to_end_s[k], r.accept_stage[k]};
        o.p95_s = r.p95_s;
        o.throughput_rps = r.throughput_rps;
        for (int q = 0; q < r.num_scales; ++q) o.attainment.push_back({r.attainment_scale[q], r.attainment_fraction[q]});
        if (r.has_min_scale_95) o.min_scale_95 = r.min_scale_95;
        o.slo_base_s = r.slo_base_s;
        for (int q = 0; q < r.num_unstable; ++q) o.unstable_stages.push_back(r.unstable_stages[q]);
    }
    cg_sim_result_free(res);
    return reps;
}

}  // namespace

SimReport run(const CascadePlan& plan, const std::vector<TraceRecord>& trace, const std::vector<ModelSpec>& models,
              const HardwareSpec& hw, const costmodel::CostModelParams& params, const SimConfig& cfg) {
    return simulate({plan}, trace, models, hw, params, cfg, false).front();
}

CompareResult compare(const std::vector<CascadePlan>& plans, const std::vector<TraceRecord>& trace,
                      const std::vector<ModelSpec>& models, const HardwareSpec& hw,
                      const costmodel::CostModelParams& params, const SimConfig& cfg) {
    CompareResult result;
    result.reports = simulate(plans, trace, models, hw, params, cfg, true);
    for (const auto& rep : result.reports) result.rows.push_back({rep.p95_s, rep.throughput_rps, rep.min_scale_95});
    return result;
}

}  // namespace cascade::sim
