// SweepResult -> flattened cg_sweep_result -> cg_sweep_result_json (GPU).
// The nlohmann build this translation unit is compiled against decides the
// integer-array layout (probed once), so the text matches that build's dump.
#include "output_gpu.hpp"

#include <cstdlib>
#include <vector>

#include "cascade_gpu.h"
#include "gpu_engine.hpp"

namespace cascade::outerplan {

namespace {

int json_flags() {
    static const int flags = nlohmann::json(std::vector<int>{1, 2}).dump(1) == "[1,2]" ? CG_JSON_COMPACT_INT_ARRAYS : 0;
    return flags;
}

std::string render(const SweepResult& res, int indent, int what) {
    const std::size_t E = res.evaluations.size(), F = res.front.points.size();
    const int c = E ? static_cast<int>(res.evaluations[0].plan_ref.allocations.size())
                    : (F ? static_cast<int>(res.front.points[0].plan_ref.allocations.size()) : 1);
    const int D = E ? static_cast<int>(res.evaluations[0].thresholds.thresholds.size())
                    : (F ? static_cast<int>(res.front.points[0].thresholds.thresholds.size())
                         : (res.skipped.empty() ? c - 1 : static_cast<int>(res.skipped[0].thresholds.size())));
    const int C = D + 1;
    // evaluations followed by the front points (front[k] = E + k)
    std::vector<double> thr, lat, qual, ratios;
    std::vector<int32_t> alloc;
    std::vector<int64_t> eplan, front, cand;
    std::vector<cg_plan> plans;
    std::vector<cg_replica> reps;
    auto add = [&](const ObjectivePoint& p) {
        thr.insert(thr.end(), p.thresholds.thresholds.begin(), p.thresholds.thresholds.end());
        lat.push_back(p.plan_ref.predicted_max_p95_s);
        qual.push_back(p.plan_ref.predicted_quality);
        for (int i = 0; i < C; ++i) {
            ratios.push_back(p.plan_ref.processing_ratios[i]);
            alloc.push_back(p.plan_ref.allocations[i]);
            const auto& pl = p.plan_ref.plans[i];
            if (!pl) {
                eplan.push_back(-1);
                continue;
            }
            eplan.push_back(static_cast<int64_t>(plans.size()));
            plans.push_back(cg_plan{pl->gpus_used, static_cast<int32_t>(pl->replicas.size()),
                                    static_cast<int64_t>(reps.size())});
            for (const auto& r : pl->replicas) reps.push_back(cg_replica{r.tp, r.pp});
        }
    };
    for (const auto& p : res.evaluations) add(p);
    for (std::size_t k = 0; k < F; ++k) {
        add(res.front.points[k]);
        front.push_back(static_cast<int64_t>(E + k));
    }
    std::vector<double> skipped;
    for (const auto& h : res.skipped) skipped.insert(skipped.end(), h.thresholds.begin(), h.thresholds.end());
    std::vector<double> weights;
    std::vector<int32_t> sel(res.weight_selection.begin(), res.weight_selection.end());
    for (const auto& w : res.weights) {
        weights.push_back(w.lambda1);
        weights.push_back(w.lambda2);
    }
    cand.assign(E, 0);
    cg_sweep_result r{};
    r.stages = C;
    r.z1_star = res.utopia.z1_star;
    r.z2_star = res.utopia.z2_star;
    r.num_evaluations = static_cast<int64_t>(E);
    r.eval_candidate = cand.data();
    r.eval_thresholds = thr.data();
    r.eval_latency = lat.data();
    r.eval_quality = qual.data();
    r.eval_ratios = ratios.data();
    r.eval_allocations = alloc.data();
    r.eval_plan = eplan.data();
    r.num_plans = static_cast<int64_t>(plans.size());
    r.plans = plans.data();
    r.num_replicas = static_cast<int64_t>(reps.size());
    r.replicas = reps.data();
    r.num_weights = static_cast<int32_t>(res.weights.size());
    r.weights = weights.data();
    r.weight_selection = sel.data();
    r.front_size = static_cast<int64_t>(F);
    r.front = front.data();
    r.num_skipped = static_cast<int64_t>(res.skipped.size());
    r.skipped_thresholds = skipped.data();
    char* text = nullptr;
    int64_t len = 0;
    const cg_status st = cg_sweep_result_json(gpu_binding::engine(), &r, indent, what, json_flags(), &text, &len);
    if (st.code != CG_OK) gpu_binding::raise(st);
    std::string s(text, static_cast<std::size_t>(len));
    cg_text_free(text);
    return s;
}

}  // namespace

std::string sweep_json(const SweepResult& res, int indent) { return render(res, indent, 0); }
std::string front_json(const SweepResult& res, int indent) { return render(res, indent, 1); }

}  // namespace cascade::outerplan
