// Host half of the validation simulator: validate_plan (proj/src/domain.cpp:
// 73-148) restated on the C-ABI plan layout, with the reference's messages.
#include <string>
#include <vector>

#include "cg_simrun.h"

namespace cg {

std::vector<std::string> validate_cascade_plan(const cg_cascade_plan& p, const cg_hardware& hw, const cg_model* models,
                                               int C) {
    std::vector<std::string> report;
    // allocations / plans / ratios always have C entries in this layout
    long long total = 0;
    for (int i = 0; i < C; ++i) {
        if (p.allocations[i] < 0) report.push_back("allocation negative");
        total += p.allocations[i];
    }
    if (total != hw.gpu_count)
        report.push_back("budget: sum of allocations " + std::to_string(total) + " != N " +
                         std::to_string(hw.gpu_count));
    long long off = 0;
    for (int i = 0; i < C; ++i) {
        const int f = p.allocations[i];
        const bool has_plan = p.has_plan[i] != 0;
        const double ratio = p.processing_ratios[i];
        const std::string stage = "stage " + std::to_string(i + 1);
        if ((f == 0) != !has_plan) report.push_back(stage + ": allocation/plan coupling violated");
        if ((f == 0) != (ratio == 0.0)) report.push_back(stage + ": allocation/ratio coupling violated");
        if (ratio < 0.0 || ratio > 1.0) report.push_back(stage + ": ratio outside [0,1]");
        const int dp = has_plan ? p.dp[i] : 0;
        if (has_plan) {
            if (dp == 0) report.push_back(stage + ": plan has no replicas");
            int used = 0;
            bool sorted = true;
            for (int k = 0; k < dp; ++k) {
                const cg_replica& r = p.replicas[off + k];
                used += r.tp * r.pp;
                if (r.tp < 1 || r.pp < 1) report.push_back(stage + ": replica degrees below 1");
                const double per_gpu = (models[i].param_count * models[i].bytes_per_param) / (r.tp * r.pp);
                if (per_gpu > hw.mem_capacity_per_gpu) report.push_back(stage + ": replica weights exceed GPU memory");
                if (k > 0) {  // canonical order: gpus desc, then tp desc (stable)
                    const cg_replica& q = p.replicas[off + k - 1];
                    const int gq = q.tp * q.pp, gr = r.tp * r.pp;
                    if (gr > gq || (gr == gq && r.tp > q.tp)) sorted = false;
                }
            }
            if (used != p.gpus_used[i]) report.push_back(stage + ": gpus_used inconsistent with replicas");
            if (used > f) report.push_back(stage + ": plan uses more GPUs than allocated");
            if (!sorted || used != p.gpus_used[i]) report.push_back(stage + ": replicas not in canonical order");
        }
        off += dp;
    }
    bool seen = false;
    double prev = 1.0;
    for (int i = 0; i < C; ++i) {
        if (p.allocations[i] == 0) continue;
        const double ratio = p.processing_ratios[i];
        if (!seen && ratio != 1.0) report.push_back("first deployed stage has ratio != 1");
        if (seen && ratio > prev)
            report.push_back("stage " + std::to_string(i + 1) + ": ratio exceeds upstream deployed stage");
        prev = ratio;
        seen = true;
    }
    for (int d = 0; d + 1 < C; ++d) {
        const double h = p.thresholds[d];
        if (h < 0.0 || h > 101.0) report.push_back("threshold outside [0," + std::to_string(101.0) + "]");
    }
    return report;
}

}  // namespace cg
