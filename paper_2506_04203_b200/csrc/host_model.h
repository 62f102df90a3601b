// Host-side reference semantics that stay on the CPU by design: input
// validation messages, shape legality / plan-space counting tables, the CRN
// log1p table and the weight ladder (glibc libm values, hazard H3).
#pragma once

#include <cmath>
#include <cstdint>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "cascade_gpu.h"
#include "cg_cuda.h"
#include "cg_internal.h"

namespace cg {

[[noreturn]] inline void fail(int code, const std::string& msg) { throw EngineError(code, msg); }

inline void throw_if_any(const std::vector<std::string>& problems, const char* what) {
    if (problems.empty()) return;
    std::ostringstream msg;
    msg << what << ":";
    for (const auto& p : problems) msg << " " << p << ";";
    fail(CG_ERR_INVALID_INPUT, msg.str());
}

// require_valid(HardwareSpec)  domain.cpp:150-162
inline void validate_hw(const cg_hardware& hw) {
    std::vector<std::string> p;
    if (hw.gpu_count <= 0) p.push_back("gpu_count must be positive");
    if (hw.flops_per_gpu <= 0) p.push_back("flops_per_gpu must be positive");
    if (hw.mem_bandwidth_per_gpu <= 0) p.push_back("mem_bandwidth_per_gpu must be positive");
    if (hw.mem_capacity_per_gpu <= 0) p.push_back("mem_capacity_per_gpu must be positive");
    if (hw.intra_node_bw <= 0) p.push_back("intra_node_bw must be positive");
    if (hw.inter_node_bw <= 0) p.push_back("inter_node_bw must be positive");
    if (hw.gpus_per_node <= 0) p.push_back("gpus_per_node must be positive");
    throw_if_any(p, "invalid HardwareSpec");
}

// require_valid(std::vector<ModelSpec>)  domain.cpp:164-182
inline void validate_models(const cg_model* models, int c) {
    std::vector<std::string> p;
    if (c <= 0) p.push_back("model cascade is empty");
    for (int i = 0; i < c; ++i) {
        const auto& m = models[i];
        const std::string id = m.id ? m.id : "";
        if (id.empty()) p.push_back("model id empty");
        if (m.param_count < 0) p.push_back(id + ": param_count negative");
        if (m.bytes_per_param < 0) p.push_back(id + ": bytes_per_param negative");
        if (m.kv_bytes_per_token < 0) p.push_back(id + ": kv_bytes_per_token negative");
        if (m.min_gpus < 1) p.push_back(id + ": min_gpus below 1");
        if (m.stage_index != i + 1) p.push_back(id + ": stage_index not ordinal " + std::to_string(i + 1));
        if (i > 0 && m.param_count < models[i - 1].param_count)
            p.push_back(id + ": param_count decreases along the cascade");
    }
    throw_if_any(p, "invalid model cascade");
}

// costmodel::require_valid(CostModelParams)  costmodel.cpp:42-63
inline void validate_params(const cg_cost_params& q) {
    std::vector<std::string> p;
    auto fraction = [&](double v, const char* name) {
        if (!(v > 0.0 && v <= 1.0)) p.push_back(std::string(name) + " must be in (0,1]");
    };
    fraction(q.prefill_efficiency, "prefill_efficiency");
    fraction(q.decode_bw_efficiency, "decode_bw_efficiency");
    fraction(q.kv_memory_fraction, "kv_memory_fraction");
    if (q.pipeline_bubble_factor < 0.0) p.push_back("pipeline_bubble_factor must be >= 0");
    if (q.comm_overhead_per_stage < 0.0) p.push_back("comm_overhead_per_stage must be >= 0");
    if (q.queueing_sim_requests <= 0) p.push_back("queueing_sim_requests must be positive");
    throw_if_any(p, "invalid CostModelParams");
}

// require_valid(WorkloadStats)  domain.cpp:184-195; returns the message or "".
inline std::string workload_problems(const double* w) {
    std::vector<std::string> p;
    if (w[0] < 0) p.push_back("arrival_rate negative");
    if (w[1] < 0 || w[2] < 0 || w[3] < 0 || w[4] < 0) p.push_back("token statistic negative");
    if (w[3] < w[1]) p.push_back("p95_input_tokens below mean");
    if (w[4] < w[2]) p.push_back("p95_output_tokens below mean");
    if (p.empty()) return "";
    std::ostringstream msg;
    msg << "invalid WorkloadStats:";
    for (const auto& s : p) msg << " " << s << ";";
    return msg.str();
}

// memory_feasible  costmodel.cpp:79-88 (same operation order; host doubles)
inline bool memory_feasible(int tp, int pp, const cg_model& m, const cg_hardware& hw,
                            const cg_cost_params& q, double kv_tokens) {
    const double gpus = tp * pp;
    const double weights = m.param_count * m.bytes_per_param;
    if (weights / gpus > hw.mem_capacity_per_gpu) return false;
    const double kv_budget = q.kv_memory_fraction * (gpus * hw.mem_capacity_per_gpu - weights);
    return kv_budget >= m.kv_bytes_per_token * kv_tokens;
}

// legal_shapes at kv_tokens = 1 in canonical order (gpus desc, tp desc),
// costmodel.cpp:92-116
inline std::vector<ShapeDesc> legal_shapes(const cg_model& m, const cg_hardware& hw,
                                           const cg_cost_params& q) {
    std::vector<ShapeDesc> all;
    for (int tp = 1; tp <= hw.gpus_per_node; tp *= 2)
        for (int pp = 1; pp <= 8; ++pp) all.push_back({tp, pp, tp * pp});
    std::stable_sort(all.begin(), all.end(), [](const ShapeDesc& a, const ShapeDesc& b) {
        if (a.gpus != b.gpus) return a.gpus > b.gpus;
        return a.tp > b.tp;
    });
    std::vector<ShapeDesc> out;
    for (const auto& s : all)
        if (memory_feasible(s.tp, s.pp, m, hw, q, 1.0)) out.push_back(s);
    return out;
}

struct HostPlanSpace {
    std::vector<ShapeDesc> shapes;
    int N = 0;
    std::vector<unsigned long long> ways;  // (S+1)*(N+1)
    unsigned long long num_plans = 0;
    int min_gpus = 0;

    unsigned long long w(int i, int b) const { return ways[(size_t)i * (N + 1) + b]; }

    void build(std::vector<ShapeDesc> s, int budget) {
        shapes = std::move(s);
        N = budget < 0 ? 0 : budget;
        const int S = (int)shapes.size();
        ways.assign((size_t)(S + 1) * (N + 1), 0ull);
        for (int b = 0; b <= N; ++b) ways[(size_t)S * (N + 1) + b] = 1;
        for (int i = S - 1; i >= 0; --i) {
            const int size = shapes[i].gpus;
            for (int b = 0; b <= N; ++b) {
                unsigned __int128 acc = 0;
                for (int k = 0; k * size <= b; ++k) acc += w(i + 1, b - k * size);
                if (acc > (unsigned __int128)0x7fffffffffffffffull)
                    fail(CG_ERR_UNSUPPORTED, "plan space too large for 64-bit plan indices");
                ways[(size_t)i * (N + 1) + b] = (unsigned long long)acc;
            }
        }
        num_plans = ways[N] - 1;  // ways[0][N] minus the empty multiset
        min_gpus = 0;
        for (const auto& sh : shapes)
            if (min_gpus == 0 || sh.gpus < min_gpus) min_gpus = sh.gpus;
    }

    // Number of plans in each replica-count class (dp <= 4, 8, 16, 32, 64,
    // 128, 255): knapsack over (GPUs, replicas), the empty plan excluded.
    void class_counts(unsigned long long out[7]) const {
        for (int c = 0; c < 7; ++c) out[c] = 0;
        const int D = 256;
        std::vector<unsigned long long> f((size_t)(N + 1) * D, 0ull);
        f[0] = 1;
        for (const auto& sh : shapes)
            for (int b = sh.gpus; b <= N; ++b)
                for (int d = 1; d < D; ++d) f[(size_t)b * D + d] += f[(size_t)(b - sh.gpus) * D + d - 1];
        static const int His[7] = {4, 8, 16, 32, 64, 128, 255};
        for (int b = 1; b <= N; ++b)
            for (int d = 1; d < D; ++d) {
                int c = 0;
                while (c < 6 && d > His[c]) ++c;
                out[c] += f[(size_t)b * D + d];
            }
    }

    // plan index -> counts (mirror of the device unrank)
    void unrank(unsigned long long p, std::vector<int>& c) const {
        const int S = (int)shapes.size();
        c.assign(S, 0);
        unsigned long long q = p + 1;
        int b = N;
        for (int i = 0; i < S; ++i) {
            int k = 0;
            while (true) {
                const unsigned long long ww = w(i + 1, b - k * shapes[i].gpus);
                if (q < ww) break;
                q -= ww;
                ++k;
            }
            c[i] = k;
            b -= k * shapes[i].gpus;
        }
    }
};

// CRN stream of costmodel.cpp:331-342: L[k] = log1p(-u_k), u_k = (x>>11)*2^-53
// from std::mt19937_64(seed), k < 2*n_req (glibc log1p; identical libm).
inline std::vector<double> crn_log1p_table(uint64_t seed, int n_req) {
    std::mt19937_64 eng(seed);
    std::vector<double> L((size_t)2 * n_req);
    for (auto& v : L) {
        const double u = static_cast<double>(eng() >> 11) * 0x1.0p-53;
        v = std::log1p(-u);
    }
    return L;
}

// weight_ladder  outerplan.cpp:134-151
inline std::vector<double> weight_ladder(double rmin, double rmax, int count) {
    if (count < 1 || rmin <= 0 || rmax < rmin) fail(CG_ERR_INVALID_INPUT, "invalid weight ladder config");
    std::vector<double> w;
    for (int k = 0; k < count; ++k) {
        double t = count == 1 ? 0.0 : static_cast<double>(k) / (count - 1);
        double ratio = rmin * std::pow(rmax / rmin, t);
        w.push_back(ratio / (1.0 + ratio));
        w.push_back(1.0 / (1.0 + ratio));
    }
    return w;
}

}  // namespace cg
