// cg_generate_trace: synthetic request traces with the reference
// generator's semantics (proj/src/cli.cpp:336-460, util.hpp:16-54), so the
// benchmark inputs are bit-identical to the reference's `gen-trace`.
// Host code: the samplers depend on glibc log1p/sqrt/cos (hazard H3) and on
// std::mt19937_64, both identical to the reference build.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include <json.hpp>

#include "cascade_gpu.h"

namespace {

using nlohmann::json;

struct Dist {
    std::string dist = "fixed";
    double value = 0, min = 0, max = 0, mean = 0, std = 0;
    bool has_min = false, has_max = false;
    std::vector<double> values, weights;
};

struct Fail {
    int code;
    std::string msg;
};

Dist parse_dist(const json& j) {
    Dist d;
    j.at("dist").get_to(d.dist);
    d.value = j.value("value", 0.0);
    d.mean = j.value("mean", 0.0);
    d.std = j.value("std", 0.0);
    d.has_min = j.contains("min");
    d.has_max = j.contains("max");
    d.min = j.value("min", 0.0);
    d.max = j.value("max", 0.0);
    d.values = j.value("values", std::vector<double>{});
    d.weights = j.value("weights", std::vector<double>{});
    return d;
}

void validate(const Dist& d) {
    if (d.dist == "fixed" || d.dist == "uniform" || d.dist == "normal") return;
    if (d.dist == "exponential") {
        if (d.mean < 0) throw Fail{CG_ERR_INVALID_INPUT, "exponential mean must be >= 0"};
        return;
    }
    if (d.dist == "choice") {
        if (d.values.empty()) throw Fail{CG_ERR_INVALID_INPUT, "choice needs values"};
        if (!d.weights.empty() && d.weights.size() != d.values.size())
            throw Fail{CG_ERR_INVALID_INPUT, "choice weights length != values length"};
        for (double w : d.weights)
            if (w < 0) throw Fail{CG_ERR_INVALID_INPUT, "choice weights must be >= 0"};
        return;
    }
    throw Fail{CG_ERR_INVALID_INPUT, "unknown distribution: " + d.dist};
}

// util::Rng samplers
struct Rng {
    std::mt19937_64 eng;
    explicit Rng(uint64_t seed) : eng(seed) {}
    double uniform() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double exponential_mean(double mean) {
        double u = uniform();
        return -mean * std::log1p(-u);
    }
    double normal(double mu, double sigma) {
        double u1 = uniform();
        double u2 = uniform();
        double r = std::sqrt(-2.0 * std::log1p(-u1));
        return mu + sigma * r * std::cos(2.0 * M_PI * u2);
    }
};

double sample(const Dist& d, Rng& rng) {
    double x;
    if (d.dist == "fixed") {
        x = d.value;
    } else if (d.dist == "uniform") {
        x = rng.uniform(d.min, d.max);
    } else if (d.dist == "exponential") {
        x = rng.exponential_mean(d.mean);
    } else if (d.dist == "normal") {
        x = rng.normal(d.mean, d.std);
    } else {
        double total = 0;
        for (size_t i = 0; i < d.values.size(); ++i) total += d.weights.empty() ? 1.0 : d.weights[i];
        double u = rng.uniform() * total;
        x = d.values.back();
        for (size_t i = 0; i < d.values.size(); ++i) {
            u -= d.weights.empty() ? 1.0 : d.weights[i];
            if (u < 0) {
                x = d.values[i];
                break;
            }
        }
    }
    if (d.has_min) x = std::max(x, d.min);
    if (d.has_max) x = std::min(x, d.max);
    return x;
}

}  // namespace

extern "C" cg_status cg_generate_trace(const char* spec_json, uint64_t seed, double* arrival_s,
                                       double* input_tokens, double* output_tokens, double* scores,
                                       int64_t capacity, int64_t* n_out, int32_t* stages_out) {
    cg_status st;
    st.code = CG_OK;
    st.message[0] = 0;
    try {
        json j = json::parse(spec_json);
        const int count = j.at("count").get<int>();
        const double rate = j.at("arrival_rate").get<double>();
        const Dist in = parse_dist(j.at("input_tokens"));
        std::vector<std::pair<Dist, Dist>> stages;
        for (const auto& s : j.at("stages")) stages.emplace_back(parse_dist(s.at("output_tokens")), parse_dist(s.at("score")));
        if (count < 0) throw Fail{CG_ERR_INVALID_INPUT, "trace count must be >= 0"};
        if (rate <= 0) throw Fail{CG_ERR_INVALID_INPUT, "arrival_rate must be positive"};
        if (stages.empty()) throw Fail{CG_ERR_INVALID_INPUT, "trace spec needs stages"};
        validate(in);
        for (const auto& s : stages) {
            validate(s.first);
            validate(s.second);
        }
        if (count > capacity) throw Fail{CG_ERR_INVALID_INPUT, "output capacity too small"};
        const int c = (int)stages.size();
        if (n_out) *n_out = count;
        if (stages_out) *stages_out = c;
        Rng rng(seed);
        double t = 0;
        for (int i = 0; i < count; ++i) {
            t += rng.exponential_mean(1.0) / rate;
            arrival_s[i] = t;
            input_tokens[i] = std::max(0.0, std::round(sample(in, rng)));
            for (int k = 0; k < c; ++k) {
                output_tokens[(int64_t)k * count + i] = std::max(0.0, std::round(sample(stages[k].first, rng)));
                scores[(int64_t)k * count + i] = std::clamp(sample(stages[k].second, rng), 0.0, 100.0);
            }
        }
    } catch (const Fail& f) {
        st.code = f.code;
        std::snprintf(st.message, sizeof(st.message), "%s", f.msg.c_str());
    } catch (const std::exception& e) {
        st.code = CG_ERR_INVALID_INPUT;
        std::snprintf(st.message, sizeof(st.message), "bad trace spec: %s", e.what());
    }
    return st;
}
