// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// extern "C" harness over the UNMODIFIED reference planner (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  Tests,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// call it through ctypes to (a) obtain ground-truth results of the
// reference's own entry points and (b) time the reference CPU scheduler.
//
// Entry points wrapped (reference file:line):
//   cascade::outerplan::sweep            proj/include/cascade/outerplan.hpp:89-92
//   cascade::routing::route_trace        proj/include/cascade/routing.hpp:26-28
//   cascade::costmodel::StageEvaluator::row  proj/include/cascade/costmodel.hpp:110-111
//   cascade::innerplan::solve_min_max    proj/include/cascade/innerplan.hpp:63
//   cascade::cli::generate_trace         proj/include/cascade/cli.hpp:171-172
//   cascade::read_trace_jsonl / write_trace_jsonl  proj/include/cascade/domain.hpp:162-164
//
// Every function returns a malloc'd JSON string (free with ref_free):
//   {"ok":true,"result":<reference to_json of the result>,"elapsed_s":t}
//   {"ok":false,"code":<int Errc>,"code_name":"...","message":"..."}
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <atomic>
#include <map>
#include <thread>
#include <string>
#include <vector>

#include "cascade/cli.hpp"
#include "cascade/costmodel.hpp"
#include "cascade/innerplan.hpp"
#include "cascade/outerplan.hpp"
#include "cascade/routing.hpp"
#include "cascade/simulator.hpp"
#include "cascade/util.hpp"

using nlohmann::json;
using namespace cascade;

namespace {

char* dup(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.data(), s.size() + 1);
    return p;
}

char* ok(json result, double elapsed) {
    json j;
    j["ok"] = true;
    j["result"] = std::move(result);
    j["elapsed_s"] = elapsed;
    return dup(j.dump(-1, ' ', false, json::error_handler_t::replace));
}

char* fail(const CascadeError& e) {
    json j;
    j["ok"] = false;
    j["code"] = static_cast<int>(e.code());
    j["code_name"] = e.code_name();
    j["message"] = e.what();
    return dup(j.dump(-1, ' ', false, json::error_handler_t::replace));
}

char* fail_std(const std::exception& e) {
    json j;
    j["ok"] = false;
    j["code"] = 100;
    j["code_name"] = "STD_EXCEPTION";
    j["message"] = e.what();
    return dup(j.dump(-1, ' ', false, json::error_handler_t::replace));
}

std::vector<TraceRecord> make_trace(const double* arrival, const double* in_tok,
                                    const double* out_tok, const double* scores,
                                    std::int64_t n, int c) {
    std::vector<TraceRecord> trace(static_cast<std::size_t>(n));
    for (std::int64_t r = 0; r < n; ++r) {
        auto& rec = trace[r];
        rec.arrival_s = arrival[r];
        rec.input_tokens = in_tok[r];
        rec.per_stage.resize(c);
        for (int i = 0; i < c; ++i) {
            rec.per_stage[i].output_tokens = out_tok[static_cast<std::int64_t>(i) * n + r];
            rec.per_stage[i].score = scores[static_cast<std::int64_t>(i) * n + r];
        }
    }
    return trace;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

extern "C" {

void ref_free(char* p) { std::free(p); }

/// config_json: {"hardware":{..},"models":[..],"cost_model":{..},"sweep":{..}}
/// (the reference PlannerConfig schema, cli.cpp:48-80).  Times sweep() only.
char* ref_sweep(const double* arrival, const double* in_tok, const double* out_tok,
                const double* scores, std::int64_t n, int c, const char* config_json,
                int total_gpus) {
    try {
        auto cfg = json::parse(config_json).get<cli::PlannerConfig>();
        auto trace = make_trace(arrival, in_tok, out_tok, scores, n, c);
        auto t0 = std::chrono::steady_clock::now();
        auto res = outerplan::sweep(trace, cfg.models, cfg.hardware, cfg.cost_model,
                                    total_gpus, cfg.sweep);
        double el = seconds_since(t0);
        return ok(json(res), el);
    } catch (const CascadeError& e) {
        return fail(e);
    } catch (const std::exception& e) {
        return fail_std(e);
    }
}

/// sweep + select_plan + the CLI file payloads (cli.cpp:165-175), dumped
/// exactly as cmd_plan writes them (dump(2) + "\n", front_to_csv).
char* ref_plan_outputs(const double* arrival, const double* in_tok,
                       const double* out_tok, const double* scores, std::int64_t n,
                       int c, const char* config_json, int total_gpus,
                       const char* requirement_json) {
    try {
        auto cfg = json::parse(config_json).get<cli::PlannerConfig>();
        auto rq = json::parse(requirement_json);
        outerplan::PlanRequirement req;
        if (rq.contains("min_quality")) req.min_quality = rq["min_quality"].get<double>();
        if (rq.contains("max_latency")) req.max_latency = rq["max_latency"].get<double>();
        auto trace = make_trace(arrival, in_tok, out_tok, scores, n, c);
        auto res = outerplan::sweep(trace, cfg.models, cfg.hardware, cfg.cost_model,
                                    total_gpus, cfg.sweep);
        auto plan = outerplan::select_plan(res.front, req);
        json files;
        files["plan.json"] = json(plan).dump(2) + "\n";
        files["front.json"] = json(res.front).dump(2) + "\n";
        files["front.csv"] = outerplan::front_to_csv(res.front);
        files["sweep.json"] = json(res).dump(2) + "\n";
        return ok(files, 0.0);
    } catch (const CascadeError& e) {
        return fail(e);
    } catch (const std::exception& e) {
        return fail_std(e);
    }
}

char* ref_route(const double* arrival, const double* in_tok, const double* out_tok,
                const double* scores, std::int64_t n, int c, const double* thresholds,
                const int* deployed) {
    try {
        auto trace = make_trace(arrival, in_tok, out_tok, scores, n, c);
        RoutingThresholds h;
        h.thresholds.assign(thresholds, thresholds + (c > 0 ? c - 1 : 0));
        std::vector<bool> dep(c);
        for (int i = 0; i < c; ++i) dep[i] = deployed[i] != 0;
        auto t0 = std::chrono::steady_clock::now();
        auto out = routing::route_trace(trace, h, dep);
        double el = seconds_since(t0);
        json j;
        j["ratios"] = out.ratios;
        j["stage_workloads"] = out.stage_workloads;
        j["quality"] = out.quality;
        j["per_request_accept_stage"] = out.per_request_accept_stage;
        return ok(j, el);
    } catch (const CascadeError& e) {
        return fail(e);
    } catch (const std::exception& e) {
        return fail_std(e);
    }
}

/// One StageEvaluator::row (costmodel.cpp:296-414).
char* ref_row(const char* hw_json, const char* params_json, const char* model_json,
              const char* workload_json, int max_budget) {
    try {
        auto hw = json::parse(hw_json).get<HardwareSpec>();
        auto params = json::parse(params_json).get<costmodel::CostModelParams>();
        auto model = json::parse(model_json).get<ModelSpec>();
        auto w = json::parse(workload_json).get<WorkloadStats>();
        costmodel::StageEvaluator ev(hw, params);
        auto t0 = std::chrono::steady_clock::now();
        auto row = ev.row(model, w, max_budget);
        double el = seconds_since(t0);
        json lat = json::array();
        for (double v : row.latency) {
            if (std::isinf(v)) lat.push_back(nullptr);
            else lat.push_back(v);
        }
        json plans = json::array();
        for (const auto& p : row.plan) {
            if (p) plans.push_back(*p);
            else plans.push_back(nullptr);
        }
        json j;
        j["latency"] = lat;
        j["plan"] = plans;
        return ok(j, el);
    } catch (const CascadeError& e) {
        return fail(e);
    } catch (const std::exception& e) {
        return fail_std(e);
    }
}

/// innerplan::solve_min_max on a LatencyTable in its JSON "profile" format
/// (innerplan.cpp:14-56; null = infeasible).
char* ref_solve(const char* table_json, int total_gpus) {
    try {
        auto table = json::parse(table_json).get<innerplan::LatencyTable>();
        auto sol = innerplan::solve_min_max(table, total_gpus);
        json j;
        j["allocations"] = sol.allocations;
        j["objective_L"] = sol.objective_L;
        j["per_stage_latency"] = sol.per_stage_latency;
        return ok(j, 0.0);
    } catch (const CascadeError& e) {
        return fail(e);
    } catch (const std::exception& e) {
        return fail_std(e);
    }
}

char* ref_export_milp(const char* table_json, int total_gpus) {
    try {
        auto table = json::parse(table_json).get<innerplan::LatencyTable>();
        return ok(json(innerplan::export_milp(table, total_gpus)), 0.0);
    } catch (const CascadeError& e) {
        return fail(e);
    } catch (const std::exception& e) {
        return fail_std(e);
    }
}

/// cli::generate_trace (cli.cpp:428-460) into caller-owned SoA buffers
/// sized count and stages*count (stage-major).  Returns the error JSON or
/// an ok JSON with the count.
char* ref_generate_trace(const char* spec_json, std::uint64_t seed, double* arrival,
                         double* in_tok, double* out_tok, double* scores,
                         std::int64_t capacity) {
    try {
        auto spec = json::parse(spec_json).get<cli::TraceGenSpec>();
        auto trace = cli::generate_trace(spec, seed);
        const std::int64_t n = static_cast<std::int64_t>(trace.size());
        if (n > capacity) throw std::runtime_error("capacity too small");
        const int c = static_cast<int>(spec.stages.size());
        for (std::int64_t r = 0; r < n; ++r) {
            arrival[r] = trace[r].arrival_s;
            in_tok[r] = trace[r].input_tokens;
            for (int i = 0; i < c; ++i) {
                out_tok[static_cast<std::int64_t>(i) * n + r] =
                    trace[r].per_stage[i].output_tokens;
                scores[static_cast<std::int64_t>(i) * n + r] = trace[r].per_stage[i].score;
            }
        }
        return ok(json(n), 0.0);
    } catch (const CascadeError& e) {
        return fail(e);
    } catch (const std::exception& e) {
        return fail_std(e);
    }
}

/// cmd_plan's sweep.json / front.json payloads (cli.cpp:121,167-172) of a
/// SweepResult given as JSON: from_json, then json(res).dump(2) timed.
char* ref_dump_sweep(const char* sweep_json) {
    try {
        const json j = json::parse(sweep_json);
        outerplan::SweepResult res;  // no from_json(SweepResult) in the reference: member-wise
        j.at("front").get_to(res.front);
        j.at("evaluations").get_to(res.evaluations);
        j.at("weights").get_to(res.weights);
        j.at("weight_selection").get_to(res.weight_selection);
        j.at("utopia").get_to(res.utopia);
        j.at("skipped").get_to(res.skipped);
        const auto t0 = std::chrono::steady_clock::now();
        std::string sweep_text = json(res).dump(2) + "\n";
        std::string front_text = json(res.front).dump(2) + "\n";
        const double el = seconds_since(t0);
        json files;
        files["sweep.json"] = std::move(sweep_text);
        files["front.json"] = std::move(front_text);
        return ok(files, el);
    } catch (const CascadeError& e) {
        return fail(e);
    } catch (const std::exception& e) {
        return fail_std(e);
    }
}

/// sim::run of one plan (compare == 0, plans_json = [plan]) or sim::compare
/// of a plan list: json(SimReport) / json(CompareResult) (simulator.cpp).
char* ref_simulate(const double* arrival, const double* in_tok, const double* out_tok,
                   const double* scores, std::int64_t n, int c, const char* config_json,
                   const char* plans_json, const char* sim_json, int compare) {
    try {
        auto cfg = json::parse(config_json).get<cli::PlannerConfig>();
        std::vector<CascadePlan> plans;
        for (const auto& p : json::parse(plans_json)) plans.push_back(p.get<CascadePlan>());
        auto sc = json::parse(sim_json).get<sim::SimConfig>();
        auto trace = make_trace(arrival, in_tok, out_tok, scores, n, c);
        const auto t0 = std::chrono::steady_clock::now();
        json out;
        if (compare) {
            out = sim::compare(plans, trace, cfg.models, cfg.hardware, cfg.cost_model, sc);
        } else {
            out = sim::run(plans.at(0), trace, cfg.models, cfg.hardware, cfg.cost_model, sc);
        }
        return ok(std::move(out), seconds_since(t0));
    } catch (const CascadeError& e) {
        return fail(e);
    } catch (const std::exception& e) {
        return fail_std(e);
    }
}

/// cli::cmd_drift (cli.cpp:216-334, replan off) on a stream given as SoA
/// columns: the files it reads are written into work_dir; returns the
/// drift_report.json document.  Also compute_baseline of the same stream
/// with h1 (has_h1) as "baseline_of_stream".
char* ref_drift(const double* arrival, const double* in_tok, const double* out_tok, const double* scores,
                std::int64_t n, int c, const char* config_json, const char* baseline_json, const char* work_dir,
                int has_h1, double h1) {
    try {
        namespace fs = std::filesystem;
        fs::create_directories(work_dir);
        const std::string dir(work_dir);
        { std::ofstream(dir + "/config.json") << config_json; }
        { std::ofstream(dir + "/baseline.json") << baseline_json; }
        auto trace = make_trace(arrival, in_tok, out_tok, scores, n, c);
        write_trace_jsonl(dir + "/stream.jsonl", trace);
        cli::DriftArgs args;
        args.config_path = dir + "/config.json";
        args.baseline_path = dir + "/baseline.json";
        args.trace_path = dir + "/stream.jsonl";
        args.out_dir = dir + "/out";
        const auto t0 = std::chrono::steady_clock::now();
        auto res = cli::cmd_drift(args);
        const double el = seconds_since(t0);
        std::ifstream rep(res.report_path);
        json out;
        out["report"] = json::parse(rep);
        CascadePlan plan;
        if (has_h1) plan.thresholds.thresholds = {h1};
        out["baseline_of_stream"] = cli::compute_baseline(trace, plan);
        return ok(std::move(out), el);
    } catch (const CascadeError& e) {
        return fail(e);
    } catch (const std::exception& e) {
        return fail_std(e);
    }
}

/// write_trace_jsonl (domain.cpp:389-394) of SoA columns.
char* ref_write_trace_jsonl(const double* arrival, const double* in_tok, const double* out_tok,
                            const double* scores, std::int64_t n, int c, const char* path) {
    try {
        write_trace_jsonl(path, make_trace(arrival, in_tok, out_tok, scores, n, c));
        return ok(json(n), 0.0);
    } catch (const CascadeError& e) {
        return fail(e);
    } catch (const std::exception& e) {
        return fail_std(e);
    }
}

/// read_trace_jsonl (domain.cpp:361-387) into caller-owned SoA buffers
/// (capacity records, stage-major with stride n).  ok JSON {"n":..,"stages":..}.
char* ref_read_trace_jsonl(const char* path, double* arrival, double* in_tok, double* out_tok,
                           double* scores, std::int64_t capacity, int max_stages) {
    try {
        const auto t0 = std::chrono::steady_clock::now();
        auto trace = read_trace_jsonl(path);
        const double el = seconds_since(t0);
        const std::int64_t n = static_cast<std::int64_t>(trace.size());
        const int c = n ? static_cast<int>(trace.front().per_stage.size()) : 0;
        if (n > capacity || c > max_stages) throw std::runtime_error("capacity too small");
        for (std::int64_t r = 0; r < n; ++r) {
            arrival[r] = trace[r].arrival_s;
            in_tok[r] = trace[r].input_tokens;
            for (int i = 0; i < c; ++i) {
                out_tok[static_cast<std::int64_t>(i) * n + r] = trace[r].per_stage[i].output_tokens;
                scores[static_cast<std::int64_t>(i) * n + r] = trace[r].per_stage[i].score;
            }
        }
        return ok(json{{"n", n}, {"stages", c}}, el);
    } catch (const CascadeError& e) {
        return fail(e);
    } catch (const std::exception& e) {
        return fail_std(e);
    }
}

/// Weight ladder, default grid and utopia helpers, for unit-level parity.
char* ref_weight_ladder(double rmin, double rmax, int count) {
    try {
        outerplan::SweepConfig cfg;
        cfg.weight_ratio_min = rmin;
        cfg.weight_ratio_max = rmax;
        cfg.weight_count = count;
        return ok(json(outerplan::weight_ladder(cfg)), 0.0);
    } catch (const CascadeError& e) {
        return fail(e);
    } catch (const std::exception& e) {
        return fail_std(e);
    }
}

char* ref_pareto(const double* latency, const double* quality, std::int64_t n) {
    try {
        std::vector<ObjectivePoint> pts(static_cast<std::size_t>(n));
        for (std::int64_t i = 0; i < n; ++i) {
            pts[i].latency_s = latency[i];
            pts[i].quality = quality[i];
            pts[i].plan_ref.predicted_max_p95_s = static_cast<double>(i);  // index tag
        }
        auto front = outerplan::pareto_filter(pts);
        json idx = json::array();
        for (const auto& p : front.points)
            idx.push_back(static_cast<std::int64_t>(p.plan_ref.predicted_max_p95_s));
        return ok(idx, 0.0);
    } catch (const std::exception& e) {
        return fail_std(e);
    }
}

/// Counts what one sweep() must decide, with the reference's own APIs: the
/// unique (stage, WorkloadStats) rows of its row cache (outerplan.cpp:191-203,
/// live stages only) and the sum of their plan-set sizes (enumerate_plans).
char* ref_plan_count(const double* arrival, const double* in_tok, const double* out_tok,
                     const double* scores, std::int64_t n, int c, const char* config_json,
                     int total_gpus) {
    try {
        auto cfg = json::parse(config_json).get<cli::PlannerConfig>();
        auto trace = make_trace(arrival, in_tok, out_tok, scores, n, c);
        auto grid = cfg.sweep.threshold_grid.empty()
                        ? outerplan::default_threshold_grid(trace, static_cast<std::size_t>(c))
                        : cfg.sweep.threshold_grid;
        std::vector<bool> deployed(c, true);
        std::map<std::string, int> rows;
        std::vector<std::size_t> cursor(grid.size(), 0);
        long long candidates = 0;
        bool done = false;
        while (!done) {
            RoutingThresholds h;
            for (std::size_t d = 0; d < grid.size(); ++d) h.thresholds.push_back(grid[d][cursor[d]]);
            auto out = routing::route_trace(trace, h, deployed);
            ++candidates;
            for (int i = 0; i < c; ++i) {
                if (!(out.ratios[i] > 0.0)) continue;
                const auto& w = out.stage_workloads[i];
                double f[5] = {w.arrival_rate, w.mean_input_tokens, w.mean_output_tokens,
                               w.p95_input_tokens, w.p95_output_tokens};
                std::string key(sizeof(int) + sizeof(f), '\0');
                std::memcpy(key.data(), &i, sizeof(int));
                std::memcpy(key.data() + sizeof(int), f, sizeof(f));
                rows.emplace(key, i);
            }
            done = true;
            for (std::size_t d = grid.size(); d-- > 0;) {
                if (++cursor[d] < grid[d].size()) { done = false; break; }
                cursor[d] = 0;
            }
            if (grid.empty()) break;
        }
        std::vector<long long> per_stage(c, -1);
        long long plans = 0;
        for (const auto& kv : rows) {
            int i = kv.second;
            if (per_stage[i] < 0)
                per_stage[i] = total_gpus >= 1
                    ? static_cast<long long>(costmodel::enumerate_plans(total_gpus, cfg.models[i],
                                                                        cfg.hardware, cfg.cost_model).size())
                    : 0;
            plans += per_stage[i];
        }
        json j;
        j["unique_rows"] = rows.size();
        j["plans"] = plans;
        j["candidates"] = candidates;
        return ok(j, 0.0);
    } catch (const CascadeError& e) {
        return fail(e);
    } catch (const std::exception& e) {
        return fail_std(e);
    }
}

/// The unique (stage, WorkloadStats) rows of a sweep -- the reference's own
/// row-cache keys (outerplan.cpp:155-162, 191-203) -- from route_trace over
/// every grid candidate (outerplan.cpp:221-239), the candidates routed
/// concurrently on `threads` std::threads (route_trace is a pure function).
/// Used only to size the CPU-baseline extrapolation in bench.py.  Reports
/// the summed per-call route_trace time (what the sequential sweep spends).
char* ref_unique_rows(const double* arrival, const double* in_tok, const double* out_tok,
                      const double* scores, std::int64_t n, int c, const char* config_json,
                      int total_gpus, int threads) {
    try {
        auto cfg = json::parse(config_json).get<cli::PlannerConfig>();
        auto trace = make_trace(arrival, in_tok, out_tok, scores, n, c);
        auto grid = cfg.sweep.threshold_grid.empty()
                        ? outerplan::default_threshold_grid(trace, static_cast<std::size_t>(c))
                        : cfg.sweep.threshold_grid;
        std::vector<std::vector<double>> cands;
        std::vector<std::size_t> cursor(grid.size(), 0);
        for (bool done = false; !done;) {
            std::vector<double> h;
            for (std::size_t d = 0; d < grid.size(); ++d) h.push_back(grid[d][cursor[d]]);
            cands.push_back(std::move(h));
            done = true;
            for (std::size_t d = grid.size(); d-- > 0;) {
                if (++cursor[d] < grid[d].size()) { done = false; break; }
                cursor[d] = 0;
            }
            if (grid.empty()) break;
        }
        std::vector<bool> deployed(c, true);
        std::vector<routing::RoutingOutcome> outs(cands.size());
        std::vector<double> secs(cands.size(), 0.0);
        if (threads < 1) threads = 1;
        std::vector<std::thread> pool;
        std::atomic<std::size_t> next{0};
        for (int t = 0; t < threads; ++t)
            pool.emplace_back([&] {
                for (std::size_t i; (i = next.fetch_add(1)) < cands.size();) {
                    RoutingThresholds h;
                    h.thresholds = cands[i];
                    auto t0 = std::chrono::steady_clock::now();
                    outs[i] = routing::route_trace(trace, h, deployed);
                    secs[i] = seconds_since(t0);
                }
            });
        for (auto& t : pool) t.join();
        std::map<std::string, std::pair<int, WorkloadStats>> rows;
        double route_s = 0.0;
        for (std::size_t k = 0; k < cands.size(); ++k) {
            route_s += secs[k];
            for (int i = 0; i < c; ++i) {
                if (!(outs[k].ratios[i] > 0.0)) continue;
                const auto& w = outs[k].stage_workloads[i];
                double f[5] = {w.arrival_rate, w.mean_input_tokens, w.mean_output_tokens,
                               w.p95_input_tokens, w.p95_output_tokens};
                std::string key(sizeof(int) + sizeof(f), '\0');
                std::memcpy(key.data(), &i, sizeof(int));
                std::memcpy(key.data() + sizeof(int), f, sizeof(f));
                rows.emplace(key, std::make_pair(i, w));
            }
        }
        json list = json::array();
        for (const auto& kv : rows) list.push_back({{"stage", kv.second.first}, {"workload", kv.second.second}});
        json j;
        j["rows"] = std::move(list);
        j["candidates"] = cands.size();
        j["route_calls_s"] = route_s;
        j["total_gpus"] = total_gpus;
        return ok(j, route_s);
    } catch (const CascadeError& e) {
        return fail(e);
    } catch (const std::exception& e) {
        return fail_std(e);
    }
}

int ref_max_threads() { return util::max_threads(); }

}  // extern "C"
