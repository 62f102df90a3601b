// Drop-in check: the reference planner with cascade::outerplan::sweep and
// cascade::read_trace_jsonl served by the GPU engine (integration/*_gpu.cpp)
// vs. the reference's own CPU bodies (outerplan.cpp / domain.cpp compiled
// with -Dsweep=cpu_sweep / -Dread_trace_jsonl=cpu_read_trace_jsonl, see
// oracle/Makefile target `dropin`).  Runs the CLI's plan pipeline and
// compares the output files byte for byte.
//
//   dropin_check <config.json> <trace-spec.json> <seed> <out_dir> [min_quality]
//   dropin_check <config.json> <trace.jsonl> 0 <out_dir> <min_quality> --gpu-only [reps]
//
// Writes <out_dir>/{gpu,cpu}/{plan.json,front.json,front.csv,sweep.json} and
// prints one JSON line {"identical": bool, "files": {...}, "gpu_s":..,"cpu_s":..}.
// --gpu-only times the GPU-served pipeline alone (the CPU sweep of a large
// config takes tens of minutes): cmd_plan end to end (JSONL ingest, sweep,
// output files) and outerplan::sweep through the C++ binding on the parsed
// records (AoS -> SoA, pageable copies, SweepResult rebuild), `reps` times.
#include <chrono>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <sstream>

#include "cascade/cli.hpp"
#include "cascade/outerplan.hpp"
#include "cascade/simulator.hpp"
#include "output_gpu.hpp"

namespace cascade {
std::vector<TraceRecord> cpu_read_trace_jsonl(const std::string& path);
}
namespace cascade::sim {
SimReport cpu_run(const CascadePlan& plan, const std::vector<TraceRecord>& trace, const std::vector<ModelSpec>& models,
                  const HardwareSpec& hw, const costmodel::CostModelParams& params, const SimConfig& cfg);
}
namespace cascade::outerplan {
SweepResult cpu_sweep(const std::vector<TraceRecord>& trace, const std::vector<ModelSpec>& models,
                      const HardwareSpec& hw, const costmodel::CostModelParams& params, int total_gpus,
                      const SweepConfig& cfg);
}

using namespace cascade;
using nlohmann::json;

static std::string slurp(const std::string& p) {
    std::ifstream in(p);
    std::stringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

int main(int argc, char** argv) {
    if (argc < 5) {
        std::fprintf(stderr, "usage: %s config.json spec.json seed out_dir [min_quality]\n", argv[0]);
        return 2;
    }
    const std::string cfg_path = argv[1], spec_path = argv[2], out = argv[4];
    const uint64_t seed = std::stoull(argv[3]);
    const double min_q = argc > 5 ? std::stod(argv[5]) : 0.0;
    const bool gpu_only = argc > 6 && std::string(argv[6]) == "--gpu-only";
    const int reps = argc > 7 ? std::stoi(argv[7]) : 3;
    namespace fs = std::filesystem;
    fs::create_directories(out + "/gpu");
    fs::create_directories(out + "/cpu");
    std::string trace_path = out + "/trace.jsonl";
    if (spec_path.size() > 6 && spec_path.substr(spec_path.size() - 6) == ".jsonl") {
        trace_path = spec_path;  // a prepared trace (e.g. C3's concatenated bursty segments)
    } else {
        auto spec = json::parse(slurp(spec_path)).get<cli::TraceGenSpec>();
        auto trace = cli::generate_trace(spec, seed);
        write_trace_jsonl(trace_path, trace);
    }
    if (gpu_only) {
        cli::PlanArgs args;
        args.config_path = cfg_path;
        args.trace_path = trace_path;
        args.out_dir = out + "/gpu";
        args.min_quality = min_q;
        json report;
        std::vector<double> plan_s, sweep_s;
        auto cfg = cli::load_planner_config(cfg_path);
        auto tr = read_trace_jsonl(trace_path);  // GPU ingest (warm-up of the engine too)
        for (int i = 0; i < reps + 1; ++i) {
            auto t0 = std::chrono::steady_clock::now();
            cli::cmd_plan(args);
            const double a = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            t0 = std::chrono::steady_clock::now();
            auto res = outerplan::sweep(tr, cfg.models, cfg.hardware, cfg.cost_model, cfg.hardware.gpu_count, cfg.sweep);
            const double b = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (i > 0) {  // the first pass warms up the engine's buffers
                plan_s.push_back(a);
                sweep_s.push_back(b);
            }
            if (res.evaluations.empty() && res.skipped.empty()) std::fprintf(stderr, "empty sweep\n");
        }
        report["records"] = tr.size();
        report["cmd_plan_s"] = plan_s;
        report["sweep_binding_s"] = sweep_s;
        std::cout << report.dump() << std::endl;
        return 0;
    }

    // GPU: the reference CLI pipeline, whose sweep() call now lands in the engine.
    cli::PlanArgs args;
    args.config_path = cfg_path;
    args.trace_path = trace_path;
    args.out_dir = out + "/gpu";
    args.min_quality = min_q;
    auto t0 = std::chrono::steady_clock::now();
    cli::cmd_plan(args);
    const double gpu_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

    // CPU: the reference's own sweep body, same writers as cmd_plan.
    auto cfg = cli::load_planner_config(cfg_path);
    t0 = std::chrono::steady_clock::now();
    auto tr = cpu_read_trace_jsonl(trace_path);
    const double cpu_read_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    t0 = std::chrono::steady_clock::now();
    auto tr_gpu = read_trace_jsonl(trace_path);
    const double gpu_read_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const bool trace_identical = tr_gpu == tr;
    t0 = std::chrono::steady_clock::now();
    auto res = outerplan::cpu_sweep(tr, cfg.models, cfg.hardware, cfg.cost_model, cfg.hardware.gpu_count, cfg.sweep);
    const double cpu_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    outerplan::PlanRequirement req;
    req.min_quality = min_q;
    auto plan = outerplan::select_plan(res.front, req);
    cli::write_output_file(out + "/cpu", "plan.json", json(plan).dump(2) + "\n");
    cli::write_output_file(out + "/cpu", "front.json", json(res.front).dump(2) + "\n");
    cli::write_output_file(out + "/cpu", "front.csv", outerplan::front_to_csv(res.front));
    cli::write_output_file(out + "/cpu", "sweep.json", json(res).dump(2) + "\n");

    // GPU output writer vs the reference's nlohmann dump of the same result
    t0 = std::chrono::steady_clock::now();
    const std::string cpu_sweep_text = json(res).dump(2) + "\n";
    const double cpu_dump_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    t0 = std::chrono::steady_clock::now();
    const std::string gpu_sweep_text = outerplan::sweep_json(res, 2) + "\n";
    const std::string gpu_front_text = outerplan::front_json(res, 2) + "\n";
    const double gpu_dump_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const bool writer_identical = gpu_sweep_text == cpu_sweep_text &&
                                  gpu_front_text == json(res.front).dump(2) + "\n";

    // validation simulator: cmd_simulate's report.json (GPU sim::run) vs the
    // reference body on the selected plan
    bool sim_identical = true;
    double gpu_sim_s = 0, cpu_sim_s = 0;
    {
        cli::SimulateArgs sargs;
        sargs.config_path = cfg_path;
        sargs.plan_path = out + "/gpu/plan.json";
        sargs.trace_path = trace_path;
        sargs.out_dir = out + "/gpu_sim";
        t0 = std::chrono::steady_clock::now();
        cli::cmd_simulate(sargs);
        gpu_sim_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        sim::SimConfig sc;
        t0 = std::chrono::steady_clock::now();
        auto rep = sim::cpu_run(plan, tr, cfg.models, cfg.hardware, cfg.cost_model, sc);
        cpu_sim_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        sim_identical = slurp(out + "/gpu_sim/report.json") == json(rep).dump(2) + "\n";
    }

    if (!writer_identical) {  // keep both texts for inspection
        cli::write_output_file(out, "writer_gpu_sweep.json", gpu_sweep_text);
        cli::write_output_file(out, "writer_ref_sweep.json", cpu_sweep_text);
    }

    json report;
    bool all = true;
    for (const char* f : {"plan.json", "front.json", "front.csv", "sweep.json"}) {
        const std::string a = slurp(out + "/gpu/" + f), b = slurp(out + "/cpu/" + f);
        report["files"][f] = {{"identical", a == b}, {"bytes", a.size()}};
        all = all && a == b;
    }
    all = all && trace_identical && writer_identical && sim_identical;
    report["sim_identical"] = sim_identical;
    report["gpu_sim_s"] = gpu_sim_s;
    report["cpu_sim_s"] = cpu_sim_s;
    report["writer_identical"] = writer_identical;
    report["cpu_dump_s"] = cpu_dump_s;
    report["gpu_dump_s"] = gpu_dump_s;
    report["trace_identical"] = trace_identical;
    report["gpu_read_s"] = gpu_read_s;
    report["cpu_read_s"] = cpu_read_s;
    report["identical"] = all;
    report["gpu_s"] = gpu_s;
    report["cpu_s"] = cpu_s;
    std::cout << report.dump() << std::endl;
    return all ? 0 : 1;
}
