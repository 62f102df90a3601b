// Reference-side binding of the GPU output writer (cg_sweep_result_json):
// the bytes nlohmann::json(res).dump(indent) / json(res.front).dump(indent)
// produce, rendered on the B200.  cmd_plan's sweep.json / front.json
// (proj/src/cli.cpp:167-172) become
//     write_output_file(dir, "sweep.json", outerplan::sweep_json(result.sweep, 2) + "\n");
//     write_output_file(dir, "front.json", outerplan::front_json(result.sweep, 2) + "\n");
#pragma once

#include <string>

#include "cascade/outerplan.hpp"

namespace cascade::outerplan {

std::string sweep_json(const SweepResult& res, int indent);
std::string front_json(const SweepResult& res, int indent);

}  // namespace cascade::outerplan
