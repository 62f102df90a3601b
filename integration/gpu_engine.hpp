// Process-wide B200 engine shared by the reference-side bindings
// (outerplan_gpu.cpp, domain_gpu.cpp): one cg_engine on CASCADE_PLANNER_GPU
// (default 0), and cg_status -> CascadeError with the reference's Errc/message.
#pragma once

#include "cascade/errors.hpp"
#include "cascade_gpu.h"

namespace cascade::gpu_binding {

cg_engine* engine();
[[noreturn]] void raise(const cg_status& st);

}  // namespace cascade::gpu_binding
