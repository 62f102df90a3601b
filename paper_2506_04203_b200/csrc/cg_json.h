// Output serialisation (k_json.cu): the reference's JSON result files.
#pragma once

#include <string>

#include "cascade_gpu.h"
#include "cg_cuda.h"

namespace cg {

struct JsonBuffers {
    DevBuf thr, lat, qual, ratios, alloc, eplan, pg, pd, po, rt, rp, front, skip, len, off, text;
};

// what = 0: json(SweepResult).dump(step); what = 1: json(result.front).dump(step).
std::string result_json(JsonBuffers& B, cudaStream_t s, const cg_sweep_result& r, int step, int what, int flags,
                        int* launches);

}  // namespace cg
