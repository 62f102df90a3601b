// Drift windows (k_drift.cu): internal interface.
#pragma once

#include <vector>

#include "cg_cuda.h"

namespace cg {

struct DriftWindowOut {
    long long k, first, requests, sampled;
    double start, span, rate, mean_in, mean_out, accept;
    int valid;  // span > 0
};

struct DriftArgs {
    long long n;
    const double* arrival;
    const double* in;
    const double* out0;     // stage-1 output tokens
    const double* score0;   // stage-1 scores
    double t0, stream_end, interval;
    long long window_requests;
    int has_h1;
    double h1;
    const long long* win;   // [n] window index per record
    const long long* first;
    const long long* count;
    long long nwin;
    DriftWindowOut* out;
};

struct DriftBuffers {
    DevBuf win, heads, cnt, first, count, out, res, arr, in, out0, sc0;
};

void drift_windows(DriftBuffers& B, cudaStream_t s, DriftArgs a, std::vector<DriftWindowOut>& out, int* launches);
// stats_of_records over the whole trace: mean input, mean stage-1 output, accept rate
void trace_baseline(DriftBuffers& B, cudaStream_t s, DriftArgs a, double res[3], int* launches);

}  // namespace cg
