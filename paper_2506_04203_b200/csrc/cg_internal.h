// Internal host/device definitions of the plan-search engine.
//
// Layout in HBM (one sweep):
//   trace     : scores f64[C][n], input f64[n], output f64[C][n]  (caller SoA, stage-major)
//   ranks     : u64[n]   16-bit rank of each request per threshold dimension
//   hist      : u64[cells][Q]  count, sum_in, sum_out[0..C-1] per rank cell
//   lists     : (key u64, ranks u64)[C+1][n]  tokens sorted ascending (p95 scans)
//   workloads : per (stage, threshold prefix): count, sums, p95 -> WorkloadStats
//   rows      : per unique row: shape service table, CRN stream T/O f64[n_req],
//               per-budget best (latency bits, plan index), final row
//   candidates: per distinct threshold tuple: quality, L, allocation, plan refs
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace cg {

constexpr int kMaxStages = 5;    // threshold dims <= 4, 16-bit ranks packed in a u64
constexpr int kMaxShapes = 32;   // tp in {1,2,4,8..} x pp in 1..8
constexpr int kMaxDp = 256;      // replicas per plan handled by the JSQ kernels
constexpr int kHistQ = 2 + kMaxStages;

struct ShapeDesc {
    int tp, pp, gpus;
};

// One model's plan space: shapes legal at kv_tokens = 1 in the reference's
// canonical order (costmodel.cpp:92-116) and the multiset counting table
// ways[i][b] = #count vectors over shapes i..S-1 using <= b GPUs (incl. empty).
struct PlanSpace {
    int S;
    int N;
    ShapeDesc shapes[kMaxShapes];
    const unsigned long long* ways;   // device, (S+1)*(N+1)
    unsigned long long num_plans;     // ways[0][N] - 1
};

// Per unique latency row (one (stage, WorkloadStats) cache entry).
struct RowDesc {
    int stage;            // model index
    int space;            // PlanSpace index
    int cls;              // JSQ kernel class
    int dpmax;            // max replicas over plans with only ok shapes
    double rate, mean_in, mean_out, p95_in, p95_out;
};

// Per-row derived tables (device), indexed [row][shape].
struct RowTables {
    unsigned char* shape_ok;
    double* prefill;
    double* decode;
    double* mean_service;
    double* inv_service;  // fl(1 / mean_service), NaN for infeasible shapes: the filter's fast stability test
    double* svc_k;        // prefill + o_(K) * decode: the filter's per-part service bound term
    double* T;            // [row][ld] CRN arrivals (first n_req used)
    double* O;            // [row][ld] CRN outputs
    int ld;               // row stride: n_req rounded up to a multiple of 4 (32-byte rows)
    // future-service bound: requests ranked by output (largest first) in
    // blocks of 32; Pv[row][i] = the smallest output among the top 32(i+1),
    // fut[c][i] = #{requests j >= 32c among the top 32(i+1)}
    int nc;
    const int* probe_req; // [nc] request index of block i's smallest output
    double* Pv;           // [row][nc]
    const unsigned* fut;  // [(na+1)][nc], na = arrival blocks of fut_ab = 2^fut_sh requests
    int fut_ab, fut_sh;
};

struct SimItem {
    int row;
    int pad;
    unsigned long long lo, hi;   // plan index range [lo, hi)
};

struct TieEntry {
    int row;
    int g;
    unsigned long long lat_bits;
    unsigned long long plan;
};

// Device-side sortable transform of doubles (ascending order of keys ==
// ascending numeric order; NaN-free inputs).
__host__ __device__ inline unsigned long long dbl_to_key(double x) {
    unsigned long long b;
#ifdef __CUDA_ARCH__
    b = static_cast<unsigned long long>(__double_as_longlong(x));
#else
    __builtin_memcpy(&b, &x, 8);
#endif
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ inline double key_to_dbl(unsigned long long k) {
    unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
#ifdef __CUDA_ARCH__
    return __longlong_as_double(static_cast<long long>(b));
#else
    double x;
    __builtin_memcpy(&x, &b, 8);
    return x;
#endif
}

// nearest-rank index (util.cpp:11-17): element ceil(q*n) (1-based), clamped.
__host__ __device__ inline long long p95_index(long long n) {
    double r = ceil(0.95 * static_cast<double>(n));
    long long rank = static_cast<long long>(r);
    if (rank < 1) rank = 1;
    if (rank > n) rank = n;
    return rank - 1;
}

}  // namespace cg
