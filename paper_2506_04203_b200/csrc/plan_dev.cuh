// Device-side plan-space helpers shared by the cost-model kernels and the
// cross-rank merge: unranking, lexicographic successor, parts comparator.
//
// Plan order = the reference's enumerate_multisets recursion
// (proj/src/costmodel.cpp:132-146): count vectors (c_0..c_{S-1}) over the
// canonical shape list in lexicographic order, the empty multiset skipped.
#pragma once

#include "cg_internal.h"

namespace cg {

__host__ __device__ __forceinline__ unsigned long long ways_at(const PlanSpace& sp, int i, int b) {
    return sp.ways[(long long)i * (sp.N + 1) + b];
}

// plan index p (0-based) -> counts; returns the GPUs used
__host__ __device__ inline int unrank_plan(const PlanSpace& sp, unsigned long long p, unsigned char* c) {
    unsigned long long q = p + 1;  // lexicographic rank including the empty multiset
    int b = sp.N;
    int used = 0;
    for (int i = 0; i < sp.S; ++i) {
        const int size = sp.shapes[i].gpus;
        int k = 0;
        while (true) {
            const unsigned long long w = ways_at(sp, i + 1, b - k * size);
            if (q < w) break;
            q -= w;
            ++k;
        }
        c[i] = (unsigned char)k;
        b -= k * size;
        used += k * size;
    }
    return used;
}

// successor in the recursion order (last shape fastest); false at the end.
// `used` (GPUs) and `dp` (replicas) are maintained incrementally.
__host__ __device__ inline bool next_plan(const PlanSpace& sp, unsigned char* c, int& used, int& dp) {
    for (int i = sp.S - 1; i >= 0; --i) {
        const int size = sp.shapes[i].gpus;
        if (used + size <= sp.N) {
            c[i] = (unsigned char)(c[i] + 1);
            used += size;
            dp += 1;
            return true;
        }
        used -= c[i] * size;
        dp -= c[i];
        c[i] = 0;
    }
    return false;
}

// Merge rule of per-budget bests across shards / ranks (the reference's
// `better`, costmodel.cpp:347-352): smaller latency, then parts-lexicographic.
// `ways` must point at the table the caller's memory space can read.
__host__ __device__ inline bool merge_take(const PlanSpace& sp, unsigned long long lat, unsigned long long plan,
                                           unsigned long long best_lat, unsigned long long best_plan);

// '<' of CompactPlan::parts (vector<pair<shape, count>>, costmodel.cpp:351)
// evaluated on dense count vectors.
// Sharded calls: local work chunk l of `rank` is global chunk l*world + rank
// of the sweep's chunk list (64 consecutive plan indices per chunk, rows in
// list order, each row's chunks from its last to its first).
__host__ __device__ __forceinline__ unsigned long long shard_global_chunk(unsigned long long l, int rank, int world) {
    return l * (unsigned long long)(world > 0 ? world : 1) + (unsigned long long)rank;
}

__host__ __device__ inline bool parts_less(const unsigned char* A, const unsigned char* B, int S) {
    for (int s = 0; s < S; ++s) {
        if (A[s] == B[s]) continue;
        if (A[s] > 0 && B[s] > 0) return A[s] < B[s];
        if (A[s] == 0) {  // A's next pair has a larger shape index, or A ended
            for (int t = s + 1; t < S; ++t)
                if (A[t]) return false;
            return true;
        }
        for (int t = s + 1; t < S; ++t)
            if (B[t]) return true;
        return false;
    }
    return false;
}

__host__ __device__ inline bool merge_take(const PlanSpace& sp, unsigned long long lat, unsigned long long plan,
                                           unsigned long long best_lat, unsigned long long best_plan) {
    if (plan == ~0ull) return false;
    if (best_plan == ~0ull || lat < best_lat) return true;
    if (lat != best_lat || plan == best_plan) return false;
    unsigned char A[kMaxShapes], B[kMaxShapes];
    unrank_plan(sp, plan, A);
    unrank_plan(sp, best_plan, B);
    return parts_less(A, B, sp.S);
}

}  // namespace cg
