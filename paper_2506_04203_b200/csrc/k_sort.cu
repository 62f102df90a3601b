// Stable LSD radix sort of u64 keys (optionally with u64 payloads), 8-bit
// digits, with digits that are constant over the input skipped.
//
// Used by the routing pass for nearest-rank p95 selection (token columns sorted
// once per sweep), by the default threshold grid (score quantiles,
// outerplan.cpp:114-132) and by the Pareto filter ordering (outerplan.cpp:93-112).
//
// Per pass: (1) per-tile digit histograms (warp-private, match_any-aggregated,
// no shared-memory atomics), (2) exclusive scan in digit-major order (three coalesced kernels),
// (3) stable scatter: per-warp ranks from __match_any_sync + warp prefix
// counters, tiles of 4096 keys held in registers between the two walks.
#include <cuda_runtime.h>

#include "cg_cuda.h"
#include "cg_kernels.h"

namespace cg {

namespace {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;

__global__ void k_or_and(const unsigned long long* __restrict__ keys, long long n,
                         unsigned long long* __restrict__ out /* [2]: or, and */) {
    unsigned long long o = 0, a = ~0ull;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        unsigned long long k = keys[i];
        o |= k;
        a &= k;
    }
    for (int off = 16; off > 0; off >>= 1) {
        o |= __shfl_xor_sync(0xffffffffu, o, off);
        a &= __shfl_xor_sync(0xffffffffu, a, off);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicOr(&out[0], o);
        atomicAnd(&out[1], a);
    }
}

__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const unsigned long long* __restrict__ keys,
                                                        long long n, int shift,
                                                        unsigned int* __restrict__ hist, int nblocks) {
    __shared__ unsigned int sh[RS_WARPS][256];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < RS_WARPS * 256; i += RS_THREADS) (&sh[0][0])[i] = 0;
    __syncthreads();
    const long long base = (long long)blockIdx.x * RS_TILE + (long long)w * (32 * RS_ITEMS);
#pragma unroll 4
    for (int it = 0; it < RS_ITEMS; ++it) {
        long long idx = base + it * 32 + lane;
        bool valid = idx < n;
        unsigned act = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            unsigned d = (unsigned)((keys[idx] >> shift) & 255ull);
            unsigned peers = __match_any_sync(act, d);
            if (lane == __ffs(peers) - 1) sh[w][d] += __popc(peers);
        }
        __syncwarp();
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += RS_THREADS) {
        unsigned t = 0;
#pragma unroll
        for (int ww = 0; ww < RS_WARPS; ++ww) t += sh[ww][d];
        hist[(long long)d * nblocks + blockIdx.x] = t;
    }
}

// Exclusive scan in place over the digit-major histogram, three coalesced
// steps: per-CTA chunk sums, one CTA scans those, each CTA rescans its chunk
// with its offset (a single-CTA scan walked strided columns: 0.57 ms at 10M
// keys per pass).
constexpr int SC_THREADS = 256;
constexpr int SC_ITEMS = 16;
constexpr int SC_CHUNK = SC_THREADS * SC_ITEMS;

__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned* total) {
    __shared__ unsigned wsum[SC_THREADS / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        unsigned t = lane < SC_THREADS / 32 ? wsum[lane] : 0u;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, t, off);
            if (lane >= off) t += y;
        }
        if (lane < SC_THREADS / 32) wsum[lane] = t;
    }
    __syncthreads();
    const unsigned before = (w > 0 ? wsum[w - 1] : 0u) + x - v;
    if (total) *total = wsum[SC_THREADS / 32 - 1];
    __syncthreads();
    return before;
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_sums(const unsigned int* __restrict__ a, long long len,
                                                         unsigned int* __restrict__ sums) {
    const long long base = (long long)blockIdx.x * SC_CHUNK;
    unsigned v = 0;
#pragma unroll
    for (int i = 0; i < SC_ITEMS; ++i) {
        const long long k = base + (long long)i * SC_THREADS + threadIdx.x;
        v += k < len ? a[k] : 0u;
    }
    unsigned tot = 0;
    block_excl_scan(v, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_top(unsigned int* __restrict__ sums, int nchunks) {
    unsigned run = 0;
    for (int b0 = 0; b0 < nchunks; b0 += SC_THREADS) {
        const int k = b0 + threadIdx.x;
        const unsigned v = k < nchunks ? sums[k] : 0u;
        unsigned tot = 0;
        const unsigned e = block_excl_scan(v, &tot);
        if (k < nchunks) sums[k] = run + e;
        run += tot;
    }
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_down(unsigned int* __restrict__ a, long long len,
                                                         const unsigned int* __restrict__ sums) {
    const long long base = (long long)blockIdx.x * SC_CHUNK + (long long)threadIdx.x * SC_ITEMS;
    unsigned v[SC_ITEMS];
    unsigned t = 0;
#pragma unroll
    for (int i = 0; i < SC_ITEMS; ++i) {
        const long long k = base + i;
        v[i] = k < len ? a[k] : 0u;
        t += v[i];
    }
    unsigned run = sums[blockIdx.x] + block_excl_scan(t, nullptr);
#pragma unroll
    for (int i = 0; i < SC_ITEMS; ++i) {
        const long long k = base + i;
        if (k < len) a[k] = run;
        run += v[i];
    }
}

void scan_excl(unsigned int* a, long long len, cudaStream_t s, int* launches) {
    const int nchunks = (int)((len + SC_CHUNK - 1) / SC_CHUNK);
    unsigned int* sums = a + len;  // radix_hist_entries leaves room after the histogram
    k_scan_sums<<<nchunks, SC_THREADS, 0, s>>>(a, len, sums);
    CG_LAUNCH_CHECK();
    k_scan_top<<<1, SC_THREADS, 0, s>>>(sums, nchunks);
    CG_LAUNCH_CHECK();
    k_scan_down<<<nchunks, SC_THREADS, 0, s>>>(a, len, sums);
    CG_LAUNCH_CHECK();
    if (launches) *launches += 3;
}

template <bool HAS_VALS>
__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(
    const unsigned long long* __restrict__ kin, const unsigned long long* __restrict__ vin,
    unsigned long long* __restrict__ kout, unsigned long long* __restrict__ vout, long long n,
    int shift, const unsigned int* __restrict__ offs, int nblocks) {
    __shared__ unsigned int wcnt[RS_WARPS][256];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
    for (int i = threadIdx.x; i < RS_WARPS * 256; i += RS_THREADS) (&wcnt[0][0])[i] = 0;
    __syncthreads();
    const long long base = (long long)blockIdx.x * RS_TILE + (long long)w * (32 * RS_ITEMS);
    unsigned long long k[RS_ITEMS], v[RS_ITEMS];
#pragma unroll
    for (int it = 0; it < RS_ITEMS; ++it) {
        long long idx = base + it * 32 + lane;
        if (idx < n) {
            k[it] = kin[idx];
            if (HAS_VALS) v[it] = vin[idx];
        } else {
            k[it] = 0;
            v[it] = 0;
        }
    }
    // walk 1: warp digit counts
#pragma unroll
    for (int it = 0; it < RS_ITEMS; ++it) {
        long long idx = base + it * 32 + lane;
        bool valid = idx < n;
        unsigned act = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            unsigned d = (unsigned)((k[it] >> shift) & 255ull);
            unsigned peers = __match_any_sync(act, d);
            if (lane == __ffs(peers) - 1) wcnt[w][d] += __popc(peers);
        }
        __syncwarp();
    }
    __syncthreads();
    // warp bases: global offset of (digit, block) + counts of earlier warps
    for (int d = threadIdx.x; d < 256; d += RS_THREADS) {
        unsigned run = offs[(long long)d * nblocks + blockIdx.x];
#pragma unroll
        for (int ww = 0; ww < RS_WARPS; ++ww) {
            unsigned c = wcnt[ww][d];
            wcnt[ww][d] = run;
            run += c;
        }
    }
    __syncthreads();
    // walk 2: stable scatter
#pragma unroll
    for (int it = 0; it < RS_ITEMS; ++it) {
        long long idx = base + it * 32 + lane;
        bool valid = idx < n;
        unsigned act = __ballot_sync(0xffffffffu, valid);
        unsigned d = 0, peers = 0, pos = 0;
        if (valid) {
            d = (unsigned)((k[it] >> shift) & 255ull);
            peers = __match_any_sync(act, d);
            pos = wcnt[w][d] + __popc(peers & lt_mask);
            kout[pos] = k[it];
            if (HAS_VALS) vout[pos] = v[it];
        }
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) wcnt[w][d] += __popc(peers);
        __syncwarp();
    }
}

}  // namespace

void launch_or_and(const unsigned long long* keys, long long n, unsigned long long* out2,
                   cudaStream_t s, int* launches) {
    unsigned long long init[2] = {0ull, ~0ull};
    CG_CUDA(cudaMemcpyAsync(out2, init, sizeof(init), cudaMemcpyHostToDevice, s));
    if (n <= 0) return;
    long long blocks = (n + 255) / 256;
    if (blocks > 1184) blocks = 1184;
    k_or_and<<<(unsigned)blocks, 256, 0, s>>>(keys, n, out2);
    CG_LAUNCH_CHECK();
    if (launches) ++*launches;
}

int radix_sort_u64(unsigned long long* keys, unsigned long long* vals, unsigned long long* keys_tmp,
                   unsigned long long* vals_tmp, long long n, unsigned long long varying_bits,
                   unsigned int* hist_scratch, cudaStream_t s, int* launches) {
    if (n <= 1) return 0;
    const int nblocks = (int)((n + RS_TILE - 1) / RS_TILE);
    unsigned long long *ki = keys, *vi = vals, *ko = keys_tmp, *vo = vals_tmp;
    int parity = 0;
    for (int byte = 0; byte < 8; ++byte) {
        if (((varying_bits >> (8 * byte)) & 255ull) == 0) continue;  // constant digit
        const int shift = 8 * byte;
        k_rs_hist<<<nblocks, RS_THREADS, 0, s>>>(ki, n, shift, hist_scratch, nblocks);
        CG_LAUNCH_CHECK();
        scan_excl(hist_scratch, 256LL * nblocks, s, launches);
        if (vals)
            k_rs_scatter<true><<<nblocks, RS_THREADS, 0, s>>>(ki, vi, ko, vo, n, shift, hist_scratch,
                                                             nblocks);
        else
            k_rs_scatter<false><<<nblocks, RS_THREADS, 0, s>>>(ki, vi, ko, vo, n, shift,
                                                              hist_scratch, nblocks);
        CG_LAUNCH_CHECK();
        if (launches) *launches += 3;
        std::swap(ki, ko);
        std::swap(vi, vo);
        parity ^= 1;
    }
    return parity;
}

size_t radix_hist_entries(long long n) {
    const size_t len = 256ull * (size_t)((n + RS_TILE - 1) / RS_TILE);
    return len + (len + SC_CHUNK - 1) / SC_CHUNK + 256;  // histogram, then the scan's chunk sums
}

}  // namespace cg
