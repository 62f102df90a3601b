// Drift windows on the GPU: the windowing and
// per-window statistics of cli::cmd_drift (proj/src/cli.cpp:216-300) and
// compute_baseline / stats_of_records (cli.cpp:101-131).
//
// cmd_drift walks the (non-decreasing) stream with windows
// [t0 + k*I, t0 + k*I + I): record r lands in the first window whose end
// exceeds its arrival.  end_k is a monotone function of k in floating point,
// so every record finds its window independently (k_dw_index, exact end_k
// checks around the estimate); windows are the runs of equal k.  Each window's
// statistics are trace-order sums over its first window_requests records,
// one thread per window (k_dw_stats) -- the same sequential additions.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "cg_cuda.h"
#include "cg_drift.h"

namespace cg {

namespace {

__device__ __forceinline__ double end_of(double t0, double interval, long long k) {
    return __dadd_rn(__dadd_rn(t0, __dmul_rn((double)k, interval)), interval);
}

// window index of every record: the smallest k with arrival < end_k
__global__ void k_dw_index(const double* __restrict__ arrival, long long n, double t0, double interval,
                           long long* __restrict__ win) {
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= n) return;
    const double x = arrival[r];
    double est = floor(__ddiv_rn(__dsub_rn(x, t0), interval));
    long long k = est > 0 ? (long long)est : 0;
    while (k > 0 && x < end_of(t0, interval, k - 1)) --k;
    while (!(x < end_of(t0, interval, k))) ++k;
    win[r] = k;
}

// window starts: records whose window differs from the previous record's
__global__ void k_dw_heads(const long long* __restrict__ win, long long n, unsigned long long* __restrict__ heads,
                           unsigned long long* __restrict__ count) {
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= n) return;
    if (r == 0 || win[r] != win[r - 1]) {
        const unsigned long long k = atomicAdd(count, 1ull);
        heads[k] = (unsigned long long)r;
    }
}

}  // namespace

__global__ void k_dw_stats(DriftArgs a) {
    const long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (w >= a.nwin) return;
    const long long first = a.first[w];
    const long long cnt = a.count[w];
    const long long k = a.win[first];
    const double start = __dadd_rn(a.t0, __dmul_rn((double)k, a.interval));
    const double rest = __dsub_rn(a.stream_end, start);
    const double span = a.interval < rest ? a.interval : rest;  // std::min(interval, end - start)
    DriftWindowOut& o = a.out[w];
    o.k = k;
    o.first = first;
    o.start = start;
    o.span = span;
    o.requests = cnt;
    o.valid = span > 0.0 ? 1 : 0;
    const long long ns = cnt < a.window_requests ? cnt : a.window_requests;
    o.sampled = ns;
    double in_sum = 0.0, out_sum = 0.0;
    long long accepted = 0;
    for (long long r = first; r < first + ns; ++r) {
        in_sum = __dadd_rn(in_sum, a.in[r]);
        out_sum = __dadd_rn(out_sum, a.out0[r]);
        if (!a.has_h1 || a.score0[r] >= a.h1) ++accepted;
    }
    const double nd = (double)ns;
    o.rate = __ddiv_rn((double)cnt, span);
    o.mean_in = __ddiv_rn(in_sum, nd);
    o.mean_out = __ddiv_rn(out_sum, nd);
    o.accept = __ddiv_rn((double)accepted, nd);
}

// stats_of_records over the whole trace (compute_baseline): block-staged
// tiles, thread 0 adds in trace order.
__global__ void __launch_bounds__(1024) k_dw_baseline(DriftArgs a, double* __restrict__ res) {
    constexpr int TILE = 1024;
    __shared__ double s_in[TILE], s_out[TILE];
    __shared__ unsigned char s_acc[TILE];
    double in_sum = 0.0, out_sum = 0.0;
    unsigned long long accepted = 0;
    for (long long b0 = 0; b0 < a.n; b0 += TILE) {
        const long long r = b0 + threadIdx.x;
        if (r < a.n) {
            s_in[threadIdx.x] = a.in[r];
            s_out[threadIdx.x] = a.out0[r];
            s_acc[threadIdx.x] = (!a.has_h1 || a.score0[r] >= a.h1) ? 1 : 0;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const int len = (int)(a.n - b0 < TILE ? a.n - b0 : TILE);
            for (int i = 0; i < len; ++i) {
                in_sum = __dadd_rn(in_sum, s_in[i]);
                out_sum = __dadd_rn(out_sum, s_out[i]);
                accepted += s_acc[i];
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double n = (double)a.n;
        res[0] = __ddiv_rn(in_sum, n);
        res[1] = __ddiv_rn(out_sum, n);
        res[2] = __ddiv_rn((double)accepted, n);
    }
}

void drift_windows(DriftBuffers& B, cudaStream_t s, DriftArgs a, std::vector<DriftWindowOut>& out, int* launches) {
    const long long n = a.n;
    a.win = B.win.as<long long>((size_t)n);
    unsigned long long* heads = B.heads.as<unsigned long long>((size_t)n + 1);
    unsigned long long* cnt = B.cnt.as<unsigned long long>(1);
    CG_CUDA(cudaMemsetAsync(cnt, 0, 8, s));
    const unsigned g = (unsigned)((n + 255) / 256);
    k_dw_index<<<g, 256, 0, s>>>(a.arrival, n, a.t0, a.interval, const_cast<long long*>(a.win));
    k_dw_heads<<<g, 256, 0, s>>>(a.win, n, heads, cnt);
    CG_LAUNCH_CHECK();
    *launches += 2;
    unsigned long long nw = 0;
    CG_CUDA(cudaMemcpyAsync(&nw, cnt, 8, cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaStreamSynchronize(s));
    std::vector<unsigned long long> h(nw);
    CG_CUDA(cudaMemcpyAsync(h.data(), heads, nw * 8, cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaStreamSynchronize(s));
    std::sort(h.begin(), h.end());
    std::vector<long long> first(nw), count(nw);
    for (size_t i = 0; i < nw; ++i) {
        first[i] = (long long)h[i];
        count[i] = (long long)((i + 1 < nw ? h[i + 1] : (unsigned long long)n) - h[i]);
    }
    long long* dfirst = B.first.as<long long>(nw + 1);
    long long* dcount = B.count.as<long long>(nw + 1);
    CG_CUDA(cudaMemcpyAsync(dfirst, first.data(), nw * 8, cudaMemcpyHostToDevice, s));
    CG_CUDA(cudaMemcpyAsync(dcount, count.data(), nw * 8, cudaMemcpyHostToDevice, s));
    a.first = dfirst;
    a.count = dcount;
    a.nwin = (long long)nw;
    a.out = B.out.as<DriftWindowOut>(nw + 1);
    k_dw_stats<<<(unsigned)((nw + 127) / 128), 128, 0, s>>>(a);
    CG_LAUNCH_CHECK();
    ++*launches;
    out.resize(nw);
    CG_CUDA(cudaMemcpyAsync(out.data(), a.out, nw * sizeof(DriftWindowOut), cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaStreamSynchronize(s));
}

void trace_baseline(DriftBuffers& B, cudaStream_t s, DriftArgs a, double res[3], int* launches) {
    double* d = B.res.as<double>(3);
    k_dw_baseline<<<1, 1024, 0, s>>>(a, d);
    CG_LAUNCH_CHECK();
    ++*launches;
    CG_CUDA(cudaMemcpyAsync(res, d, 24, cudaMemcpyDeviceToHost, s));
    CG_CUDA(cudaStreamSynchronize(s));
}

}  // namespace cg
