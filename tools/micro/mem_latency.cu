// Dependent-load (pointer chase) latency at a given working-set size, one thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 mem_latency.cu -o mem_latency
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
__global__ void chase(const unsigned* __restrict__ next, int steps, unsigned* out, long long* cyc) {
    unsigned p = 0;
    for (int i = 0; i < 64; ++i) p = next[p];  // warm
    const long long t0 = clock64();
    for (int i = 0; i < steps; ++i) p = next[p];
    const long long t1 = clock64();
    *out = p;
    *cyc = t1 - t0;
}
int main() {
    const size_t sizes[] = {16 << 10, 128 << 10, 4 << 20, 64 << 20, 1024ull << 20};
    unsigned* out; long long* cyc; cudaMalloc(&out, 4); cudaMalloc(&cyc, 8);
    for (size_t bytes : sizes) {
        const size_t n = bytes / 4, stride = 128 / 4;  // one element per 128-byte line
        std::vector<unsigned> h(n);
        const size_t lines = n / stride;
        // random cyclic permutation over lines
        std::vector<size_t> perm(lines);
        for (size_t i = 0; i < lines; ++i) perm[i] = i;
        unsigned long long s = 88172645463325252ull;
        for (size_t i = lines - 1; i > 0; --i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; size_t j = s % (i + 1); std::swap(perm[i], perm[j]); }
        for (size_t i = 0; i < lines; ++i) h[perm[i] * stride] = (unsigned)(perm[(i + 1) % lines] * stride);
        unsigned* d; cudaMalloc(&d, bytes); cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice);
        const int steps = 4096;
        long long c = 0;
        for (int rep = 0; rep < 2; ++rep) { chase<<<1, 1>>>(d, steps, out, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); }
        printf("working set %8zu KB: %.0f cycles per dependent load\n", bytes >> 10, c / (double)steps);
        cudaFree(d);
    }
    return 0;
}
