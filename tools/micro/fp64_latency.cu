// Dependent-chain latency of fp64 / fp32 / int ops on the running GPU (one warp).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false fp64_latency.cu -o fp64_latency
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain_dadd(double* out, double a, long long* cyc) {
    double x = a;
    const long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < 4096; ++i) x = __dadd_rn(x, a);
    const long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void chain_dmul(double* out, double a, long long* cyc) {
    double x = a;
    const long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < 4096; ++i) x = __dmul_rn(x, a);
    const long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void chain_dsetp(double* out, double a, long long* cyc) {
    double x = a, y = a * 0.5;
    const long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < 4096; ++i) x = (x <= y) ? y : x + 0.0;  // compare + select feeding the next compare
    const long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void chain_fadd(float* out, float a, long long* cyc) {
    float x = a;
    const long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < 4096; ++i) x = __fadd_rn(x, a);
    const long long t1 = clock64();
    out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void tput_dadd(double* out, double a, long long* cyc) {
    double x0 = a, x1 = a, x2 = a, x3 = a, x4 = a, x5 = a, x6 = a, x7 = a;
    const long long t0 = clock64();
#pragma unroll 4
    for (int i = 0; i < 4096; ++i) {
        x0 = __dadd_rn(x0, a); x1 = __dadd_rn(x1, a); x2 = __dadd_rn(x2, a); x3 = __dadd_rn(x3, a);
        x4 = __dadd_rn(x4, a); x5 = __dadd_rn(x5, a); x6 = __dadd_rn(x6, a); x7 = __dadd_rn(x7, a);
    }
    const long long t1 = clock64();
    out[threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7; if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    double* d; float* f; long long* c; long long h;
    cudaMalloc(&d, 1024 * 8); cudaMalloc(&f, 1024 * 4); cudaMalloc(&c, 8);
    for (int rep = 0; rep < 2; ++rep) {
        chain_dadd<<<1, 32>>>(d, 1.0000001, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("DADD dependent chain: %.1f cycles/op\n", h / 4096.0);
        chain_dmul<<<1, 32>>>(d, 1.0000001, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("DMUL dependent chain: %.1f cycles/op\n", h / 4096.0);
        chain_dsetp<<<1, 32>>>(d, 1.0000001, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("DSETP+DADD+select chain: %.1f cycles/iter\n", h / 4096.0);
        chain_fadd<<<1, 32>>>(f, 1.0001f, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("FADD dependent chain: %.1f cycles/op\n", h / 4096.0);
        tput_dadd<<<1, 32>>>(d, 1.0000001, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("DADD 8 independent chains, one warp: %.2f cycles/op\n", h / (4096.0 * 8));
    }
    return 0;
}
