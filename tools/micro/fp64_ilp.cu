// FP64 pipe micro-benchmark (B200 design data for the CI-test kernels): achieved DMUL/DADD
// throughput vs resident warps per SM and independent chains per thread (ILP), -fmad=false style
// (separate mul and add, the reference's rounding).  Prints GFLOP-instr/s and % of the DFMA probe.
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void chains(double* out, int iters, double seed) {
    double a[K], m[K];
#pragma unroll
    for (int k = 0; k < K; ++k) { a[k] = seed + threadIdx.x + k; m[k] = 0.999999 + 1e-9 * k; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int k = 0; k < K; ++k) a[k] = __dadd_rn(__dmul_rn(a[k], m[k]), 1e-7);
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) s += a[k];
    if (s == 12345.678) out[0] = s;
}

template <int K>
void run(int warps_per_sm, int sms, double* out) {
    const int threads = 128;
    const int blocks = sms * (warps_per_sm / 4);
    const int iters = 2048 / K * 4;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    chains<K><<<blocks, threads>>>(out, 16, 1.0);
    cudaEventRecord(e0);
    chains<K><<<blocks, threads>>>(out, iters, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    const double inst = 2.0 * 8 * K * (double)iters * blocks * threads;  // DMUL + DADD per chain step
    printf("warps/SM %2d  ILP %2d : %7.1f G fp64-inst/s  (%.1f%% of 64 lanes/clk/SM at 1.965 GHz)\n", warps_per_sm, K,
           inst / (ms * 1e-3) / 1e9, 100.0 * inst / (ms * 1e-3) / (64.0 * sms * 1.965e9));
}

int main() {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, 8);
    const int W[] = {4, 8, 12, 16, 24, 32};
    for (int w : W) { run<1>(w, sms, out); run<2>(w, sms, out); run<4>(w, sms, out); run<8>(w, sms, out); }
    return 0;
}
