// Which rounding sequence does DMMA (mma.sync.m8n8k4.f64) implement?  Compares the device
// result of D = A(8x4) B(4x8) + C with host restatements built from correctly rounded
// fma() / two-rounding a*b+c, over random and cancellation-heavy inputs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o dmma_semantics dmma_semantics.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

__global__ void dmma_kernel(const double* A, const double* B, const double* C, double* D, int trials) {
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    for (int tr = blockIdx.x; tr < trials; tr += gridDim.x) {
        const double* a = A + tr * 32;  // row-major 8x4
        const double* b = B + tr * 32;  // col-major 4x8: b[n*4 + k]
        const double* c = C + tr * 64;  // row-major 8x8
        double d0 = c[g * 8 + 2 * t], d1 = c[g * 8 + 2 * t + 1];
        const double fa = a[g * 4 + t], fb = b[g * 4 + t];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(d0), "+d"(d1) : "d"(fa), "d"(fb));
        D[tr * 64 + g * 8 + 2 * t] = d0;
        D[tr * 64 + g * 8 + 2 * t + 1] = d1;
    }
}

int main(int argc, char** argv) {
    const int trials = argc > 1 ? atoi(argv[1]) : 200000;
    std::mt19937_64 rng(12345);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    std::uniform_int_distribution<int> ex(-30, 30);
    double *A = new double[trials * 32], *B = new double[trials * 32], *C = new double[trials * 64], *D = new double[trials * 64];
    for (int tr = 0; tr < trials; ++tr) {
        const int mode = tr % 4;
        for (int k = 0; k < 32; ++k) {
            A[tr * 32 + k] = mode == 0 ? u(rng) : std::ldexp(u(rng), ex(rng));
            B[tr * 32 + k] = mode == 0 ? u(rng) : std::ldexp(u(rng), ex(rng));
        }
        for (int k = 0; k < 64; ++k) C[tr * 64 + k] = mode == 3 ? 0.0 : std::ldexp(u(rng), mode == 0 ? 0 : ex(rng));
        if (mode == 2)  // heavy cancellation: c = -(a0 b0 + a1 b1) roughly
            for (int i = 0; i < 8; ++i)
                for (int j = 0; j < 8; ++j) {
                    double s = 0;
                    for (int k = 0; k < 4; ++k) s += A[tr * 32 + i * 4 + k] * B[tr * 32 + j * 4 + k];
                    C[tr * 64 + i * 8 + j] = -s;
                }
    }
    double *dA, *dB, *dC, *dD;
    cudaMalloc(&dA, sizeof(double) * trials * 32);
    cudaMalloc(&dB, sizeof(double) * trials * 32);
    cudaMalloc(&dC, sizeof(double) * trials * 64);
    cudaMalloc(&dD, sizeof(double) * trials * 64);
    cudaMemcpy(dA, A, sizeof(double) * trials * 32, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B, sizeof(double) * trials * 32, cudaMemcpyHostToDevice);
    cudaMemcpy(dC, C, sizeof(double) * trials * 64, cudaMemcpyHostToDevice);
    dmma_kernel<<<1024, 32>>>(dA, dB, dC, dD, trials);
    cudaMemcpy(D, dD, sizeof(double) * trials * 64, cudaMemcpyDeviceToHost);
    if (cudaGetLastError() != cudaSuccess) { printf("cuda error\n"); return 1; }
    const char* names[] = {"fma chain k=0..3 from c", "fma chain k=3..0 from c", "two-rounding chain k=0..3",
                           "fma chain from a0b0, c added last", "pairwise fma((a0b0+a1b1)+(a2b2+a3b3))+c, long double"};
    long long match[5] = {0, 0, 0, 0, 0}, total = 0;
    for (int tr = 0; tr < trials; ++tr)
        for (int i = 0; i < 8; ++i)
            for (int j = 0; j < 8; ++j) {
                const double* a = A + tr * 32 + i * 4;
                const double* b = B + tr * 32 + j * 4;
                const double c = C[tr * 64 + i * 8 + j], d = D[tr * 64 + i * 8 + j];
                double h[5];
                h[0] = c;
                for (int k = 0; k < 4; ++k) h[0] = std::fma(a[k], b[k], h[0]);
                h[1] = c;
                for (int k = 3; k >= 0; --k) h[1] = std::fma(a[k], b[k], h[1]);
                h[2] = c;
                for (int k = 0; k < 4; ++k) h[2] = h[2] + a[k] * b[k];
                h[3] = a[0] * b[0];
                for (int k = 1; k < 4; ++k) h[3] = std::fma(a[k], b[k], h[3]);
                h[3] = h[3] + c;
                long double e = ((long double)a[0] * b[0] + (long double)a[1] * b[1]) +
                                ((long double)a[2] * b[2] + (long double)a[3] * b[3]) + (long double)c;
                h[4] = (double)e;
                for (int q = 0; q < 5; ++q) match[q] += memcmp(&h[q], &d, 8) == 0;
                ++total;
            }
    for (int q = 0; q < 5; ++q) printf("%-55s %lld / %lld\n", names[q], match[q], total);
    return 0;
}
