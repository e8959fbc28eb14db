// datagen_dev.cu -- sample_linear_gaussian (datagen.hpp:62-82) with the structural equations on the
// device (the generator is O(m p deg) and runs at C5 scale before the path).
//
// The noise is the reference stream (xoshiro256++ / polar, rng.hpp), generated on the host threads in
// jump-ahead chunks (datagen.cpp noise_stream: the polar method's log stays the host libm's, so every
// normal equals the reference generator's bit for bit).  The equations then run here:
//   sem_kernel           x_i = n_i + sum_j w_ij x_j, one thread per sample, parents ascending
//                        (datagen.hpp:75-78), two roundings per term (-fmad=false)
//   sem_rescaled_kernel  the overflow-safe variant of pcs_sample_linear_gaussian_rescaled (datagen.cpp):
//                        unit-RMS columns, scales as mant * 2^exp, the sum of squares over 16 fixed
//                        sample chunks added in chunk order -- cooperative grid, three grid-wide
//                        barriers per variable (its scale feeds every later variable)
// Both are bit-identical to the host generators (tests/test_gpu_datagen.py).
#include <cooperative_groups.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "pcs_internal.h"
#include "pcstable_b200.h"

namespace cg = cooperative_groups;

namespace pcs {

constexpr int kSemThreads = 128;
constexpr int kSemUnroll = 8;

__global__ void __launch_bounds__(kSemThreads) sem_kernel(const int64_t* __restrict__ start, const int32_t* __restrict__ par,
                                                          const double* __restrict__ pw, int p, int m,
                                                          double* __restrict__ x) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    for (int i = 0; i < p; ++i) {
        double v = x[(size_t)i * m + r];  // the noise draw of (sample r, variable i)
        const int64_t b = __ldg(start + i), e = __ldg(start + i + 1);
        int64_t k = b;
        for (; k + kSemUnroll <= e; k += kSemUnroll) {  // loads first, then the ordered sum
            double xv[kSemUnroll], wv[kSemUnroll];
#pragma unroll
            for (int u = 0; u < kSemUnroll; ++u) {
                xv[u] = x[(size_t)__ldg(par + k + u) * m + r];
                wv[u] = __ldg(pw + k + u);
            }
#pragma unroll
            for (int u = 0; u < kSemUnroll; ++u) v = v + wv[u] * xv[u];
        }
        for (; k < e; ++k) v = v + __ldg(pw + k) * x[(size_t)__ldg(par + k) * m + r];
        x[(size_t)i * m + r] = v;
    }
}

constexpr int kRsChunks = 16;  // datagen.cpp's fixed sum-of-squares chunks

__global__ void __launch_bounds__(kSemThreads) sem_rescaled_kernel(const int64_t* __restrict__ start,
                                                                   const int32_t* __restrict__ par,
                                                                   const double* __restrict__ pw, int p, int m,
                                                                   double* __restrict__ x, double* smant,
                                                                   long long* sexp, double* part, double* inv_out,
                                                                   int* err) {
    cg::grid_group grid = cg::this_grid();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int gsize = gridDim.x * blockDim.x;
    for (int i = 0; i < p; ++i) {
        const int64_t b = start[i], e = start[i + 1];
        // F = the largest contributing scale (noise: 1 = 0.5 * 2^1), the same on every thread
        double Fm = 0.5;
        long long Fe = 1;
        for (int64_t k = b; k < e; ++k) {
            const int j = par[k];
            const long long ej = sexp[j];
            const double mj = smant[j];
            if (ej > Fe || (ej == Fe && mj > Fm)) { Fm = mj; Fe = ej; }
        }
        if (r < m) {
            const double nz = 1 - Fe < -2200 ? 0.0 : ldexp(0.5 / Fm, (int)(1 - Fe));
            double v = x[(size_t)i * m + r] * nz;
            for (int64_t k = b; k < e; ++k) {
                const int j = par[k];
                const long long d = sexp[j] - Fe;
                const double c = pw[k] * (d < -2200 ? 0.0 : ldexp(smant[j] / Fm, (int)d));
                v = v + c * x[(size_t)j * m + r];
            }
            x[(size_t)i * m + r] = v;
        }
        grid.sync();
        for (int c = r; c < kRsChunks; c += gsize) {  // chunk sums in sample order
            const int r0 = (int)((long long)m * c / kRsChunks), r1 = (int)((long long)m * (c + 1) / kRsChunks);
            double ss = 0.0;
            for (int q = r0; q < r1; ++q) {
                const double v = x[(size_t)i * m + q];
                ss += v * v;
            }
            part[c] = ss;
        }
        grid.sync();
        if (r == 0) {
            double ss = 0.0;
            for (int c = 0; c < kRsChunks; ++c) ss += part[c];
            const double rms = sqrt(ss / m);
            if (!(rms > 0.0) || !isfinite(rms)) *err = 1;
            *inv_out = 1.0 / rms;
            int ex = 0;
            smant[i] = frexp(Fm * rms, &ex);
            sexp[i] = Fe + ex;
        }
        grid.sync();
        if (r < m) x[(size_t)i * m + r] *= *inv_out;
    }
}

}  // namespace pcs

extern "C" {

pcs_status pcs_sample_linear_gaussian_device(const double* weights, int32_t n, int32_t m, uint64_t seed,
                                             int32_t rescaled, double* d_x, double* log_scale, uint64_t stream) {
    using namespace pcs;
    if (m < 4 || n < 2 || !weights || !d_x) return PCS_EINVAL;
    std::vector<int64_t> start((size_t)n + 1);
    std::vector<int32_t> par;
    std::vector<double> pw;
    for (int i = 0; i < n; ++i) {
        start[i] = (int64_t)par.size();
        for (int j = 0; j < n; ++j) {
            const double w = weights[(size_t)i * n + j];
            if (w == 0.0) continue;
            if (j >= i) return PCS_EINVAL;  // strictly lower triangular (datagen.hpp:66-69)
            par.push_back(j);
            pw.push_back(w);
        }
    }
    start[n] = (int64_t)par.size();
    const size_t nm = (size_t)n * m;
    double* noise = nullptr;
    if (cudaMallocHost(reinterpret_cast<void**>(&noise), sizeof(double) * nm) != cudaSuccess) return PCS_ENOMEM;
    pcs_status st = pcs_noise_stream(seed, (int64_t)nm, n, m, noise);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int64_t* dStart = nullptr;
    int32_t* dPar = nullptr;
    double *dPw = nullptr, *dMant = nullptr, *dPart = nullptr, *dInv = nullptr;
    long long* dExp = nullptr;
    int* dErr = nullptr;
    auto ok = [](cudaError_t e) { return e == cudaSuccess; };
    if (!st && !(ok(cudaMalloc(&dStart, sizeof(int64_t) * start.size())) &&
                 ok(cudaMalloc(&dPar, sizeof(int32_t) * std::max<size_t>(par.size(), 1))) &&
                 ok(cudaMalloc(&dPw, sizeof(double) * std::max<size_t>(pw.size(), 1))) &&
                 ok(cudaMalloc(&dMant, sizeof(double) * n)) && ok(cudaMalloc(&dExp, sizeof(long long) * n)) &&
                 ok(cudaMalloc(&dPart, sizeof(double) * kRsChunks)) && ok(cudaMalloc(&dInv, sizeof(double))) &&
                 ok(cudaMalloc(&dErr, sizeof(int)))))
        st = PCS_ENOMEM;
    int err = 0;
    std::vector<double> hm;
    std::vector<long long> he;
    if (!st) {
        cudaMemcpyAsync(dStart, start.data(), sizeof(int64_t) * start.size(), cudaMemcpyHostToDevice, s);
        if (!par.empty()) {
            cudaMemcpyAsync(dPar, par.data(), sizeof(int32_t) * par.size(), cudaMemcpyHostToDevice, s);
            cudaMemcpyAsync(dPw, pw.data(), sizeof(double) * pw.size(), cudaMemcpyHostToDevice, s);
        }
        cudaMemcpyAsync(d_x, noise, sizeof(double) * nm, cudaMemcpyHostToDevice, s);
        cudaMemsetAsync(dErr, 0, sizeof(int), s);
        const int blocks = (m + kSemThreads - 1) / kSemThreads;
        if (!rescaled) {
            ++g_kernel_launches;
            sem_kernel<<<blocks, kSemThreads, 0, s>>>(dStart, dPar, dPw, n, m, d_x);
        } else {
            int per_sm = 0, sms = 0, dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sem_rescaled_kernel, kSemThreads, 0);
            if ((long long)per_sm * sms < blocks) {
                st = PCS_EUNSUPPORTED;  // every sample's thread must be resident for the grid barriers
            } else {
                int nn = n, mm = m;
                double* dx = d_x;
                void* args[] = {&dStart, &dPar, &dPw, &nn, &mm, &dx, &dMant, &dExp, &dPart, &dInv, &dErr};
                ++g_kernel_launches;
                if (cudaLaunchCooperativeKernel(reinterpret_cast<void*>(sem_rescaled_kernel), blocks, kSemThreads,
                                                args, 0, s) != cudaSuccess)
                    st = PCS_ECUDA;
            }
            hm.resize(n);
            he.resize(n);
            if (!st) {
                cudaMemcpyAsync(hm.data(), dMant, sizeof(double) * n, cudaMemcpyDeviceToHost, s);
                cudaMemcpyAsync(he.data(), dExp, sizeof(long long) * n, cudaMemcpyDeviceToHost, s);
                cudaMemcpyAsync(&err, dErr, sizeof(int), cudaMemcpyDeviceToHost, s);
            }
        }
        if (cudaStreamSynchronize(s) != cudaSuccess || cudaGetLastError() != cudaSuccess) st = PCS_ECUDA;
        if (!st && err) st = PCS_EINVAL;
        if (!st && rescaled && log_scale)
            for (int i = 0; i < n; ++i) log_scale[i] = std::log(hm[i]) + (double)he[i] * 0.69314718055994530942;
    }
    cudaFree(dStart); cudaFree(dPar); cudaFree(dPw); cudaFree(dMant); cudaFree(dExp); cudaFree(dPart);
    cudaFree(dInv); cudaFree(dErr);
    cudaFreeHost(noise);
    return st;
}

}  // extern "C"
