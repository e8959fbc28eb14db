// corr.cu -- correlation build (stats::compute_correlation, stats.hpp:132-156) and
// CorrelationMatrix validation (core.hpp:73-95) on the device.
//
//   colmean_kernel   column means of the m x p (Eigen column-major) data + finiteness
//   center_kernel    Xc = X - mean  (the centred temporary of stats.hpp:136)
//   gram_dmma_kernel G = Xc' Xc on the FP64 tensor cores (mma.sync m8n8k4 f64 ->
//                    SASS DMMA), upper-triangular 64x64 tiles only (SYRK)
//   corr_finalize    sd = sqrt(diag G) (ZeroVarianceError), c = clamp(g/(sd_i sd_j))
//   normalize_kernel CorrelationMatrix ctor for user-supplied correlation input
#include <cuda.h>

#include <cstdlib>

#include "pcs_internal.h"

namespace pcs {

// err flag bits
constexpr int kErrNonFinite = 1;
constexpr int kErrDiag = 2;
constexpr int kErrAsym = 4;
constexpr int kErrRange = 8;

// ------------------------------------------------ CorrelationMatrix ctor
__global__ void normalize_kernel(double* C, long long ldc, int p, int* err) {
    const long long n = (long long)p * p;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(k / p), j = (int)(k % p);
        if (i == j) {
            if (fabs(C[(size_t)i * ldc + i] - 1.0) > 1e-12) atomicOr(err, kErrDiag);
            continue;
        }
        if (i > j) continue;
        const double a = C[(size_t)i * ldc + j], b = C[(size_t)j * ldc + i];
        if (!isfinite(a) || !isfinite(b) || fabs(a - b) > 1e-12) { atomicOr(err, kErrAsym); continue; }
        double v = 0.5 * (a + b);
        if (fabs(v) > 1.0 + 1e-12) { atomicOr(err, kErrRange); continue; }
        v = v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);
        C[(size_t)i * ldc + j] = v;
        C[(size_t)j * ldc + i] = v;
    }
}

__global__ void set_diag_kernel(double* C, long long ldc, int p) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < p) C[(size_t)i * ldc + i] = 1.0;
}

void launch_normalize_corr(double* C, long long ldc, int p, int* err, cudaStream_t s) {
    long long n = (long long)p * p;
    long long blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    ++g_kernel_launches;
    normalize_kernel<<<(int)blocks, 256, 0, s>>>(C, ldc, p, err);
    ++g_kernel_launches;
    set_diag_kernel<<<(p + 255) / 256, 256, 0, s>>>(C, ldc, p);
}

// exact invariants the kernels rely on (a matrix this library built has them): flag = 1 otherwise
__global__ void check_corr_kernel(const double* C, long long ldc, int p, int* flag) {
    const long long n = (long long)p * p;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(k / p), j = (int)(k % p);
        const double a = C[(size_t)i * ldc + j];
        bool bad = i == j ? a != 1.0 : !(fabs(a) <= 1.0);  // NaN fails too
        if (!bad && i < j) bad = __double_as_longlong(a) != __double_as_longlong(C[(size_t)j * ldc + i]);
        if (bad) atomicOr(flag, 1);
    }
}

void launch_check_corr(const double* C, long long ldc, int p, int* flag, cudaStream_t s) {
    long long n = (long long)p * p;
    long long blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    ++g_kernel_launches;
    check_corr_kernel<<<(int)blocks, 256, 0, s>>>(C, ldc, p, flag);
}

// ------------------------------------------------ correlation build
__global__ void colmean_kernel(const double* __restrict__ X, int m, int p, double* mean, int* err) {
    const int j = blockIdx.x;
    const double* col = X + (size_t)j * m;
    double s = 0.0;
    bool bad = false;
    for (int r = threadIdx.x; r < m; r += blockDim.x) {
        const double v = col[r];
        bad |= !isfinite(v);
        s += v;
    }
    __shared__ double red[256];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int d = blockDim.x / 2; d > 0; d >>= 1) {
        if (threadIdx.x < d) red[threadIdx.x] += red[threadIdx.x + d];
        __syncthreads();
    }
    if (threadIdx.x == 0) mean[j] = red[0] / m;
    if (bad) atomicOr(err, kErrNonFinite);
}

// Xc row-major p x ldk (ldk = m rounded up to the k-tile; the tail is zero)
__global__ void center_kernel(const double* __restrict__ X, int m, int p, const double* __restrict__ mean,
                              double* __restrict__ Xc, int ldk) {
    const long long n = (long long)p * ldk;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const int j = (int)(k / ldk), r = (int)(k % ldk);
        Xc[k] = r < m ? X[(size_t)j * m + r] - mean[j] : 0.0;
    }
}

constexpr int kGT = 64;      // output tile
constexpr int kGK = 32;      // k chunk
constexpr int kGPad = 36;    // smem row stride (doubles): 4 mod 16 -> conflict-free 8x4 fragment loads

__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// 4 warps (2 x 2), each owning a 32 x 32 sub-tile = 4 x 4 DMMA tiles of 8 x 8.
// bi0 / full: the row-band variant (multi-GPU correlation split) computes every tile of row tiles
// bi0 + blockIdx.y, both triangles; G(j, i) = G(i, j) bit for bit (the FMA chain of x_i[k] x_j[k] is
// commutative per step), so the rows of different ranks assemble into a symmetric matrix.
__global__ void __launch_bounds__(128) gram_dmma_kernel(const double* __restrict__ Xc, int p, int ldk,
                                                        double* __restrict__ G, long long ldg, int bi0, int full) {
    const int bi = bi0 + blockIdx.y, bj = blockIdx.x;
    if (!full && bi > bj) return;  // symmetric: upper tiles only
    __shared__ __align__(16) double sA[kGT * kGPad];
    __shared__ __align__(16) double sB[kGT * kGPad];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 1, wn = warp & 1;
    const int g = lane >> 2, t = lane & 3;
    const int i0 = bi * kGT, j0 = bj * kGT;
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int k0 = 0; k0 < ldk; k0 += kGK) {
        // 64 rows x 32 doubles per operand = 1024 double2; 8 per thread
#pragma unroll
        for (int v = 0; v < 8; ++v) {
            const int idx = tid + v * 128;
            const int r = idx >> 4, c = (idx & 15) * 2;
            double2 xa = make_double2(0.0, 0.0), xb = make_double2(0.0, 0.0);
            if (i0 + r < p) xa = *reinterpret_cast<const double2*>(Xc + (size_t)(i0 + r) * ldk + k0 + c);
            if (j0 + r < p) xb = *reinterpret_cast<const double2*>(Xc + (size_t)(j0 + r) * ldk + k0 + c);
            *reinterpret_cast<double2*>(sA + r * kGPad + c) = xa;
            *reinterpret_cast<double2*>(sB + r * kGPad + c) = xb;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kGK; kk += 4) {
            double fa[4], fb[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) fa[a] = sA[(wm * 32 + a * 8 + g) * kGPad + kk + t];
#pragma unroll
            for (int b = 0; b < 4; ++b) fb[b] = sB[(wn * 32 + b * 8 + g) * kGPad + kk + t];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b], fa[a], fb[b]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int r = i0 + wm * 32 + a * 8 + g;
            const int c = j0 + wn * 32 + b * 8 + 2 * t;
            if (r < p && c < p) G[(size_t)r * ldg + c] = acc[a][b][0];
            if (r < p && c + 1 < p) G[(size_t)r * ldg + c + 1] = acc[a][b][1];
        }
}

// sd, ZeroVarianceError (lowest column index wins, like the reference loop), clamp
__global__ void corr_sd_kernel(const double* G, long long ldg, int p, double* sd, int* zero_col) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p) return;
    const double ss = G[(size_t)i * ldg + i];
    if (!(ss > 0.0)) atomicMin(zero_col, i);
    sd[i] = sqrt(ss);
}

__global__ void corr_finalize_kernel(const double* __restrict__ G, long long ldg, int p, const double* __restrict__ sd,
                                     double* __restrict__ C, long long ldc) {
    const long long n = (long long)p * p;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(k / p), j = (int)(k % p);
        double v;
        if (i == j) v = 1.0;
        else {
            const int a = i < j ? i : j, b = i < j ? j : i;  // gram(i, j) with i < j (stats.hpp:150)
            v = G[(size_t)a * ldg + b] / (sd[a] * sd[b]);
            v = v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);
        }
        C[(size_t)i * ldc + j] = v;
    }
}

// ---- Gram v2: 128 x 128 tiles, 8 warps (4 x 2, 32 x 64 each), TMA-staged k-chunks of 16 in a
// 3-stage mbarrier ring.  Same accumulation order as gram_dmma_kernel (every output is the FMA chain
// over k = 0 .. ldk-1, DMMA = FMA chain, tools/micro/dmma_semantics.cu), so the bits are identical.
// TMA box = 20 k x 128 rows: the 4 extra k columns pad each smem row to 20 doubles (160 B), which
// makes the 8 x 4 fragment loads bank-conflict free (rows 4 banks apart); they are simply not used.
constexpr int kG2T = 128, kG2K = 16, kG2Box = 20, kG2Stages = 3, kG2Threads = 256;

struct __align__(128) Gram2Smem {
    double A[kG2Stages][kG2T * kG2Box];
    double B[kG2Stages][kG2T * kG2Box];
    unsigned long long full[kG2Stages];
};

__device__ __forceinline__ uint32_t g2_smem(const void* q) { return (uint32_t)__cvta_generic_to_shared(q); }

__global__ void __launch_bounds__(kG2Threads, 1)
    gram_dmma2_kernel(const __grid_constant__ CUtensorMap mapX, int p, int ldk, double* __restrict__ G, long long ldg,
                      int bi0, int full, int nb) {
    extern __shared__ __align__(128) unsigned char g2raw[];
    Gram2Smem& S = *reinterpret_cast<Gram2Smem*>(g2raw);
    int bi, bj;
    if (full) {
        bi = bi0 + blockIdx.x / nb;
        bj = blockIdx.x % nb;
    } else {  // upper-triangular tile pairs (bi <= bj), row by row
        int t = blockIdx.x, r = 0;
        while (t >= nb - r) { t -= nb - r; ++r; }
        bi = r;
        bj = r + t;
    }
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 1, wn = warp & 1;  // 4 x 2 warps: rows wm*32, cols wn*64
    const int g = lane >> 2, t = lane & 3;
    const int i0 = bi * kG2T, j0 = bj * kG2T;
    const int nk = ldk / kG2K;
    const uint32_t bytes = 2u * kG2T * kG2Box * sizeof(double);
    if (tid == 0) {
        for (int s = 0; s < kG2Stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(g2_smem(&S.full[s])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int s = 0; s < kG2Stages && s < nk; ++s) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(g2_smem(&S.full[s])), "r"(bytes)
                         : "memory");
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
                    "r"(g2_smem(S.A[s])), "l"(reinterpret_cast<unsigned long long>(&mapX)), "r"(g2_smem(&S.full[s])),
                "r"(s * kG2K), "r"(i0)
                : "memory");
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
                    "r"(g2_smem(S.B[s])), "l"(reinterpret_cast<unsigned long long>(&mapX)), "r"(g2_smem(&S.full[s])),
                "r"(s * kG2K), "r"(j0)
                : "memory");
        }
    }
    __syncthreads();
    double acc[4][8][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % kG2Stages;
        const uint32_t parity = (uint32_t)((kc / kG2Stages) & 1);
        asm volatile(
            "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n}" ::"r"(
                g2_smem(&S.full[s])),
            "r"(parity)
            : "memory");
        const double* sA = S.A[s];
        const double* sB = S.B[s];
#pragma unroll
        for (int kk = 0; kk < kG2K; kk += 4) {
            double fa[4], fb[8];
#pragma unroll
            for (int a = 0; a < 4; ++a) fa[a] = sA[(wm * 32 + a * 8 + g) * kG2Box + kk + t];
#pragma unroll
            for (int b = 0; b < 8; ++b) fb[b] = sB[(wn * 64 + b * 8 + g) * kG2Box + kk + t];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 8; ++b) dmma_8x8x4(acc[a][b], fa[a], fb[b]);
        }
        __syncthreads();  // stage s consumed by every warp
        if (tid == 0 && kc + kG2Stages < nk) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(g2_smem(&S.full[s])), "r"(bytes)
                         : "memory");
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
                    "r"(g2_smem(S.A[s])), "l"(reinterpret_cast<unsigned long long>(&mapX)), "r"(g2_smem(&S.full[s])),
                "r"((kc + kG2Stages) * kG2K), "r"(i0)
                : "memory");
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
                    "r"(g2_smem(S.B[s])), "l"(reinterpret_cast<unsigned long long>(&mapX)), "r"(g2_smem(&S.full[s])),
                "r"((kc + kG2Stages) * kG2K), "r"(j0)
                : "memory");
        }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const int r = i0 + wm * 32 + a * 8 + g;
            const int c = j0 + wn * 64 + b * 8 + 2 * t;
            if (r < p && c < p) G[(size_t)r * ldg + c] = acc[a][b][0];
            if (r < p && c + 1 < p) G[(size_t)r * ldg + c + 1] = acc[a][b][1];
        }
}

typedef CUresult (*G2EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// Xc (p x ldk, row-major) as a TMA tensor; 0 on success
static int gram2_map(CUtensorMap* m, const double* Xc, int p, int ldk) {
    static const G2EncodeFn fn = [] {  // thread-safe one-time lookup
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<G2EncodeFn>(nullptr);
        return reinterpret_cast<G2EncodeFn>(f);
    }();
    if (!fn) return 1;
    cuuint64_t dims[2] = {(cuuint64_t)ldk, (cuuint64_t)p};
    cuuint64_t strides[1] = {(cuuint64_t)ldk * sizeof(double)};
    cuuint32_t box[2] = {(cuuint32_t)kG2Box, (cuuint32_t)kG2T};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(Xc), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
               ? 0
               : 2;
}

// PCS_GRAM=1: the round-1 kernel (64 x 64 tiles, synchronous staging); default the TMA-staged v2
static bool gram_v1() {
    static const int v = [] {
        const char* e = std::getenv("PCS_GRAM");
        return e ? std::atoi(e) : 2;
    }();
    return v == 1;
}

// G tiles of rows [bi0 * 128, ...): full = 0: upper triangle of the whole matrix; 1: every tile of
// row-tile range [bi0, bi1).  Returns false when the TMA path is unavailable (caller uses v1).
static bool launch_gram2(const double* Xc, int p, int ldk, double* G, long long ldg, int bi0, int bi1, int full,
                         cudaStream_t s) {
    if (gram_v1() || ldk % kG2K) return false;
    CUtensorMap map;
    if (gram2_map(&map, Xc, p, ldk)) return false;
    const int nb = (p + kG2T - 1) / kG2T;
    const size_t smem = sizeof(Gram2Smem);
    if (cudaFuncSetAttribute(gram_dmma2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return false;
    const long long blocks = full ? (long long)(bi1 - bi0) * nb : (long long)nb * (nb + 1) / 2;
    ++g_kernel_launches;
    gram_dmma2_kernel<<<(unsigned)blocks, kG2Threads, smem, s>>>(map, p, ldk, G, ldg, bi0, full, nb);
    return true;
}

// sd_j = sqrt(G(j, j)) for every column from the same FMA chain as the Gram's diagonal (k = 0 .. ldk-1,
// from +0.0; the DMMA diagonal is that chain, tools/micro/dmma_semantics.cu), ZeroVarianceError check
__global__ void sumsq_sd_kernel(const double* __restrict__ Xc, int p, int ldk, double* sd, int* zero_col) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= p) return;
    const double* x = Xc + (size_t)j * ldk;
    double s = 0.0;
    for (int k = 0; k < ldk; ++k) s = fma(x[k], x[k], s);
    if (!(s > 0.0)) atomicMin(zero_col, j);
    sd[j] = sqrt(s);
}

// rows [r0, r1) of C from row-band Gram tiles (G holds rows (r0 / kGT) * kGT .. of the band at row 0)
__global__ void corr_finalize_rows_kernel(const double* __restrict__ G, long long ldg, int p, int g_row0, int r0, int r1,
                                          const double* __restrict__ sd, double* __restrict__ C, long long ldc) {
    const long long n = (long long)(r1 - r0) * p;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const int i = r0 + (int)(k / p), j = (int)(k % p);
        double v;
        if (i == j) v = 1.0;
        else {
            const int a = i < j ? i : j, b = i < j ? j : i;
            v = G[(size_t)(i - g_row0) * ldg + j] / (sd[a] * sd[b]);
            v = v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);
        }
        C[(size_t)i * ldc + j] = v;
    }
}

// Rows [r0, r1) of the correlation matrix (the others untouched): every rank of a multi-GPU run builds
// its row band and the bands are all-gathered (bit-identical to launch_correlation's rows).
// Scratch: Xc (p x ldk), G (band rows x ldg), sd (p), err_flags[2].
void launch_correlation_rows(const double* X, int m, int p, int r0, int r1, double* Xc, double* G, long long ldg,
                             double* mean, double* C, long long ldc, int* err_flags, cudaStream_t s) {
    const int ldk = (m + kGK - 1) / kGK * kGK;
    ++g_kernel_launches;
    colmean_kernel<<<p, 256, 0, s>>>(X, m, p, mean, err_flags);
    long long n = (long long)p * ldk;
    long long blocks = (n + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    ++g_kernel_launches;
    center_kernel<<<(int)blocks, 256, 0, s>>>(X, m, p, mean, Xc, ldk);
    if (r1 <= r0) return;
    const int nb = (p + kGT - 1) / kGT, bi0 = r0 / kGT, bi1 = (r1 + kGT - 1) / kGT;
    double* sd = mean;  // mean is dead after centring
    ++g_kernel_launches;
    sumsq_sd_kernel<<<(p + 255) / 256, 256, 0, s>>>(Xc, p, ldk, sd, err_flags + 1);
    // the row band in 128-row tiles (v2) or 64-row tiles (v1); G's row 0 is the band's first tile row
    const int b2lo = r0 / kG2T, b2hi = (r1 + kG2T - 1) / kG2T;
    int g_row0 = bi0 * kGT;
    if (launch_gram2(Xc, p, ldk, G - (size_t)b2lo * kG2T * ldg, ldg, b2lo, b2hi, 1, s)) {
        g_row0 = b2lo * kG2T;
    } else {
        ++g_kernel_launches;
        gram_dmma_kernel<<<dim3(nb, bi1 - bi0), 128, 0, s>>>(Xc, p, ldk, G - (size_t)bi0 * kGT * ldg, ldg, bi0, 1);
    }
    n = (long long)(r1 - r0) * p;
    blocks = (n + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    ++g_kernel_launches;
    corr_finalize_rows_kernel<<<(int)blocks, 256, 0, s>>>(G, ldg, p, g_row0, r0, r1, sd, C, ldc);
}

// X: m x p column-major (device).  Scratch: Xc (p x ldk), G (p x ldg), mean (p), err_flags[2] = {flags, zero_col}
void launch_correlation(const double* X, int m, int p, double* Xc, double* G, long long ldg, double* mean, double* C,
                        long long ldc, int* err_flags, cudaStream_t s) {
    const int ldk = (m + kGK - 1) / kGK * kGK;
    ++g_kernel_launches;
    colmean_kernel<<<p, 256, 0, s>>>(X, m, p, mean, err_flags);
    long long n = (long long)p * ldk;
    long long blocks = (n + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    ++g_kernel_launches;
    center_kernel<<<(int)blocks, 256, 0, s>>>(X, m, p, mean, Xc, ldk);
    if (!launch_gram2(Xc, p, ldk, G, ldg, 0, 0, 0, s)) {
        const int nb = (p + kGT - 1) / kGT;
        ++g_kernel_launches;
        gram_dmma_kernel<<<dim3(nb, nb), 128, 0, s>>>(Xc, p, ldk, G, ldg, 0, 0);
    }
    double* sd = mean;  // mean is dead after centring
    ++g_kernel_launches;
    corr_sd_kernel<<<(p + 255) / 256, 256, 0, s>>>(G, ldg, p, sd, err_flags + 1);
    n = (long long)p * p;
    blocks = (n + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    ++g_kernel_launches;
    corr_finalize_kernel<<<(int)blocks, 256, 0, s>>>(G, ldg, p, sd, C, ldc);
}

}  // namespace pcs
