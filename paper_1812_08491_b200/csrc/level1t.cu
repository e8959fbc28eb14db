// level1t.cu -- level 1 (ell = 1) on dense snapshots as a TMA-tiled sweep.
//
// At ell = 1 every conditioning set is one vertex k of the tested row, M2^+ = [1] exactly, and the
// reference's partial correlation (stats.hpp:292-307) collapses to
//     h01 = c_ij - c_ik c_jk,   denom = (1 - c_ik^2)(1 - c_jk^2)
// (d01 == d10 bit for bit, so 0.5 (d01 + d10) is exact).  The serial strategy (skeleton.hpp:140-160)
// stops every directed pair (i, j) at its first separating k in row i's order; with one sweep over k
// in ascending vertex order every pair meets its k's in exactly that order, so the first hit is the
// serial one.
//
// A block owns a tile of 32 rows i x 64 target columns j (both edge directions at once: dir 0 when
// i < j, dir 1 when i > j; keys are MIN-merged) and walks k in chunks of 32:
//   * TMA (cp.async.bulk.tensor.2d) brings C(k0:k0+32, j0:j0+64) and C(i0:i0+32, k0:k0+32) into
//     shared memory, one chunk ahead of the compute (mbarrier transaction counts);
//   * a transform pass builds (c_jk, h11 = 1 - c_jk^2) per (k, j) and (c_ik, g_ik = RN(hi2' (1 - c_ik^2)))
//     per (i, k), each reused by all 32 rows / 64 targets of the tile; a factor that is exactly 0 is
//     stored as NaN;
//   * every thread owns 8 rows x 2 targets and per k evaluates, in the reference's rounding,
//     h01 = RN(c_ij - RN(c_ik c_jk)) and the certified-dependent filter  !(RN(h01^2) < RN(g_ik h11 + 1e-240))
//     (5 FP64 instructions per test); tests that the filter cannot certify are decided exactly, in k
//     order, after the chunk (decide_fast, the same code as the other kernels).
// Certification: g_ik = RN(h00 * hi2 (1 + 1e-14)) makes RN(g h11 + 1e-240) >= RN(RN(h00 h11) hi2) whenever
// h00, h11 > 0 (three roundings lose < 4 ulp << 1e-14), so the filter implies decide_fast's "A >= denom
// hi2" branch, as in surely_dependent (pcs_device.cuh).  Degenerate denominators (stats.hpp:301-305:
// !(h00 h11 > 0), "dependent") are certified too: a zero factor is NaN, so the comparison is false;
// one negative factor makes the right-hand side negative (|h| >= 2^-53 when nonzero, no underflow);
// two negative factors give the true positive product and are tested like positive ones.  On
// rank-truncated inputs (C2, the C5 generator: most |c| round to 1) zero factors are the common case.
// Compiled with -fmad=false like level.cu.
//
// Roofline: 5 FP64 instructions per test on the FP64 pipe; C is read from HBM about once per 32-row
// band (0.25 B per test) and otherwise served by L2 (blocks of the same target band run together).
#include <cuda.h>

#include "pcs_internal.h"

namespace pcs {

namespace {

constexpr int kTI = 32;        // rows per tile
constexpr int kTJ = 64;        // target columns per tile
constexpr int kKC = 32;        // k per chunk
constexpr int kThreads = 128;  // 4 warps x (8 rows x 2 targets per lane)
constexpr int kRowsPerWarp = 8;
constexpr int kJG = 16;        // target bands per L2 group (16 x 64 columns of C: 8 KB x p)

__device__ __noinline__ int decide_slow1(double h01, double denom, Thresholds th) { return decide_fast(h01, denom, th); }

// near-threshold decision: counted per level, listed per run (as level.cu's record_near)
__device__ __noinline__ void record_near1(const LevelArgs& A, int i, int j, int d, double h01, double denom) {
    atomicAdd(&A.cnt->near, 1ull);
    if (!A.near_rec || !A.near_total) return;
    const unsigned long long k = atomicAdd(A.near_total, 1ull);
    if (k >= (unsigned long long)kNearCap) return;
    double z = 0.0, rho = 0.0;
    decide_exact(h01, denom, A.th.tau, &z, &rho);
    A.near_rec[k] = NearRec{1, i, j, d, rho, z, 0, 0};
}

struct __align__(128) L1TSmem {
    double rawJ[kKC][kTJ];     // TMA destination: C(k0 + kk, j0 + jj)
    double rawI[kTI][kKC];     // TMA destination: C(i0 + r, k0 + kk)
    double2 J2[kKC][kTJ];      // (c_jk, h11)
    double2 I2[kKC][kTI];      // (c_ik, g_ik), k-major so a warp's 8 rows are contiguous
    unsigned long long bar;    // mbarrier
    uint32_t mw[2][kTI];       // row bitmask words of the chunk being computed / prefetched
    int kbase[kTI];            // neighbours of row i below k0 (full-row rank base)
    int jbase[kTI];            // position of the first neighbour >= j0 in row i
    int any_live;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}

// issue the two tile loads of chunk kc (one thread)
__device__ __forceinline__ void issue_chunk(L1TSmem& S, const CUtensorMap* mapJ, const CUtensorMap* mapI, int kc,
                                            int i0, int j0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&S.bar, (uint32_t)(sizeof(S.rawJ) + sizeof(S.rawI)));
    tma_load_2d(&S.rawJ[0][0], mapJ, j0, kc * kKC, &S.bar);
    tma_load_2d(&S.rawI[0][0], mapI, kc * kKC, i0, &S.bar);
}

}  // namespace

__global__ void __launch_bounds__(kThreads, 3)
    level1_tile_kernel(LevelArgs A, const uint32_t* __restrict__ adj, int W, int nI, int shard, int nsh,
                       const __grid_constant__ CUtensorMap mapJ, const __grid_constant__ CUtensorMap mapI,
                       double g_scale) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    L1TSmem& S = *reinterpret_cast<L1TSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // block order: groups of kJG target bands; inside a group the kJG blocks of one row band run
    // back to back (its C(I, k) tiles are L2 hits for all but the first) and the group's target bands
    // C(k, J) stay L2-resident while the row bands stream past: C is read from HBM about
    // (p / (kJG * kTJ)) + 1 times per pass instead of once per target band
    const int nJ = (A.p + kTJ - 1) / kTJ;
    const int grp = blockIdx.x / (nI * kJG), in = blockIdx.x % (nI * kJG);
    const int gw = min(kJG, nJ - grp * kJG);  // bands in this (possibly last, narrower) group
    const int jb = grp * kJG + in % gw, ib = shard + (in / gw) * nsh;  // this shard's nI row blocks (cyclic)
    const int i0 = ib * kTI, j0 = jb * kTJ;
    const int p = A.p;
    const int nchunks = (p + kKC - 1) / kKC;

    // ---- pair setup: rows r = warp*8 + a (a < 8), targets t = lane + 32 b (b < 2)
    const int jw0 = j0 >> 5;  // first bitmask word of the target band (j0 is a multiple of 64)
    uint32_t live = 0;        // bit (a * 2 + b): pair still looking for its first separating k
#pragma unroll
    for (int a = 0; a < kRowsPerWarp; ++a) {
        const int i = i0 + warp * kRowsPerWarp + a;
        if (i >= p) continue;
        const uint32_t w0 = __ldg(adj + (size_t)i * W + jw0);
        const uint32_t w1 = jw0 + 1 < W ? __ldg(adj + (size_t)i * W + jw0 + 1) : 0u;
        if ((w0 >> lane) & 1u) live |= 1u << (a * 2 + 0);
        if ((w1 >> lane) & 1u) live |= 1u << (a * 2 + 1);
    }
    if (tid == 0) S.any_live = 0;
    __syncthreads();
    if (live) S.any_live = 1;
    __syncthreads();
    if (!S.any_live) return;

    double cij[kRowsPerWarp][2];
#pragma unroll
    for (int a = 0; a < kRowsPerWarp; ++a) {
        const int i = i0 + warp * kRowsPerWarp + a;
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const int j = j0 + lane + 32 * b;
            cij[a][b] = ((live >> (a * 2 + b)) & 1u) ? __ldg(A.C + (size_t)i * A.ldc + j) : 0.0;
        }
    }
    if (tid < kTI) {
        const int i = i0 + tid;
        int jb0 = 0;
        if (i < p) {  // lower_bound(row i, j0)
            const int o = A.off[i], w = A.off[i + 1] - o;
            int lo = 0, hi = w;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (__ldg(A.nbr + o + mid) < j0) lo = mid + 1; else hi = mid;
            }
            jb0 = lo;
        }
        S.jbase[tid] = jb0;
        S.kbase[tid] = 0;
        S.mw[0][tid] = i < p ? __ldg(adj + (size_t)i * W) : 0u;
    }
    if (tid == 0) {
        mbar_init(&S.bar, 1);
        issue_chunk(S, &mapJ, &mapI, 0, i0, j0);
    }
    __syncthreads();

    constexpr double kTiny = 1e-240;
    const unsigned long long dir_lo = 0ull, dir_hi = 1ull << kDirShift;
    unsigned long long tests = 0;
    int nan = 0;
    uint32_t parity = 0;

    for (int kc = 0; kc < nchunks; ++kc) {
        const int cur = kc & 1;
        mbar_wait(&S.bar, parity);
        parity ^= 1u;
        // transform: (c_jk, 1 - c_jk^2) and (c_ik, g_ik)
        for (int q = tid; q < kKC * kTJ; q += kThreads) {
            const int kk = q / kTJ, jj = q % kTJ;
            const double c = S.rawJ[kk][jj];
            const double h11 = 1.0 - c * c;
            S.J2[kk][jj] = make_double2(c, h11 == 0.0 ? __longlong_as_double(0x7ff8000000000000ll) : h11);
        }
        for (int q = tid; q < kTI * kKC; q += kThreads) {
            const int r = q / kKC, kk = q % kKC;
            const double c = S.rawI[r][kk];
            const double h00 = 1.0 - c * c;
            S.I2[kk][r] = make_double2(c, h00 == 0.0 ? __longlong_as_double(0x7ff8000000000000ll) : h00 * g_scale);
        }
        if (tid < kTI && kc + 1 < nchunks) {
            const int i = i0 + tid;
            S.mw[cur ^ 1][tid] = i < p ? __ldg(adj + (size_t)i * W + kc + 1) : 0u;
        }
        __syncthreads();
        if (tid == 0 && kc + 1 < nchunks) issue_chunk(S, &mapJ, &mapI, kc + 1, i0, j0);

        uint32_t mwr[kRowsPerWarp];
#pragma unroll
        for (int a = 0; a < kRowsPerWarp; ++a) mwr[a] = S.mw[cur][warp * kRowsPerWarp + a];
        uint32_t rowany = 0;
#pragma unroll
        for (int a = 0; a < kRowsPerWarp; ++a) rowany |= mwr[a];
        if (live && rowany) {
            // cand[a*2+b]: bit kk = test (i, j | k0 + kk) not certified dependent
            uint32_t cand[kRowsPerWarp * 2];
#pragma unroll
            for (int q = 0; q < kRowsPerWarp * 2; ++q) cand[q] = 0u;
#pragma unroll 1
            for (int kg = 0; kg < kKC / 8; ++kg) {
                uint32_t g[kRowsPerWarp * 2];
#pragma unroll
                for (int q = 0; q < kRowsPerWarp * 2; ++q) g[q] = 0u;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int kk = kg * 8 + u;
                    const double2 jv0 = S.J2[kk][lane], jv1 = S.J2[kk][lane + 32];
#pragma unroll
                    for (int a = 0; a < kRowsPerWarp; ++a) {
                        const double2 iv = S.I2[kk][warp * kRowsPerWarp + a];
                        const double x0 = iv.x * jv0.x, x1 = iv.x * jv1.x;
                        const double h0 = cij[a][0] - x0, h1 = cij[a][1] - x1;
                        const bool d0 = !(h0 * h0 < fma(iv.y, jv0.y, kTiny));
                        const bool d1 = !(h1 * h1 < fma(iv.y, jv1.y, kTiny));
                        if (!d0) g[a * 2 + 0] |= 1u << u;
                        if (!d1) g[a * 2 + 1] |= 1u << u;
                    }
                }
#pragma unroll
                for (int q = 0; q < kRowsPerWarp * 2; ++q) cand[q] |= g[q] << (kg * 8);
            }
            // validity (k in row i, k != j, pair live), serial order, exact decision
#pragma unroll
            for (int a = 0; a < kRowsPerWarp; ++a) {
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                    const int q = a * 2 + b;
                    if (!((live >> q) & 1u)) continue;
                    const int j = j0 + lane + 32 * b;
                    uint32_t valid = mwr[a];
                    if ((j >> 5) == kc) valid &= ~(1u << (j & 31));
                    uint32_t cw = cand[q] & valid;
                    uint32_t tested = valid;
                    while (cw) {
                        const int kk = __ffs(cw) - 1;
                        cw &= cw - 1u;
                        const int r = warp * kRowsPerWarp + a;
                        const double2 iv = S.I2[kk][r];
                        const double2 jv = S.J2[kk][lane + 32 * b];
                        const double h01 = cij[a][b] - iv.x * jv.x;
                        const double den = (1.0 - iv.x * iv.x) * (1.0 - jv.x * jv.x);
                        int d = decide_slow1(h01, den, A.th);
                        if (d & kNearBit) {
                            d &= ~kNearBit;
                            record_near1(A, i0 + r, j, d, h01, den);
                        }
                        if (d == kDependent) continue;
                        tested = valid & ((2u << kk) - 1u);
                        live &= ~(1u << q);
                        if (d == kNanError) { nan = 1; break; }
                        const int i = i0 + r;
                        const int rank = S.kbase[r] + __popc(mwr[a] & ((1u << kk) - 1u));
                        const uint32_t wj0 = __ldg(adj + (size_t)i * W + jw0);
                        const int posj = S.jbase[r] + (b == 0 ? __popc(wj0 & ((1u << lane) - 1u))
                                                              : __popc(wj0) + __popc(__ldg(adj + (size_t)i * W + jw0 + 1) &
                                                                                     ((1u << lane) - 1u)));
                        const int e = __ldg(A.eid + A.off[i] + posj);
                        atomicMin(A.keys + e, (i < j ? dir_lo : dir_hi) | (unsigned long long)rank);
                        break;
                    }
                    tests += (unsigned)__popc(tested);
                }
            }
        }
        __syncthreads();  // J2 / I2 / kbase reads done before the next transform
        if (tid < kTI) S.kbase[tid] += __popc(S.mw[cur][tid]);
        if (!__syncthreads_or(live != 0)) {
            // every pair of the tile has its first separating k: the next chunk's load is still in
            // flight into this CTA's shared memory -- let it land before the CTA exits
            if (kc + 1 < nchunks) mbar_wait(&S.bar, parity);
            break;
        }
    }
    {
        unsigned long long v = tests;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
        if (lane == 0 && v) {
            atomicAdd(&A.cnt->gpu_tests, v);
            atomicAdd(&A.cnt->gpu_exact, v);
        }
    }
    if (nan) atomicOr(&A.cnt->err_nan, 1);
}

}  // namespace pcs

namespace pcs {

size_t level1_tile_smem_bytes() { return sizeof(L1TSmem) + 128; }

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda at link time)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static const EncodeTiledFn fn = [] {  // thread-safe one-time lookup
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<EncodeTiledFn>(f);
        return static_cast<EncodeTiledFn>(nullptr);
    }();
    return fn;
}

static int make_map(CUtensorMap* m, const double* C, long long ldc, int p, int box_x, int box_y) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return 1;
    cuuint64_t dims[2] = {(cuuint64_t)ldc, (cuuint64_t)p};
    cuuint64_t strides[1] = {(cuuint64_t)ldc * sizeof(double)};
    cuuint32_t box[2] = {(cuuint32_t)box_x, (cuuint32_t)box_y};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(C), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : 2;
}

// the level-1 pairs of row blocks shard, shard + nsh, ... (32 rows each), both directions; returns
// nonzero if the tensor maps cannot be built
int launch_level1_tile(const LevelArgs& A, const uint32_t* adj, int W, int shard, int nsh, cudaStream_t s) {
    CUtensorMap mapJ, mapI;
    if (make_map(&mapJ, A.C, A.ldc, A.p, kTJ, kKC) || make_map(&mapI, A.C, A.ldc, A.p, kKC, kTI)) return 1;
    const int nIall = (A.p + kTI - 1) / kTI;
    const int nI = shard < nIall ? (nIall - shard + nsh - 1) / nsh : 0, nJ = (A.p + kTJ - 1) / kTJ;
    if (nI == 0) return 0;
    const size_t smem = level1_tile_smem_bytes();
    if (cudaFuncSetAttribute(level1_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 3;
    // g_ik = RN(h00 * g_scale), g_scale >= hi2 (1 + 1e-14) (certification margin, see the header)
    const long double gs = (long double)A.th.hi2 * (1.0L + 1e-14L);
    double g_scale = (double)gs;
    if ((long double)g_scale < gs) g_scale = nextafter(g_scale, INFINITY);
    ++g_kernel_launches;
    level1_tile_kernel<<<(unsigned)(nI * nJ), kThreads, smem, s>>>(A, adj, W, nI, shard, nsh, mapJ, mapI, g_scale);
    return cudaGetLastError() == cudaSuccess ? 0 : 4;
}

}  // namespace pcs
