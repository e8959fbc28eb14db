// level.cu -- per-level kernels of the B200 PC-stable skeleton.
//
//   level0_kernel       Alg. 2 / run_level_zero (skeleton.hpp:262-288) -> live bitmask
//   snapshot_*          compact() (core.hpp:227-239) as popc + scan + warp-ballot fill
//   edge_index_kernel   undirected edge ids of the snapshot (key / sepset slots)
//   level1_kernel       ell = 1, cuPC-S arrangement (skeleton.hpp:175-222) specialised:
//                       M2^+ = [1] exactly, so only the closed form is evaluated
//   level_set_kernel<L> ell >= 2, cuPC-S: 32 conditioning sets per warp, one
//                       pseudo-inverse per lane, shared by every target of the row
//   level_edge_kernel<L> ell >= 2, cuPC-E (skeleton.hpp:135-170): warp per edge,
//                       lanes over ranks, per-test pseudo-inverse, ballot early exit
//   commit_kernel       claim_removal (skeleton.hpp:123-129): apply removals, decode
//                       sepsets, serial-equivalent counters
//
// Keys: key[e] = (dir << 62) | full-row rank of the first separating set found for
// undirected edge e (dir 0 = row a, dir 1 = row b, a < b); atomicMin keeps the
// serial strategy's choice regardless of schedule.
//
// Compiled with -fmad=false: decisions are bit-identical to oracle/pcs_oracle.c.
#include <cstddef>
#include <cstdlib>

#include "pcs_internal.h"

namespace pcs {

std::atomic<unsigned long long> g_kernel_launches{0};

#ifndef PCS_SET_DBUF
#define PCS_SET_DBUF 0      // 1: two unrolled step copies ping-ponging the prefetch registers
#endif

// The rare candidates' exact decision, out of line: inlined, its log/sqrt/div sequences would be
// copied into every step instance and crowd the hot loop out of the instruction cache.
__device__ __noinline__ int decide_slow(double h01, double denom, Thresholds th) { return decide_fast(h01, denom, th); }

// A near-threshold decision (rare): counted per level and listed per run with its statistic
__device__ __noinline__ void record_near(NearRec* rec, unsigned long long* total, unsigned long long* level_count,
                                         int level, int i, int j, int d, double h01, double denom, double tau) {
    atomicAdd(level_count, 1ull);
    if (!rec || !total) return;
    const unsigned long long k = atomicAdd(total, 1ull);
    if (k >= (unsigned long long)kNearCap) return;
    double z = 0.0, rho = 0.0;
    decide_exact(h01, denom, tau, &z, &rho);
    rec[k] = NearRec{level, i, j, d, rho, z, 0, 0};
}

// strips kNearBit off a decision and records the near-threshold test
__device__ __forceinline__ int take_near(int d, const LevelArgs& A, int i, int j, double h01, double denom) {
    if (d & kNearBit)
        record_near(A.near_rec, A.near_total, &A.cnt->near, A.ell, i, j, d & ~kNearBit, h01, denom, A.th.tau);
    return d & ~kNearBit;
}

// the cuPC-S sweeps store the raw facts inline (no call in the hot loop: a call's register saves cost
// spills there); launch_near_fixup finds the row from its CSR offset and evaluates rho / z at level end
__device__ __forceinline__ int take_near_row(int d, const LevelArgs& A, int oi, int j, double h01, double denom) {
    if (d & kNearBit) {
        d &= ~kNearBit;
        atomicAdd(&A.cnt->near, 1ull);
        const unsigned long long k = atomicAdd(A.near_total, 1ull);
        if (k < (unsigned long long)kNearCap) A.near_rec[k] = NearRec{A.ell, -1, j, d, h01, denom, oi, 1};
    }
    return d;
}

__global__ void near_fixup_kernel(LevelArgs A) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= kNearCap || (unsigned long long)k >= *A.near_total) return;
    NearRec r = A.near_rec[k];
    if (!r.raw) return;
    int lo = 0, hi = A.p - 1;  // the row with off[row] == oi < off[row + 1]
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (A.off[mid + 1] <= r.oi) lo = mid + 1; else hi = mid;
    }
    double z = 0.0, rho = 0.0;
    decide_exact(r.rho, r.z, A.th.tau, &z, &rho);
    r.i = lo;
    r.rho = rho;
    r.z = z;
    r.raw = 0;
    A.near_rec[k] = r;
}

void launch_near_fixup(const LevelArgs& A, cudaStream_t s) {
    ++g_kernel_launches;
    near_fixup_kernel<<<kNearCap / 128, 128, 0, s>>>(A);
}

#ifndef PCS_SET_NT_SMALL
#define PCS_SET_NT_SMALL 4  // targets per lane per set for L = 3 (tuning knob, results identical; 4: -5% on C2 L3 with the pinv table)
#endif
#ifndef PCS_UNRANK_BSEARCH
#define PCS_UNRANK_BSEARCH 0  // 1: phase-1 unrank by per-member binary search over the binomial table
#endif
#ifndef PCS_FMA_SIGN_FILTER
#define PCS_FMA_SIGN_FILTER 1  // the step loop's filter as sign(fma(h2, h2, -g)), one FP64 op fewer; 0: A/B
#endif
#if PCS_FMA_SIGN_FILTER
#define SURELY_DEP surely_dependent2f
#else
#define SURELY_DEP surely_dependent2
#endif
#ifndef PCS_SBASE_OPAQUE
#define PCS_SBASE_OPAQUE 1  // the step loop's shared slot base pinned in a register (no per-step
                            // rematerialisation); 0: A/B
#endif
#ifndef PCS_SMEM_PTX
#define PCS_SMEM_PTX 1      // 1: the step loop reads the set slots by 32-bit shared addresses (inline PTX)
#endif
#ifndef PCS_COUNT_CAND
#define PCS_COUNT_CAND 0    // 1: diagnostics counters of the common-path filter (PCS_TRACE prints them)
#endif
#ifndef PCS_NT2_SP
#define PCS_NT2_SP 1        // sets per step for two-targets-per-lane batches (L <= 3); 1: plain set_sweep
#endif
#ifndef PCS_SET_SP
#define PCS_SET_SP 2        // sets per step for one-target-per-lane batches (L <= 3)
#endif
#ifndef PCS_SET_NT_L2
#define PCS_SET_NT_L2 3     // targets per lane per set at L = 2 (short tests: per-step overhead dominates)
#endif
#ifndef PCS_SET_MINB_DEEP
#define PCS_SET_MINB_DEEP 2  // the same at L >= 6: 255 registers, fewer pinv spills (C3 levels 6-8 0.56 -> 0.45 ms)
#endif
#ifndef PCS_SET_MINB_L2
#define PCS_SET_MINB_L2 6   // the same at L = 2 (80 registers: 24 warps per SM; C5 p=2000 level 2 -4 to -6% vs 4)
#endif
#ifndef PCS_SET_MINB
#define PCS_SET_MINB 4      // resident blocks per SM the set kernel is register-budgeted for
#endif


namespace {

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

__device__ __forceinline__ void add_counter(unsigned long long* dst, unsigned long long v) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(dst, v);
}

// largest r in [0, n) with prefix[r] <= u (prefix non-decreasing, prefix[0] = 0)
__device__ __forceinline__ int find_row(const unsigned long long* prefix, int n, unsigned long long u) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(prefix + mid) <= u) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Same, for a warp whose units only increase: `hint` is the row of its previous unit.  The hint's
// bracket is two independent loads (one round trip) and almost always hits (a C2 level-3 row has
// ~20k units); otherwise a binary search over the rows after the hint.
__device__ __forceinline__ int find_row_from(const unsigned long long* prefix, int n, unsigned long long u, int hint) {
    const unsigned long long a = __ldg(prefix + hint), b = __ldg(prefix + hint + 1);
    if (a <= u && u < b) return hint;
    int lo = u < a ? 0 : hint + 1, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(prefix + mid) <= u) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// ---- runtime-ell unrank/rank (commit path; ell up to kMaxKeyLevel)
constexpr int kMaxKeyLevel = 64;
__device__ void unrank_rt(const BinomTable& C, int w, int ell, unsigned long long t, int* pos) {
    int start = 0;
    for (int c = 0; c < ell; ++c) {
        const int k = ell - c;
        const unsigned long long total = C(w - start, k);
        const unsigned long long need = total - t;
        int lo = start, hi = w - k;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (C(w - mid, k) >= need) lo = mid; else hi = mid - 1;
        }
        pos[c] = lo;
        t -= total - C(w - lo, k);
        start = lo + 1;
    }
}
__device__ unsigned long long rank_rt(const BinomTable& C, int w, int ell, const int* pos) {
    unsigned long long s = 0;
    for (int a = 0; a < ell; ++a) s += C(w - 1 - pos[a], ell - a);
    return C(w, ell) - 1ull - s;
}

}  // namespace

// =========================================================== level 0
// and_live: keep only pairs already live in adj (pcs_run_level on an incomplete graph; run_pc_stable
// starts from the complete graph and overwrites)
__global__ void level0_kernel(const double* __restrict__ C, long long ldc, int p, int W, uint32_t* __restrict__ adj,
                              Thresholds th, Counters* cnt, int and_live, NearRec* near_rec,
                              unsigned long long* near_total) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    unsigned long long removed = 0;
    int nan = 0;
    for (long long item = warp; item < (long long)p * W; item += nwarps) {
        const int i = (int)(item / W), w = (int)(item % W);
        const int j = w * 32 + lane;
        const bool was = and_live ? ((adj[(size_t)i * W + w] >> lane) & 1u) != 0 : true;
        bool live = false;
        if (j < p && j != i) {
            const double cv = __ldg(C + (size_t)i * ldc + j);
            int d = decide0(cv, th);
            if (d & kNearBit) {  // level 0: rho = clamp(c_ij), i.e. h01 = c_ij over denom = 1
                d &= ~kNearBit;
                if (j > i) record_near(near_rec, near_total, &cnt->near, 0, i, j, d, cv, 1.0, th.tau);
            }
            nan |= d == kNanError;
            live = d == kDependent && was;
            if (j > i && d == kIndependent && was) ++removed;
        }
        __syncwarp();
        const unsigned word = __ballot_sync(0xffffffffu, live);
        if (lane == 0) adj[(size_t)i * W + w] = word;
    }
    add_counter(&cnt->removed, removed);
    if (nan) atomicOr(&cnt->err_nan, 1);
}

void launch_level0(const double* C, long long ldc, int p, int W, uint32_t* adj, Thresholds th, Counters* cnt,
                   cudaStream_t s, bool and_live, NearRec* near_rec, unsigned long long* near_total) {
    const long long items = (long long)p * W;
    long long blocks = (items * 32 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    ++g_kernel_launches;
    level0_kernel<<<(int)blocks, 256, 0, s>>>(C, ldc, p, W, adj, th, cnt, and_live ? 1 : 0, near_rec, near_total);
}

// =========================================================== snapshot
__global__ void snapshot_degree_kernel(const uint32_t* __restrict__ adj, int p, int W, int32_t* deg,
                                       int32_t* lowcnt) {
    const int lane = threadIdx.x & 31;
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= p) return;
    int d = 0, lc = 0;
    const int wi = i >> 5;
    for (int w = lane; w < W; w += 32) {
        const uint32_t x = adj[(size_t)i * W + w];
        d += __popc(x);
        if (w < wi) lc += __popc(x);
        else if (w == wi) lc += __popc(x & ((1u << (i & 31)) - 1u));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        d += __shfl_xor_sync(0xffffffffu, d, o);
        lc += __shfl_xor_sync(0xffffffffu, lc, o);
    }
    if (lane == 0) { deg[i] = d; lowcnt[i] = lc; }
}

void launch_snapshot_degrees(const uint32_t* adj, int p, int W, int32_t* deg, int32_t* lowcnt, cudaStream_t s) {
    ++g_kernel_launches;
    snapshot_degree_kernel<<<(p * 32 + 255) / 256, 256, 0, s>>>(adj, p, W, deg, lowcnt);
}

// single-block exclusive scans of deg and (deg - lowcnt); p <= 46340
__global__ void snapshot_scan_kernel(const int32_t* __restrict__ deg, const int32_t* __restrict__ lowcnt, int p,
                                     int32_t* off, int32_t* upoff, SnapInfo* info) {
    __shared__ long long s1[1024], s2[1024];
    __shared__ int smax[1024];
    __shared__ double sc2[1024], sc3[1024];
    const int t = threadIdx.x, nt = blockDim.x;
    const int per = (p + nt - 1) / nt;
    const int beg = min(t * per, p), end = min(beg + per, p);
    long long a = 0, b = 0;
    int mx = 0;
    double c2 = 0.0, c3 = 0.0;
    for (int k = beg; k < end; ++k) {
        a += deg[k];
        b += deg[k] - lowcnt[k];
        mx = max(mx, deg[k]);
        const double w = (double)deg[k];
        c2 += 0.5 * w * (w - 1.0);
        c3 += w * (w - 1.0) * (w - 2.0) / 6.0;
    }
    s1[t] = a; s2[t] = b; smax[t] = mx;
    sc2[t] = c2; sc3[t] = c3;
    __syncthreads();
    for (int d = nt / 2; d > 0; d >>= 1) {  // totals only (a sizing estimate)
        if (t < d) { sc2[t] += sc2[t + d]; sc3[t] += sc3[t + d]; }
        __syncthreads();
    }
    __syncthreads();
    for (int d = 1; d < nt; d <<= 1) {  // Hillis-Steele inclusive scan
        long long x1 = 0, x2 = 0;
        int xm = 0;
        if (t >= d) { x1 = s1[t - d]; x2 = s2[t - d]; xm = smax[t - d]; }
        __syncthreads();
        if (t >= d) { s1[t] += x1; s2[t] += x2; smax[t] = max(smax[t], xm); }
        __syncthreads();
    }
    long long r1 = s1[t] - a, r2 = s2[t] - b;
    for (int k = beg; k < end; ++k) {
        off[k] = (int32_t)r1;
        upoff[k] = (int32_t)r2;
        r1 += deg[k];
        r2 += deg[k] - lowcnt[k];
    }
    if (t == nt - 1) {
        off[p] = (int32_t)s1[t];
        upoff[p] = (int32_t)s2[t];
        info->e_dir = s1[t];
        info->e_und = s2[t];
        info->max_width = smax[t];
        info->pad = 0;  // the whole struct is copied to the host (compute-sanitizer initcheck)
        info->sets2 = sc2[0];
        info->sets3 = sc3[0];
    }
}

void launch_snapshot_scan(const int32_t* deg, const int32_t* lowcnt, int p, int32_t* off, int32_t* upoff,
                          SnapInfo* info, cudaStream_t s) {
    ++g_kernel_launches;
    snapshot_scan_kernel<<<1, 1024, 0, s>>>(deg, lowcnt, p, off, upoff, info);
}

__global__ void snapshot_fill_kernel(const uint32_t* __restrict__ adj, int p, int W, const int32_t* __restrict__ off,
                                     int32_t* __restrict__ nbr) {
    const int lane = threadIdx.x & 31;
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= p) return;
    int base = off[i];
    for (int w0 = 0; w0 < W; w0 += 32) {
        const int w = w0 + lane;
        uint32_t x = w < W ? adj[(size_t)i * W + w] : 0u;
        const int c = __popc(x);
        int incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += y;
        }
        int at = base + incl - c;
        while (x) {
            const int bit = __ffs(x) - 1;
            nbr[at++] = w * 32 + bit;
            x &= x - 1;
        }
        base += __shfl_sync(0xffffffffu, incl, 31);
    }
}

void launch_snapshot_fill(const uint32_t* adj, int p, int W, const int32_t* off, int32_t* nbr, cudaStream_t s) {
    ++g_kernel_launches;
    snapshot_fill_kernel<<<(p * 32 + 255) / 256, 256, 0, s>>>(adj, p, W, off, nbr);
}

__global__ void edge_index_kernel(LevelArgs A, int32_t* eid, int32_t* eu_a, int32_t* eu_qa, int32_t* eu_qb,
                                  double* cnbr) {
    const int lane = threadIdx.x & 31;
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= A.p) return;
    const int oi = A.off[i], w = A.off[i + 1] - oi, lci = A.lowcnt[i];
    for (int q = lane; q < w; q += 32) {
        const int j = A.nbr[oi + q];
        if (cnbr) cnbr[oi + q] = __ldg(A.C + (size_t)i * A.ldc + j);
        if (j > i) {
            const int e = A.upoff[i] + (q - lci);
            eid[oi + q] = e;
            eu_a[e] = i;
            eu_qa[e] = q;
        } else {  // entry (i -> j), j < i: position of i among row j's upper part
            const int oj = A.off[j];
            int lo = A.lowcnt[j], hi = A.off[j + 1] - oj - 1;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (A.nbr[oj + mid] < i) lo = mid + 1; else hi = mid;
            }
            const int e = A.upoff[j] + (lo - A.lowcnt[j]);
            eid[oi + q] = e;
            eu_qb[e] = q;
        }
    }
}

void launch_edge_index(const LevelArgs& A, int32_t* eid, int32_t* eu_a, int32_t* eu_qa, int32_t* eu_qb,
                       double* cnbr, cudaStream_t s) {
    ++g_kernel_launches;
    edge_index_kernel<<<(A.p * 32 + 255) / 256, 256, 0, s>>>(A, eid, eu_a, eu_qa, eu_qb, cnbr);
}

__global__ void refresh_kdir_kernel(const int32_t* __restrict__ eid, const unsigned long long* __restrict__ keys,
                                    unsigned long long* kdir, long long n) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        kdir[k] = keys[eid[k]];
}

void launch_refresh_kdir(const LevelArgs& A, long long e_dir, cudaStream_t s) {
    if (e_dir <= 0) return;
    long long blocks = (e_dir + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    ++g_kernel_launches;
    refresh_kdir_kernel<<<(int)blocks, 256, 0, s>>>(A.eid, A.keys, A.kdir, e_dir);
}

__global__ void fill_keys_kernel(unsigned long long* keys, long long n) {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        keys[k] = (unsigned long long)kNoneKey;
}
void launch_fill_keys(unsigned long long* keys, long long n, cudaStream_t s) {
    if (n <= 0) return;
    long long blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    ++g_kernel_launches;
    fill_keys_kernel<<<(int)blocks, 256, 0, s>>>(keys, n);
}

// =========================================================== work prefix
constexpr int kL1Threads = 128;   // targets per ell=1 tile
constexpr int kSetBand = 32;      // conditioning sets per ell>=2 unit

// units[i]: work units of row i in this pass; cost[i] (optional, multi-GPU sharding): units[i] times
// the relative cost of one of its units -- an ell = 1 tile tests its targets against the row's w
// candidate sets, an ell >= 2 band tests the row's ntar targets against 32 sets (+ 32 pseudo-inverses
// and the staging, the constant term)
__global__ void row_work_kernel(LevelArgs A, int pass, int variant, int row_begin, int row_end,
                                unsigned long long* units, unsigned long long* cost) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.p) return;
    unsigned long long u = 0, c = 0;
    const int w = A.off[i + 1] - A.off[i];
    const int lc = A.lowcnt[i];
    const int ntar = pass == 2 ? w : (pass == 0 ? w - lc : lc);  // pass 2: both directions at once
    if (i >= row_begin && i < row_end && w >= A.ell + 1 && ntar > 0) {
        if (A.ell == 1) {
            u = (unsigned long long)((ntar + kL1Threads - 1) / kL1Threads);
            c = u * (unsigned long long)(w + 8);
        } else {
            // a band's sweep walks its 32 sets once per staged batch of targets (a step costs about the
            // same whatever the batch's fill), plus a fixed part (cursor, staging, 32 pseudo-inverses)
            const int stage = A.ell <= 3 ? 32 * PCS_SET_NT_SMALL : 64;
            u = (A.binom(w, A.ell) + kSetBand - 1) / kSetBand;
            c = u * (unsigned long long)(8 * ((ntar + stage - 1) / stage) + 3);
        }
    }
    units[i] = u;
    if (cost) cost[i] = c;
}

// per-edge cost of a cuPC-E pass (multi-GPU sharding): C(w - 1, ell) tests in the tested row
__global__ void edge_cost_kernel(LevelArgs A, int pass, long long E, unsigned long long* cost) {
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (long long)gridDim.x * blockDim.x) {
        const int a = A.eu_a[e];
        const int x = pass == 0 ? a : A.nbr[A.off[a] + A.eu_qa[e]];
        const int w = A.off[x + 1] - A.off[x];
        const unsigned long long b = w >= A.ell + 1 ? A.binom(w - 1, A.ell) : 0ull;
        cost[e] = (b > (1ull << 40) ? (1ull << 40) : b) + 1ull;
    }
}

// unit index at cost position b: pc = cost prefix (n+1 entries), pu = unit prefix (n+1) or null
// (unit k = entry k).  Inside an entry the units are equally expensive; monotone in b, 0 at b = 0
// and the total unit count at b = pc[n], so consecutive shards tile [0, units) exactly.
__device__ unsigned long long unit_at_cost(const unsigned long long* pu, const unsigned long long* pc, long long n,
                                           unsigned long long b) {
    if (b >= pc[n]) return pu ? pu[n] : (unsigned long long)n;
    long long lo = 0, hi = n - 1;
    while (lo < hi) {
        const long long mid = (lo + hi + 1) >> 1;
        if (pc[mid] <= b) lo = mid; else hi = mid - 1;
    }
    const unsigned long long rc = pc[lo + 1] - pc[lo], d = b - pc[lo];  // pc[lo] <= b < pc[lo + 1]
    const unsigned long long nu = pu ? pu[lo + 1] - pu[lo] : 1ull;
    unsigned long long k = (unsigned long long)((double)d / (double)rc * (double)nu + 0.5);
    if (k > nu) k = nu;
    return (pu ? pu[lo] : (unsigned long long)lo) + k;
}

__global__ void shard_bounds_kernel(const unsigned long long* pu, const unsigned long long* pc, long long n, int shard,
                                    int nsh, unsigned long long* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const unsigned long long T = pc[n];
    const unsigned long long b0 = (unsigned long long)((unsigned __int128)T * shard / nsh);
    const unsigned long long b1 = (unsigned long long)((unsigned __int128)T * (shard + 1) / nsh);
    out[0] = shard == 0 ? 0ull : unit_at_cost(pu, pc, n, b0);
    out[1] = shard == nsh - 1 ? (pu ? pu[n] : (unsigned long long)n) : unit_at_cost(pu, pc, n, b1);
}

// exclusive scan in place over n+1 entries (entry n receives the total); one block
__global__ void scan_u64_kernel(unsigned long long* a, int n) {
    __shared__ unsigned long long s[1024];
    const int t = threadIdx.x, nt = blockDim.x;
    const int per = (n + nt - 1) / nt;
    const int beg = min(t * per, n), end = min(beg + per, n);
    unsigned long long x = 0;
    for (int k = beg; k < end; ++k) x += a[k];
    s[t] = x;
    __syncthreads();
    for (int d = 1; d < nt; d <<= 1) {
        unsigned long long y = t >= d ? s[t - d] : 0ull;
        __syncthreads();
        s[t] += y;
        __syncthreads();
    }
    unsigned long long r = s[t] - x;
    for (int k = beg; k < end; ++k) {
        const unsigned long long v = a[k];
        a[k] = r;
        r += v;
    }
    if (t == nt - 1) a[n] = s[t];
}

void launch_row_work(const LevelArgs& A, int pass, int variant, int row_begin, int row_end,
                     unsigned long long* prefix, cudaStream_t s) {
    ++g_kernel_launches;
    row_work_kernel<<<(A.p + 255) / 256, 256, 0, s>>>(A, pass, variant, row_begin, row_end, prefix, nullptr);
    ++g_kernel_launches;
    scan_u64_kernel<<<1, 1024, 0, s>>>(prefix, A.p);
}

void launch_row_work_sharded(const LevelArgs& A, int pass, int variant, unsigned long long* prefix,
                             unsigned long long* cost, int shard, int nsh, unsigned long long* bounds,
                             cudaStream_t s) {
    ++g_kernel_launches;
    row_work_kernel<<<(A.p + 255) / 256, 256, 0, s>>>(A, pass, variant, 0, A.p, prefix, cost);
    g_kernel_launches += 3;
    scan_u64_kernel<<<1, 1024, 0, s>>>(prefix, A.p);
    scan_u64_kernel<<<1, 1024, 0, s>>>(cost, A.p);
    shard_bounds_kernel<<<1, 32, 0, s>>>(prefix, cost, A.p, shard, nsh, bounds);
}

void launch_edge_bounds(const LevelArgs& A, int pass, long long E, unsigned long long* cost, int shard, int nsh,
                        unsigned long long* bounds, cudaStream_t s) {
    long long blocks = (E + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    g_kernel_launches += 3;
    edge_cost_kernel<<<(int)blocks, 256, 0, s>>>(A, pass, E, cost);
    scan_u64_kernel<<<1, 1024, 0, s>>>(cost, (int)E);
    shard_bounds_kernel<<<1, 32, 0, s>>>(nullptr, cost, E, shard, nsh, bounds);
}

// =========================================================== ell = 1
// One block = one row i and a tile of up to 128 targets q (threads).  The row's
// candidate sets {row[s]} are staged in shared memory in chunks; every thread
// walks s in ascending order and stops at its first separating s, which is the
// serial strategy's first passing rank for that edge direction.
constexpr int kL1Chunk = 1024;
constexpr int kL1Unroll = 8;

// Grid-stride over tiles [tile_base, min(tile_end, prefix[p])): the tile count is read on the device,
// so the host launches without waiting for the prefix scan.
// Multi-GPU: shard `shard` of `nsh` takes every nsh-th tile (cyclic: a row's tiles and neighbouring rows
// spread over the ranks, whose early exits then balance statistically).
__global__ void __launch_bounds__(kL1Threads) level1_kernel(LevelArgs A, int pass, const unsigned long long* prefix,
                                                            unsigned long long tile_base, unsigned long long tile_end,
                                                            int shard, int nsh) {
    // per candidate set k of the chunk: the row offset k * ldc of C(k, .) and (c_ik, 1 - c_ik^2), so a
    // test costs one LDS, one LDS.128, one coalesced gather C(k, j) and its FP64 arithmetic
    __shared__ int s_koff[kL1Chunk + kL1Unroll];
    __shared__ double2 s_ch[kL1Chunk + kL1Unroll];
    const unsigned long long t_end = min(tile_end, prefix[A.p]);
    unsigned long long tests = 0;
    int nan = 0;
    for (unsigned long long tile = tile_base + shard + (unsigned long long)blockIdx.x * nsh; tile < t_end;
         tile += (unsigned long long)gridDim.x * nsh) {
    const int i = find_row(prefix, A.p, tile);
    const int t_in_row = (int)(tile - prefix[i]);
    const int oi = A.off[i], w = A.off[i + 1] - oi, lc = A.lowcnt[i];
    const int qbeg = pass == 0 ? lc : 0, qend = pass == 0 ? w : lc;
    const int q = qbeg + t_in_row * kL1Threads + threadIdx.x;
    const double* __restrict__ C = A.C;
    const long long ldc = A.ldc;
    bool active = q < qend;
    int j = 0, e = 0;
    double cij = 0.0;
    if (active) {
        j = A.nbr[oi + q];
        e = A.eid[oi + q];
        cij = __ldg(C + (size_t)i * ldc + j);
        if (pass == 1 && A.keys[e] != (unsigned long long)kNoneKey) active = false;
    }
    const unsigned long long dirbits = (unsigned long long)pass << kDirShift;
    const double hi2 = A.th.hi2;
    const double* __restrict__ Cj = C + j;
    for (int s0 = 0; s0 < w; s0 += kL1Chunk) {
        if (!__syncthreads_or(active)) break;
        const int n = min(kL1Chunk, w - s0);
        for (int t = threadIdx.x; t < n + kL1Unroll; t += kL1Threads) {
            if (t < n) {
                const int k = A.nbr[oi + s0 + t];
                const double cik = __ldg(C + (size_t)i * ldc + k);
                s_koff[t] = k * (int)ldc;  // p * ldc < 2^31 (p <= 46340)
                s_ch[t] = make_double2(cik, 1.0 - cik * cik);
            } else {  // padding read by the last unrolled group: a valid address, masked below
                s_koff[t] = 0;
                s_ch[t] = make_double2(0.0, 1.0);
            }
        }
        __syncthreads();
        if (active) {
            const int qrel = q - s0;  // the target's own position inside this chunk (not a test)
            for (int t = 0; t < n && active; t += kL1Unroll) {
                double cjk[kL1Unroll];
#pragma unroll
                for (int u = 0; u < kL1Unroll; ++u) cjk[u] = __ldg(Cj + s_koff[t + u]);
                // branch-free common path: h01 = c_ij - c_ik c_jk and denom = (1 - c_ik^2)(1 - c_jk^2)
                // in the reference's rounding (M2^+ = [1] exactly, the symmetrised h01 collapses:
                // d01 == d10), certified-dependent filter, exact decision only for the rare
                // candidates, in set order
                double h01[kL1Unroll], den[kL1Unroll];
                unsigned valid = 0, cand = 0;
#pragma unroll
                for (int u = 0; u < kL1Unroll; ++u) {
                    const double2 ch = s_ch[t + u];
                    const bool ok = (t + u < n) & (t + u != qrel);
                    const double h11 = 1.0 - cjk[u] * cjk[u];
                    h01[u] = cij - ch.x * cjk[u];
                    den[u] = ch.y * h11;
                    valid |= (unsigned)ok << u;
                    cand |= (unsigned)(ok & !surely_dependent(h01[u], den[u], hi2)) << u;
                }
                unsigned done = valid;
                if (cand) {
#pragma unroll
                    for (int u = 0; u < kL1Unroll; ++u) {
                        if (!((cand >> u) & 1u)) continue;
                        const int d = take_near(decide_slow(h01[u], den[u], A.th), A, i, j, h01[u], den[u]);
                        if (d != kDependent) {
                            active = false;
                            if (d == kNanError) nan = 1;
                            else atomicMin(A.keys + e, dirbits | (unsigned long long)(s0 + t + u));
                            done = valid & ((2u << u) - 1u);  // tests up to and including the find
                            break;
                        }
                    }
                }
                tests += (unsigned)__popc(done);
            }
        }
        __syncthreads();
    }
    __syncthreads();  // the next tile re-stages s_koff / s_ch
    }
    add_counter(&A.cnt->gpu_tests, tests);
    add_counter(&A.cnt->gpu_exact, tests);
    if (nan) atomicOr(&A.cnt->err_nan, 1);
}

// tiles [u_begin, min(u_end, prefix[p])); `bound` is a host upper bound of the tile count (grid size)
void launch_level1(const LevelArgs& A, int pass, const unsigned long long* prefix, unsigned long long u_begin,
                   unsigned long long u_end, unsigned long long bound, int shard, int nsh, cudaStream_t s) {
    unsigned long long n = (bound + nsh - 1) / nsh;
    if (u_end != ~0ull && u_end - u_begin < n) n = u_end - u_begin;
    if (n > 148ull * 16) n = 148ull * 16;
    if (n == 0) return;
    ++g_kernel_launches;
    level1_kernel<<<(unsigned)n, kL1Threads, 0, s>>>(A, pass, prefix, u_begin, u_end, shard, nsh);
}

// =========================================================== ell >= 2, cuPC-S
// Unit = (row i, band of 32 consecutive conditioning-set ranks t0 .. t0+31).
//
// Phase 1 (once per unit): lane k unranks set t0+k, gathers M2 and computes its
// pseudo-inverse and the per-set parts of the test (P0 = C(i,S) M2^+, h00;
// stats.hpp:292-300) into shared slot k.
//
// Phase 2: the row's live targets (edges whose key is still above the band's
// first rank) are compacted into shared memory and dealt out NT per lane
// (interleaved, so lanes hold neighbouring vertex ids).  The warp then walks the
// 32 sets in rank order; per set every lane evaluates its NT targets as
// independent straight-line chains (ILP NT).  Consecutive ranks share their first
// L-1 members, so the gathers C(j, S) of those members stay in registers until the
// prefix changes and only the last member is gathered per test -- one L2 load per
// test instead of L -- and that load is issued one set ahead (software prefetch).
// A target stops at its first separating set (its relative key drops to that set).
//
// A unit that finds no live target proves every later unit of the row dead
// (keys only decrease, ranks only increase) and advances the work cursor past the
// row.
// ---- per-level pseudo-inverse table (l = 2, 3): M2^+ depends only on the set, and a set recurs in
// every row that contains it (C2 level 3: 2.7e9 (row, set) pseudo-inverses over C(1000, 3) = 1.7e8
// distinct sets), so when the level's (row, set) pairs outnumber the vertex l-subsets the host builds the
// table of all of them once (pinv_table_kernel) and phase 1 loads its set's entry by colex rank
// (C(c, 3) + C(b, 2) + a for a < b < c) instead of gathering M2 and running the pseudo-inverse.
template <int L>
struct PinvStride {
    static constexpr int v = (L * L + 1) / 2 * 2;  // doubles per entry, 16-B aligned
};

__device__ __forceinline__ unsigned long long ch2(unsigned long long n) { return n * (n - 1) / 2; }
__device__ __forceinline__ unsigned long long ch3(unsigned long long n) { return n * (n - 1) * (n - 2) / 6; }

template <int L>
__device__ __forceinline__ unsigned long long colex_rank(const int (&mem)[L]) {
    if constexpr (L == 2) return ch2((unsigned long long)mem[1]) + (unsigned long long)mem[0];
    else return ch3((unsigned long long)mem[2]) + ch2((unsigned long long)mem[1]) + (unsigned long long)mem[0];
}

// largest n with f(n) <= t, starting from a floating estimate (f = C(., k), k = 2, 3)
template <int K>
__device__ __forceinline__ int colex_top(unsigned long long t) {
    double est = K == 2 ? sqrt(2.0 * (double)t) : cbrt(6.0 * (double)t);
    long long n = (long long)est + K - 1;
    auto f = [](long long x) -> unsigned long long {
        if (x < K) return 0ull;
        return K == 2 ? ch2((unsigned long long)x) : ch3((unsigned long long)x);
    };
    while (n > 0 && f(n) > t) --n;
    while (f(n + 1) <= t) ++n;
    return (int)n;
}

template <int L>
__global__ void __launch_bounds__(128) pinv_table_kernel(const double* __restrict__ C, long long ldc,
                                                         unsigned long long count, double* __restrict__ table) {
    for (unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; t < count;
         t += (unsigned long long)gridDim.x * blockDim.x) {
        int mem[L];
        unsigned long long r = t;
        if constexpr (L == 3) {
            mem[2] = colex_top<3>(r);
            r -= ch3((unsigned long long)mem[2]);
        }
        mem[1] = colex_top<2>(r);
        r -= ch2((unsigned long long)mem[1]);
        mem[0] = (int)r;
        double m2[L * L], minv[L * L];
#pragma unroll
        for (int a = 0; a < L; ++a)
#pragma unroll
            for (int b = 0; b < L; ++b) m2[a * L + b] = __ldg(C + (size_t)mem[a] * ldc + mem[b]);
        pinv<L>(m2, minv);
        double* e = table + t * (unsigned long long)PinvStride<L>::v;
#pragma unroll
        for (int q = 0; q < L * L; ++q) e[q] = minv[q];
    }
}

int pinv_table_stride(int ell) { return ell == 2 ? PinvStride<2>::v : PinvStride<3>::v; }

int launch_pinv_table(const double* C, long long ldc, int p, int ell, double* table, cudaStream_t s) {
    const unsigned long long n = (unsigned long long)p;
    const unsigned long long count = ell == 2 ? n * (n - 1) / 2 : n * (n - 1) * (n - 2) / 6;
    unsigned long long blocks = (count + 127) / 128;
    if (blocks > 148ull * 64) blocks = 148ull * 64;
    ++g_kernel_launches;
    if (ell == 2) pinv_table_kernel<2><<<(unsigned)blocks, 128, 0, s>>>(C, ldc, count, table);
    else if (ell == 3) pinv_table_kernel<3><<<(unsigned)blocks, 128, 0, s>>>(C, ldc, count, table);
    else return -1;
    return 0;
}

template <int L>
struct alignas(16) SetSlot {
    // column c of the set's test data, 16 B aligned for LDS.128:
    //   {M2^+[0][c], ..., M2^+[L-1][c], C(i,S)[c], P0[c], (pad)}
    static constexpr int CW = (L + 3) / 2 * 2;
    double col[L][CW];
    double h00, pad;
    int pos[L];
    int roff[L];  // row offsets mem[a] * ldc of the set's members
};

constexpr int kSetWarps = 4;

template <int L>
struct SetCfg {
    static constexpr int NT = L == 2 ? PCS_SET_NT_L2 : (L <= 3 ? PCS_SET_NT_SMALL : 2);  // targets per lane per set
    static constexpr int kStage = 32 * NT;     // live targets staged per pass over the band
};

template <int L>
struct SetWarpSmem {
    SetSlot<L> slot[32];
    unsigned long long tkey[SetCfg<L>::kStage];
    double tcij[SetCfg<L>::kStage];
    int tq[SetCfg<L>::kStage];
    int tj[SetCfg<L>::kStage];
    int te[SetCfg<L>::kStage];
};

// h_terms<L> (stats.hpp:292-307) for NT targets against one shared set, streamed one column
// of M2^+ at a time: P1[col] is consumed as soon as it exists, so only one column of M2^+
// (plus C(i,S)[col], P0[col]) is live.  Every accumulator (P1[col], d11, d01, d10) sees
// exactly the reference's sequence of roundings (-fmad=false), so h01 / denom are
// bit-identical to h_terms<L>.
//
// Outputs s01 = d01 + d10 and h2 = RN(2 c_ij - s01) = 2 h01 exactly (see surely_dependent2), so the
// common path skips the reference's 0.5 * (.) multiply; the rare exact path rebuilds
// h01 = c_ij - 0.5 * s01 bit for bit (c_ij = 0.5 * cij2 is exact).
template <int L, int NT, int LP>
__device__ __forceinline__ void h_terms_stream(const SetSlot<L>& sl, const double (&cp)[NT][LP],
                                               const double (&cur)[NT], const double (&cij2)[NT],
                                               double (&s01)[NT], double (&h2)[NT], double (&den)[NT]) {
    double d11[NT], d01[NT], d10[NT];
#pragma unroll
    for (int col = 0; col < L; ++col) {
        double cv[SetSlot<L>::CW];  // one column: M2^+[.][col], C(i,S)[col], P0[col]
#pragma unroll
        for (int k = 0; k < SetSlot<L>::CW; k += 2) {
            const double2 v = *reinterpret_cast<const double2*>(&sl.col[col][k]);
            cv[k] = v.x;
            cv[k + 1] = v.y;
        }
        const double* mc = cv;
        const double ci = cv[L], pc = cv[L + 1];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            double x[L];
#pragma unroll
            for (int a = 0; a < L - 1; ++a) x[a] = cp[t][a];
            x[L - 1] = cur[t];
            double pcol = x[0] * mc[0];
#pragma unroll
            for (int k = 1; k < L; ++k) pcol = pcol + x[k] * mc[k];
            if (col == 0) {
                d11[t] = pcol * x[0];
                d01[t] = pc * x[0];
                d10[t] = pcol * ci;
            } else {
                d11[t] = d11[t] + pcol * x[col];
                d01[t] = d01[t] + pc * x[col];
                d10[t] = d10[t] + pcol * ci;
            }
        }
    }
    const double h00 = sl.h00;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const double h11 = 1.0 - d11[t];
        s01[t] = d01[t] + d10[t];
        h2[t] = cij2[t] - s01[t];
        den[t] = h00 * h11;
    }
}

// Key of a find: the target's direction (q < lc: j < i, direction 1 of edge (j, i)) and the set's
// full-row rank; both directions' mirror entries of the edge are lowered with the key.
__device__ __forceinline__ void record_find(const LevelArgs& A, int oi, int q, int e, int j, bool dir1,
                                            unsigned long long key) {
    atomicMin(A.keys + e, key);
    atomicMin(A.kdir + oi + q, key);
    atomicMin(A.kdir + A.off[j] + (dir1 ? A.eu_qa[e] : A.eu_qb[e]), key);
}

// h_terms for NT targets per lane against SP sets of the same run (shared leading members cp[t],
// per-(target, set) last-member gather cur[t][k]): the same per-accumulator rounding sequence as
// h_terms_stream; each set's column data is loaded once and shared by the NT targets.
template <int L, int NT, int SP, int LP>
__device__ __forceinline__ void h_terms_tsp(const SetSlot<L>* const (&sl)[SP], const double (&cp)[NT][LP],
                                            const double (&cur)[NT][SP], const double (&cij2)[NT],
                                            double (&s01)[NT][SP], double (&h2)[NT][SP], double (&den)[NT][SP]) {
    double d11[NT][SP], d01[NT][SP], d10[NT][SP];
#pragma unroll
    for (int col = 0; col < L; ++col) {
#pragma unroll
        for (int k = 0; k < SP; ++k) {
            double cv[SetSlot<L>::CW];
#pragma unroll
            for (int c = 0; c < SetSlot<L>::CW; c += 2) {
                const double2 v = *reinterpret_cast<const double2*>(&sl[k]->col[col][c]);
                cv[c] = v.x;
                cv[c + 1] = v.y;
            }
            const double ci = cv[L], pc = cv[L + 1];
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                double x[L];
#pragma unroll
                for (int a = 0; a < L - 1; ++a) x[a] = cp[t][a];
                x[L - 1] = cur[t][k];
                double pcol = x[0] * cv[0];
#pragma unroll
                for (int q = 1; q < L; ++q) pcol = pcol + x[q] * cv[q];
                if (col == 0) {
                    d11[t][k] = pcol * x[0];
                    d01[t][k] = pc * x[0];
                    d10[t][k] = pcol * ci;
                } else {
                    d11[t][k] = d11[t][k] + pcol * x[col];
                    d01[t][k] = d01[t][k] + pc * x[col];
                    d10[t][k] = d10[t][k] + pcol * ci;
                }
            }
        }
    }
#pragma unroll
    for (int k = 0; k < SP; ++k) {
        const double h00 = sl[k]->h00;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const double h11 = 1.0 - d11[t][k];
            s01[t][k] = d01[t][k] + d10[t][k];
            h2[t][k] = cij2[t] - s01[t][k];
            den[t][k] = h00 * h11;
        }
    }
}

// Phase 2 for a partially filled batch (NT targets per lane, NT below the kernel's full NT): a step
// tests the lane's NT targets against SP consecutive live sets of the current run (NT x SP independent
// chains instead of NT, and one step's bookkeeping for SP sets).  Sets are still settled in rank
// order per target: the first separating set among a step's SP wins and later ones are discarded.
// Same results and counters as set_sweep<L, NT>.
template <int L, int NT, int SP>
__device__ __forceinline__ void set_sweep_tsp(const LevelArgs& A, SetWarpSmem<L>& S, int lane, int oi, int lc,
                                              int nlive, int nvalid, unsigned segmask, unsigned livemask,
                                              unsigned long long K0, unsigned long long& tests,
                                              unsigned long long& degen, int& nan) {
    const double* __restrict__ C = A.C;
    const double hi2x4 = A.th.hi2x4;
    int rel[NT], q[NT];
    const double* Cj[NT];
    double cij2[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const int kk = t * 32 + lane;
        rel[t] = -1;
        Cj[t] = C;
        cij2[t] = 0.0;
        q[t] = -1;
        if (kk < nlive) {
            q[t] = S.tq[kk];
            const unsigned long long kb = q[t] < lc ? (K0 | (1ull << kDirShift)) : K0;
            const unsigned long long d = S.tkey[kk] - kb;
            rel[t] = d > 0x3fffffffull ? 0x3fffffff : (int)d;
            Cj[t] = C + S.tj[kk];
            const double c = S.tcij[kk];
            cij2[t] = c + c;
        }
    }
    constexpr int LP = L > 1 ? L - 1 : 1;
    const unsigned valid_mask = nvalid >= 32 ? 0xffffffffu : ((1u << nvalid) - 1u);
    segmask &= valid_mask;
    const unsigned live = livemask & valid_mask, dead = valid_mask & ~livemask;
    auto next_live = [&](int x) -> int {
        const unsigned m = live & ~((2u << x) - 1u);
        return m ? __ffs(m) - 1 : nvalid;
    };
    auto run_end = [&](int x) -> int {
        const unsigned m = segmask & ~((2u << x) - 1u);
        return m ? __ffs(m) - 1 : nvalid;
    };
    // a group: up to SP consecutive live sets of one run (g[k] = nvalid: empty item); returns the
    // first live set after the group
    auto gather_group = [&](int first, int (&g)[SP], double (&buf)[NT][SP]) -> int {
        const int re = first < nvalid ? run_end(first) : nvalid;
        int x = first;
#pragma unroll
        for (int k = 0; k < SP; ++k) {
            const bool ok = x < re;
            g[k] = ok ? x : nvalid;
            const int ro = S.slot[ok ? x : (first < nvalid ? first : nvalid - 1)].roff[L - 1];
#pragma unroll
            for (int t = 0; t < NT; ++t) buf[t][k] = __ldg(Cj[t] + ro);
            if (ok) x = next_live(x);
        }
        return x;
    };
    double cp[NT][LP];
    int g[SP];
    double nxt[NT][SP];
    int after = gather_group(live ? __ffs(live) - 1 : nvalid, g, nxt);
    int sg = 0;
    while (sg < nvalid) {
        const int sg0 = sg;
        const int seg_end = run_end(sg0);
        const SetSlot<L>& sl0 = S.slot[sg0];
        const int base = sl0.pos[L - 1];
        if (g[0] < seg_end) {
#pragma unroll
            for (int a = 0; a < L - 1; ++a)
#pragma unroll
                for (int t = 0; t < NT; ++t) cp[t][a] = __ldg(Cj[t] + sl0.roff[a]);
        }
        int lim[NT], dm[NT];
        unsigned hit = 0;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            bool pm = false;
#pragma unroll
            for (int a = 0; a < L - 1; ++a) pm |= sl0.pos[a] == q[t];
            lim[t] = pm ? -1 : rel[t];
            dm[t] = sg0 + q[t] - base;
        }
        while (g[0] < seg_end) {
            int gn[SP];
            double alt[NT][SP];
            const int after2 = gather_group(after, gn, alt);
            const SetSlot<L>* sls[SP];
#pragma unroll
            for (int k = 0; k < SP; ++k) sls[k] = &S.slot[g[k] < nvalid ? g[k] : g[0]];
            double s01[NT][SP], h2[NT][SP], den[NT][SP];
            h_terms_tsp<L, NT, SP, LP>(sls, cp, nxt, cij2, s01, h2, den);
            unsigned cand = 0;
#pragma unroll
            for (int t = 0; t < NT; ++t)
#pragma unroll
                for (int k = 0; k < SP; ++k)
                    cand |= (unsigned)((g[k] < seg_end) & (g[k] < lim[t]) & (g[k] != dm[t]) &
                                       !SURELY_DEP(h2[t][k], den[t][k], hi2x4)) << (t * SP + k);
            if (__any_sync(0xffffffffu, cand)) {
#pragma unroll
                for (int t = 0; t < NT; ++t) {
#pragma unroll
                    for (int k = 0; k < SP; ++k) {
                        if (((cand >> (t * SP + k)) & 1u) && g[k] < lim[t]) {
                            const double h01 = 0.5 * cij2[t] - 0.5 * s01[t][k];
                            const int d = take_near_row(decide_slow(h01, den[t][k], A.th), A, oi, S.tj[t * 32 + lane], h01, den[t][k]);
                            if (d != kDependent) {
                                const int kk = t * 32 + lane;
                                const bool dir1 = q[t] < lc;
                                if (d == kNanError) nan = 1;
                                else record_find(A, oi, q[t], S.te[kk], S.tj[kk], dir1,
                                                 (dir1 ? (K0 | (1ull << kDirShift)) : K0) + (unsigned long long)g[k]);
                                rel[t] = g[k];
                                lim[t] = g[k];
                                hit |= 1u << t;
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < SP; ++k) {
                g[k] = gn[k];
#pragma unroll
                for (int t = 0; t < NT; ++t) nxt[t][k] = alt[t][k];
            }
            after = after2;
        }
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int hi = ((hit >> t) & 1u) ? lim[t] + 1 : min(seg_end, lim[t]);
            const int n = max(0, hi - sg0);
            const bool in = dm[t] >= sg0 && dm[t] < sg0 + n;
            tests += (unsigned)(n - (in ? 1 : 0));
            const unsigned rm = n >= 32 ? 0xffffffffu : (((1u << n) - 1u) << sg0);
            degen += (unsigned)(__popc(dead & rm) - ((in && ((dead >> dm[t]) & 1u)) ? 1 : 0));
        }
        sg = seg_end;
    }
}

// Shared-state-space loads by 32-bit address (PCS_SMEM_PTX): the step loop then carries one 32-bit
// slot base instead of rematerialising a generic (cluster-window) pointer every step.
__device__ __forceinline__ double2 lds_f64x2(uint32_t a) {
    double2 v;
    asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int lds_s32(uint32_t a) {
    int v;
    asm("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

template <int L, int NT, int LP>
__device__ __forceinline__ void h_terms_stream_sa(uint32_t sla, const double (&cp)[NT][LP],
                                                  const double (&cur)[NT], const double (&cij2)[NT],
                                                  double (&s01)[NT], double (&h2)[NT], double (&den)[NT]) {
    double d11[NT], d01[NT], d10[NT];
#pragma unroll
    for (int col = 0; col < L; ++col) {
        double cv[SetSlot<L>::CW];
#pragma unroll
        for (int k = 0; k < SetSlot<L>::CW; k += 2) {
            const double2 v = lds_f64x2(sla + (uint32_t)offsetof(SetSlot<L>, col) +
                                        (uint32_t)((col * SetSlot<L>::CW + k) * sizeof(double)));
            cv[k] = v.x;
            cv[k + 1] = v.y;
        }
        const double* mc = cv;
        const double ci = cv[L], pc = cv[L + 1];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            double x[L];
#pragma unroll
            for (int a = 0; a < L - 1; ++a) x[a] = cp[t][a];
            x[L - 1] = cur[t];
            double pcol = x[0] * mc[0];
#pragma unroll
            for (int k = 1; k < L; ++k) pcol = pcol + x[k] * mc[k];
            if (col == 0) {
                d11[t] = pcol * x[0];
                d01[t] = pc * x[0];
                d10[t] = pcol * ci;
            } else {
                d11[t] = d11[t] + pcol * x[col];
                d01[t] = d01[t] + pc * x[col];
                d10[t] = d10[t] + pcol * ci;
            }
        }
    }
    const double h00 = lds_f64(sla + (uint32_t)offsetof(SetSlot<L>, h00));
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const double h11 = 1.0 - d11[t];
        s01[t] = d01[t] + d10[t];
        h2[t] = cij2[t] - s01[t];
        den[t] = h00 * h11;
    }
}

// Phase 2 for one staged batch of targets, NT (<= SetCfg<L>::NT) per lane.
// segmask: bit s set when set s starts a new run of equal leading L-1 members.  Inside a
// run (lexicographic order) the last member's position advances by one per set: set
// sg0 + d has last position base + d, so "target is a member" is one compare per set.
// livemask: bit s set when set s has h00 != 0.  h00 == 0 (exactly) makes denom = h00 * h11 a
// zero or NaN for every target, so every test of such a set is the reference's degenerate
// "dependent" (stats.hpp:301-305) without any arithmetic: those sets are counted, never visited
// (rank-truncated inputs hit this often: ~29% of C2's level-3 sets), and the last-member
// prefetch always targets the next LIVE set, so skipped sets cost no L2 round trip either.
template <int L, int NT>
__device__ __forceinline__ void set_sweep(const LevelArgs& A, SetWarpSmem<L>& S, int lane, int oi, int lc, int nlive,
                                          int nvalid, unsigned segmask, unsigned livemask, unsigned long long K0,
                                          unsigned long long& tests, unsigned long long& degen, int& nan) {
    const double* __restrict__ C = A.C;
#if PCS_SMEM_PTX
    uint32_t slot0 = (uint32_t)__cvta_generic_to_shared(&S.slot[0]);
#if PCS_SBASE_OPAQUE
    asm volatile("" : "+r"(slot0));  // keep it in a register: rematerialising costs two S2R per step
#endif
#endif
    const double hi2x4 = A.th.hi2x4;  // 4 hi2, exact (power-of-two scaling), precomputed on the host
    int rel[NT];           // tested while the set index is below rel (relative key)
    const double* Cj[NT];  // C + j: gathers C(mem, j) = Cj[t][mem * ldc] (one IMAD.WIDE each)
    double cij2[NT];       // 2 c_ij (exact)
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const int k = t * 32 + lane;
        if (k < nlive) {
            const unsigned long long kb = S.tq[k] < lc ? (K0 | (1ull << kDirShift)) : K0;  // target's key base
            const unsigned long long d = S.tkey[k] - kb;  // > 0 (staged targets are live)
            rel[t] = d > 0x3fffffffull ? 0x3fffffff : (int)d;
            Cj[t] = C + S.tj[k];
            const double c = S.tcij[k];
            cij2[t] = c + c;
        } else {
            rel[t] = -1;
            Cj[t] = C;  // valid address: loads stay unconditional
            cij2[t] = 0.0;
        }
    }
    constexpr int LP = L > 1 ? L - 1 : 1;
    const unsigned valid_mask = nvalid >= 32 ? 0xffffffffu : ((1u << nvalid) - 1u);
    segmask &= valid_mask;
    const unsigned live = livemask & valid_mask, dead = valid_mask & ~livemask;
    auto next_live = [&](int s) -> int {  // first live set after s (nvalid: none)
        const unsigned m = live & ~((2u << s) - 1u);
        return m ? __ffs(m) - 1 : nvalid;
    };
    double cp[NT][LP];
    double nxt[NT], alt[NT];
    int nl = live ? __ffs(live) - 1 : nvalid;  // next live set to test
    if (nl < nvalid) {
        const int ro = S.slot[nl].roff[L - 1];
#pragma unroll
        for (int t = 0; t < NT; ++t) nxt[t] = __ldg(Cj[t] + ro);
    }
    int sg = 0;
    while (sg < nvalid) {
        const int sg0 = sg;
        const unsigned later = segmask & ~((2u << sg0) - 1u);
        const int seg_end = later ? __ffs(later) - 1 : nvalid;
        int lim[NT], dm[NT];  // lim: tested while sg < lim; dm: the set whose last member is the target
        unsigned hit = 0;     // bit t: target t found its separating set in this run (at set lim[t])
        {
            // new run of sets sharing their first L-1 members: gather those once per target
            const SetSlot<L>& sl = S.slot[sg0];
            const int base = sl.pos[L - 1];
            if (nl < seg_end) {
#pragma unroll
                for (int a = 0; a < L - 1; ++a) {
                    const int ro = sl.roff[a];
#pragma unroll
                    for (int t = 0; t < NT; ++t) cp[t][a] = __ldg(Cj[t] + ro);
                }
            }
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int k = t * 32 + lane;
                const int q = k < nlive ? S.tq[k] : -1;
                bool pm = false;
#pragma unroll
                for (int a = 0; a < L - 1; ++a) pm |= sl.pos[a] == q;
                lim[t] = pm ? -1 : rel[t];  // a shared member is never tested in this run
                dm[t] = sg0 + q - base;
            }
        }
        // double-buffered last-member gathers: step(s, n, cur, pre) tests live set s with `cur` while
        // prefetching live set n (the next one, possibly in a later run) into `pre`
        auto step = [&](int sgx, int nxs, const double (&cur)[NT], double (&pre)[NT]) {
#if PCS_SMEM_PTX
            {  // clamped: always a valid slot
                const int ro = lds_s32(slot0 + (uint32_t)(min(nxs, nvalid - 1) * (int)sizeof(SetSlot<L>)) +
                                       (uint32_t)(offsetof(SetSlot<L>, roff) + (L - 1) * sizeof(int)));
#pragma unroll
                for (int t = 0; t < NT; ++t) pre[t] = __ldg(Cj[t] + ro);
            }
            double s01[NT], h2[NT], den[NT];
            h_terms_stream_sa<L, NT, LP>(slot0 + (uint32_t)(sgx * (int)sizeof(SetSlot<L>)), cp, cur, cij2, s01, h2,
                                         den);
#else
            const SetSlot<L>& sl = S.slot[sgx];
            {  // clamped: always a valid slot
                const int ro = S.slot[min(nxs, nvalid - 1)].roff[L - 1];
#pragma unroll
                for (int t = 0; t < NT; ++t) pre[t] = __ldg(Cj[t] + ro);
            }
            double s01[NT], h2[NT], den[NT];
            h_terms_stream<L, NT, LP>(sl, cp, cur, cij2, s01, h2, den);
#endif
            // branch-free common path: flag the (rare) tests not certainly dependent
            unsigned cand = 0;
#pragma unroll
            for (int t = 0; t < NT; ++t)
                cand |= (unsigned)((sgx < lim[t]) & (sgx != dm[t]) & !SURELY_DEP(h2[t], den[t], hi2x4)) << t;
#if PCS_COUNT_CAND  // diagnostics build only: steps, candidate tests, steps whose vote fired
            {
                const unsigned nc = __reduce_add_sync(0xffffffffu, (unsigned)__popc(cand));
                if (lane == 0) {
                    atomicAdd(&A.cnt->dbg[0], 1ull);
                    atomicAdd(&A.cnt->dbg[1], (unsigned long long)nc);
                    if (nc) atomicAdd(&A.cnt->dbg[2], 1ull);
                }
            }
#endif
            if (__any_sync(0xffffffffu, cand)) {
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    if ((cand >> t) & 1u) {
                        const double h01 = 0.5 * cij2[t] - 0.5 * s01[t];  // == c_ij - 0.5 * (d01 + d10)
                        const int d = take_near_row(decide_slow(h01, den[t], A.th), A, oi, S.tj[t * 32 + lane], h01, den[t]);
                        if (d != kDependent) {
                            if (d == kNanError) nan = 1;
                            else {
                                const int k = t * 32 + lane;
                                const bool dir1 = S.tq[k] < lc;
                                record_find(A, oi, S.tq[k], S.te[k], S.tj[k], dir1,
                                            (dir1 ? (K0 | (1ull << kDirShift)) : K0) + (unsigned long long)sgx);
                            }
                            rel[t] = sgx;
                            lim[t] = sgx;
                            hit |= 1u << t;
                        }
                    }
                }
            }
        };
#if PCS_SET_DBUF
        while (nl < seg_end) {
            int s = nl;
            nl = next_live(s);
            step(s, nl, nxt, alt);
            if (nl >= seg_end) {
#pragma unroll
                for (int t = 0; t < NT; ++t) nxt[t] = alt[t];
                break;
            }
            s = nl;
            nl = next_live(s);
            step(s, nl, alt, nxt);
        }
#else
        // one copy of the step body (instruction-cache footprint); the prefetched gathers move to
        // `nxt` with NT register moves
        while (nl < seg_end) {
            const int s = nl;
            nl = next_live(s);
            step(s, nl, nxt, alt);
#pragma unroll
            for (int t = 0; t < NT; ++t) nxt[t] = alt[t];
        }
#endif
        // tests of this run, per target: sets [sg0, hi) minus the member set (serial order); the
        // dead (h00 == 0) ones among them were decided without arithmetic
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int hi = ((hit >> t) & 1u) ? lim[t] + 1 : min(seg_end, lim[t]);
            const int n = max(0, hi - sg0);
            const bool in = dm[t] >= sg0 && dm[t] < sg0 + n;
            tests += (unsigned)(n - (in ? 1 : 0));
            const unsigned rm = n >= 32 ? 0xffffffffu : (((1u << n) - 1u) << sg0);
            degen += (unsigned)(__popc(dead & rm) - ((in && ((dead >> dm[t]) & 1u)) ? 1 : 0));
        }
        sg = seg_end;
    }
}

template <int L>
__global__ void __launch_bounds__(kSetWarps * 32, L == 2 ? PCS_SET_MINB_L2 : (L >= 6 ? PCS_SET_MINB_DEEP : PCS_SET_MINB)) level_set_kernel(LevelArgs A, int pass,
                                                                     const unsigned long long* prefix,
                                                                     unsigned long long u_begin,
                                                                     unsigned long long u_end) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int kStage = SetCfg<L>::kStage;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    SetWarpSmem<L>& S = reinterpret_cast<SetWarpSmem<L>*>(smem_raw)[wib];
    const double* __restrict__ C = A.C;
    const long long ldc = A.ldc;
    // pass 2: both directions in one sweep (every set's pseudo-inverse computed once per level);
    // a target's key base carries its own direction bit, dir-0 (K0) or dir-1 (K0 | 1 << 62)
    const unsigned long long dirbits = pass == 1 ? (1ull << kDirShift) : 0ull;
    const unsigned lt_mask = (1u << lane) - 1u;
    unsigned long long tests = 0, pinvs = 0, degen = 0;
    int nan = 0;
    unsigned long long* cursor = &A.cnt->units[pass & 1];
    u_end = min(u_end, prefix[A.p]);
    int row_hint = 0;
    // the next unit is grabbed one unit ahead (lane 0's atomic result is only read at the top of the
    // next iteration), so the cursor round trip overlaps the current unit's work
    unsigned long long grabbed = 0;
    if (lane == 0) grabbed = atomicAdd(cursor, 1ull);
    for (;;) {
        const unsigned long long u = u_begin + __shfl_sync(0xffffffffu, grabbed, 0);
        if (u >= u_end) break;
        if (lane == 0) grabbed = atomicAdd(cursor, 1ull);
        const int i = find_row_from(prefix, A.p, u, row_hint);
        row_hint = i;
        const unsigned long long t0 = (u - prefix[i]) * kSetBand;
        const int oi = A.off[i], w = A.off[i + 1] - oi, lc = A.lowcnt[i];
        const int qbeg = pass == 2 ? 0 : (pass == 0 ? lc : 0), qend = pass == 2 ? w : (pass == 0 ? w : lc);
        const unsigned long long K0 = dirbits | t0;
        const unsigned long long total = A.binom(w, L);
        const int nvalid = (int)min(32ull, total - t0);
        bool have_sets = false;
        unsigned segmask = 1u, livemask = 0u;
        for (int tb = qbeg; tb < qend; tb += kStage) {
            const int tend = min(tb + kStage, qend);
            // ---- stage the live targets of [tb, tend), compacted: per directed entry the key mirror,
            // edge id, neighbour and C(i, j) are independent coalesced loads (one round trip)
            int nlive = 0;
#ifdef PCS_STAGE_REPS  // cost probe (tools/variants.py): staging repeated, results unchanged
            for (int rep = 0; rep < PCS_STAGE_REPS; ++rep) {
            asm volatile("" ::: "memory");
            nlive = 0;
#endif
            {
                constexpr int NC = kStage / 32;
                unsigned long long kk[NC];
                int ee[NC], jj[NC];
                double cc[NC];
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const int q = tb + c * 32 + lane;
                    kk[c] = 0;
                    if (q < tend) {
                        kk[c] = A.kdir[oi + q];
                        ee[c] = A.eid[oi + q];
                        jj[c] = A.nbr[oi + q];
                        cc[c] = A.cnbr[oi + q];
                    }
                }
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    // a target's key base: K0 with the target's own direction bit (q < lc: j < i)
                    const bool live = kk[c] > (K0 | (tb + c * 32 + lane < lc ? (1ull << kDirShift) : 0ull));
                    const unsigned bal = __ballot_sync(0xffffffffu, live);
                    if (live) {
                        const int at = nlive + __popc(bal & lt_mask);
                        S.tkey[at] = kk[c];
                        S.tq[at] = tb + c * 32 + lane;
                        S.tj[at] = jj[c];
                        S.te[at] = ee[c];
                        S.tcij[at] = cc[c];
                    }
                    nlive += __popc(bal);
                }
            }
#ifdef PCS_STAGE_REPS
            }
#endif
            if (nlive == 0) continue;
            // ---- phase 1 (once per unit): lane-parallel pseudo-inverses of the band's sets
            if (!have_sets) {
                have_sets = true;
#ifdef PCS_PHASE1_REPS  // cost probe (tools/variants.py): phase 1 repeated, results unchanged
                for (int rep = 0; rep < PCS_PHASE1_REPS; ++rep) {
                asm volatile("" ::: "memory");
#endif
                if (lane < nvalid) {
                    int pos[L];
#if PCS_UNRANK_BSEARCH
                    unrank<L>(A.binom, w, t0 + lane, pos);
#else
                    unrank_est<L>(A.binom, w, t0 + lane, pos);
#endif
                    int mem[L];
                    double m2[L * L], minv[L * L], ciS[L], p0[L], h00;
#pragma unroll
                    for (int a = 0; a < L; ++a) {
                        mem[a] = A.nbr[oi + pos[a]];
                        ciS[a] = __ldg(C + (size_t)i * ldc + mem[a]);
                    }
                    if (L <= 3 && A.pinv_table) {  // the set's M2^+ from the per-level table (same bits)
                        const double* e = A.pinv_table + colex_rank<L>(mem) * (unsigned long long)PinvStride<L>::v;
#pragma unroll
                        for (int q = 0; q < L * L; q += 2) {
                            if (q + 1 < L * L) {
                                const double2 v2 = __ldg(reinterpret_cast<const double2*>(e + q));
                                minv[q] = v2.x;
                                minv[q + 1] = v2.y;
                            } else {
                                minv[q] = __ldg(e + q);
                            }
                        }
                    } else {
#pragma unroll
                        for (int a = 0; a < L; ++a)
#pragma unroll
                            for (int b = 0; b < L; ++b) m2[a * L + b] = __ldg(C + (size_t)mem[a] * ldc + mem[b]);
                        pinv<L>(m2, minv);
                    }
                    p0_terms<L>(minv, ciS, p0, h00);
                    SetSlot<L>& sl = S.slot[lane];
#pragma unroll
                    for (int c = 0; c < L; ++c) {
#pragma unroll
                        for (int k = 0; k < L; ++k) sl.col[c][k] = minv[k * L + c];
                        sl.col[c][L] = ciS[c];
                        sl.col[c][L + 1] = p0[c];
                    }
#pragma unroll
                    for (int a = 0; a < L; ++a) {
                        sl.pos[a] = pos[a];
                        sl.roff[a] = mem[a] * (int)ldc;  // p * ldc < 2^31 (p <= 46340)
                    }
                    sl.h00 = h00;
                }
#ifdef PCS_PHASE1_REPS
                }
#endif
                if (lane == 0) pinvs += nvalid;
                // runs of consecutive sets with equal leading L-1 members (lexicographic order)
                bool starts = lane == 0;
                if (L > 1) {
                    const int prev = lane > 0 ? lane - 1 : 0;
#pragma unroll
                    for (int a = 0; a < L - 1; ++a) {
                        const int mine = lane < nvalid ? S.slot[lane].pos[a] : -1;
                        const int theirs = __shfl_sync(0xffffffffu, mine, prev);
                        starts = starts || mine != theirs;
                    }
                }
                segmask = __ballot_sync(0xffffffffu, starts);
                livemask = __ballot_sync(0xffffffffu, lane < nvalid && S.slot[lane].h00 != 0.0);
            }
            __syncwarp();
            // ---- phase 2: sets in rank order, NT targets per lane
            const int nt = (nlive + 31) >> 5;
            if constexpr (SetCfg<L>::NT >= 4 && L <= 3) {  // partially filled batches as in the NT = 3 case
                constexpr int NTM = SetCfg<L>::NT;
                if (nt > 3) set_sweep<L, NTM>(A, S, lane, oi, lc, nlive, nvalid, segmask, livemask, K0, tests, degen, nan);
                else if (nt == 3) set_sweep<L, 3>(A, S, lane, oi, lc, nlive, nvalid, segmask, livemask, K0, tests, degen, nan);
#if PCS_NT2_SP > 1
                else if (nt == 2) set_sweep_tsp<L, 2, PCS_NT2_SP>(A, S, lane, oi, lc, nlive, nvalid, segmask, livemask, K0, tests, degen, nan);
#else
                else if (nt == 2) set_sweep<L, 2>(A, S, lane, oi, lc, nlive, nvalid, segmask, livemask, K0, tests, degen, nan);
#endif
                else set_sweep_tsp<L, 1, PCS_SET_SP>(A, S, lane, oi, lc, nlive, nvalid, segmask, livemask, K0, tests, degen, nan);
            } else if constexpr (SetCfg<L>::NT >= 4) {
                constexpr int NTM = SetCfg<L>::NT;
                if (nt > 3) set_sweep<L, NTM>(A, S, lane, oi, lc, nlive, nvalid, segmask, livemask, K0, tests, degen, nan);
                else if (nt == 3) set_sweep<L, 3>(A, S, lane, oi, lc, nlive, nvalid, segmask, livemask, K0, tests, degen, nan);
                else if (nt == 2) set_sweep<L, 2>(A, S, lane, oi, lc, nlive, nvalid, segmask, livemask, K0, tests, degen, nan);
                else set_sweep<L, 1>(A, S, lane, oi, lc, nlive, nvalid, segmask, livemask, K0, tests, degen, nan);
            } else if constexpr (SetCfg<L>::NT == 3) {
                if (nt == 3) set_sweep<L, 3>(A, S, lane, oi, lc, nlive, nvalid, segmask, livemask, K0, tests, degen, nan);
#if PCS_NT2_SP > 1
                else if (nt == 2) set_sweep_tsp<L, 2, PCS_NT2_SP>(A, S, lane, oi, lc, nlive, nvalid, segmask, livemask, K0, tests, degen, nan);
#else
                else if (nt == 2) set_sweep<L, 2>(A, S, lane, oi, lc, nlive, nvalid, segmask, livemask, K0, tests, degen, nan);
#endif
                else set_sweep_tsp<L, 1, PCS_SET_SP>(A, S, lane, oi, lc, nlive, nvalid, segmask, livemask, K0, tests, degen, nan);
            } else {
                if (nt == 2) set_sweep<L, 2>(A, S, lane, oi, lc, nlive, nvalid, segmask, livemask, K0, tests, degen, nan);
                else set_sweep_tsp<L, 1, 2>(A, S, lane, oi, lc, nlive, nvalid, segmask, livemask, K0, tests, degen, nan);
            }
            __syncwarp();
        }
        if (!have_sets && lane == 0) {
            // no live target at rank t0: none at any later rank of this row either
            const unsigned long long next_row = prefix[i + 1] - u_begin;
            atomicMax(cursor, next_row);
        }
    }
    add_counter(&A.cnt->gpu_tests, tests);
    add_counter(&A.cnt->gpu_exact, tests - degen);  // evaluated in the reference's operation order
    if (lane == 0 && pinvs) atomicAdd(&A.cnt->gpu_pinv, pinvs);
    if (nan) atomicOr(&A.cnt->err_nan, 1);
}

template <int L>
static int launch_set_L(const LevelArgs& A, int pass, const unsigned long long* prefix, unsigned long long u_begin,
                        unsigned long long u_end, int num_sms, cudaStream_t s) {
    const size_t smem = sizeof(SetWarpSmem<L>) * kSetWarps;
    // per launch (the attribute is per device; one launch per level pass, so the call is negligible)
    if (cudaFuncSetAttribute(level_set_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return -2;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, level_set_kernel<L>, kSetWarps * 32, smem);
    if (per_sm < 1) per_sm = 1;
    ++g_kernel_launches;
    level_set_kernel<L><<<num_sms * per_sm, kSetWarps * 32, smem, s>>>(A, pass, prefix, u_begin, u_end);
    return 0;
}

int launch_level_set(const LevelArgs& A, int pass, const unsigned long long* prefix, unsigned long long u_begin,
                     unsigned long long u_end, int num_sms, cudaStream_t s) {
    switch (A.ell) {
        case 2: return launch_set_L<2>(A, pass, prefix, u_begin, u_end, num_sms, s);
        case 3: return launch_set_L<3>(A, pass, prefix, u_begin, u_end, num_sms, s);
        case 4: return launch_set_L<4>(A, pass, prefix, u_begin, u_end, num_sms, s);
        case 5: return launch_set_L<5>(A, pass, prefix, u_begin, u_end, num_sms, s);
        case 6: return launch_set_L<6>(A, pass, prefix, u_begin, u_end, num_sms, s);
        case 7: return launch_set_L<7>(A, pass, prefix, u_begin, u_end, num_sms, s);
        case 8: return launch_set_L<8>(A, pass, prefix, u_begin, u_end, num_sms, s);
        default: return -1;
    }
}

// =========================================================== ell >= 2, cuPC-E
template <int L>
__global__ void __launch_bounds__(128) level_edge_kernel(LevelArgs A, int pass, long long e_begin, long long e_end) {
    const int lane = threadIdx.x & 31;
    const double* __restrict__ C = A.C;
    const long long ldc = A.ldc;
    const unsigned long long dirbits = (unsigned long long)pass << kDirShift;
    unsigned long long tests = 0, pinvs = 0;
    int nan = 0;
    unsigned long long* cursor = &A.cnt->units[pass];
    for (;;) {
        unsigned long long ue = 0;
        if (lane == 0) ue = atomicAdd(cursor, 1ull);
        ue = __shfl_sync(0xffffffffu, ue, 0);
        const long long e = e_begin + (long long)ue;
        if (e >= e_end) break;
        if (pass == 1 && A.keys[e] != (unsigned long long)kNoneKey) continue;
        const int a = A.eu_a[e], qa = A.eu_qa[e];
        const int b = A.nbr[A.off[a] + qa];
        const int i = pass == 0 ? a : b;
        const int q = pass == 0 ? qa : A.eu_qb[e];
        const int j = pass == 0 ? b : a;
        const int oi = A.off[i], w = A.off[i + 1] - oi;
        if (w < L + 1) continue;
        const unsigned long long total = A.binom(w - 1, L);
        const double cij = __ldg(C + (size_t)i * ldc + j);
        for (unsigned long long base = 0; base < total; base += 32) {
            const unsigned long long t = base + lane;
            const bool valid = t < total;
            int d = kDependent;
            int pos[L];
            if (valid) {
                unrank<L>(A.binom, w - 1, t, pos);
                int mem[L];
                double ciS[L], cjS[L], m2[L * L], minv[L * L], p0[L], h00, h01, denom;
#pragma unroll
                for (int k = 0; k < L; ++k) {
                    pos[k] += pos[k] >= q;  // skip the target position (skeleton.hpp:146-149)
                    mem[k] = A.nbr[oi + pos[k]];
                    ciS[k] = __ldg(C + (size_t)i * ldc + mem[k]);
                    cjS[k] = __ldg(C + (size_t)j * ldc + mem[k]);
                }
                if (L <= 3 && A.pinv_table) {  // the level's pseudo-inverse table (same bits)
                    const double* te = A.pinv_table + colex_rank<L>(mem) * (unsigned long long)PinvStride<L>::v;
#pragma unroll
                    for (int q2 = 0; q2 < L * L; ++q2) minv[q2] = __ldg(te + q2);
                } else {
#pragma unroll
                    for (int x = 0; x < L; ++x)
#pragma unroll
                        for (int y = 0; y < L; ++y) m2[x * L + y] = __ldg(C + (size_t)mem[x] * ldc + mem[y]);
                    pinv<L>(m2, minv);
                }
                p0_terms<L>(minv, ciS, p0, h00);
                h_terms<L>(minv, ciS, p0, h00, cjS, cij, h01, denom);
                d = take_near(decide_fast(h01, denom, A.th), A, i, j, h01, denom);
                ++tests;
                ++pinvs;
            }
            const unsigned hit = __ballot_sync(0xffffffffu, d != kDependent);
            if (hit) {
                const int first = __ffs(hit) - 1;
                if (lane == first) {
                    if (d == kNanError) nan = 1;
                    else atomicMin(A.keys + e, dirbits | rank_of<L>(A.binom, w, pos));
                }
                break;
            }
        }
    }
    add_counter(&A.cnt->gpu_tests, tests);
    add_counter(&A.cnt->gpu_exact, tests);
    add_counter(&A.cnt->gpu_pinv, pinvs);
    if (nan) atomicOr(&A.cnt->err_nan, 1);
}

// ----------------------------------------------------------- cuPC-E, staged operands
// The same warp-per-edge schedule (lanes over the edge's conditioning sets in rank order, 32 per
// round, ballot early exit at the first separating set), with the edge's correlation sub-block in
// shared memory instead of 2L + 1 L2 gathers per test:
//   ci[k] = C(i, nbr_i[k])  the contiguous C(i, nbr) segment of row i (A.cnbr), one 1-D TMA bulk copy
//                           (cp.async.bulk, mbarrier transaction count) issued by lane 0;
//   cj[k] = C(j, nbr_i[k])  a gather (the other lanes, concurrently with the bulk copy);
//   nb[k] = nbr_i[k].
// A test then reads its members, C(i, S) and C(j, S) from shared memory; its set comes from
// unrank_est (one estimate + fix-up per member instead of a binary search) and, at l = 2, 3, its
// M2^+ from the level's pseudo-inverse table.  Decisions, keys and counters are those of
// level_edge_kernel (same h_terms / decide_fast, same ranks).
namespace {
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(unsigned long long* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_wait(unsigned long long* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "EWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra EWAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
// one bulk copy of `bytes` (a multiple of 16, both addresses 16-B aligned) completing on `bar`
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(reinterpret_cast<unsigned long long>(src)), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}
}  // namespace

constexpr int kEdgeWarps = 4;
// per-warp shared bytes for rows up to wcap entries (wcap a multiple of 4): barrier, ci (+2 for the
// aligned superset the bulk copy brings), cj, nb
__host__ __device__ inline size_t edge_warp_smem(int wcap) { return 16 + (size_t)(wcap + 2) * 8 + (size_t)wcap * 12; }
constexpr size_t kEdgeSmemMax = 200 * 1024;  // per block; wider rows use level_edge_kernel

#ifndef PCS_EDGE_SPL
#define PCS_EDGE_SPL 1  // staged cuPC-E: conditioning sets per lane per round at l <= 3 (2: same time, 4: +12%)
#endif
template <int L>
struct EdgeSpl {
    static constexpr int v = L <= 3 ? PCS_EDGE_SPL : 1;
};

#ifndef PCS_EDGE_MINB
#define PCS_EDGE_MINB 1  // resident blocks per SM the staged cuPC-E kernel is register-budgeted for
#endif

template <int L>
__global__ void __launch_bounds__(kEdgeWarps * 32, PCS_EDGE_MINB) level_edge_staged_kernel(LevelArgs A, int pass, long long e_begin,
                                                                            long long e_end, int wcap) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    unsigned char* base = smem_raw + (size_t)wib * edge_warp_smem(wcap);
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(base);
    double* cibuf = reinterpret_cast<double*>(base + 16);
    double* cj = cibuf + wcap + 2;
    int* nb = reinterpret_cast<int*>(cj + wcap);
    const double* __restrict__ C = A.C;
    const long long ldc = A.ldc;
    const unsigned long long dirbits = (unsigned long long)pass << kDirShift;
    unsigned long long tests = 0, pinvs = 0;
    int nan = 0;
    uint32_t parity = 0;
    if (lane == 0) bar_init(bar);
    __syncwarp();
    unsigned long long* cursor = &A.cnt->units[pass];
    for (;;) {
        unsigned long long ue = 0;
        if (lane == 0) ue = atomicAdd(cursor, 1ull);
        ue = __shfl_sync(0xffffffffu, ue, 0);
        const long long e = e_begin + (long long)ue;
        if (e >= e_end) break;
        if (pass == 1 && A.keys[e] != (unsigned long long)kNoneKey) continue;
        const int a = A.eu_a[e], qa = A.eu_qa[e];
        const int b = A.nbr[A.off[a] + qa];
        const int i = pass == 0 ? a : b;
        const int q = pass == 0 ? qa : A.eu_qb[e];
        const int j = pass == 0 ? b : a;
        const int oi = A.off[i], w = A.off[i + 1] - oi;
        if (w < L + 1) continue;
        // ---- stage: C(i, nbr_i) by bulk copy (an even-aligned superset of the segment), the rest by lanes
        const int o0 = oi & ~1;
        if (lane == 0) bulk_load(cibuf, A.cnbr + o0, (uint32_t)((((oi + w + 1) & ~1) - o0) * sizeof(double)), bar);
        const double* __restrict__ Cj = C + (size_t)j * ldc;
        for (int k = lane; k < w; k += 32) {
            const int m = A.nbr[oi + k];
            nb[k] = m;
            cj[k] = __ldg(Cj + m);
        }
        bar_wait(bar, parity);
        parity ^= 1u;
        __syncwarp();
        const double* ci = cibuf + (oi - o0);
        const double cij = ci[q];
        const unsigned long long total = A.binom(w - 1, L);
        // rounds of 32 * SPL ranks: lane l tests ranks base_t + 32 s + l (s < SPL), SPL independent
        // chains per lane; the round's first separating set in rank order wins.  At l = 2, 3 a lane
        // unranks its first set once per edge and then steps its positions by 32 SPL ranks per round
        // (advance_lex), no binomial-table loads in the loop.
        constexpr int SPL = EdgeSpl<L>::v;
        constexpr bool kIncr = L <= 3;
        int cur[SPL][L];
        if (kIncr) {
#pragma unroll
            for (int sp = 0; sp < SPL; ++sp)
                if ((unsigned long long)(32 * sp + lane) < total) unrank_est<L>(A.binom, w - 1, 32 * sp + lane, cur[sp]);
        }
        for (unsigned long long base_t = 0; base_t < total; base_t += 32 * SPL) {
            int d[SPL];
            int pos[SPL][L];
#pragma unroll
            for (int sp = 0; sp < SPL; ++sp) {
                const unsigned long long t = base_t + 32 * sp + lane;
                d[sp] = kDependent;
                if (t < total) {
                    if (kIncr) {
#pragma unroll
                        for (int k = 0; k < L; ++k) pos[sp][k] = cur[sp][k];
                        advance_lex<L>(cur[sp], w - 1, 32 * SPL);
                    } else {
                        unrank_est<L>(A.binom, w - 1, t, pos[sp]);
                    }
                    int mem[L];
                    double ciS[L], cjS[L], minv[L * L], p0[L], h00, h01, denom;
#pragma unroll
                    for (int k = 0; k < L; ++k) {
                        pos[sp][k] += pos[sp][k] >= q;  // skip the target position (skeleton.hpp:146-149)
                        mem[k] = nb[pos[sp][k]];
                        ciS[k] = ci[pos[sp][k]];
                        cjS[k] = cj[pos[sp][k]];
                    }
                    if (L <= 3 && A.pinv_table) {  // the level's pseudo-inverse table (same bits)
                        const double* te = A.pinv_table + colex_rank<L>(mem) * (unsigned long long)PinvStride<L>::v;
#pragma unroll
                        for (int q2 = 0; q2 < L * L; ++q2) minv[q2] = __ldg(te + q2);
                    } else {
                        double m2[L * L];
#pragma unroll
                        for (int x = 0; x < L; ++x)
#pragma unroll
                            for (int y = 0; y < L; ++y) m2[x * L + y] = __ldg(C + (size_t)mem[x] * ldc + mem[y]);
                        pinv<L>(m2, minv);
                    }
                    p0_terms<L>(minv, ciS, p0, h00);
                    h_terms<L>(minv, ciS, p0, h00, cjS, cij, h01, denom);
                    d[sp] = take_near(decide_fast(h01, denom, A.th), A, i, j, h01, denom);
                    ++tests;
                    ++pinvs;
                }
            }
            bool found = false;
#pragma unroll
            for (int sp = 0; sp < SPL; ++sp) {
                const unsigned hit = __ballot_sync(0xffffffffu, d[sp] != kDependent);
                if (hit && !found) {
                    found = true;
                    const int first = __ffs(hit) - 1;
                    if (lane == first) {
                        if (d[sp] == kNanError) nan = 1;
                        else atomicMin(A.keys + e, dirbits | rank_of<L>(A.binom, w, pos[sp]));
                    }
                }
            }
            if (found) break;
        }
        __syncwarp();  // the buffers are rewritten for the next edge
    }
    add_counter(&A.cnt->gpu_tests, tests);
    add_counter(&A.cnt->gpu_exact, tests);
    add_counter(&A.cnt->gpu_pinv, pinvs);
    if (nan) atomicOr(&A.cnt->err_nan, 1);
}

#ifndef PCS_EDGE_STAGED
#define PCS_EDGE_STAGED 1  // 0: cuPC-E always on the unstaged kernel (A/B)
#endif

template <int L>
static int launch_edge_L(const LevelArgs& A, int pass, long long e_begin, long long e_end, int maxw, int num_sms,
                         cudaStream_t s) {
    // PCS_EDGE_STAGED=0 in the environment forces the unstaged kernel (tests cover both)
    static const bool staged = [] {
        const char* e = std::getenv("PCS_EDGE_STAGED");
        return PCS_EDGE_STAGED && !(e && std::atoi(e) == 0);
    }();
    int per_sm = 0;
    const int wcap = (maxw + 3) & ~3;
    const size_t smem = edge_warp_smem(wcap) * kEdgeWarps;
    if (staged && smem <= kEdgeSmemMax) {
        if (cudaFuncSetAttribute(level_edge_staged_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
            return -2;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, level_edge_staged_kernel<L>, kEdgeWarps * 32, smem);
        if (per_sm < 1) per_sm = 1;
        ++g_kernel_launches;
        level_edge_staged_kernel<L><<<num_sms * per_sm, kEdgeWarps * 32, smem, s>>>(A, pass, e_begin, e_end, wcap);
        return 0;
    }
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, level_edge_kernel<L>, 128, 0);
    if (per_sm < 1) per_sm = 1;
    ++g_kernel_launches;
    level_edge_kernel<L><<<num_sms * per_sm, 128, 0, s>>>(A, pass, e_begin, e_end);
    return 0;
}

int launch_level_edge(const LevelArgs& A, int pass, long long e_begin, long long e_end, int maxw, int num_sms,
                      cudaStream_t s) {
    switch (A.ell) {
        case 2: return launch_edge_L<2>(A, pass, e_begin, e_end, maxw, num_sms, s);
        case 3: return launch_edge_L<3>(A, pass, e_begin, e_end, maxw, num_sms, s);
        case 4: return launch_edge_L<4>(A, pass, e_begin, e_end, maxw, num_sms, s);
        case 5: return launch_edge_L<5>(A, pass, e_begin, e_end, maxw, num_sms, s);
        case 6: return launch_edge_L<6>(A, pass, e_begin, e_end, maxw, num_sms, s);
        case 7: return launch_edge_L<7>(A, pass, e_begin, e_end, maxw, num_sms, s);
        case 8: return launch_edge_L<8>(A, pass, e_begin, e_end, maxw, num_sms, s);
        default: return -1;
    }
}

// =========================================================== ell > 8 (generic)
// cuPC-S with runtime ell: lane-parallel pseudo-inverses as in level_set_kernel,
// all per-set matrices in a per-lane slice of global scratch (L1/L2 resident).
// Serves both device variants above kMaxTemplLevel (results are identical).
__host__ __device__ inline long long rt_lane_doubles(int n) { return 7ll * n * n + 4ll * n + 1; }

__global__ void __launch_bounds__(128) level_set_rt_kernel(LevelArgs A, int pass, const unsigned long long* prefix,
                                                           unsigned long long u_begin, unsigned long long u_end,
                                                           double* scratch, int* iscratch) {
    const int n = A.ell;
    const int lane = threadIdx.x & 31;
    const long long gwarp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long SD = rt_lane_doubles(n);
    double* wbase = scratch + gwarp * 32 * SD;
    int* ibase = iscratch + gwarp * 32 * 2 * n;
    // per-lane regions
    double* m2 = wbase + lane * SD;
    double* minv = m2 + n * n;
    double* ws = minv + n * n;
    double* ciS = ws + 5 * n * n;
    double* p0 = ciS + n;
    double* h00p = p0 + n;
    double* P1 = h00p + 1;
    double* cjS = P1 + n;
    int* pos = ibase + lane * 2 * n;
    int* mem = pos + n;
    const double* __restrict__ C = A.C;
    const long long ldc = A.ldc;
    // pass 2: both directions in one sweep (each set's pseudo-inverse once per level), a target's key
    // base carrying its own direction bit, as in level_set_kernel
    const unsigned long long dirbits = pass == 1 ? (1ull << kDirShift) : 0ull;
    unsigned long long tests = 0, pinvs = 0, degen = 0;
    int nan = 0;
    unsigned long long* cursor = &A.cnt->units[pass & 1];
    u_end = min(u_end, prefix[A.p]);
    int row_hint = 0;
    for (;;) {
        unsigned long long u = 0;
        if (lane == 0) u = u_begin + atomicAdd(cursor, 1ull);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= u_end) break;
        const int i = find_row_from(prefix, A.p, u, row_hint);
        row_hint = i;
        const unsigned long long t0 = (u - prefix[i]) * kSetBand;
        const int oi = A.off[i], w = A.off[i + 1] - oi, lc = A.lowcnt[i];
        const int qbeg = pass == 2 ? 0 : (pass == 0 ? lc : 0), qend = pass == 2 ? w : (pass == 0 ? w : lc);
        auto dbits = [&](int q) -> unsigned long long {  // q < lc: j < i, direction 1 of edge (j, i)
            return pass == 2 ? (q < lc ? (1ull << kDirShift) : 0ull) : dirbits;
        };
        bool open = false;
        for (int q = qbeg + lane; q < qend; q += 32) open |= A.keys[A.eid[oi + q]] > (dbits(q) | t0);
        if (!__any_sync(0xffffffffu, open)) {
            // no open target at rank t0: none at any later rank of this row (keys only decrease)
            if (lane == 0) atomicMax(cursor, prefix[i + 1] - u_begin);
            continue;
        }
        const unsigned long long total = A.binom(w, n);
        const unsigned long long t = t0 + lane;
        const bool valid = t < total;
        if (valid) {
            unrank_rt(A.binom, w, n, t, pos);
            for (int a = 0; a < n; ++a) {
                mem[a] = A.nbr[oi + pos[a]];
                ciS[a] = __ldg(C + (size_t)i * ldc + mem[a]);
            }
            for (int a = 0; a < n; ++a)
                for (int b = 0; b < n; ++b) m2[a * n + b] = __ldg(C + (size_t)mem[a] * ldc + mem[b]);
            pinv_rt(m2, n, minv, ws);
            double h00;
            p0_terms_rt(minv, ciS, n, p0, h00);
            *h00p = h00;
        }
        const int nvalid = __popc(__ballot_sync(0xffffffffu, valid));
        if (lane == 0) pinvs += nvalid;
        __syncwarp();
        __threadfence_block();
        for (int qc = qbeg; qc < qend; qc += 32) {
            const int q = qc + lane;
            bool live = q < qend;
            int j = 0, e = 0;
            unsigned long long key = 0;
            double cij = 0.0;
            if (live) {
                j = A.nbr[oi + q];
                e = A.eid[oi + q];
                key = A.keys[e];
                live = key > (dbits(q) | t0);
                if (live) cij = __ldg(C + (size_t)i * ldc + j);
            }
            if (!__any_sync(0xffffffffu, live)) continue;
            for (int sg = 0; sg < nvalid; ++sg) {
                if (!live) break;
                const double* S = wbase + sg * SD;
                const int* Spos = ibase + sg * 2 * n;
                const unsigned long long Kc = dbits(q) | (t0 + sg);
                if (key <= Kc) { live = false; break; }
                bool member = false;
                for (int a = 0; a < n; ++a) member |= Spos[a] == q;
                if (member) continue;
                const double* Sminv = S + n * n;
                const double* SciS = S + 7 * n * n;
                ++tests;
                if (SciS[2 * n] == 0.0) { ++degen; continue; }  // h00 == 0: degenerate (see set_sweep)
                for (int a = 0; a < n; ++a) cjS[a] = __ldg(C + (size_t)Spos[n + a] * ldc + j);
                double h01, denom;
                h_terms_rt(Sminv, SciS, SciS + n, SciS[2 * n], cjS, n, cij, P1, h01, denom);
                const int d = take_near(decide_fast(h01, denom, A.th), A, i, j, h01, denom);
                if (d != kDependent) {
                    live = false;
                    if (d == kNanError) nan = 1;
                    else atomicMin(A.keys + e, Kc);
                }
            }
        }
        __syncwarp();
    }
    add_counter(&A.cnt->gpu_tests, tests);
    add_counter(&A.cnt->gpu_exact, tests - degen);
    if (lane == 0 && pinvs) atomicAdd(&A.cnt->gpu_pinv, pinvs);
    if (nan) atomicOr(&A.cnt->err_nan, 1);
}

long long level_rt_scratch_bytes(int ell, int num_sms, int* blocks_out) {
    const long long per_lane = rt_lane_doubles(ell) * 8 + 2ll * ell * 4;
    long long blocks = (long long)num_sms * 8;
    const long long budget = 2ll << 30;
    while (blocks > num_sms && blocks * 128 * per_lane > budget) blocks -= num_sms;
    if (blocks_out) *blocks_out = (int)blocks;
    return blocks * 128 * per_lane;
}

int launch_level_set_rt(const LevelArgs& A, int pass, const unsigned long long* prefix, unsigned long long u_begin,
                        unsigned long long u_end, int num_sms, void* scratch, cudaStream_t s) {
    if (A.ell > kMaxRtLevel) return -1;
    int blocks = 0;
    level_rt_scratch_bytes(A.ell, num_sms, &blocks);
    const long long lanes = (long long)blocks * 128;
    double* sd = static_cast<double*>(scratch);
    int* si = reinterpret_cast<int*>(sd + lanes * rt_lane_doubles(A.ell));
    ++g_kernel_launches;
    level_set_rt_kernel<<<blocks, 128, 0, s>>>(A, pass, prefix, u_begin, u_end, sd, si);
    return 0;
}

// generic-ell parity helpers (one test / block per thread, global scratch)
__global__ void ci_batch_rt_kernel(const double* C, long long ldc, int n, long long cnt, const int32_t* ij,
                                   const int32_t* sets, double tau, uint8_t* indep, double* zout, double* rhoout,
                                   uint8_t* degen, int* err, double* scratch) {
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= cnt) return;
    double* m2 = scratch + k * rt_lane_doubles(n);
    double* minv = m2 + n * n;
    double* ws = minv + n * n;
    double* ciS = ws + 5 * n * n;
    double* p0 = ciS + n;
    double* P1 = p0 + n + 1;
    double* cjS = P1 + n;
    const int i = ij[2 * k], j = ij[2 * k + 1];
    const int32_t* mem = sets + k * n;
    for (int a = 0; a < n; ++a) {
        ciS[a] = C[(size_t)i * ldc + mem[a]];
        cjS[a] = C[(size_t)j * ldc + mem[a]];
        for (int b = 0; b < n; ++b) m2[a * n + b] = C[(size_t)mem[a] * ldc + mem[b]];
    }
    pinv_rt(m2, n, minv, ws);
    double h00, h01, denom, z, rho;
    p0_terms_rt(minv, ciS, n, p0, h00);
    h_terms_rt(minv, ciS, p0, h00, cjS, n, C[(size_t)i * ldc + j], P1, h01, denom);
    const int d = decide_exact(h01, denom, tau, &z, &rho);
    if (d == kNanError) atomicOr(err, 1);
    indep[k] = d == kIndependent;
    zout[k] = z;
    rhoout[k] = rho;
    degen[k] = !(denom > 0.0);
}

__global__ void pinv_batch_rt_kernel(const double* a, int n, long long cnt, double* out, double* scratch) {
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= cnt) return;
    pinv_rt(a + k * n * n, n, out + k * n * n, scratch + k * 5ll * n * n);
}

int launch_ci_batch_rt(const double* C, long long ldc, int ell, long long n, const int32_t* ij, const int32_t* sets,
                       double tau, uint8_t* indep, double* z, double* rho, uint8_t* degen, int* err, double* scratch,
                       cudaStream_t s) {
    if (n <= 0) return 0;
    ++g_kernel_launches;
    ci_batch_rt_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(C, ldc, ell, n, ij, sets, tau, indep, z, rho,
                                                                   degen, err, scratch);
    return 0;
}

int launch_pinv_batch_rt(const double* a, int ell, long long n, double* out, double* scratch, cudaStream_t s) {
    if (n <= 0) return 0;
    ++g_kernel_launches;
    pinv_batch_rt_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(a, ell, n, out, scratch);
    return 0;
}

// =========================================================== commit
// One thread per undirected snapshot edge: decode the key (full-row rank in
// the deciding row), clear the edge in the live bitmask, append the sepset
// record (a, b, ell, members...) and accumulate the serial strategy's ci_tests
// (test_edge_over_sets counts, skeleton.hpp:140-158).
__global__ void commit_kernel(LevelArgs A, uint32_t* adj, int W, long long e_und, int32_t* rec) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long tests = 0, removed = 0;
    const int ell = A.ell;
    if (e < e_und) {
        const int a = A.eu_a[e], qa = A.eu_qa[e], qb = A.eu_qb[e];
        const int b = A.nbr[A.off[a] + qa];
        const int wa = A.off[a + 1] - A.off[a], wb = A.off[b + 1] - A.off[b];
        const unsigned long long T0 = wa >= ell + 1 ? A.binom(wa - 1, ell) : 0ull;
        const unsigned long long T1 = wb >= ell + 1 ? A.binom(wb - 1, ell) : 0ull;
        const unsigned long long key = A.keys[e];
        if (key == (unsigned long long)kNoneKey) {
            tests = T0 + T1;
        } else {
            const int dir = (int)(key >> kDirShift);
            const unsigned long long t = key & kRankMask;
            const int r = dir ? b : a, q = dir ? qb : qa, w = dir ? wb : wa;
            int pos[kMaxKeyLevel];
            unrank_rt(A.binom, w, ell, t, pos);
            int red[kMaxKeyLevel];
            for (int k = 0; k < ell; ++k) red[k] = pos[k] - (pos[k] > q);
            const unsigned long long rr = rank_rt(A.binom, w - 1, ell, red);
            tests = dir ? T0 + rr + 1ull : rr + 1ull;
            removed = 1;
            atomicAnd(adj + (size_t)a * W + (b >> 5), ~(1u << (b & 31)));
            atomicAnd(adj + (size_t)b * W + (a >> 5), ~(1u << (a & 31)));
            const unsigned long long slot = atomicAdd(&A.cnt->rec_count, 1ull);
            int32_t* out = rec + slot * (size_t)(3 + ell);  // the result's final layout: no host re-layout
            out[0] = a;
            out[1] = b;
            out[2] = ell;
            const int orow = A.off[r];
            for (int k = 0; k < ell; ++k) out[3 + k] = A.nbr[orow + pos[k]];
        }
    }
    add_counter(&A.cnt->ci_serial, tests);
    add_counter(&A.cnt->removed, removed);
}

void launch_commit(const LevelArgs& A, uint32_t* adj, int W, long long e_und, int32_t* rec, cudaStream_t s) {
    if (e_und <= 0) return;
    ++g_kernel_launches;
    commit_kernel<<<(unsigned)((e_und + 255) / 256), 256, 0, s>>>(A, adj, W, e_und, rec);
}

// =========================================================== parity helpers
template <int L>
__global__ void ci_batch_kernel(const double* C, long long ldc, long long n, const int32_t* ij, const int32_t* sets,
                                double tau, uint8_t* indep, double* zout, double* rhoout, uint8_t* degen, int* err) {
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int i = ij[2 * k], j = ij[2 * k + 1];
    double z, rho, h01 = 0.0, denom = 1.0;
    int d;
    if (L == 0) {
        const double c = C[(size_t)i * ldc + j];
        const double v = c < -kRhoClamp ? -kRhoClamp : (c > kRhoClamp ? kRhoClamp : c);
        rho = v;
        z = fabs(0.5 * log((1.0 + v) / (1.0 - v)));
        d = z <= tau ? kIndependent : kDependent;
        if (!(v > -1.0 && v < 1.0)) d = kNanError;
    } else {
        constexpr int LL = L > 0 ? L : 1;
        int mem[LL];
        double ciS[LL], cjS[LL], m2[LL * LL], minv[LL * LL], p0[LL], h00;
#pragma unroll
        for (int a = 0; a < LL; ++a) {
            mem[a] = sets[k * LL + a];
            ciS[a] = C[(size_t)i * ldc + mem[a]];
            cjS[a] = C[(size_t)j * ldc + mem[a]];
        }
#pragma unroll
        for (int a = 0; a < LL; ++a)
#pragma unroll
            for (int b = 0; b < LL; ++b) m2[a * LL + b] = C[(size_t)mem[a] * ldc + mem[b]];
        pinv<LL>(m2, minv);
        p0_terms<LL>(minv, ciS, p0, h00);
        h_terms<LL>(minv, ciS, p0, h00, cjS, C[(size_t)i * ldc + j], h01, denom);
        d = decide_exact(h01, denom, tau, &z, &rho);
    }
    if (d == kNanError) atomicOr(err, 1);
    indep[k] = d == kIndependent;
    zout[k] = z;
    rhoout[k] = rho;
    degen[k] = (L > 0) && !(denom > 0.0);
}

int launch_ci_batch(const double* C, long long ldc, int p, int ell, long long n, const int32_t* ij,
                    const int32_t* sets, double tau, uint8_t* indep, double* z, double* rho, uint8_t* degen,
                    int* err, cudaStream_t s) {
    if (n <= 0) return 0;
    const unsigned blocks = (unsigned)((n + 127) / 128);
#define PCS_CI_CASE(LV) \
    case LV: ci_batch_kernel<LV><<<blocks, 128, 0, s>>>(C, ldc, n, ij, sets, tau, indep, z, rho, degen, err); return 0;
    switch (ell) {
        PCS_CI_CASE(0) PCS_CI_CASE(1) PCS_CI_CASE(2) PCS_CI_CASE(3) PCS_CI_CASE(4)
        PCS_CI_CASE(5) PCS_CI_CASE(6) PCS_CI_CASE(7) PCS_CI_CASE(8)
        default: return -1;
    }
#undef PCS_CI_CASE
}

template <int L>
__global__ void pinv_batch_kernel(const double* a, long long n, double* out) {
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double m[L * L], r[L * L];
#pragma unroll
    for (int q = 0; q < L * L; ++q) m[q] = a[k * L * L + q];
    pinv<L>(m, r);
#pragma unroll
    for (int q = 0; q < L * L; ++q) out[k * L * L + q] = r[q];
}

int launch_pinv_batch(const double* a, int ell, long long n, double* out, cudaStream_t s) {
    if (n <= 0) return 0;
    const unsigned blocks = (unsigned)((n + 127) / 128);
#define PCS_PINV_CASE(LV) \
    case LV: pinv_batch_kernel<LV><<<blocks, 128, 0, s>>>(a, n, out); return 0;
    switch (ell) {
        PCS_PINV_CASE(1) PCS_PINV_CASE(2) PCS_PINV_CASE(3) PCS_PINV_CASE(4)
        PCS_PINV_CASE(5) PCS_PINV_CASE(6) PCS_PINV_CASE(7) PCS_PINV_CASE(8)
        default: return -1;
    }
#undef PCS_PINV_CASE
}

}  // namespace pcs
