// host.cu -- host driver and C ABI of libpcstable_b200.so.
//
// The level loop of run_pc_stable (skeleton.hpp:341-391) runs on the host; every
// level's work runs on the device:
//   level 0   : level0_kernel (bitmask)                               skeleton.hpp:262-288
//   level >= 1: snapshot (degree, scan, fill, edge index)             core.hpp:227-239
//               pass 0 / pass 1 CI-test kernels (keys, atomicMin)     skeleton.hpp:131-222
//               commit (removals, sepsets, serial-equivalent counts)  skeleton.hpp:123-129
// Stop conditions in the reference's order: level cap, sample size, max degree
// (skeleton.hpp:353-373).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "../../include/pcstable_b200.h"
#include "pcs_internal.h"

using namespace pcs;

namespace {

thread_local std::string g_err;

pcs_status fail(pcs_status st, const std::string& msg) {
    g_err = msg;
    return st;
}

#define CUDA_TRY(expr)                                                                      \
    do {                                                                                    \
        cudaError_t e_ = (expr);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return fail(PCS_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));     \
    } while (0)

// PCS_TRACE=1: per-phase host timings on stderr (observability; no effect on results)
void trace(const char* fmt, ...) {
    static const bool on = [] {
        const char* e = std::getenv("PCS_TRACE");
        return e && *e && *e != '0';
    }();
    if (!on) return;
    va_list ap;
    va_start(ap, fmt);
    std::fprintf(stderr, "[pcs] ");
    std::vfprintf(stderr, fmt, ap);
    std::fprintf(stderr, "\n");
    va_end(ap);
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// ----------------------------------------------------------- stats on the host
// Wichura AS 241, same coefficients and Horner order as stats.hpp:19-108
const double kA[8] = {3.3871328727963666080e0, 1.3314166789178437745e2, 1.9715909503065514427e3,
                      1.3731693765509461125e4, 4.5921953931549871457e4, 6.7265770927008700853e4,
                      3.3430575583588128105e4, 2.5090809287301226727e3};
const double kB[8] = {1.0, 4.2313330701600911252e1, 6.8718700749205790830e2, 5.3941960214247511077e3,
                      2.1213794301586595867e4, 3.9307895800092710610e4, 2.8729085735721942674e4,
                      5.2264952788528545610e3};
const double kC[8] = {1.42343711074968357734e0, 4.63033784615654529590e0, 5.76949722146069140550e0,
                      3.64784832476320460504e0, 1.27045825245236838258e0, 2.41780725177450611770e-1,
                      2.27238449892691845833e-2, 7.74545014278341407640e-4};
const double kD[8] = {1.0, 2.05319162663775882187e0, 1.67638483018380384940e0, 6.89767334985100004550e-1,
                      1.48103976427480074590e-1, 1.51986665636164571966e-2, 5.47593808499534494600e-4,
                      1.05075007164441684324e-9};
const double kE[8] = {6.65790464350110377720e0, 5.46378491116411436990e0, 1.78482653991729133580e0,
                      2.96560571828504891230e-1, 2.65321895265761230930e-2, 1.24266094738807843860e-3,
                      2.71155556874348757815e-5, 2.01033439929228813265e-7};
const double kF[8] = {1.0, 5.99832206555887937690e-1, 1.36929880922735805310e-1, 1.48753612908506148525e-2,
                      7.86869131145613259100e-4, 1.84631831751005468180e-5, 1.42151175831644588870e-7,
                      2.04426310338993978564e-15};

double horner7(const double* k, double r) {
    double acc = k[7] * r + k[6];
    for (int d = 5; d >= 0; --d) acc = acc * r + k[d];
    return acc;
}

double normal_quantile(double p) {  // caller guarantees 0 < p < 1
    const double q = p - 0.5;
    if (std::fabs(q) <= 0.425) {
        const double r = 0.180625 - q * q;
        return q * horner7(kA, r) / horner7(kB, r);
    }
    double r = q < 0.0 ? p : 1.0 - p;
    r = std::sqrt(-std::log(r));
    double z;
    if (r <= 5.0) {
        r -= 1.6;
        z = horner7(kC, r) / horner7(kD, r);
    } else {
        r -= 5.0;
        z = horner7(kE, r) / horner7(kF, r);
    }
    return q < 0.0 ? -z : z;
}

pcs_status threshold_tau(double alpha, int m, int ell, double* tau) {
    if (!(alpha > 0.0 && alpha <= 1.0)) return fail(PCS_EINVAL, "threshold_tau: alpha must lie in (0, 1]");
    if (ell < 0) return fail(PCS_EINVAL, "threshold_tau: ell must be >= 0");
    const double dof = static_cast<double>(m) - ell - 3;
    if (dof < 1.0)
        return fail(PCS_ELEVEL, "threshold_tau: need m - ell - 3 >= 1, got m = " + std::to_string(m) +
                                    ", ell = " + std::to_string(ell));
    *tau = normal_quantile(1.0 - alpha / 2.0) / std::sqrt(dof);
    return PCS_OK;
}

// Certain-decision bands around tanh(tau): z <= tau - delta  <=>  |rho| <= tanh(tau - delta).
Thresholds make_thresholds(double tau) {
    Thresholds th;
    th.tau = tau;
    const long double delta = std::max<long double>(1e-9L * tau, 1e-14L);
    const long double tl = (long double)tau - delta, tu = (long double)tau + delta;
    const long double zclamp = 0.5L * std::log((2.0L - 1e-12L) / 1e-12L);  // z at the rho clamp
    if (tl > 0) {
        const long double t = std::tanh(tl);
        th.lo = (double)t;
        th.lo2 = (double)(t * t);
    } else {
        th.lo = -1.0;
        th.lo2 = -1.0;
    }
    if (tu < zclamp - 1e-6L) {
        const long double t = std::tanh(tu);
        th.hi = (double)t;
        th.hi2 = (double)(t * t);
    } else {
        th.hi = INFINITY;
        th.hi2 = INFINITY;
    }
    th.hi2x4 = 4.0 * th.hi2;
    return th;
}

// exact C(n, k) with overflow report (comb.hpp:35-46)
bool binomial_exact(int n, int k, unsigned long long* out) {
    if (k < 0 || k > n) { *out = 0; return true; }
    if (n - k < k) k = n - k;
    unsigned __int128 r = 1;
    for (int i = 1; i <= k; ++i) {
        r = r * (unsigned)(n - k + i) / (unsigned)i;
        if (r > (unsigned __int128)UINT64_MAX) return false;
    }
    *out = (unsigned long long)r;
    return true;
}

}  // namespace

// ================================================================ result
template <class T>
struct NoInitAlloc : std::allocator<T> {
    template <class U>
    struct rebind { using other = NoInitAlloc<U>; };
    NoInitAlloc() = default;
    template <class U>
    NoInitAlloc(const NoInitAlloc<U>&) noexcept {}
    template <class U>
    void construct(U* ptr) noexcept { ::new (static_cast<void*>(ptr)) U; }
    template <class U, class... Args>
    void construct(U* ptr, Args&&... args) { ::new (static_cast<void*>(ptr)) U(std::forward<Args>(args)...); }
};

struct pcs_result {
    int p = 0;
    int W = 0;
    int stop_reason = PCS_STOP_MAX_DEGREE;
    std::vector<pcs_level_stats> levels;
    std::vector<uint32_t> adj;                 // final live bitmask, p x W
    // flattened (a, b, ell, members...) of level >= 1 removals, copied straight from the device pool
    // (default-initialised elements: no zero fill before the copy)
    std::vector<int32_t, NoInitAlloc<int32_t>> recs;
    double device_seconds = 0.0;
    unsigned long long near_total = 0;         // near-threshold decisions of the run (all levels)
    std::vector<NearRec> near;                 // the first kNearCap of them
};

// ================================================================ session
struct pcs_session {
    int p = 0, m = 0, W = 0;
    long long ldc = 0;
    pcs_config cfg{};
    int device = 0, num_sms = 148;
    cudaStream_t st = nullptr;
    cudaEvent_t ev_begin = nullptr, ev_end = nullptr, ev_k0 = nullptr, ev_k1 = nullptr;
    bool own_c = true, own_stream = true;
    double* dC = nullptr;
    uint32_t* dAdj = nullptr;
    int32_t *dDeg = nullptr, *dLow = nullptr, *dOff = nullptr, *dUp = nullptr;
    SnapInfo* dInfo = nullptr;
    Counters* dCnt = nullptr;
    unsigned long long* dPrefix = nullptr;
    int32_t *dNbr = nullptr, *dEid = nullptr;
    unsigned long long* dKdir = nullptr;  // per directed entry: mirror of its edge's key (cuPC-S staging)
    double* dCnbr = nullptr;              // per directed entry: C(i, nbr)
    long long capDir = 0;
    int32_t *dEuA = nullptr, *dEuQa = nullptr, *dEuQb = nullptr;
    unsigned long long* dKeys = nullptr;
    long long capUnd = 0;
    int32_t* dRec = nullptr;       // record pool: per level, count x (3 + ell) ints
    long long capRec = 0, recUsed = 0;
    unsigned long long* dBinom = nullptr;
    size_t capBinom = 0;
    unsigned char* dScratch = nullptr;  // generic-ell per-lane scratch
    long long capScratch = 0;
    unsigned long long* dShardCost = nullptr;  // multi-GPU: per-row / per-edge cost prefix of a pass
    long long capShardCost = 0;
    unsigned long long* dBounds = nullptr;     // multi-GPU: this shard's [first, end) work unit
    // level state
    int ell = -1;
    bool stopped = false, in_level = false;
    double tau_override = NAN;     // pcs_run_level: the caller's threshold instead of threshold_tau
    double* dPinv = nullptr;       // l = 2, 3 pseudo-inverse table (level_set_kernel phase 1)
    NearRec* dNear = nullptr;      // near-threshold list of the run
    unsigned long long* dNearTotal = nullptr;
    long long capPinv = 0;         // doubles
    bool use_pinv = false;
    Counters* hCnt = nullptr;      // pinned copy of the level's counters (deferred level end)
    bool pending_end = false;      // run_session: the level's counters are in flight to hCnt
    double pending_t0 = 0.0;
    int pending_ell = 0;
    bool pending_timing = false;
    bool level0_and = false;       // pcs_run_level at ell = 0: the input graph may be incomplete
    int stop_reason = PCS_STOP_MAX_DEGREE;
    SnapInfo info{};
    Thresholds th{};
    int binom_stride = 0;
    double t_level = 0.0;
    float kernel_ms = 0.f;
    bool kernel_timing = false;
    std::vector<pcs_level_stats> levels;
};

namespace {

// Pinned host slots for the deferred counter copies, recycled across sessions (cudaMallocHost costs
// milliseconds; a run creates and frees a session).
static std::mutex g_pinned_mu;
static std::vector<Counters*> g_pinned_free;
static Counters* pinned_counters() {
    {
        std::lock_guard<std::mutex> g(g_pinned_mu);
        if (!g_pinned_free.empty()) {
            Counters* c = g_pinned_free.back();
            g_pinned_free.pop_back();
            return c;
        }
    }
    Counters* c = nullptr;
    return cudaMallocHost(reinterpret_cast<void**>(&c), sizeof(Counters)) == cudaSuccess ? c : nullptr;
}
static void pinned_counters_release(Counters* c) {
    if (!c) return;
    std::lock_guard<std::mutex> g(g_pinned_mu);
    g_pinned_free.push_back(c);
}

void free_session(pcs_session* s) {
    if (!s) return;
    cudaSetDevice(s->device);
    // stream-ordered frees back into the device pool (no implicit device synchronisation)
    auto rel = [&](void* ptr) {
        if (!ptr) return;
        if (s->st) cudaFreeAsync(ptr, s->st);
        else cudaFree(ptr);
    };
    if (s->own_c) rel(s->dC);
    rel(s->dAdj); rel(s->dDeg); rel(s->dLow); rel(s->dOff); rel(s->dUp);
    rel(s->dInfo); rel(s->dCnt); rel(s->dPrefix); rel(s->dNbr); rel(s->dEid); rel(s->dKdir); rel(s->dCnbr);
    rel(s->dEuA); rel(s->dEuQa); rel(s->dEuQb); rel(s->dKeys); rel(s->dRec);
    rel(s->dBinom);
    rel(s->dScratch);
    rel(s->dShardCost);
    rel(s->dBounds);
    rel(s->dPinv);
    rel(s->dNear);
    rel(s->dNearTotal);
    if (s->st) cudaStreamSynchronize(s->st);
    pinned_counters_release(s->hCnt);
    if (s->ev_begin) cudaEventDestroy(s->ev_begin);
    if (s->ev_end) cudaEventDestroy(s->ev_end);
    if (s->ev_k0) cudaEventDestroy(s->ev_k0);
    if (s->ev_k1) cudaEventDestroy(s->ev_k1);
    if (s->st && s->own_stream) cudaStreamDestroy(s->st);
    delete s;
}

pcs_status validate_config(const pcs_config* c) {  // core.hpp:370-383
    if (!c) return fail(PCS_EINVAL, "null config");
    if (!(c->alpha > 0.0 && c->alpha < 1.0)) return fail(PCS_EINVAL, "SkeletonConfig: alpha must lie in (0, 1)");
    if (c->max_level < -1) return fail(PCS_EINVAL, "SkeletonConfig: max_level must be >= 0");
    if (c->edges_per_unit < 1) return fail(PCS_EINVAL, "SkeletonConfig: edges_per_unit must be >= 1");
    if (c->workers_per_edge < 1) return fail(PCS_EINVAL, "SkeletonConfig: workers_per_edge must be >= 1");
    if (c->set_groups < 1) return fail(PCS_EINVAL, "SkeletonConfig: set_groups must be >= 1");
    if (c->unit_width < 1) return fail(PCS_EINVAL, "SkeletonConfig: unit_width must be >= 1");
    if (c->variant != PCS_VARIANT_SET && c->variant != PCS_VARIANT_EDGE)
        return fail(PCS_EINVAL, "SkeletonConfig: unknown device variant");
    if (c->shard_count < 1 || c->shard_index < 0 || c->shard_index >= c->shard_count)
        return fail(PCS_EINVAL, "SkeletonConfig: bad shard index/count");
    return PCS_OK;
}

cudaError_t dev_malloc(void** ptr, size_t bytes, cudaStream_t st);

template <class T>
pcs_status realloc_dev(pcs_session* s, T** ptr, long long n) {
    if (*ptr) cudaFreeAsync(*ptr, s->st);
    *ptr = nullptr;
    CUDA_TRY(dev_malloc(reinterpret_cast<void**>(ptr), sizeof(T) * (size_t)std::max<long long>(n, 1), s->st));
    return PCS_OK;
}

// Device buffers come from the stream-ordered pool: frees do not synchronise the device and
// the pool keeps its memory between calls (release threshold = unlimited), so repeated runs
// neither pay cudaMalloc/cudaFree latency nor stall on the driver's deferred reclamation.
// A private stream-ordered pool per device: session buffers stay cached across runs (release
// threshold = max) without touching the device's default pool, which the host application (PyTorch,
// ...) may use with its own release policy.
static cudaMemPool_t lib_pool(int device) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    if (device < 0 || device >= 64) return nullptr;
    std::lock_guard<std::mutex> g(mu);
    if (!pools[device]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        cudaMemPool_t pool = nullptr;
        if (cudaMemPoolCreate(&pool, &props) == cudaSuccess) {
            unsigned long long thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            pools[device] = pool;
        }
    }
    return pools[device];
}

cudaError_t dev_malloc(void** ptr, size_t bytes, cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool = lib_pool(dev);
    return pool ? cudaMallocFromPoolAsync(ptr, bytes, pool, st) : cudaMallocAsync(ptr, bytes, st);
}

pcs_status session_alloc(pcs_session* s) {
    const int p = s->p;
    s->W = (p + 31) / 32;
    if (s->cfg.stream) {
        s->st = reinterpret_cast<cudaStream_t>(s->cfg.stream);
        s->own_stream = false;
    } else {
        CUDA_TRY(cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking));
    }
    CUDA_TRY(cudaEventCreate(&s->ev_begin));
    CUDA_TRY(cudaEventCreate(&s->ev_end));
    CUDA_TRY(cudaEventCreate(&s->ev_k0));
    CUDA_TRY(cudaEventCreate(&s->ev_k1));
    CUDA_TRY(dev_malloc(reinterpret_cast<void**>(&s->dAdj), sizeof(uint32_t) * (size_t)p * s->W, s->st));
    CUDA_TRY(dev_malloc(reinterpret_cast<void**>(&s->dDeg), sizeof(int32_t) * (size_t)(p + 1), s->st));
    CUDA_TRY(dev_malloc(reinterpret_cast<void**>(&s->dLow), sizeof(int32_t) * (size_t)(p + 1), s->st));
    CUDA_TRY(dev_malloc(reinterpret_cast<void**>(&s->dOff), sizeof(int32_t) * (size_t)(p + 1), s->st));
    CUDA_TRY(dev_malloc(reinterpret_cast<void**>(&s->dUp), sizeof(int32_t) * (size_t)(p + 1), s->st));
    CUDA_TRY(dev_malloc(reinterpret_cast<void**>(&s->dInfo), sizeof(SnapInfo), s->st));
    CUDA_TRY(dev_malloc(reinterpret_cast<void**>(&s->dCnt), sizeof(Counters), s->st));
    CUDA_TRY(dev_malloc(reinterpret_cast<void**>(&s->dPrefix), sizeof(unsigned long long) * (size_t)(p + 1), s->st));
    CUDA_TRY(dev_malloc(reinterpret_cast<void**>(&s->dNear), sizeof(NearRec) * kNearCap, s->st));
    CUDA_TRY(dev_malloc(reinterpret_cast<void**>(&s->dNearTotal), sizeof(unsigned long long), s->st));
    CUDA_TRY(cudaMemsetAsync(s->dNearTotal, 0, sizeof(unsigned long long), s->st));
    return PCS_OK;
}

pcs_status session_new(int p, int m, const pcs_config* cfg, pcs_session** out) {
    *out = nullptr;
    pcs_status st = validate_config(cfg);
    if (st) return st;
    if (m < 4) return fail(PCS_EINVAL, "run_pc_stable: need at least 4 samples");
    if (p < 2) return fail(PCS_EINVAL, "CorrelationMatrix: need a square matrix, n >= 2");
    if (p > 46340) return fail(PCS_EINVAL, "AdjacencyMatrix: n * n must fit Index (int32), n <= 46340");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(PCS_ECUDA, "no CUDA device available");
    if (cfg->device < 0 || cfg->device >= ndev) return fail(PCS_EINVAL, "bad CUDA device ordinal");
    CUDA_TRY(cudaSetDevice(cfg->device));
    auto* s = new pcs_session();
    s->p = p;
    s->m = m;
    s->cfg = *cfg;
    s->device = cfg->device;
    cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, s->device);
    st = session_alloc(s);
    if (st) { free_session(s); return st; }
    *out = s;
    return PCS_OK;
}

pcs_status check_level_errors(pcs_session* s, const Counters& c) {
    if (c.err_nan) return fail(PCS_ENAN, "fisher_z: rho must lie in (-1, 1)");
    (void)s;
    return PCS_OK;
}

pcs_status build_binomials(pcs_session* s, int ell, int maxw) {
    const int stride = maxw + 1;
    std::vector<unsigned long long> t((size_t)(ell + 1) * stride, 0ull);
    for (int n = 0; n < stride; ++n) t[n] = 1ull;
    for (int k = 1; k <= ell; ++k)
        for (int n = 1; n < stride; ++n) {
            const unsigned long long a = t[(size_t)(k - 1) * stride + n - 1], b = t[(size_t)k * stride + n - 1];
            t[(size_t)k * stride + n] = (a > UINT64_MAX - b) ? UINT64_MAX : a + b;
        }
    if (t.size() > s->capBinom) {
        pcs_status st = realloc_dev(s, &s->dBinom, (long long)t.size());
        if (st) return st;
        s->capBinom = t.size();
    }
    CUDA_TRY(cudaMemcpyAsync(s->dBinom, t.data(), sizeof(unsigned long long) * t.size(), cudaMemcpyHostToDevice,
                             s->st));
    s->binom_stride = stride;
    return PCS_OK;
}

// PCS_MERGE_PASSES=0: cuPC-S levels >= 2 as two direction passes (as the cuPC-E and generic-ell
// kernels run); default 1 (one sweep over both directions).  No effect on results.
bool merge_passes() {
    static const bool on = [] {
        const char* e = std::getenv("PCS_MERGE_PASSES");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

LevelArgs level_args(pcs_session* s) {
    LevelArgs A{};
    A.C = s->dC;
    A.ldc = s->ldc;
    A.p = s->p;
    A.ell = s->ell;
    A.off = s->dOff;
    A.nbr = s->dNbr;
    A.lowcnt = s->dLow;
    A.upoff = s->dUp;
    A.eid = s->dEid;
    A.eu_a = s->dEuA;
    A.eu_qa = s->dEuQa;
    A.eu_qb = s->dEuQb;
    A.keys = s->dKeys;
    A.kdir = s->dKdir;
    A.cnbr = s->dCnbr;
    A.pinv_table = s->use_pinv ? s->dPinv : nullptr;
    A.near_rec = s->dNear;
    A.near_total = s->dNearTotal;
    A.binom.t = s->dBinom;
    A.binom.stride = s->binom_stride;
    A.th = s->th;
    A.cnt = s->dCnt;
    return A;
}

void stop(pcs_session* s, int reason) {
    s->stopped = true;
    s->stop_reason = reason;
}

}  // namespace

namespace pcs {
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace pcs

// ================================================================ C ABI
extern "C" {

const char* pcs_version(void) { return "pcstable_b200 0.2 (sm_100a, abi 2)"; }
const char* pcs_last_error(void) { return g_err.c_str(); }

void pcs_config_default(pcs_config* cfg) {  // core.hpp:357-368
    std::memset(cfg, 0, sizeof *cfg);
    cfg->alpha = 0.05;
    cfg->max_level = -1;
    cfg->variant = PCS_VARIANT_SET;
    cfg->edges_per_unit = 2;
    cfg->workers_per_edge = 32;
    cfg->set_groups = 2;
    cfg->unit_width = 64;
    cfg->device = 0;
    cfg->shard_index = 0;
    cfg->shard_count = 1;
}

pcs_status pcs_threshold_tau(double alpha, int32_t m, int32_t ell, double* tau) {
    return threshold_tau(alpha, m, ell, tau);
}

static pcs_status session_upload_corr(pcs_session* s, const double* c) {
    s->ldc = (s->p + 3) / 4 * 4;
    CUDA_TRY(dev_malloc(reinterpret_cast<void**>(&s->dC), sizeof(double) * (size_t)s->p * s->ldc, s->st));
    CUDA_TRY(cudaEventRecord(s->ev_begin, s->st));
    CUDA_TRY(cudaMemcpy2DAsync(s->dC, sizeof(double) * s->ldc, c, sizeof(double) * s->p, sizeof(double) * s->p, s->p,
                               cudaMemcpyHostToDevice, s->st));
    int* dErr = nullptr;
    CUDA_TRY(dev_malloc(reinterpret_cast<void**>(&dErr), sizeof(int), s->st));
    CUDA_TRY(cudaMemsetAsync(dErr, 0, sizeof(int), s->st));
    launch_normalize_corr(s->dC, s->ldc, s->p, dErr, s->st);
    int err = 0;
    CUDA_TRY(cudaMemcpyAsync(&err, dErr, sizeof(int), cudaMemcpyDeviceToHost, s->st));
    cudaFreeAsync(dErr, s->st);
    CUDA_TRY(cudaStreamSynchronize(s->st));
    if (err & 2) return fail(PCS_EINVAL, "CorrelationMatrix: diagonal must be 1");
    if (err & 4) return fail(PCS_EINVAL, "CorrelationMatrix: matrix must be symmetric");
    if (err & 8) return fail(PCS_EINVAL, "CorrelationMatrix: entries must lie in [-1, 1]");
    return PCS_OK;
}

pcs_status pcs_session_create(const double* c, int32_t p, int32_t m, const pcs_config* cfg, pcs_session** out) {
    pcs_session* s = nullptr;
    pcs_status st = session_new(p, m, cfg, &s);
    if (st) return st;
    st = session_upload_corr(s, c);
    if (st) { free_session(s); return st; }
    *out = s;
    return PCS_OK;
}

pcs_status pcs_session_create_device(const double* d_c, int64_t ldc, int32_t p, int32_t m, const pcs_config* cfg,
                                     pcs_session** out) {
    if (!d_c) return fail(PCS_EINVAL, "CorrelationMatrix: null device pointer");
    if (ldc < p) return fail(PCS_EINVAL, "CorrelationMatrix: leading dimension must be >= n");
    if ((long long)p * ldc >= (1ll << 31)) return fail(PCS_EUNSUPPORTED, "CorrelationMatrix: n * ldc must be < 2^31");
    pcs_session* s = nullptr;
    pcs_status st = session_new(p, m, cfg, &s);
    if (st) return st;
    // The kernels need the CorrelationMatrix invariants exactly (core.hpp:73-95): unit diagonal, bitwise
    // symmetry, finite entries in [-1, 1].  A caller buffer that already has them (every matrix this
    // library builds) is used in place; anything else is copied into a session buffer and run through
    // the constructor's validation + symmetrisation, like session_upload_corr.
    int* dFlag = nullptr;
    int flag = 0;
    CUDA_TRY(dev_malloc(reinterpret_cast<void**>(&dFlag), sizeof(int), s->st));
    CUDA_TRY(cudaMemsetAsync(dFlag, 0, sizeof(int), s->st));
    launch_check_corr(d_c, ldc, p, dFlag, s->st);
    CUDA_TRY(cudaMemcpyAsync(&flag, dFlag, sizeof(int), cudaMemcpyDeviceToHost, s->st));
    cudaFreeAsync(dFlag, s->st);
    CUDA_TRY(cudaStreamSynchronize(s->st));
    if (!flag) {
        s->own_c = false;
        s->dC = const_cast<double*>(d_c);
        s->ldc = ldc;
        cudaEventRecord(s->ev_begin, s->st);
        *out = s;
        return PCS_OK;
    }
    s->ldc = (p + 3) / 4 * 4;
    st = [&]() -> pcs_status {
        CUDA_TRY(dev_malloc(reinterpret_cast<void**>(&s->dC), sizeof(double) * (size_t)p * s->ldc, s->st));
        CUDA_TRY(cudaEventRecord(s->ev_begin, s->st));
        CUDA_TRY(cudaMemcpy2DAsync(s->dC, sizeof(double) * s->ldc, d_c, sizeof(double) * ldc, sizeof(double) * p, p,
                                   cudaMemcpyDeviceToDevice, s->st));
        int* dErr = nullptr;
        CUDA_TRY(dev_malloc(reinterpret_cast<void**>(&dErr), sizeof(int), s->st));
        CUDA_TRY(cudaMemsetAsync(dErr, 0, sizeof(int), s->st));
        launch_normalize_corr(s->dC, s->ldc, p, dErr, s->st);
        int err = 0;
        CUDA_TRY(cudaMemcpyAsync(&err, dErr, sizeof(int), cudaMemcpyDeviceToHost, s->st));
        cudaFreeAsync(dErr, s->st);
        CUDA_TRY(cudaStreamSynchronize(s->st));
        if (err & 2) return fail(PCS_EINVAL, "CorrelationMatrix: diagonal must be 1");
        if (err & 4) return fail(PCS_EINVAL, "CorrelationMatrix: matrix must be symmetric");
        if (err & 8) return fail(PCS_EINVAL, "CorrelationMatrix: entries must lie in [-1, 1]");
        return PCS_OK;
    }();
    if (st) { free_session(s); return st; }
    *out = s;
    return PCS_OK;
}

static pcs_status finalize_pending(pcs_session* s);
static pcs_status maybe_pinv_table(pcs_session* s, int ell);


pcs_status pcs_session_level_begin(pcs_session* s, int32_t* running, int32_t* ell_out, int64_t* num_keys) {
    if (!s) return fail(PCS_EINVAL, "null session");
    CUDA_TRY(cudaSetDevice(s->device));
    *running = 0;
    *num_keys = 0;
    if (s->stopped) { *ell_out = s->ell; return finalize_pending(s); }
    if (s->in_level) return fail(PCS_EINVAL, "level already started");
    const int ell = s->ell + 1;
    *ell_out = ell;
    if (s->cfg.max_level >= 0 && ell > s->cfg.max_level) { stop(s, PCS_STOP_LEVEL_CAP); return finalize_pending(s); }
    double tau;
    pcs_status st = PCS_OK;
    if (!std::isnan(s->tau_override)) tau = s->tau_override;
    else {
        st = threshold_tau(s->cfg.alpha, s->m, ell, &tau);
        if (st == PCS_ELEVEL) { stop(s, PCS_STOP_SAMPLE_SIZE); return finalize_pending(s); }
        if (st) return st;
    }
    s->ell = ell;
    s->th = make_thresholds(tau);
    s->t_level = now_s();
    s->kernel_timing = false;
    CUDA_TRY(cudaMemsetAsync(s->dCnt, 0, sizeof(Counters), s->st));
    if (ell == 0) {
        CUDA_TRY(cudaEventRecord(s->ev_k0, s->st));
        launch_level0(s->dC, s->ldc, s->p, s->W, s->dAdj, s->th, s->dCnt, s->st, s->level0_and, s->dNear,
                      s->dNearTotal);
        CUDA_TRY(cudaEventRecord(s->ev_k1, s->st));
        s->kernel_timing = true;
        CUDA_TRY(cudaGetLastError());
        s->in_level = true;
        *running = 1;
        return PCS_OK;
    }
    // snapshot of the live graph (compact(), core.hpp:227-239)
    launch_snapshot_degrees(s->dAdj, s->p, s->W, s->dDeg, s->dLow, s->st);
    launch_snapshot_scan(s->dDeg, s->dLow, s->p, s->dOff, s->dUp, s->dInfo, s->st);
    CUDA_TRY(cudaMemcpyAsync(&s->info, s->dInfo, sizeof(SnapInfo), cudaMemcpyDeviceToHost, s->st));
    CUDA_TRY(cudaStreamSynchronize(s->st));
    if ((st = finalize_pending(s))) return st;  // the previous level's statistics (record pool offset)
    const int maxw = s->info.max_width;
    if (maxw - 1 < ell) {  // skeleton.hpp:370-373 (level not recorded)
        s->ell = ell - 1;
        stop(s, PCS_STOP_MAX_DEGREE);
        return PCS_OK;
    }
    unsigned long long tmp;
    if (!binomial_exact(maxw - 1, ell, &tmp)) return fail(PCS_EOVERFLOW, "binomial: C(n, k) exceeds 64 bits");
    if (!binomial_exact(maxw, ell, &tmp) || tmp >= (1ull << 62))
        return fail(PCS_EUNSUPPORTED, "level " + std::to_string(ell) + ": C(" + std::to_string(maxw) + ", " +
                                          std::to_string(ell) + ") conditioning sets per row exceed 2^62");
    if (ell > kMaxRtLevel)
        return fail(PCS_EUNSUPPORTED, "conditioning level " + std::to_string(ell) + " > " +
                                          std::to_string(kMaxRtLevel) + " not supported on the device");
    if (ell > kMaxTemplLevel) {
        const long long need = level_rt_scratch_bytes(ell, s->num_sms, nullptr);
        if (need > s->capScratch) {
            if ((st = realloc_dev(s, &s->dScratch, need))) return st;
            s->capScratch = need;
        }
    }
    if (s->info.e_dir > s->capDir) {
        if ((st = realloc_dev(s, &s->dNbr, s->info.e_dir))) return st;
        if ((st = realloc_dev(s, &s->dEid, s->info.e_dir))) return st;
        if ((st = realloc_dev(s, &s->dKdir, s->info.e_dir))) return st;
        if ((st = realloc_dev(s, &s->dCnbr, s->info.e_dir + 2))) return st;  // +2: the staged cuPC-E bulk copy's even-aligned superset
        s->capDir = s->info.e_dir;
    }
    if (s->info.e_und > s->capUnd) {
        if ((st = realloc_dev(s, &s->dEuA, s->info.e_und))) return st;
        if ((st = realloc_dev(s, &s->dEuQa, s->info.e_und))) return st;
        if ((st = realloc_dev(s, &s->dEuQb, s->info.e_und))) return st;
        if ((st = realloc_dev(s, &s->dKeys, s->info.e_und))) return st;
        s->capUnd = s->info.e_und;
    }
    {
        const long long need = s->recUsed + s->info.e_und * (3 + ell);
        if (need > s->capRec) {  // grow the record pool, keeping earlier levels' records
            const long long cap = std::max(need, s->capRec * 3 / 2);
            int32_t* np = nullptr;
            CUDA_TRY(dev_malloc(reinterpret_cast<void**>(&np), sizeof(int32_t) * (size_t)cap, s->st));
            if (s->recUsed)
                CUDA_TRY(cudaMemcpyAsync(np, s->dRec, sizeof(int32_t) * (size_t)s->recUsed, cudaMemcpyDeviceToDevice,
                                         s->st));
            if (s->dRec) cudaFreeAsync(s->dRec, s->st);
            s->dRec = np;
            s->capRec = cap;
        }
    }
    if ((st = build_binomials(s, ell, maxw))) return st;
    if ((st = maybe_pinv_table(s, ell))) return st;
    launch_snapshot_fill(s->dAdj, s->p, s->W, s->dOff, s->dNbr, s->st);
    LevelArgs A = level_args(s);
    launch_edge_index(A, s->dEid, s->dEuA, s->dEuQa, s->dEuQb, ell >= 2 ? s->dCnbr : nullptr, s->st);
    launch_fill_keys(s->dKeys, s->info.e_und, s->st);
    CUDA_TRY(cudaGetLastError());
    s->in_level = true;
    *running = 1;
    *num_keys = s->info.e_und;
    return PCS_OK;
}

// PCS_L1_TILE: 0 never, 1 always, unset/other: when the level-1 snapshot is dense (at least half of all
// pairs live), where the TMA-tiled sweep (level1t.cu) tests every (i, j, k) of a 32 x 64 x 32 tile from
// shared memory.  Sparse snapshots keep level1_kernel (a tile would mostly test absent pairs).
static bool level1_tile(const pcs_session* s) {
    static const int mode = [] {
        const char* e = std::getenv("PCS_L1_TILE");
        return e ? std::atoi(e) : -1;
    }();
    if (s->ell != 1 || mode == 0) return false;
    if (mode == 1) return true;
    // measured (profiles/r2s03_l1tile.log): 2.2-4.8x faster than level1_kernel at p = 5000-20000 (C beyond
    // L2), 1.3x slower at p = 1643 (C3: L2-resident, 73% dense, most pairs separate within a few k)
    const double pairs = (double)s->p * (double)(s->p - 1);
    return s->p >= 2048 && (double)s->info.e_dir >= 0.5 * pairs;
}

// PCS_PINV_TABLE: 0 never, 1 whenever it fits, unset/other: when the level's (row, set) pairs outnumber
// the vertex l-subsets 4:1 and the table takes at most a quarter of the free device memory (32 GB cap).
// C2: level 2 3.8e7 pairs / 5.0e5 subsets, level 3 2.7e9 / 1.7e8 (13 GB table).
static pcs_status maybe_pinv_table(pcs_session* s, int ell) {
    static const int mode = [] {
        const char* e = std::getenv("PCS_PINV_TABLE");
        return e ? std::atoi(e) : -1;
    }();
    s->use_pinv = false;
    if (mode == 0 || (ell != 2 && ell != 3)) return PCS_OK;  // both variants (cuPC-E: one lookup per test)
    const double n = (double)s->p;
    const double subsets = ell == 2 ? n * (n - 1) / 2 : n * (n - 1) * (n - 2) / 6;
    const double pairs = ell == 2 ? s->info.sets2 : s->info.sets3;
    const double doubles = subsets * (double)pinv_table_stride(ell);
    if ((mode != 1 && pairs < 4.0 * subsets) || doubles > 32e9 / 8.0) return PCS_OK;
    if ((long long)doubles > s->capPinv) {  // a new allocation: leave 3/4 of the free memory alone
        size_t free_b = 0, total_b = 0;
        cudaMemGetInfo(&free_b, &total_b);
        if (doubles > 0.25 * (double)free_b / 8.0) return PCS_OK;
    }
    if ((long long)doubles > s->capPinv) {
        pcs_status st = realloc_dev(s, &s->dPinv, (long long)doubles);
        if (st) return st;
        s->capPinv = (long long)doubles;
    }
    if (launch_pinv_table(s->dC, s->ldc, s->p, ell, s->dPinv, s->st)) return fail(PCS_EUNSUPPORTED, "pinv table");
    s->use_pinv = true;
    return PCS_OK;
}

static bool merged_level(const pcs_session* s) {
    // the generic-ell kernel (l > 8) serves both variants and merges its passes too
    return (s->cfg.variant == PCS_VARIANT_SET && s->ell >= 2 && s->ell <= kMaxTemplLevel && merge_passes()) ||
           (s->ell > kMaxTemplLevel && merge_passes()) || level1_tile(s);
}

pcs_status pcs_session_level_passes(pcs_session* s, int32_t* passes) {
    if (!s || !passes) return fail(PCS_EINVAL, "null argument");
    *passes = (s->in_level && merged_level(s)) ? 1 : 2;
    return PCS_OK;
}

pcs_status pcs_session_level_pass(pcs_session* s, int32_t pass) {
    if (!s || !s->in_level) return fail(PCS_EINVAL, "no level in progress");
    if (pass != 0 && pass != 1) return fail(PCS_EINVAL, "pass must be 0 or 1");
    if (s->ell == 0) return PCS_OK;
    // cuPC-S with a register-template kernel tests both directions in ONE sweep (pass 0 does it as
    // "pass 2"; pass 1 has nothing left): every set's pseudo-inverse is computed once per level instead
    // of once per direction, at the price of testing direction 1 of edges that direction 0 separates
    // in the same level (their keys stay the direction-0 ones: MIN).  Results are unchanged.
    const bool merged = merged_level(s);
    if (merged && pass == 1) return PCS_OK;
    const int kpass = merged ? 2 : pass;
    CUDA_TRY(cudaSetDevice(s->device));
    LevelArgs A = level_args(s);
    const int shard = s->cfg.shard_index, nsh = s->cfg.shard_count;
    if (!s->kernel_timing) { CUDA_TRY(cudaEventRecord(s->ev_k0, s->st)); }
    // Multi-GPU: every rank derives the same cost-weighted split of the pass's work units (contiguous
    // ranges, so a row's early exits stay on one GPU); units are not equally expensive (a band of row i
    // tests its ntar targets, which differ by orders of magnitude between rows), so splitting by unit
    // count would leave the ranks up to ~1.8x apart at 8 GPUs (C2 level 3).
    pcs_status st = PCS_OK;
    if (nsh > 1) {
        const long long need = std::max<long long>(s->p + 1, s->info.e_und + 1);
        if (need > s->capShardCost) {
            if ((st = realloc_dev(s, &s->dShardCost, need))) return st;
            s->capShardCost = need;
        }
        if (!s->dBounds && (st = realloc_dev(s, &s->dBounds, 2))) return st;
    }
    if (level1_tile(s)) {
        // multi-GPU: cyclic 32-row blocks (no host round trip for bounds)
        if (launch_level1_tile(A, s->dAdj, s->W, shard, nsh, s->st))
            return fail(PCS_ECUDA, "level-1 tile kernel: tensor map / launch failed");
    } else if (s->ell == 1) {
        // level1_kernel: cyclic tiles of 128 targets over the ranks; the tile total stays on the device
        launch_row_work(A, pass, s->cfg.variant, 0, s->p, s->dPrefix, s->st);
        launch_level1(A, pass, s->dPrefix, 0, ~0ull, (unsigned long long)(s->info.e_dir / 128 + s->p), shard, nsh,
                      s->st);
    } else if (s->cfg.variant == PCS_VARIANT_SET || s->ell == 1 || s->ell > kMaxTemplLevel) {
        unsigned long long u0 = 0, u1 = 0;
        if (nsh > 1) {
            unsigned long long b[2] = {0, 0};
            launch_row_work_sharded(A, kpass, s->cfg.variant, s->dPrefix, s->dShardCost, shard, nsh, s->dBounds, s->st);
            CUDA_TRY(cudaMemcpyAsync(b, s->dBounds, sizeof(b), cudaMemcpyDeviceToHost, s->st));
            CUDA_TRY(cudaStreamSynchronize(s->st));
            u0 = b[0];
            u1 = b[1];
        } else {
            // the kernels read the unit total (prefix[p]) on the device: no host round trip
            launch_row_work(A, kpass, s->cfg.variant, 0, s->p, s->dPrefix, s->st);
            u1 = ~0ull;
        }
        if (u1 > u0) {
            if (s->ell > kMaxTemplLevel) {
                CUDA_TRY(cudaMemsetAsync(&s->dCnt->units[pass], 0, sizeof(unsigned long long), s->st));
                if (launch_level_set_rt(A, kpass, s->dPrefix, u0, u1, s->num_sms, s->dScratch, s->st))
                    return fail(PCS_EUNSUPPORTED, "level not supported by the generic set kernel");
            } else {
                launch_refresh_kdir(A, s->info.e_dir, s->st);
                if (launch_level_set(A, kpass, s->dPrefix, u0, u1, s->num_sms, s->st))
                    return fail(PCS_EUNSUPPORTED, "level not supported by the set kernel");
            }
        }
    } else {
        const long long E = s->info.e_und;
        long long e0 = 0, e1 = E;
        if (nsh > 1) {  // cost-weighted: an edge's pass costs C(w - 1, ell) tests in the tested row
            unsigned long long b[2] = {0, 0};
            launch_edge_bounds(A, pass, E, s->dShardCost, shard, nsh, s->dBounds, s->st);
            CUDA_TRY(cudaMemcpyAsync(b, s->dBounds, sizeof(b), cudaMemcpyDeviceToHost, s->st));
            CUDA_TRY(cudaStreamSynchronize(s->st));
            e0 = (long long)b[0];
            e1 = (long long)b[1];
        }
        if (e1 > e0 && launch_level_edge(A, pass, e0, e1, s->info.max_width, s->num_sms, s->st))
            return fail(PCS_EUNSUPPORTED, "level not supported by the edge kernel");
    }
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(s->ev_k1, s->st));
    s->kernel_timing = true;
    return PCS_OK;
}

pcs_status pcs_session_snapshot(pcs_session* s, int32_t* offsets, int32_t* indices) {
    if (!s || !s->in_level || s->ell < 1) return fail(PCS_EINVAL, "no level >= 1 in progress");
    CUDA_TRY(cudaSetDevice(s->device));
    CUDA_TRY(cudaMemcpyAsync(offsets, s->dOff, sizeof(int32_t) * (size_t)(s->p + 1), cudaMemcpyDeviceToHost, s->st));
    if (indices && s->info.e_dir > 0)
        CUDA_TRY(cudaMemcpyAsync(indices, s->dNbr, sizeof(int32_t) * (size_t)s->info.e_dir, cudaMemcpyDeviceToHost,
                                 s->st));
    CUDA_TRY(cudaStreamSynchronize(s->st));
    return PCS_OK;
}

unsigned long long pcs_kernel_launches(void) { return g_kernel_launches.load(std::memory_order_relaxed); }

pcs_status pcs_session_set_shard(pcs_session* s, int32_t shard_index, int32_t shard_count) {
    if (!s || shard_count < 1 || shard_index < 0 || shard_index >= shard_count)
        return fail(PCS_EINVAL, "bad shard index/count");
    s->cfg.shard_index = shard_index;
    s->cfg.shard_count = shard_count;
    return PCS_OK;
}

pcs_status pcs_session_keys(pcs_session* s, void** device_ptr, int64_t* count) {
    if (!s) return fail(PCS_EINVAL, "null session");
    *device_ptr = s->dKeys;
    *count = (s->in_level && s->ell >= 1) ? s->info.e_und : 0;
    CUDA_TRY(cudaStreamSynchronize(s->st));  // keys are complete when the caller reduces them
    return PCS_OK;
}

// LevelStats from the level's counters (after the stream has passed the counter copy)
static pcs_status level_stats_from(pcs_session* s, const Counters& c, double t_level, int ell, bool timing) {
    CUDA_TRY(cudaGetLastError());
    pcs_status st = check_level_errors(s, c);
    if (st) return st;
    pcs_level_stats L{};
    L.level = ell;
    if (ell == 0) {
        const unsigned long long p = (unsigned long long)s->p;
        L.ci_tests = p * (p - 1) / 2;  // skeleton.hpp:274-276
        L.pseudo_inverses = 0;
        L.device_ci_tests = L.ci_tests;
        L.device_near_threshold = c.near;
    } else {
        L.ci_tests = c.ci_serial;
        L.pseudo_inverses = c.ci_serial;  // skeleton.hpp:151-152
        L.device_ci_tests = c.gpu_tests;
        L.device_pseudo_inverses = c.gpu_pinv;
        L.device_exact_tests = c.gpu_exact;
        L.device_near_threshold = c.near;
        if (c.rec_count) {
            s->recUsed += (long long)c.rec_count * (3 + ell);
        }
    }
    L.edges_removed = c.removed;
    if (timing) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, s->ev_k0, s->ev_k1);
        L.kernel_ms = ms;
    }
    L.elapsed_s = now_s() - t_level;
    if (c.dbg[0])
        trace("level %d filter: %llu steps, %llu candidate tests, %llu steps with a candidate", ell,
              (unsigned long long)c.dbg[0], (unsigned long long)c.dbg[1], (unsigned long long)c.dbg[2]);
    trace("level %d: %.3f ms host (kernels %.3f ms), %llu serial / %llu device tests, %llu removed", L.level,
          L.elapsed_s * 1e3, L.kernel_ms, (unsigned long long)L.ci_tests, (unsigned long long)L.device_ci_tests,
          (unsigned long long)L.edges_removed);
    s->levels.push_back(L);
    return PCS_OK;
}

// the deferred level end of run_session: the counters were copied to pinned memory asynchronously;
// this runs after the stream's next synchronisation (level_begin's snapshot summary or finish)
static pcs_status finalize_pending(pcs_session* s) {
    if (!s->pending_end) return PCS_OK;
    CUDA_TRY(cudaStreamSynchronize(s->st));  // usually already passed
    s->pending_end = false;
    return level_stats_from(s, *s->hCnt, s->pending_t0, s->pending_ell, s->pending_timing);
}

// deferred = true (run_session only): commit + counter copy are enqueued and the level's statistics are
// read at the next synchronisation point, so a level costs one host round trip (the snapshot summary)
static pcs_status level_end_impl(pcs_session* s, bool deferred) {
    if (!s || !s->in_level) return fail(PCS_EINVAL, "no level in progress");
    CUDA_TRY(cudaSetDevice(s->device));
    LevelArgs A = level_args(s);
    if (s->ell >= 1) launch_commit(A, s->dAdj, s->W, s->info.e_und, s->dRec + s->recUsed, s->st);
    if (s->ell >= 2) launch_near_fixup(A, s->st);  // before the next snapshot replaces off[]
    s->in_level = false;
    if (deferred) {
        if (!s->hCnt && !(s->hCnt = pinned_counters())) return fail(PCS_ENOMEM, "pinned host memory");
        CUDA_TRY(cudaMemcpyAsync(s->hCnt, s->dCnt, sizeof(Counters), cudaMemcpyDeviceToHost, s->st));
        s->pending_end = true;
        s->pending_t0 = s->t_level;
        s->pending_ell = s->ell;
        s->pending_timing = s->kernel_timing;
        return PCS_OK;
    }
    Counters c{};
    CUDA_TRY(cudaMemcpyAsync(&c, s->dCnt, sizeof(Counters), cudaMemcpyDeviceToHost, s->st));
    CUDA_TRY(cudaStreamSynchronize(s->st));
    return level_stats_from(s, c, s->t_level, s->ell, s->kernel_timing);
}

pcs_status pcs_session_level_end(pcs_session* s) { return level_end_impl(s, false); }

pcs_status pcs_session_finish(pcs_session* s, pcs_result** out) {
    if (!s) return fail(PCS_EINVAL, "null session");
    CUDA_TRY(cudaSetDevice(s->device));
    if (pcs_status st = finalize_pending(s)) return st;
    auto* r = new pcs_result();
    r->p = s->p;
    r->W = s->W;
    r->stop_reason = s->stop_reason;
    r->levels = s->levels;
    if (s->recUsed) {  // the pool already holds (a, b, ell, members...) records, level after level
        r->recs.resize((size_t)s->recUsed);
        CUDA_TRY(cudaMemcpyAsync(r->recs.data(), s->dRec, sizeof(int32_t) * r->recs.size(), cudaMemcpyDeviceToHost,
                                 s->st));
    }
    CUDA_TRY(cudaMemcpyAsync(&r->near_total, s->dNearTotal, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s->st));
    CUDA_TRY(cudaStreamSynchronize(s->st));
    if (r->near_total) {
        r->near.resize((size_t)std::min<unsigned long long>(r->near_total, kNearCap));
        CUDA_TRY(cudaMemcpyAsync(r->near.data(), s->dNear, sizeof(NearRec) * r->near.size(), cudaMemcpyDeviceToHost, s->st));
    }
    r->adj.resize((size_t)s->p * s->W);
    CUDA_TRY(cudaMemcpyAsync(r->adj.data(), s->dAdj, sizeof(uint32_t) * r->adj.size(), cudaMemcpyDeviceToHost, s->st));
    CUDA_TRY(cudaEventRecord(s->ev_end, s->st));
    CUDA_TRY(cudaStreamSynchronize(s->st));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, s->ev_begin, s->ev_end);
    r->device_seconds = ms * 1e-3;
    *out = r;
    return PCS_OK;
}

void pcs_session_free(pcs_session* s) { free_session(s); }

static pcs_status run_session(pcs_session* s, pcs_result** out) {
    double tb = 0, tp = 0, te = 0;  // PCS_TRACE: host time in level_begin / passes / level_end
    for (;;) {
        int32_t running = 0, ell = 0;
        int64_t nk = 0;
        double t = now_s();
        pcs_status st = pcs_session_level_begin(s, &running, &ell, &nk);
        tb += now_s() - t;
        if (st) return st;
        if (!running) break;
        t = now_s();
        if ((st = pcs_session_level_pass(s, 0))) return st;
        if ((st = pcs_session_level_pass(s, 1))) return st;
        tp += now_s() - t;
        t = now_s();
        if ((st = level_end_impl(s, true))) return st;
        te += now_s() - t;
    }
    const double t = now_s();
    pcs_status st = pcs_session_finish(s, out);
    trace("run_session: level_begin %.2f ms, passes %.2f ms, level_end %.2f ms, finish %.2f ms", tb * 1e3, tp * 1e3,
          te * 1e3, (now_s() - t) * 1e3);
    return st;
}

pcs_status pcs_run_pc_stable(const double* c, int32_t p, int32_t m, const pcs_config* cfg, pcs_result** out) {
    *out = nullptr;
    pcs_session* s = nullptr;
    pcs_status st = pcs_session_create(c, p, m, cfg, &s);
    if (st) return st;
    st = run_session(s, out);
    free_session(s);
    return st;
}

// One level on a caller-given live graph (run_level_zero / run_level_serial / run_level_edge_parallel /
// run_level_set_shared, skeleton.hpp:262-333): the session starts at that graph instead of the complete
// one, takes the caller's tau, and runs exactly level ell.
pcs_status pcs_run_level(const double* c, int32_t p, int32_t ell, double tau, const pcs_config* cfg,
                         uint8_t* graph_cells, pcs_result** out) {
    *out = nullptr;
    if (!c || !graph_cells || !cfg) return fail(PCS_EINVAL, "null argument");
    if (ell < 0) return fail(PCS_EINVAL, "run_level: ell must be >= 0");
    if (!(tau >= 0.0)) return fail(PCS_EINVAL, "run_level: tau must be >= 0");
    pcs_config c2 = *cfg;
    c2.max_level = -1;
    pcs_session* s = nullptr;
    pcs_status st = pcs_session_create(c, p, 1 << 30, &c2, &s);
    if (st) return st;
    st = [&]() -> pcs_status {
        std::vector<uint32_t> bits((size_t)p * s->W, 0u);
        for (int i = 0; i < p; ++i)
            for (int j = 0; j < p; ++j) {
                if (i == j) continue;
                const uint8_t a = graph_cells[(size_t)i * p + j], b = graph_cells[(size_t)j * p + i];
                if (a != b) return fail(PCS_EINVAL, "AdjacencyMatrix: graph must be symmetric");
                if (a) bits[(size_t)i * s->W + j / 32] |= 1u << (j % 32);
            }
        CUDA_TRY(cudaMemcpyAsync(s->dAdj, bits.data(), sizeof(uint32_t) * bits.size(), cudaMemcpyHostToDevice, s->st));
        s->tau_override = tau;
        s->level0_and = true;
        s->ell = ell - 1;
        int32_t running = 0, e = 0;
        int64_t nk = 0;
        pcs_status q = pcs_session_level_begin(s, &running, &e, &nk);
        if (q) return q;
        if (running) {
            if ((q = pcs_session_level_pass(s, 0))) return q;
            if ((q = pcs_session_level_pass(s, 1))) return q;
            if ((q = pcs_session_level_end(s))) return q;
        }
        if ((q = pcs_session_finish(s, out))) return q;
        (*out)->stop_reason = PCS_STOP_LEVEL_CAP;
        const int W = (*out)->W;
        for (int i = 0; i < p; ++i)
            for (int j = 0; j < p; ++j)
                graph_cells[(size_t)i * p + j] = (uint8_t)(((*out)->adj[(size_t)i * W + j / 32] >> (j % 32)) & 1u);
        return PCS_OK;
    }();
    free_session(s);
    if (st && *out) { pcs_result_free(*out); *out = nullptr; }
    return st;
}

pcs_status pcs_run_pc_stable_device(const double* d_c, int64_t ldc, int32_t p, int32_t m, const pcs_config* cfg,
                                    pcs_result** out) {
    *out = nullptr;
    pcs_session* s = nullptr;
    pcs_status st = pcs_session_create_device(d_c, ldc, p, m, cfg, &s);
    if (st) return st;
    st = run_session(s, out);
    free_session(s);
    return st;
}

static pcs_status correlation_device(cudaStream_t stream, const double* x, int m, int p, double* dC, long long ldc,
                                     int32_t* zero_var_col, bool x_on_device = false, int r0 = -1, int r1 = -1) {
    if (m < 4) return fail(PCS_EINVAL, "DataMatrix: need at least 4 samples, got " + std::to_string(m));
    if (p < 2) return fail(PCS_EINVAL, "DataMatrix: need at least 2 variables, got " + std::to_string(p));
    const int ldk = (m + 31) / 32 * 32;
    const long long ldg = (p + 3) / 4 * 4;
    double *dX = nullptr, *dXc = nullptr, *dG = nullptr, *dMean = nullptr;
    int* dErr = nullptr;
    pcs_status st = PCS_OK;
    auto cleanup = [&]() {
        for (void* q : {(void*)dX, (void*)dXc, (void*)dG, (void*)dMean, (void*)dErr})
            if (q) cudaFreeAsync(q, stream);
    };
    auto alloc = [&](auto** ptr, size_t bytes) {
        return dev_malloc(reinterpret_cast<void**>(ptr), bytes, stream) != cudaSuccess;
    };
    if ((!x_on_device && alloc(&dX, sizeof(double) * (size_t)m * p)) || alloc(&dXc, sizeof(double) * (size_t)p * ldk) ||
        alloc(&dG, sizeof(double) * (size_t)(r0 >= 0 ? std::min<long long>(p, (long long)(r1 - r0) + 256) : p) * ldg) ||
        alloc(&dMean, sizeof(double) * (size_t)p) ||
        alloc(&dErr, sizeof(int) * 2)) {
        cleanup();
        return fail(PCS_ENOMEM, "cudaMalloc failed in compute_correlation");
    }
    int init[2] = {0, INT32_MAX};
    if (!x_on_device) cudaMemcpyAsync(dX, x, sizeof(double) * (size_t)m * p, cudaMemcpyHostToDevice, stream);
    cudaMemcpyAsync(dErr, init, sizeof(init), cudaMemcpyHostToDevice, stream);
    if (r0 >= 0)
        launch_correlation_rows(x_on_device ? x : dX, m, p, r0, r1, dXc, dG, ldg, dMean, dC, ldc, dErr, stream);
    else
        launch_correlation(x_on_device ? x : dX, m, p, dXc, dG, ldg, dMean, dC, ldc, dErr, stream);
    int err[2];
    cudaMemcpyAsync(err, dErr, sizeof(err), cudaMemcpyDeviceToHost, stream);
    cleanup();
    cudaError_t ce = cudaStreamSynchronize(stream);
    if (ce != cudaSuccess) return fail(PCS_ECUDA, std::string("compute_correlation: ") + cudaGetErrorString(ce));
    if (err[0] & 1) st = fail(PCS_EINVAL, "DataMatrix: values must be finite");
    else if (err[1] != INT32_MAX) {
        if (zero_var_col) *zero_var_col = err[1];
        st = fail(PCS_EZEROVAR, "compute_correlation: column " + std::to_string(err[1]) + " has zero variance");
    }
    return st;
}

pcs_status pcs_correlation(const double* x, int32_t m, int32_t p, double* c_out, int32_t* zero_var_col) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(PCS_ECUDA, "no CUDA device available");
    cudaStream_t stream;
    CUDA_TRY(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    double* dC = nullptr;
    if (cudaMalloc(&dC, sizeof(double) * (size_t)p * p) != cudaSuccess) {
        cudaStreamDestroy(stream);
        return fail(PCS_ENOMEM, "cudaMalloc failed");
    }
    pcs_status st = correlation_device(stream, x, m, p, dC, p, zero_var_col);
    if (!st) {
        cudaError_t ce = cudaMemcpy(c_out, dC, sizeof(double) * (size_t)p * p, cudaMemcpyDeviceToHost);
        if (ce != cudaSuccess) st = fail(PCS_ECUDA, cudaGetErrorString(ce));
    }
    cudaFree(dC);
    cudaStreamDestroy(stream);
    return st;
}

static pcs_status run_data(const double* x, bool on_device, int32_t m, int32_t p, const pcs_config* cfg,
                           pcs_result** out, int32_t* zero_var_col) {
    *out = nullptr;
    pcs_session* s = nullptr;
    const double t0 = now_s();
    pcs_status st = session_new(p, m, cfg, &s);
    if (st) return st;
    s->ldc = (p + 3) / 4 * 4;
    if (dev_malloc(reinterpret_cast<void**>(&s->dC), sizeof(double) * (size_t)p * s->ldc, s->st) != cudaSuccess) {
        free_session(s);
        return fail(PCS_ENOMEM, "cudaMalloc failed");
    }
    const double t1 = now_s();
    cudaEventRecord(s->ev_begin, s->st);
    st = correlation_device(s->st, x, m, p, s->dC, s->ldc, zero_var_col, on_device);
    const double t2 = now_s();
    if (!st) st = run_session(s, out);
    const double t3 = now_s();
    free_session(s);
    trace("run_pc_stable_data: setup %.2f ms, correlation %.2f ms, levels+finish %.2f ms, teardown %.2f ms",
          (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, (now_s() - t3) * 1e3);
    return st;
}

pcs_status pcs_correlation_device(const double* d_x, int32_t m, int32_t p, double* d_c, int64_t ldc, uint64_t stream,
                                  int32_t* zero_var_col) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(PCS_ECUDA, "no CUDA device available");
    return correlation_device(reinterpret_cast<cudaStream_t>(stream), d_x, m, p, d_c, ldc, zero_var_col, true);
}

pcs_status pcs_correlation_device_rows(const double* d_x, int32_t m, int32_t p, int32_t row_begin, int32_t row_end,
                                       double* d_c, int64_t ldc, uint64_t stream, int32_t* zero_var_col) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(PCS_ECUDA, "no CUDA device available");
    if (row_begin < 0 || row_end > p || row_begin > row_end) return fail(PCS_EINVAL, "bad row range");
    return correlation_device(reinterpret_cast<cudaStream_t>(stream), d_x, m, p, d_c, ldc, zero_var_col, true, row_begin,
                              row_end);
}

pcs_status pcs_run_pc_stable_data(const double* x, int32_t m, int32_t p, const pcs_config* cfg, pcs_result** out,
                                  int32_t* zero_var_col) {
    return run_data(x, false, m, p, cfg, out, zero_var_col);
}

pcs_status pcs_run_pc_stable_data_device(const double* d_x, int32_t m, int32_t p, const pcs_config* cfg,
                                         pcs_result** out, int32_t* zero_var_col) {
    return run_data(d_x, true, m, p, cfg, out, zero_var_col);
}

int32_t pcs_result_p(const pcs_result* r) { return r->p; }
int32_t pcs_result_levels(const pcs_result* r, pcs_level_stats* out, int32_t cap) {
    const int32_t n = (int32_t)r->levels.size();
    for (int32_t k = 0; k < n && k < cap; ++k) out[k] = r->levels[k];
    return n;
}
int32_t pcs_result_stop_reason(const pcs_result* r) { return r->stop_reason; }
static inline bool res_at(const pcs_result* r, int i, int j) {
    return (r->adj[(size_t)i * r->W + (j >> 5)] >> (j & 31)) & 1u;
}
void pcs_result_adjacency(const pcs_result* r, uint8_t* out) {
    for (int i = 0; i < r->p; ++i)
        for (int j = 0; j < r->p; ++j) out[(size_t)i * r->p + j] = res_at(r, i, j);
}
int64_t pcs_result_edge_count(const pcs_result* r) {
    int64_t n = 0;
    for (int i = 0; i < r->p; ++i)
        for (int j = i + 1; j < r->p; ++j) n += res_at(r, i, j);
    return n;
}
void pcs_result_edge_list(const pcs_result* r, int32_t* out) {
    int64_t k = 0;
    for (int i = 0; i < r->p; ++i)
        for (int j = i + 1; j < r->p; ++j)
            if (res_at(r, i, j)) { out[2 * k] = i; out[2 * k + 1] = j; ++k; }
}
int64_t pcs_result_record_ints(const pcs_result* r) { return (int64_t)r->recs.size(); }
void pcs_result_records(const pcs_result* r, int32_t* out) {
    if (!r->recs.empty()) std::memcpy(out, r->recs.data(), sizeof(int32_t) * r->recs.size());
}
void pcs_result_bitmask(const pcs_result* r, uint32_t* out) {
    if (!r->adj.empty()) std::memcpy(out, r->adj.data(), sizeof(uint32_t) * r->adj.size());
}

int64_t pcs_result_member_total(const pcs_result* r) {
    int64_t tot = 0;
    for (size_t k = 0; k < r->recs.size();) {
        const int ell = r->recs[k + 2];
        tot += ell;
        k += 3 + (size_t)ell;
    }
    return tot;
}
void pcs_result_sepsets(const pcs_result* r, int32_t* level, int64_t* offset, int32_t* members) {
    const int p = r->p;
    const size_t ns = (size_t)p * (p - 1) / 2;
    // slot -> record index (levels >= 1); other removed pairs were removed at level 0 with the empty set
    std::vector<int64_t> rec_at(ns, -1);
    for (size_t k = 0; k < r->recs.size();) {
        int a = r->recs[k], b = r->recs[k + 1];
        if (a > b) std::swap(a, b);
        const size_t slot = (size_t)a * (2 * (size_t)p - a - 1) / 2 + (size_t)(b - a - 1);
        rec_at[slot] = (int64_t)k;
        k += 3 + (size_t)r->recs[k + 2];
    }
    int64_t at = 0;
    size_t slot = 0;
    for (int i = 0; i < p; ++i)
        for (int j = i + 1; j < p; ++j, ++slot) {
            offset[slot] = at;
            if (res_at(r, i, j)) { level[slot] = -1; continue; }
            const int64_t k = rec_at[slot];
            if (k < 0) { level[slot] = 0; continue; }
            const int ell = r->recs[k + 2];
            level[slot] = ell;
            for (int q = 0; q < ell; ++q) members[at + q] = r->recs[k + 3 + q];
            at += ell;
        }
}
double pcs_result_device_seconds(const pcs_result* r) { return r->device_seconds; }

int64_t pcs_result_near_count(const pcs_result* r) { return (int64_t)r->near_total; }

int64_t pcs_result_near_records(const pcs_result* r, pcs_near_record* out, int64_t cap) {
    const int64_t n = std::min<int64_t>((int64_t)r->near.size(), cap);
    for (int64_t k = 0; k < n; ++k) {
        const NearRec& x = r->near[(size_t)k];
        out[k].level = x.level;
        out[k].i = x.i;
        out[k].j = x.j;
        out[k].independent = x.decision == kIndependent;
        out[k].rho = x.rho;
        out[k].z = x.z;
    }
    return n;
}
void pcs_result_free(pcs_result* r) { delete r; }

pcs_status pcs_ci_test_batch(const double* c, int32_t p, int32_t ell, int64_t n, const int32_t* ij,
                             const int32_t* sets, double tau, uint8_t* independent, double* z, double* rho,
                             uint8_t* degenerate) {
    if (ell < 0 || ell > kMaxRtLevel) return fail(PCS_EUNSUPPORTED, "ci_test_batch: ell out of range");
    pcs_config cfg;
    pcs_config_default(&cfg);
    pcs_session* s = nullptr;
    pcs_status st = pcs_session_create(c, p, 4, &cfg, &s);
    if (st) return st;
    int32_t *dIJ = nullptr, *dS = nullptr;
    uint8_t *dInd = nullptr, *dDeg = nullptr;
    double *dZ = nullptr, *dR = nullptr;
    int* dErr = nullptr;
    const size_t nn = (size_t)std::max<int64_t>(n, 1);
    cudaMalloc(&dIJ, sizeof(int32_t) * 2 * nn);
    cudaMalloc(&dS, sizeof(int32_t) * nn * std::max(ell, 1));
    cudaMalloc(&dInd, nn);
    cudaMalloc(&dDeg, nn);
    cudaMalloc(&dZ, sizeof(double) * nn);
    cudaMalloc(&dR, sizeof(double) * nn);
    cudaMalloc(&dErr, sizeof(int));
    cudaMemcpy(dIJ, ij, sizeof(int32_t) * 2 * n, cudaMemcpyHostToDevice);
    if (ell > 0) cudaMemcpy(dS, sets, sizeof(int32_t) * n * ell, cudaMemcpyHostToDevice);
    cudaMemset(dErr, 0, sizeof(int));
    double* dW = nullptr;
    if (ell > kMaxTemplLevel) {
        cudaMalloc(&dW, sizeof(double) * nn * (7ull * ell * ell + 4ull * ell + 1));
        launch_ci_batch_rt(s->dC, s->ldc, ell, n, dIJ, dS, tau, dInd, dZ, dR, dDeg, dErr, dW, s->st);
    } else {
        launch_ci_batch(s->dC, s->ldc, p, ell, n, dIJ, dS, tau, dInd, dZ, dR, dDeg, dErr, s->st);
    }
    cudaStreamSynchronize(s->st);
    int err = 0;
    cudaMemcpy(independent, dInd, n, cudaMemcpyDeviceToHost);
    cudaMemcpy(degenerate, dDeg, n, cudaMemcpyDeviceToHost);
    cudaMemcpy(z, dZ, sizeof(double) * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(rho, dR, sizeof(double) * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(&err, dErr, sizeof(int), cudaMemcpyDeviceToHost);
    cudaError_t ce = cudaGetLastError();
    cudaFree(dIJ); cudaFree(dS); cudaFree(dInd); cudaFree(dDeg); cudaFree(dZ); cudaFree(dR); cudaFree(dErr);
    cudaFree(dW);
    free_session(s);
    if (ce != cudaSuccess) return fail(PCS_ECUDA, cudaGetErrorString(ce));
    if (err) return fail(PCS_ENAN, "fisher_z: rho must lie in (-1, 1)");
    return PCS_OK;
}

pcs_status pcs_pseudo_inverse_batch(const double* a, int32_t ell, int64_t n, double* out) {
    if (ell < 1 || ell > kMaxRtLevel) return fail(PCS_EUNSUPPORTED, "pseudo_inverse_batch: ell out of range");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(PCS_ECUDA, "no CUDA device available");
    for (int64_t q = 0; q < n * ell * ell; ++q)
        if (!std::isfinite(a[q])) return fail(PCS_EINVAL, "pseudo_inverse: entries must be finite");
    double *dA = nullptr, *dO = nullptr;
    const size_t bytes = sizeof(double) * (size_t)std::max<int64_t>(n, 1) * ell * ell;
    CUDA_TRY(cudaMalloc(&dA, bytes));
    CUDA_TRY(cudaMalloc(&dO, bytes));
    cudaMemcpy(dA, a, sizeof(double) * n * ell * ell, cudaMemcpyHostToDevice);
    double* dW = nullptr;
    if (ell > kMaxTemplLevel) {
        CUDA_TRY(cudaMalloc(&dW, sizeof(double) * 5ull * ell * ell * (size_t)std::max<int64_t>(n, 1)));
        launch_pinv_batch_rt(dA, ell, n, dO, dW, 0);
    } else {
        launch_pinv_batch(dA, ell, n, dO, 0);
    }
    cudaError_t ce = cudaMemcpy(out, dO, sizeof(double) * n * ell * ell, cudaMemcpyDeviceToHost);
    cudaFree(dA);
    cudaFree(dO);
    cudaFree(dW);
    if (ce != cudaSuccess) return fail(PCS_ECUDA, cudaGetErrorString(ce));
    return PCS_OK;
}

}  // extern "C"
