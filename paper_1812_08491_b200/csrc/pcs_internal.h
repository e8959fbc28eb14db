// pcs_internal.h -- shared declarations between the host driver (host.cu) and
// the kernel translation units (level.cu, corr.cu).  Not part of the ABI.
#pragma once
#include <atomic>
#include <cstdint>
#include <string>
#include <cuda_runtime.h>

#include "pcs_device.cuh"

namespace pcs {

// number of kernels this library has launched (diagnostics: bench.py's gpu_launches)
// (atomic: sessions on different host threads launch concurrently)
extern std::atomic<unsigned long long> g_kernel_launches;
// message returned by pcs_last_error() (host.cu)
void set_last_error(const std::string& msg);

constexpr int kMaxTemplLevel = 8;  // ell handled by register-resident templates

// Device-side counters of one level (zeroed by the host before each level).
struct Counters {
    unsigned long long ci_serial;   // serial-equivalent ci_tests (Appendix B of SURVEY.md)
    unsigned long long removed;     // edges removed
    unsigned long long gpu_tests;   // CI tests executed on the device
    unsigned long long gpu_pinv;    // pseudo-inverses executed on the device
    unsigned long long gpu_exact;   // tests whose statistic was evaluated (not a zero-h00 set)
    unsigned long long rec_count;   // sepset records written
    unsigned long long units[2];    // persistent-grid work cursors (pass A / B)
    unsigned long long dbg[4];      // diagnostics builds only (PCS_COUNT_CAND)
    unsigned long long near;        // decisions taken by the exact comparison inside the threshold band
    int err_nan;                    // fisher_z would throw (NaN statistic)
    int err_other;
};

// One near-threshold decision (the exact comparison inside the +-1e-9 band), listed per run
struct NearRec {
    int level, i, j, decision;  // decision: kDependent / kIndependent / kNanError
    double rho, z;
    int oi, raw;                // raw = 1: written by a cuPC-S sweep as (row offset oi, h01 in rho, denom in z);
                                // finished by launch_near_fixup before the snapshot changes
};
constexpr int kNearCap = 4096;  // records kept per run (the count is exact beyond)

// Summary of a fresh snapshot (compact(), core.hpp:227-239).
struct SnapInfo {
    long long e_dir;      // directed entries (2E)
    long long e_und;      // undirected edges (E)
    int max_width;
    int pad;
    double sets2, sets3;  // sum over rows of C(w, 2), C(w, 3): the level's (row, set) pairs at l = 2, 3
};

// Everything a level kernel reads.
struct LevelArgs {
    const double* C;
    long long ldc;
    int p;
    int ell;
    const int32_t* off;      // p+1
    const int32_t* nbr;      // 2E, ascending rows
    const int32_t* lowcnt;   // p: neighbours < i
    const int32_t* upoff;    // p+1: prefix of (deg - lowcnt)
    const int32_t* eid;      // 2E: undirected id of each directed entry
    const int32_t* eu_a;     // E: row a (a < b)
    const int32_t* eu_qa;    // E: position of b in row a
    const int32_t* eu_qb;    // E: position of a in row b
    unsigned long long* keys;  // E
    unsigned long long* kdir;  // 2E: keys[eid[k]] mirrored per directed entry (cuPC-S staging reads it
                               //     coalesced, no dependent gather); refreshed before every pass
    const double* cnbr;        // 2E: C(i, nbr[k]) of the directed entry k of row i (filled per level)
    const double* pinv_table;  // l = 2, 3: M2^+ of every vertex l-subset by colex rank (null: compute per set)
    NearRec* near_rec;         // near-threshold list of the run (kNearCap records)
    unsigned long long* near_total;  // records written so far in the run
    BinomTable binom;
    Thresholds th;
    Counters* cnt;
};

// ---- corr.cu
void launch_normalize_corr(double* C, long long ldc, int p, int* err, cudaStream_t s);
// rows [r0, r1) of C only (multi-GPU split); G holds the row band's tiles: ((r1 - r0) + 256) x ldg
void launch_correlation_rows(const double* X, int m, int p, int r0, int r1, double* Xc, double* G, long long ldg,
                             double* mean, double* C, long long ldc, int* err_flags, cudaStream_t s);
// flag |= 1 unless C has a unit diagonal, bitwise symmetry and finite entries in [-1, 1]
void launch_check_corr(const double* C, long long ldc, int p, int* flag, cudaStream_t s);
void launch_correlation(const double* X, int m, int p, double* Xc, double* G, long long ldg, double* mean,
                        double* C, long long ldc, int* err_flags, cudaStream_t s);

// ---- level.cu
void launch_level0(const double* C, long long ldc, int p, int W, uint32_t* adj, Thresholds th, Counters* cnt,
                   cudaStream_t s, bool and_live = false, NearRec* near_rec = nullptr,
                   unsigned long long* near_total = nullptr);
void launch_snapshot_degrees(const uint32_t* adj, int p, int W, int32_t* deg, int32_t* lowcnt, cudaStream_t s);
void launch_snapshot_scan(const int32_t* deg, const int32_t* lowcnt, int p, int32_t* off, int32_t* upoff,
                          SnapInfo* info, cudaStream_t s);
void launch_snapshot_fill(const uint32_t* adj, int p, int W, const int32_t* off, int32_t* nbr, cudaStream_t s);
void launch_edge_index(const LevelArgs& A, int32_t* eid, int32_t* eu_a, int32_t* eu_qa, int32_t* eu_qb,
                       double* cnbr, cudaStream_t s);
// kdir[k] = keys[eid[k]] for every directed entry (before each cuPC-S pass)
void launch_refresh_kdir(const LevelArgs& A, long long e_dir, cudaStream_t s);
void launch_fill_keys(unsigned long long* keys, long long n, cudaStream_t s);
// per-row work prefix for a pass (units of work: target tiles for ell=1, set bands for ell>=2,
// restricted to [row_begin,row_end) for sharding); returns nothing, writes prefix[p+1]
void launch_row_work(const LevelArgs& A, int pass, int variant, int row_begin, int row_end,
                     unsigned long long* prefix, cudaStream_t s);
// multi-GPU: the same prefix plus a cost prefix, and this shard's cost-weighted unit range -> bounds[2]
void launch_row_work_sharded(const LevelArgs& A, int pass, int variant, unsigned long long* prefix,
                             unsigned long long* cost, int shard, int nsh, unsigned long long* bounds,
                             cudaStream_t s);
// multi-GPU cuPC-E: cost-weighted range of undirected edges for this shard -> bounds[2]
void launch_edge_bounds(const LevelArgs& A, int pass, long long E, unsigned long long* cost, int shard, int nsh,
                        unsigned long long* bounds, cudaStream_t s);
// tiles [u_begin, min(u_end, prefix[p])) (u_end = ~0: the device-side total); bound = host upper bound
void launch_level1(const LevelArgs& A, int pass, const unsigned long long* prefix, unsigned long long u_begin,
                   unsigned long long u_end, unsigned long long bound, int shard, int nsh, cudaStream_t s);
// turns the raw near-threshold records of the current level into (row, rho, z)
void launch_near_fixup(const LevelArgs& A, cudaStream_t s);
// ---- level1t.cu: ell = 1, both directions, TMA-tiled (dense snapshots); rows [row_begin, row_end)
// multi-GPU: shard `shard` of `nsh` takes every nsh-th 32-row block (cyclic)
int launch_level1_tile(const LevelArgs& A, const uint32_t* adj, int W, int shard, int nsh, cudaStream_t s);
// l = 2, 3: the pseudo-inverse of every l-subset {a < b (< c)} of the p vertices into table[colex rank *
// pinv_table_stride(l)], the same pinv<L> as the per-set path (bit-identical entries)
int pinv_table_stride(int ell);
int launch_pinv_table(const double* C, long long ldc, int p, int ell, double* table, cudaStream_t s);
int launch_level_set(const LevelArgs& A, int pass, const unsigned long long* prefix, unsigned long long u_begin,
                     unsigned long long u_end, int num_sms, cudaStream_t s);
// maxw: the snapshot's widest row (sizes the staged kernel's shared-memory row buffers)
int launch_level_edge(const LevelArgs& A, int pass, long long e_begin, long long e_end, int maxw, int num_sms,
                      cudaStream_t s);
// generic ell (> kMaxTemplLevel, <= kMaxRtLevel): cuPC-S with global per-lane scratch
long long level_rt_scratch_bytes(int ell, int num_sms, int* blocks_out);
int launch_level_set_rt(const LevelArgs& A, int pass, const unsigned long long* prefix, unsigned long long u_begin,
                        unsigned long long u_end, int num_sms, void* scratch, cudaStream_t s);
int launch_ci_batch_rt(const double* C, long long ldc, int ell, long long n, const int32_t* ij, const int32_t* sets,
                       double tau, uint8_t* indep, double* z, double* rho, uint8_t* degen, int* err, double* scratch,
                       cudaStream_t s);
int launch_pinv_batch_rt(const double* a, int ell, long long n, double* out, double* scratch, cudaStream_t s);
void launch_commit(const LevelArgs& A, uint32_t* adj, int W, long long e_und, int32_t* rec, cudaStream_t s);
// parity helpers (stats::ci_test / pseudo_inverse on the device, one test per thread)
int launch_ci_batch(const double* C, long long ldc, int p, int ell, long long n, const int32_t* ij,
                    const int32_t* sets, double tau, uint8_t* indep, double* z, double* rho, uint8_t* degen,
                    int* err, cudaStream_t s);
int launch_pinv_batch(const double* a, int ell, long long n, double* out, cudaStream_t s);

}  // namespace pcs
