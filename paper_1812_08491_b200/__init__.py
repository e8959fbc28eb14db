"""pcstable_b200 -- B200-native PC-stable skeleton discovery (cuPC), Python host side.

Mirrors the reference C++ API of proj/include/pcstable (same names, argument
meaning and error behaviour) on top of the C ABI in include/pcstable_b200.h,
implemented by the in-tree CUDA library libpcstable_b200.so (sm_100a).  There
is no CPU fallback: every call below runs the device path and raises if the
library or a GPU is missing.

    compute_correlation(data)          stats.hpp:132   (FP64 DMMA Gram on the device)
    threshold_tau(alpha, m, ell)       stats.hpp:120
    run_pc_stable(c, m, cfg)           skeleton.hpp:341 -> SkeletonResult
    run_pc_stable_data(data, cfg)      correlation + skeleton in one device pipeline
    ci_test_batch / pseudo_inverse_batch   stats.hpp:366 / :172 on the device (parity helpers)
    Session                            per-level stepping used by the multi-GPU driver
"""
from __future__ import annotations

import ctypes as ct
import enum
import os
from dataclasses import dataclass, field
from typing import Iterator, Optional

import numpy as np

__all__ = [
    "Strategy", "StopReason", "SkeletonConfig", "LevelStats", "SkeletonResult", "AdjacencyMatrix",
    "SeparationSets", "ZeroVarianceError", "LevelUnreachableError", "PcsError", "compute_correlation",
    "threshold_tau", "run_pc_stable", "run_pc_stable_data", "ci_test_batch", "pseudo_inverse_batch",
    "Session", "library", "LIB_PATH", "random_dag", "sample_linear_gaussian", "run_pc_stable_data_device",
    "run_pc_stable_device", "correlation_device", "kernel_launches", "MixedGraph", "find_v_structures",
    "apply_meek_rules", "orient_skeleton",
]

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libpcstable_b200.so")

# ----------------------------------------------------------------- errors
PCS_OK, PCS_EINVAL, PCS_EZEROVAR, PCS_EOVERFLOW, PCS_ENAN, PCS_ECUDA, PCS_ENOMEM, PCS_EUNSUPPORTED, PCS_ELEVEL = range(9)


class PcsError(RuntimeError):
    """Device-side failure (CUDA error, out of memory, unsupported level)."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class ZeroVarianceError(RuntimeError):
    """pcstable::ZeroVarianceError (core.hpp:23-31)."""

    def __init__(self, column: int, msg: str):
        super().__init__(msg)
        self.column = column


class LevelUnreachableError(RuntimeError):
    """pcstable::LevelUnreachableError (core.hpp:41-44)."""


def _raise(code: int, column: int = -1):
    msg = library().pcs_last_error().decode()
    if code == PCS_EINVAL or code == PCS_ENAN:
        raise ValueError(msg)  # std::invalid_argument
    if code == PCS_EZEROVAR:
        raise ZeroVarianceError(column, msg)
    if code == PCS_EOVERFLOW:
        raise OverflowError(msg)  # std::overflow_error
    if code == PCS_ELEVEL:
        raise LevelUnreachableError(msg)
    raise PcsError(code, msg)


# ----------------------------------------------------------------- ABI structs
class _Config(ct.Structure):
    _fields_ = [
        ("alpha", ct.c_double), ("max_level", ct.c_int32), ("variant", ct.c_int32),
        ("edges_per_unit", ct.c_int32), ("workers_per_edge", ct.c_int32), ("set_groups", ct.c_int32),
        ("unit_width", ct.c_int32), ("device", ct.c_int32), ("shard_index", ct.c_int32),
        ("shard_count", ct.c_int32), ("reserved0", ct.c_int32), ("stream", ct.c_uint64),
        ("reserved", ct.c_int32 * 4),
    ]


class _NearRec(ct.Structure):
    _fields_ = [("level", ct.c_int32), ("i", ct.c_int32), ("j", ct.c_int32), ("independent", ct.c_int32),
                ("rho", ct.c_double), ("z", ct.c_double)]


class _Level(ct.Structure):
    _fields_ = [
        ("level", ct.c_int32), ("pad", ct.c_int32), ("ci_tests", ct.c_uint64), ("pseudo_inverses", ct.c_uint64),
        ("edges_removed", ct.c_uint64), ("elapsed_s", ct.c_double), ("device_ci_tests", ct.c_uint64),
        ("device_pseudo_inverses", ct.c_uint64), ("kernel_ms", ct.c_double), ("device_exact_tests", ct.c_uint64),
        ("device_near_threshold", ct.c_uint64),
    ]


_lib = None


def library():
    """Loads libpcstable_b200.so; raises if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = ct.CDLL(LIB_PATH)
    dp, ip, vp = ct.POINTER(ct.c_double), ct.POINTER(ct.c_int32), ct.c_void_p
    u8p = ct.POINTER(ct.c_uint8)
    L.pcs_version.restype = ct.c_char_p
    L.pcs_last_error.restype = ct.c_char_p
    L.pcs_config_default.argtypes = [ct.POINTER(_Config)]
    L.pcs_threshold_tau.argtypes = [ct.c_double, ct.c_int32, ct.c_int32, dp]
    L.pcs_correlation.argtypes = [dp, ct.c_int32, ct.c_int32, dp, ip]
    L.pcs_run_pc_stable.argtypes = [dp, ct.c_int32, ct.c_int32, ct.POINTER(_Config), ct.POINTER(vp)]
    L.pcs_run_pc_stable_data.argtypes = [dp, ct.c_int32, ct.c_int32, ct.POINTER(_Config), ct.POINTER(vp), ip]
    L.pcs_run_pc_stable_data_device.argtypes = [vp, ct.c_int32, ct.c_int32, ct.POINTER(_Config), ct.POINTER(vp), ip]
    L.pcs_random_dag.argtypes = [ct.c_int32, ct.c_double, ct.c_uint64, dp]
    L.pcs_sample_linear_gaussian.argtypes = [dp, ct.c_int32, ct.c_int32, ct.c_uint64, dp]
    L.pcs_sample_linear_gaussian_rescaled.argtypes = [dp, ct.c_int32, ct.c_int32, ct.c_uint64, dp, dp]
    L.pcs_run_pc_stable_device.argtypes = [vp, ct.c_int64, ct.c_int32, ct.c_int32, ct.POINTER(_Config),
                                           ct.POINTER(vp)]
    L.pcs_result_p.argtypes = [vp]
    L.pcs_result_levels.argtypes = [vp, ct.POINTER(_Level), ct.c_int32]
    L.pcs_result_stop_reason.argtypes = [vp]
    L.pcs_result_adjacency.argtypes = [vp, u8p]
    L.pcs_result_edge_count.argtypes = [vp]
    L.pcs_result_edge_count.restype = ct.c_int64
    L.pcs_result_edge_list.argtypes = [vp, ip]
    L.pcs_result_member_total.argtypes = [vp]
    L.pcs_result_member_total.restype = ct.c_int64
    L.pcs_result_sepsets.argtypes = [vp, ip, ct.POINTER(ct.c_int64), ip]
    L.pcs_result_device_seconds.argtypes = [vp]
    L.pcs_result_device_seconds.restype = ct.c_double
    L.pcs_result_bitmask.argtypes = [vp, ct.POINTER(ct.c_uint32)]
    L.pcs_result_record_ints.argtypes = [vp]
    L.pcs_result_record_ints.restype = ct.c_int64
    L.pcs_result_records.argtypes = [vp, ip]
    L.pcs_correlation_device.argtypes = [vp, ct.c_int32, ct.c_int32, vp, ct.c_int64, ct.c_uint64, ip]
    L.pcs_result_near_count.argtypes = [vp]
    L.pcs_result_near_count.restype = ct.c_int64
    L.pcs_result_near_records.argtypes = [vp, ct.POINTER(_NearRec), ct.c_int64]
    L.pcs_result_near_records.restype = ct.c_int64
    L.pcs_noise_stream.argtypes = [ct.c_uint64, ct.c_int64, ct.c_int32, ct.c_int32, dp]
    L.pcs_sample_linear_gaussian_device.argtypes = [dp, ct.c_int32, ct.c_int32, ct.c_uint64, ct.c_int32, vp, dp,
                                                    ct.c_uint64]
    L.pcs_run_level.argtypes = [dp, ct.c_int32, ct.c_int32, ct.c_double, ct.POINTER(_Config), ct.POINTER(ct.c_uint8),
                                ct.POINTER(vp)]
    L.pcs_correlation_device_rows.argtypes = [vp, ct.c_int32, ct.c_int32, ct.c_int32, ct.c_int32, vp, ct.c_int64,
                                              ct.c_uint64, ip]
    L.pcs_kernel_launches.restype = ct.c_ulonglong
    L.pcs_probe_fp64_tflops.argtypes = [dp]
    L.pcs_session_snapshot.argtypes = [vp, ip, ip]
    L.pcs_session_set_shard.argtypes = [vp, ct.c_int32, ct.c_int32]
    L.pcs_result_free.argtypes = [vp]
    L.pcs_ci_test_batch.argtypes = [dp, ct.c_int32, ct.c_int32, ct.c_int64, ip, ip, ct.c_double, u8p, dp, dp, u8p]
    L.pcs_pseudo_inverse_batch.argtypes = [dp, ct.c_int32, ct.c_int64, dp]
    L.pcs_session_create.argtypes = [dp, ct.c_int32, ct.c_int32, ct.POINTER(_Config), ct.POINTER(vp)]
    L.pcs_session_create_device.argtypes = [vp, ct.c_int64, ct.c_int32, ct.c_int32, ct.POINTER(_Config),
                                            ct.POINTER(vp)]
    L.pcs_session_level_begin.argtypes = [vp, ip, ip, ct.POINTER(ct.c_int64)]
    L.pcs_session_level_pass.argtypes = [vp, ct.c_int32]
    L.pcs_session_keys.argtypes = [vp, ct.POINTER(vp), ct.POINTER(ct.c_int64)]
    L.pcs_session_level_end.argtypes = [vp]
    L.pcs_session_finish.argtypes = [vp, ct.POINTER(vp)]
    L.pcs_session_free.argtypes = [vp]
    L.pcs_orient_records.argtypes = [ct.c_int32, ct.POINTER(ct.c_uint32), ip, ct.c_int64, ct.c_int32, ct.POINTER(vp)]
    L.pcs_orient_skeleton.argtypes = [ct.c_int32, u8p, ip, ct.POINTER(ct.c_int64), ip, ct.c_int32, ip, ct.c_int64,
                                      ct.POINTER(vp)]
    L.pcs_mixed_directed_count.argtypes = [vp]
    L.pcs_mixed_directed_count.restype = ct.c_int64
    L.pcs_mixed_undirected_count.argtypes = [vp]
    L.pcs_mixed_undirected_count.restype = ct.c_int64
    L.pcs_mixed_directed.argtypes = [vp, ip]
    L.pcs_mixed_undirected.argtypes = [vp, ip]
    L.pcs_mixed_free.argtypes = [vp]
    _lib = L
    return L


def version() -> str:
    return library().pcs_version().decode()


# ----------------------------------------------------------------- config / results
class Strategy(enum.Enum):
    """core.hpp:341.  Every strategy yields the Serial strategy's skeleton, sepsets and counters on the
    device; EdgeParallel selects the cuPC-E kernels, SetShared (and Serial) the cuPC-S kernels."""
    Serial = "serial"
    EdgeParallel = "edge"
    SetShared = "set"


class StopReason(enum.Enum):  # skeleton.hpp:22-31
    MaxDegreeReached = "max-degree"
    LevelCapReached = "level-cap"
    SampleSizeExhausted = "sample-size"


_STOP = {0: StopReason.MaxDegreeReached, 1: StopReason.LevelCapReached, 2: StopReason.SampleSizeExhausted}


@dataclass
class SkeletonConfig:  # core.hpp:357-384
    alpha: float = 0.05
    max_level: Optional[int] = None
    strategy: Strategy = Strategy.SetShared
    edges_per_unit: int = 2
    workers_per_edge: int = 32
    set_groups: int = 2
    unit_width: int = 64
    worker_count: int = 1           # CPU knob of the reference; inert on the device
    schedule_seed: Optional[int] = None  # inert: device results never depend on schedule
    device: int = 0
    stream: int = 0                 # cudaStream_t handle to run on (0: library-owned stream)

    def validate(self):  # core.hpp:370-383
        if not (0.0 < self.alpha < 1.0):
            raise ValueError("SkeletonConfig: alpha must lie in (0, 1)")
        if self.max_level is not None and self.max_level < 0:
            raise ValueError("SkeletonConfig: max_level must be >= 0")
        for name in ("edges_per_unit", "workers_per_edge", "set_groups", "unit_width", "worker_count"):
            if getattr(self, name) < 1:
                raise ValueError(f"SkeletonConfig: {name} must be >= 1")

    def _abi(self, shard_index: int = 0, shard_count: int = 1) -> _Config:
        self.validate()
        c = _Config()
        library().pcs_config_default(ct.byref(c))
        c.alpha = self.alpha
        c.max_level = -1 if self.max_level is None else int(self.max_level)
        c.variant = 1 if Strategy(self.strategy) == Strategy.EdgeParallel else 0
        c.edges_per_unit, c.workers_per_edge = self.edges_per_unit, self.workers_per_edge
        c.set_groups, c.unit_width = self.set_groups, self.unit_width
        c.device, c.shard_index, c.shard_count = self.device, shard_index, shard_count
        c.stream = int(self.stream)
        return c


@dataclass
class LevelStats:  # core.hpp:387-393 (+ device counters)
    level: int
    ci_tests: int
    pseudo_inverses: int
    edges_removed: int
    elapsed_s: float
    device_ci_tests: int = 0
    device_pseudo_inverses: int = 0
    kernel_ms: float = 0.0
    device_exact_tests: int = 0
    device_near_threshold: int = 0  # tests decided by the exact comparison inside the threshold band


class AdjacencyMatrix:
    """Read-only skeleton with the reference's accessors (core.hpp:109-194), backed by the
    device's live bitmask (bit j of word i*W + j/32)."""

    def __init__(self, bits: np.ndarray, n: int):
        self.bits = bits
        self.n = n
        self._cells = None

    @property
    def cells(self) -> np.ndarray:
        if self._cells is None:
            b = np.unpackbits(self.bits.view(np.uint8).reshape(self.n, -1), axis=1, bitorder="little")
            self._cells = np.ascontiguousarray(b[:, : self.n])
        return self._cells

    def size(self) -> int:
        return self.n

    def at(self, i: int, j: int) -> bool:
        return bool((int(self.bits[i, j >> 5]) >> (j & 31)) & 1)

    def edge_count(self) -> int:
        # popcount of the symmetric bitmask (no diagonal bits): every edge is counted twice
        return int(np.bitwise_count(self.bits).sum(dtype=np.int64)) // 2

    def edges(self) -> np.ndarray:
        """(E, 2) array of surviving edges (i < j), ascending."""
        return np.argwhere(np.triu(self.cells, 1))

    def __eq__(self, other) -> bool:
        return isinstance(other, AdjacencyMatrix) and np.array_equal(self.cells, other.cells)


class SeparationSets:
    """Sepsets keyed by unordered pair (core.hpp:267-339).  Level-0 removals carry the empty set;
    removals at level >= 1 come from the device's records, grouped by level and looked up by
    binary search (no per-record Python work until as_dict() is asked for)."""

    def __init__(self, n: int, skeleton: AdjacencyMatrix, records: np.ndarray, levels: list):
        self.n = n
        self._skel = skeleton
        self.records = np.ascontiguousarray(records, np.int32)  # (a, b, ell, members...) of levels >= 1
        self._levels = [(lv.level, lv.edges_removed) for lv in levels]
        self._sorted = None  # per-level (ell, sorted pair keys, members), built on first lookup
        self._dict = None

    @property
    def _blocks(self):
        if self._sorted is None:
            blocks, at, n, records = [], 0, self.n, self.records
            for ell, cnt in self._levels:
                if ell < 1 or cnt == 0 or at >= len(records):
                    continue
                blk = np.asarray(records[at:at + cnt * (3 + ell)]).reshape(cnt, 3 + ell)
                at += cnt * (3 + ell)
                a = np.minimum(blk[:, 0], blk[:, 1]).astype(np.int64)
                b = np.maximum(blk[:, 0], blk[:, 1]).astype(np.int64)
                key = a * n + b
                order = np.argsort(key, kind="stable")
                blocks.append((ell, key[order], np.ascontiguousarray(blk[order, 3:])))
            self._sorted = blocks
        return self._sorted

    def size(self) -> int:
        return self.n

    def find(self, i: int, j: int):
        if i == j or not (0 <= i < self.n and 0 <= j < self.n):
            raise ValueError("SeparationSets: invalid vertex pair")
        a, b = min(i, j), max(i, j)
        if self._skel.at(a, b):
            return None
        k = a * self.n + b
        for _, keys, mem in self._blocks:
            x = int(np.searchsorted(keys, k))
            if x < len(keys) and keys[x] == k:
                return tuple(int(v) for v in mem[x])
        return ()

    def as_dict(self) -> dict:
        if self._dict is None:
            iu, ju = np.nonzero(np.triu(1 - self._skel.cells, 1))
            d = {(int(a), int(b)): () for a, b in zip(iu, ju)}
            for _, keys, mem in self._blocks:
                for k, row in zip(keys.tolist(), mem.tolist()):
                    d[(k // self.n, k % self.n)] = tuple(row)
            self._dict = d
        return self._dict

    def stored_count(self) -> int:
        n = self.n
        return n * (n - 1) // 2 - self._skel.edge_count()

    def for_each(self) -> Iterator:
        d = self.as_dict()
        for k in sorted(d):
            yield k[0], k[1], d[k]


@dataclass
class SkeletonResult:  # skeleton.hpp:33-40
    skeleton: AdjacencyMatrix
    sepsets: SeparationSets
    levels: list = field(default_factory=list)
    stop_reason: StopReason = StopReason.MaxDegreeReached
    device_seconds: float = 0.0
    near_threshold_count: int = 0   # decisions inside the +-1e-9 threshold band (exact comparison)
    near_threshold: list = field(default_factory=list)  # first 4096: dicts level, i, j, independent, rho, z

    def levels_run(self) -> int:
        return len(self.levels)

    def edge_set(self):
        return [tuple(map(int, e)) for e in self.skeleton.edges()]


def _dp(a):
    return a.ctypes.data_as(ct.POINTER(ct.c_double))


def _ip(a):
    return a.ctypes.data_as(ct.POINTER(ct.c_int32))


def _collect(h, with_sepsets: bool = True) -> SkeletonResult:
    """Copies a pcs_result into Python objects (bitmask + records; sepsets decoded lazily)."""
    L = library()
    p = L.pcs_result_p(h)
    lv = (_Level * 256)()
    n = L.pcs_result_levels(h, lv, 256)
    levels = [LevelStats(lv[k].level, lv[k].ci_tests, lv[k].pseudo_inverses, lv[k].edges_removed, lv[k].elapsed_s,
                         lv[k].device_ci_tests, lv[k].device_pseudo_inverses, lv[k].kernel_ms,
                         lv[k].device_exact_tests, lv[k].device_near_threshold) for k in range(n)]
    W = (p + 31) // 32
    bits = np.empty((p, W), np.uint32)
    L.pcs_result_bitmask(h, bits.ctypes.data_as(ct.POINTER(ct.c_uint32)))
    nrec = L.pcs_result_record_ints(h) if with_sepsets else 0  # records only when sepsets are asked for
    rec = np.empty(max(nrec, 1), np.int32)
    if nrec:
        L.pcs_result_records(h, _ip(rec))
    adj = AdjacencyMatrix(bits, p)
    sep = SeparationSets(p, adj, rec[:nrec], levels)
    nn = L.pcs_result_near_count(h)
    near = []
    if nn:
        buf = (_NearRec * min(nn, 4096))()
        got = L.pcs_result_near_records(h, buf, len(buf))
        near = [dict(level=b.level, i=b.i, j=b.j, independent=bool(b.independent), rho=b.rho, z=b.z)
                for b in buf[:got]]
    return SkeletonResult(adj, sep, levels, _STOP[L.pcs_result_stop_reason(h)], L.pcs_result_device_seconds(h),
                          nn, near)


# ----------------------------------------------------------------- API
def threshold_tau(alpha: float, m: int, ell: int) -> float:
    out = ct.c_double()
    rc = library().pcs_threshold_tau(alpha, m, ell, ct.byref(out))
    if rc:
        _raise(rc)
    return out.value


def _data_colmajor(data) -> tuple[np.ndarray, int, int]:
    """data: (m, p) samples x variables, like DataMatrix (core.hpp:48-67)."""
    x = np.asarray(data, np.float64)
    if x.ndim != 2:
        raise ValueError("DataMatrix: need a 2-D array (samples x variables)")
    m, p = x.shape
    return np.asfortranarray(x), m, p


def compute_correlation(data) -> np.ndarray:
    """stats::compute_correlation on the device; returns the p x p correlation matrix."""
    x, m, p = _data_colmajor(data)
    c = np.empty((p, p), np.float64)
    col = ct.c_int32(-1)
    rc = library().pcs_correlation(_dp(x), m, p, _dp(c), ct.byref(col))
    if rc:
        _raise(rc, col.value)
    return c


def run_pc_stable(c, sample_count: int, cfg: Optional[SkeletonConfig] = None, with_sepsets: bool = True
                  ) -> SkeletonResult:
    """run_pc_stable (skeleton.hpp:341-391) on the device."""
    cfg = cfg or SkeletonConfig()
    c = np.ascontiguousarray(c, np.float64)
    if c.ndim != 2 or c.shape[0] != c.shape[1]:
        raise ValueError("CorrelationMatrix: need a square matrix, n >= 2")
    abi = cfg._abi()
    h = ct.c_void_p()
    rc = library().pcs_run_pc_stable(_dp(c), c.shape[0], int(sample_count), ct.byref(abi), ct.byref(h))
    if rc:
        _raise(rc)
    try:
        return _collect(h, with_sepsets)
    finally:
        library().pcs_result_free(h)


def run_pc_stable_data(data, cfg: Optional[SkeletonConfig] = None, with_sepsets: bool = True) -> SkeletonResult:
    """compute_correlation + run_pc_stable in one device pipeline (bench.hpp:107-113 shape)."""
    cfg = cfg or SkeletonConfig()
    x, m, p = _data_colmajor(data)
    abi = cfg._abi()
    h = ct.c_void_p()
    col = ct.c_int32(-1)
    rc = library().pcs_run_pc_stable_data(_dp(x), m, p, ct.byref(abi), ct.byref(h), ct.byref(col))
    if rc:
        _raise(rc, col.value)
    try:
        return _collect(h, with_sepsets)
    finally:
        library().pcs_result_free(h)


def run_pc_stable_data_device(x_ptr: int, m: int, p: int, cfg: Optional[SkeletonConfig] = None,
                              with_sepsets: bool = False) -> SkeletonResult:
    """compute_correlation + run_pc_stable on m x p column-major data already in device memory."""
    cfg = cfg or SkeletonConfig()
    abi = cfg._abi()
    h = ct.c_void_p()
    col = ct.c_int32(-1)
    rc = library().pcs_run_pc_stable_data_device(ct.c_void_p(x_ptr), m, p, ct.byref(abi), ct.byref(h),
                                                 ct.byref(col))
    if rc:
        _raise(rc, col.value)
    try:
        return _collect(h, with_sepsets)
    finally:
        library().pcs_result_free(h)


def correlation_device(x_ptr: int, m: int, p: int, c_ptr: int, ldc: int, stream: int = 0):
    """compute_correlation from device-resident column-major data into a device p x ldc buffer."""
    col = ct.c_int32(-1)
    rc = library().pcs_correlation_device(ct.c_void_p(x_ptr), m, p, ct.c_void_p(c_ptr), ldc, stream, ct.byref(col))
    if rc:
        _raise(rc, col.value)


def run_level(c, graph_cells, ell: int, tau: float, cfg: Optional[SkeletonConfig] = None):
    """One level on a given live graph (run_level_zero / run_level_serial / run_level_edge_parallel /
    run_level_set_shared, skeleton.hpp:262-333; cfg.strategy picks the kernels).  graph_cells: (p, p)
    0/1 symmetric, the level-start snapshot.  Returns (graph after the level, LevelStats, {(i, j): sepset}
    of the pairs this level removed)."""
    cfg = cfg or SkeletonConfig()
    c = np.ascontiguousarray(c, np.float64)
    p = c.shape[0]
    g = np.ascontiguousarray(np.asarray(graph_cells, np.uint8)).copy()
    before = g.copy()
    h = ct.c_void_p()
    abi = cfg._abi()
    rc = library().pcs_run_level(_dp(c), p, ell, tau, ct.byref(abi), g.ctypes.data_as(ct.POINTER(ct.c_uint8)),
                                 ct.byref(h))
    if rc:
        _raise(rc)
    try:
        res = _collect(h)
    finally:
        library().pcs_result_free(h)
    lv = res.levels[0] if res.levels else LevelStats(ell, 0, 0, 0, 0.0)
    removed = np.argwhere(np.triu(before.astype(bool) & ~g.astype(bool), 1))
    sep = {}
    for i, j in removed:
        got = res.sepsets.find(int(i), int(j))
        sep[(int(i), int(j))] = tuple(got) if (got is not None and ell > 0) else ()
    return g, lv, sep


def noise_stream(seed: int, count: int, p: int, m: int) -> np.ndarray:
    """The reference generator's first `count` normals (rng.hpp), jump-ahead parallel on the host,
    as a (p, m) variable-major array (draw n -> [n % p, n / p])."""
    out = np.zeros((p, m), np.float64)
    rc = library().pcs_noise_stream(seed, count, p, m, _dp(out))
    if rc:
        _raise(rc)
    return out


def sample_linear_gaussian_device(weights: np.ndarray, m: int, seed: int, x_ptr: int, rescaled: bool = False,
                                  stream: int = 0):
    """sample_linear_gaussian (or the rescaled variant) into device memory at x_ptr (m x n column-major,
    i.e. a (n, m) row-major float64 buffer); returns log_scale for the rescaled variant."""
    w = np.ascontiguousarray(weights, np.float64)
    n = w.shape[0]
    ls = np.zeros(n, np.float64)
    rc = library().pcs_sample_linear_gaussian_device(_dp(w), n, m, seed, 1 if rescaled else 0, ct.c_void_p(x_ptr),
                                                     _dp(ls), stream)
    if rc:
        _raise(rc)
    return ls if rescaled else None


def correlation_device_rows(x_ptr: int, m: int, p: int, row_begin: int, row_end: int, c_ptr: int, ldc: int,
                            stream: int = 0):
    """Rows [row_begin, row_end) of compute_correlation into the device p x ldc buffer (the multi-GPU
    split: each rank builds its row band, then the bands are all-gathered; multigpu.correlation_sharded)."""
    col = ct.c_int32(-1)
    rc = library().pcs_correlation_device_rows(ct.c_void_p(x_ptr), m, p, row_begin, row_end, ct.c_void_p(c_ptr), ldc,
                                               stream, ct.byref(col))
    if rc:
        _raise(rc, col.value)


def probe_fp64_tflops() -> float:
    """Measured FP64 FMA peak (TFLOP/s) of the current device."""
    out = ct.c_double()
    rc = library().pcs_probe_fp64_tflops(ct.byref(out))
    if rc:
        _raise(rc)
    return out.value


def kernel_launches() -> int:
    """Kernels launched by the library so far in this process."""
    return int(library().pcs_kernel_launches())


def random_dag(n: int, density: float, seed: int) -> np.ndarray:
    """random_dag (datagen.hpp:42-56): n x n weights, weights[i, j] != 0 means j causes i (j < i)."""
    w = np.empty((n, n), np.float64)
    rc = library().pcs_random_dag(n, density, seed, _dp(w))
    if rc:
        raise ValueError("random_dag: need n >= 2 and density in (0, 1)")
    return w


def sample_linear_gaussian(weights: np.ndarray, m: int, seed: int) -> np.ndarray:
    """sample_linear_gaussian (datagen.hpp:62-82): returns the (m, n) data matrix (samples x variables),
    stored column-major like Eigen (x.T is C-contiguous)."""
    w = np.ascontiguousarray(weights, np.float64)
    n = w.shape[0]
    xt = np.empty((n, m), np.float64)  # row j = variable j == column-major m x n
    rc = library().pcs_sample_linear_gaussian(_dp(w), n, m, seed, _dp(xt))
    if rc:
        raise ValueError("sample_linear_gaussian: need m >= 4 and strictly lower-triangular weights")
    return xt.T


def sample_linear_gaussian_rescaled(weights: np.ndarray, m: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """Overflow-safe sample_linear_gaussian for the BASELINE scaling shapes: the same noise
    stream with every variable kept at unit RMS; returns ((m, n) data, log_scale[n]) with
    x_reference[:, i] == x[:, i] * exp(log_scale[i]) (to rounding) and the same correlation matrix."""
    w = np.ascontiguousarray(weights, np.float64)
    n = w.shape[0]
    xt = np.empty((n, m), np.float64)
    ls = np.empty(n, np.float64)
    rc = library().pcs_sample_linear_gaussian_rescaled(_dp(w), n, m, seed, _dp(xt), _dp(ls))
    if rc:
        raise ValueError("sample_linear_gaussian_rescaled: need m >= 4, strictly lower-triangular weights")
    return xt.T, ls


def run_pc_stable_device(c_ptr: int, ldc: int, p: int, sample_count: int, cfg: Optional[SkeletonConfig] = None,
                         with_sepsets: bool = False) -> SkeletonResult:
    """run_pc_stable on a correlation matrix already resident in device memory."""
    cfg = cfg or SkeletonConfig()
    abi = cfg._abi()
    h = ct.c_void_p()
    rc = library().pcs_run_pc_stable_device(ct.c_void_p(c_ptr), ldc, p, int(sample_count), ct.byref(abi),
                                            ct.byref(h))
    if rc:
        _raise(rc)
    try:
        return _collect(h, with_sepsets)
    finally:
        library().pcs_result_free(h)


def ci_test_batch(c, ell: int, ij, sets, tau: float):
    """stats::ci_test for many (i, j | S) of one level on the device.
    Returns (independent, z, rho, degenerate) arrays."""
    c = np.ascontiguousarray(c, np.float64)
    ij = np.ascontiguousarray(ij, np.int32).reshape(-1, 2)
    n = ij.shape[0]
    sets = np.ascontiguousarray(sets if ell > 0 else np.zeros((n, 1)), np.int32).reshape(n, max(ell, 1))
    ind = np.empty(n, np.uint8)
    deg = np.empty(n, np.uint8)
    z = np.empty(n, np.float64)
    rho = np.empty(n, np.float64)
    u8 = ct.POINTER(ct.c_uint8)
    rc = library().pcs_ci_test_batch(_dp(c), c.shape[0], ell, n, _ip(ij), _ip(sets), tau, ind.ctypes.data_as(u8),
                                     _dp(z), _dp(rho), deg.ctypes.data_as(u8))
    if rc:
        _raise(rc)
    return ind.astype(bool), z, rho, deg.astype(bool)


def pseudo_inverse_batch(a) -> np.ndarray:
    """stats::pseudo_inverse for a stack (n, ell, ell) on the device."""
    a = np.ascontiguousarray(a, np.float64)
    if a.ndim == 2:
        a = a[None]
    n, ell, _ = a.shape
    out = np.empty_like(a)
    rc = library().pcs_pseudo_inverse_batch(_dp(a), ell, n, _dp(out))
    if rc:
        _raise(rc)
    return out


class Session:
    """Level-stepped skeleton run (pcs_session_*).  Multi-GPU: every rank creates a session with
    shard_index/shard_count, runs each pass on its shard, and MIN-all-reduces keys() in between
    (see paper_1812_08491_b200/multigpu.py)."""

    def __init__(self, c=None, sample_count: int = 0, cfg: Optional[SkeletonConfig] = None, shard_index: int = 0,
                 shard_count: int = 1, device_ptr: Optional[int] = None, ldc: Optional[int] = None,
                 p: Optional[int] = None):
        cfg = cfg or SkeletonConfig()
        abi = cfg._abi(shard_index, shard_count)
        self._h = ct.c_void_p()
        L = library()
        if device_ptr is not None:
            rc = L.pcs_session_create_device(ct.c_void_p(device_ptr), ldc, p, int(sample_count), ct.byref(abi),
                                             ct.byref(self._h))
        else:
            c = np.ascontiguousarray(c, np.float64)
            rc = L.pcs_session_create(_dp(c), c.shape[0], int(sample_count), ct.byref(abi), ct.byref(self._h))
        if rc:
            self._h = None
            _raise(rc)

    def level_begin(self) -> tuple[bool, int, int]:
        running, ell, nk = ct.c_int32(), ct.c_int32(), ct.c_int64()
        rc = library().pcs_session_level_begin(self._h, ct.byref(running), ct.byref(ell), ct.byref(nk))
        if rc:
            _raise(rc)
        return bool(running.value), ell.value, nk.value

    def level_pass(self, pass_index: int):
        rc = library().pcs_session_level_pass(self._h, pass_index)
        if rc:
            _raise(rc)

    def level_passes(self) -> int:
        """1 when pass 0 tests both edge directions (cuPC-S levels >= 2), else 2."""
        n = ct.c_int32()
        rc = library().pcs_session_level_passes(self._h, ct.byref(n))
        if rc:
            _raise(rc)
        return n.value

    def keys(self) -> tuple[int, int]:
        ptr, n = ct.c_void_p(), ct.c_int64()
        rc = library().pcs_session_keys(self._h, ct.byref(ptr), ct.byref(n))
        if rc:
            _raise(rc)
        return ptr.value or 0, n.value

    def set_shard(self, shard_index: int, shard_count: int):
        rc = library().pcs_session_set_shard(self._h, shard_index, shard_count)
        if rc:
            _raise(rc)

    def snapshot(self, p: int, e_dir: Optional[int] = None):
        """CSR snapshot (offsets, indices) of the current level (compact(), core.hpp:227-239)."""
        off = np.empty(p + 1, np.int32)
        rc = library().pcs_session_snapshot(self._h, _ip(off), None)
        if rc:
            _raise(rc)
        idx = np.empty(max(int(off[-1]), 1), np.int32)
        rc = library().pcs_session_snapshot(self._h, _ip(off), _ip(idx))
        if rc:
            _raise(rc)
        return off, idx[: int(off[-1])]

    def level_end(self):
        rc = library().pcs_session_level_end(self._h)
        if rc:
            _raise(rc)

    def finish(self, with_sepsets: bool = True) -> SkeletonResult:
        h = ct.c_void_p()
        rc = library().pcs_session_finish(self._h, ct.byref(h))
        if rc:
            _raise(rc)
        try:
            return _collect(h, with_sepsets)
        finally:
            library().pcs_result_free(h)

    def close(self):
        if self._h:
            library().pcs_session_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------------------- orientation (orient.hpp)
class MixedGraph:
    """orient.hpp:15-32: directed (from, to) and undirected (a < b) pairs."""

    def __init__(self, n: int = 0, directed=(), undirected=()):
        self.n = int(n)
        self.directed = {(int(a), int(b)) for a, b in directed}
        self.undirected = {(min(int(a), int(b)), max(int(a), int(b))) for a, b in undirected}

    def has_directed(self, a: int, b: int) -> bool:
        return (a, b) in self.directed

    def has_undirected(self, a: int, b: int) -> bool:
        return (min(a, b), max(a, b)) in self.undirected

    def adjacent(self, a: int, b: int) -> bool:
        return self.has_undirected(a, b) or self.has_directed(a, b) or self.has_directed(b, a)

    def __eq__(self, other) -> bool:
        return (isinstance(other, MixedGraph) and self.n == other.n and self.directed == other.directed
                and self.undirected == other.undirected)

    def __repr__(self) -> str:
        return f"MixedGraph(n={self.n}, directed={sorted(self.directed)}, undirected={sorted(self.undirected)})"


def _collect_mixed(h) -> MixedGraph:
    L = library()
    try:
        nd, nu = L.pcs_mixed_directed_count(h), L.pcs_mixed_undirected_count(h)
        d = np.empty((max(nd, 1), 2), np.int32)
        u = np.empty((max(nu, 1), 2), np.int32)
        L.pcs_mixed_directed(h, _ip(d))
        L.pcs_mixed_undirected(h, _ip(u))
    finally:
        L.pcs_mixed_free(h)
    return d[:nd], u[:nu]


def _orient(skeleton, sepsets, stage: int, directed=()) -> MixedGraph:
    L = library()
    h = ct.c_void_p()
    if isinstance(skeleton, AdjacencyMatrix) and isinstance(sepsets, SeparationSets) and stage != 2:
        n = skeleton.n
        if sepsets.n != n:
            raise ValueError("find_v_structures: skeleton and sepsets sizes differ")
        bits = np.ascontiguousarray(skeleton.bits, np.uint32)
        rec = sepsets.records if len(sepsets.records) else np.zeros(1, np.int32)
        rc = L.pcs_orient_records(n, bits.ctypes.data_as(ct.POINTER(ct.c_uint32)), _ip(rec), len(sepsets.records),
                                  stage, ct.byref(h))
    else:
        cells = skeleton.cells if isinstance(skeleton, AdjacencyMatrix) else np.asarray(skeleton)
        n = cells.shape[0]
        adj = np.ascontiguousarray(cells != 0, np.uint8)
        sep = sepsets.as_dict() if isinstance(sepsets, SeparationSets) else dict(sepsets or {})
        if isinstance(sepsets, SeparationSets) and sepsets.n != n:
            raise ValueError("find_v_structures: skeleton and sepsets sizes differ")
        ns = max(n * (n - 1) // 2, 1)
        lvl = np.full(ns, -1, np.int32)
        off = np.zeros(ns, np.int64)
        mem = []
        for (i, j), st in sep.items():
            a, b = min(i, j), max(i, j)
            slot = a * (2 * n - a - 1) // 2 + (b - a - 1)
            lvl[slot] = len(st)
            off[slot] = len(mem)
            mem.extend(int(v) for v in st)
        mem = np.asarray(mem if mem else [0], np.int32)
        din = np.asarray(list(directed) if len(directed) else [(0, 0)], np.int32).reshape(-1, 2)
        rc = L.pcs_orient_skeleton(n, adj.ctypes.data_as(ct.POINTER(ct.c_uint8)), _ip(lvl),
                                   off.ctypes.data_as(ct.POINTER(ct.c_int64)), _ip(mem), stage, _ip(din),
                                   len(directed), ct.byref(h))
    if rc:
        _raise(rc)
    d, u = _collect_mixed(h)
    return MixedGraph(n, map(tuple, d.tolist()), map(tuple, u.tolist()))


def find_v_structures(skeleton, sepsets) -> MixedGraph:
    """orient.hpp:40-89 (unshielded-triple votes on the device)."""
    return _orient(skeleton, sepsets, 1)


def apply_meek_rules(g: MixedGraph) -> MixedGraph:
    """orient.hpp:147-167 (the reference's visiting order, on the host)."""
    adj = np.zeros((g.n, g.n), np.uint8)
    for a, b in list(g.directed) + list(g.undirected):
        adj[a, b] = adj[b, a] = 1
    return _orient(adj, None, 2, directed=sorted(g.directed))


def orient_skeleton(skeleton, sepsets) -> MixedGraph:
    """orient.hpp:170-173: v-structures then the Meek rules."""
    return _orient(skeleton, sepsets, 3)
