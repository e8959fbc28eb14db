"""ctypes binding of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module.  It loads oracle/libpcs_oracle.so (built
by oracle/Makefile, see __graft_entry__.build()).
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpcs_oracle.so")

OK, EINVAL, EZEROVAR, EOVERFLOW, ENAN, ELEVEL, ENOMEM = range(7)
SERIAL, EDGE, SET, KEYS, FAST = range(5)
STOP_NAMES = {0: "max-degree", 1: "level-cap", 2: "sample-size"}
NONE_KEY = (1 << 63) - 1


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class OrcConfig(ct.Structure):
    _fields_ = [
        ("alpha", ct.c_double),
        ("max_level", ct.c_int),
        ("strategy", ct.c_int),
        ("edges_per_unit", ct.c_int),
        ("workers_per_edge", ct.c_int),
        ("set_groups", ct.c_int),
        ("unit_width", ct.c_int),
        ("worker_count", ct.c_int),
        ("has_schedule_seed", ct.c_int),
        ("schedule_seed", ct.c_uint64),
    ]


class OrcLevel(ct.Structure):
    _fields_ = [
        ("level", ct.c_int32),
        ("pad", ct.c_int32),
        ("ci_tests", ct.c_uint64),
        ("pseudo_inverses", ct.c_uint64),
        ("edges_removed", ct.c_uint64),
        ("elapsed_s", ct.c_double),
    ]


_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ct.CDLL(LIB_PATH)
        dp = ct.POINTER(ct.c_double)
        ip = ct.POINTER(ct.c_int32)
        L.orc_last_error.restype = ct.c_char_p
        L.orc_binomial.argtypes = [ct.c_int, ct.c_int, ct.POINTER(ct.c_uint64)]
        L.orc_unrank_positions.argtypes = [ct.c_int, ct.c_int, ct.c_uint64, ip]
        L.orc_unrank_positions_excluding.argtypes = [ct.c_int, ct.c_int, ct.c_uint64, ct.c_int, ip]
        L.orc_next_combination.argtypes = [ip, ct.c_int, ct.c_int]
        L.orc_normal_quantile.argtypes = [ct.c_double, dp]
        L.orc_fisher_z.argtypes = [ct.c_double, dp]
        L.orc_threshold_tau.argtypes = [ct.c_double, ct.c_int, ct.c_int, dp]
        L.orc_compute_correlation.argtypes = [dp, ct.c_int, ct.c_int, dp, ct.POINTER(ct.c_int), ct.c_int]
        L.orc_compute_correlation_fma.argtypes = [dp, ct.c_int, ct.c_int, ct.c_int, dp, ct.POINTER(ct.c_int), ct.c_int]
        L.orc_correlation_normalize.argtypes = [dp, ct.c_int]
        L.orc_pseudo_inverse.argtypes = [dp, ct.c_int, dp]
        L.orc_partial_correlation.argtypes = [dp, ct.c_int, ct.c_int, ct.c_int, ip, ct.c_int, dp, ct.POINTER(ct.c_int)]
        L.orc_ci_test.argtypes = [dp, ct.c_int, ct.c_int, ct.c_int, ip, ct.c_int, ct.c_double,
                                  ct.POINTER(ct.c_int), dp, dp, ct.POINTER(ct.c_int)]
        L.orc_random_dag.argtypes = [ct.c_int, ct.c_double, ct.c_uint64, dp]
        L.orc_sample_linear_gaussian.argtypes = [dp, ct.c_int, ct.c_int, ct.c_uint64, dp]
        L.orc_normals.argtypes = [ct.c_uint64, dp, ct.c_int64]
        L.orc_raw.argtypes = [ct.c_uint64, ct.POINTER(ct.c_uint64), ct.c_int64]
        L.orc_config_default.argtypes = [ct.POINTER(OrcConfig)]
        L.orc_run_pc_stable.argtypes = [dp, ct.c_int, ct.c_int, ct.POINTER(OrcConfig), ct.POINTER(ct.c_void_p)]
        L.orc_result_levels.argtypes = [ct.c_void_p, ct.POINTER(OrcLevel), ct.c_int]
        L.orc_result_stop_reason.argtypes = [ct.c_void_p]
        L.orc_result_adjacency.argtypes = [ct.c_void_p, ct.POINTER(ct.c_uint8)]
        L.orc_result_member_total.argtypes = [ct.c_void_p]
        L.orc_result_member_total.restype = ct.c_int64
        L.orc_result_sepsets.argtypes = [ct.c_void_p, ip, ct.POINTER(ct.c_int64), ip]
        L.orc_result_free.argtypes = [ct.c_void_p]
        L.orc_level_keys.argtypes = [dp, ct.c_int, ip, ip, ct.c_int, ct.c_double, ct.c_int64, ct.c_int64,
                                     ct.POINTER(ct.c_int64), ct.c_int]
        L.orc_level_keys_fast.argtypes = [dp, ct.c_int, ip, ip, ct.c_int, ct.c_double, ct.POINTER(ct.c_int64),
                                          ct.c_int]
        L.orc_orient.argtypes = [ct.c_int, ct.POINTER(ct.c_uint8), ip, ct.POINTER(ct.c_int64), ip, ct.c_int, ip,
                                 ct.c_int64, ip, ct.POINTER(ct.c_int64), ip, ct.POINTER(ct.c_int64)]
        _lib = L
    return _lib


def _check(rc: int):
    if rc != OK:
        raise OracleError(rc, lib().orc_last_error().decode())


def _dp(a):
    return a.ctypes.data_as(ct.POINTER(ct.c_double))


def _ip(a):
    return a.ctypes.data_as(ct.POINTER(ct.c_int32))


# ---------------------------------------------------------------- comb / stats
def binomial(n: int, k: int) -> int:
    out = ct.c_uint64()
    _check(lib().orc_binomial(n, k, ct.byref(out)))
    return out.value


def unrank_positions(width: int, ell: int, t: int) -> list[int]:
    out = np.zeros(max(ell, 1), np.int32)
    _check(lib().orc_unrank_positions(width, ell, t, _ip(out)))
    return out[:ell].tolist()


def unrank_positions_excluding(reduced_width: int, ell: int, t: int, skip: int) -> list[int]:
    out = np.zeros(max(ell, 1), np.int32)
    _check(lib().orc_unrank_positions_excluding(reduced_width, ell, t, skip, _ip(out)))
    return out[:ell].tolist()


def next_combination(pos: list[int], width: int):
    a = np.asarray(pos, np.int32).copy()
    ok = lib().orc_next_combination(_ip(a), len(pos), width)
    return bool(ok), a.tolist()


def normal_quantile(p: float) -> float:
    out = ct.c_double()
    _check(lib().orc_normal_quantile(p, ct.byref(out)))
    return out.value


def fisher_z(rho: float) -> float:
    out = ct.c_double()
    _check(lib().orc_fisher_z(rho, ct.byref(out)))
    return out.value


def threshold_tau(alpha: float, m: int, ell: int) -> float:
    out = ct.c_double()
    _check(lib().orc_threshold_tau(alpha, m, ell, ct.byref(out)))
    return out.value


def compute_correlation(x_colmajor: np.ndarray, threads: int = 1) -> np.ndarray:
    """x: (p, m) array whose rows are the variables (== Eigen col-major m x p)."""
    x = np.ascontiguousarray(x_colmajor, np.float64)
    p, m = x.shape
    c = np.empty((p, p), np.float64)
    zc = ct.c_int(-1)
    rc = lib().orc_compute_correlation(_dp(x), m, p, _dp(c), ct.byref(zc), threads)
    if rc == EZEROVAR:
        e = OracleError(rc, lib().orc_last_error().decode())
        e.column = zc.value
        raise e
    _check(rc)
    return c


DEVICE_KPAD = 32  # the device Gram's k-chunk (csrc/corr.cu kGK)


def compute_correlation_fma(x_colmajor: np.ndarray, threads: int = 1, kpad: int = DEVICE_KPAD) -> np.ndarray:
    """compute_correlation in the device's pinned order (tree means, FMA-chain Gram); x as above."""
    x = np.ascontiguousarray(x_colmajor, np.float64)
    p, m = x.shape
    c = np.empty((p, p), np.float64)
    zc = ct.c_int(-1)
    rc = lib().orc_compute_correlation_fma(_dp(x), m, p, kpad, _dp(c), ct.byref(zc), threads)
    if rc == EZEROVAR:
        e = OracleError(rc, lib().orc_last_error().decode())
        e.column = zc.value
        raise e
    _check(rc)
    return c


def normalize_correlation(c: np.ndarray) -> np.ndarray:
    a = np.array(c, np.float64, order="C", copy=True)
    _check(lib().orc_correlation_normalize(_dp(a), a.shape[0]))
    return a


def pseudo_inverse(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, np.float64)
    n = a.shape[0]
    if a.ndim != 2 or a.shape[1] != n:
        raise OracleError(EINVAL, "pseudo_inverse: matrix must be square")
    out = np.empty_like(a)
    _check(lib().orc_pseudo_inverse(_dp(a), n, _dp(out)))
    return out


def partial_correlation(c: np.ndarray, i: int, j: int, s) -> tuple[float, bool]:
    c = np.ascontiguousarray(c, np.float64)
    s = list(s)
    return _pc(c, i, j, np.asarray(s if s else [0], np.int32), len(s))


def _pc(c, i, j, s_arr, ell=None):
    ell = len(s_arr) if ell is None else ell
    rho = ct.c_double()
    deg = ct.c_int()
    _check(lib().orc_partial_correlation(_dp(c), c.shape[0], i, j, _ip(s_arr), ell, ct.byref(rho), ct.byref(deg)))
    return rho.value, bool(deg.value)


def ci_test(c: np.ndarray, i: int, j: int, s, tau: float):
    """Returns (independent, z, rho, degenerate) like stats::ci_test."""
    c = np.ascontiguousarray(c, np.float64)
    s = list(s)
    arr = np.asarray(s if s else [0], np.int32)
    ind, deg = ct.c_int(), ct.c_int()
    z, rho = ct.c_double(), ct.c_double()
    _check(lib().orc_ci_test(_dp(c), c.shape[0], i, j, _ip(arr), len(s), tau, ct.byref(ind), ct.byref(z),
                             ct.byref(rho), ct.byref(deg)))
    return bool(ind.value), z.value, rho.value, bool(deg.value)


# ---------------------------------------------------------------- datagen
def random_dag(n: int, density: float, seed: int) -> np.ndarray:
    w = np.empty((n, n), np.float64)
    _check(lib().orc_random_dag(n, density, seed, _dp(w)))
    return w


def sample_linear_gaussian(weights: np.ndarray, m: int, seed: int) -> np.ndarray:
    """Returns (p, m): row j = samples of variable j (== Eigen col-major m x p)."""
    w = np.ascontiguousarray(weights, np.float64)
    n = w.shape[0]
    x = np.empty((n, m), np.float64)
    _check(lib().orc_sample_linear_gaussian(_dp(w), n, m, seed, _dp(x)))
    return x


def normals(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().orc_normals(seed, _dp(out), n)
    return out


def raw(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint64)
    lib().orc_raw(seed, out.ctypes.data_as(ct.POINTER(ct.c_uint64)), n)
    return out


# ---------------------------------------------------------------- skeleton
@dataclass
class LevelStats:
    level: int
    ci_tests: int
    pseudo_inverses: int
    edges_removed: int
    elapsed_s: float


@dataclass
class SkeletonResult:
    p: int
    adjacency: np.ndarray            # (p, p) uint8
    sepsets: dict = field(default_factory=dict)   # (i, j) i<j -> tuple(members)
    levels: list = field(default_factory=list)
    stop_reason: str = "max-degree"

    def levels_run(self) -> int:
        return len(self.levels)

    def edge_set(self):
        iu = np.argwhere(np.triu(self.adjacency, 1))
        return [tuple(map(int, e)) for e in iu]


def config(alpha=0.05, max_level=None, strategy=SERIAL, workers=1, edges_per_unit=2, set_groups=2,
           unit_width=64, schedule_seed=None) -> OrcConfig:
    cfg = OrcConfig()
    lib().orc_config_default(ct.byref(cfg))
    cfg.alpha = alpha
    cfg.max_level = -1 if max_level is None else max_level
    cfg.strategy = strategy
    cfg.worker_count = workers
    cfg.edges_per_unit = edges_per_unit
    cfg.set_groups = set_groups
    cfg.unit_width = unit_width
    if schedule_seed is not None:
        cfg.has_schedule_seed = 1
        cfg.schedule_seed = schedule_seed
    return cfg


def run_pc_stable(c: np.ndarray, m: int, cfg: OrcConfig | None = None, **kw) -> SkeletonResult:
    c = np.ascontiguousarray(c, np.float64)
    p = c.shape[0]
    cfg = cfg or config(**kw)
    h = ct.c_void_p()
    _check(lib().orc_run_pc_stable(_dp(c), p, m, ct.byref(cfg), ct.byref(h)))
    try:
        lv = (OrcLevel * 128)()
        n = lib().orc_result_levels(h, lv, 128)
        levels = [LevelStats(lv[k].level, lv[k].ci_tests, lv[k].pseudo_inverses, lv[k].edges_removed,
                             lv[k].elapsed_s) for k in range(n)]
        adj = np.empty((p, p), np.uint8)
        lib().orc_result_adjacency(h, adj.ctypes.data_as(ct.POINTER(ct.c_uint8)))
        tot = lib().orc_result_member_total(h)
        ns = p * (p - 1) // 2
        lvl = np.empty(ns, np.int32)
        off = np.empty(ns, np.int64)
        mem = np.empty(max(tot, 1), np.int32)
        lib().orc_result_sepsets(h, _ip(lvl), off.ctypes.data_as(ct.POINTER(ct.c_int64)), _ip(mem))
        reason = STOP_NAMES[lib().orc_result_stop_reason(h)]
    finally:
        lib().orc_result_free(h)
    sep = {}
    iu, ju = np.triu_indices(p, 1)
    for s in np.nonzero(lvl >= 0)[0]:
        sep[(int(iu[s]), int(ju[s]))] = tuple(int(v) for v in mem[off[s]:off[s] + lvl[s]])
    return SkeletonResult(p, adj, sep, levels, reason)


@dataclass
class ResultArrays:
    """A run's result without per-pair Python objects: adjacency (p, p) uint8, per unordered-pair
    slot (core.hpp:329-335, ascending (i, j), i < j) the sepset length (-1: none) and its members."""
    p: int
    adjacency: np.ndarray
    slot_len: np.ndarray      # int32[p(p-1)/2]
    slot_off: np.ndarray      # int64[p(p-1)/2]
    members: np.ndarray       # int32[total]
    levels: list
    stop_reason: str


def run_pc_stable_arrays(c: np.ndarray, m: int, cfg: OrcConfig | None = None, **kw) -> ResultArrays:
    c = np.ascontiguousarray(c, np.float64)
    p = c.shape[0]
    cfg = cfg or config(**kw)
    h = ct.c_void_p()
    _check(lib().orc_run_pc_stable(_dp(c), p, m, ct.byref(cfg), ct.byref(h)))
    try:
        lv = (OrcLevel * 128)()
        n = lib().orc_result_levels(h, lv, 128)
        levels = [LevelStats(lv[k].level, lv[k].ci_tests, lv[k].pseudo_inverses, lv[k].edges_removed,
                             lv[k].elapsed_s) for k in range(n)]
        adj = np.empty((p, p), np.uint8)
        lib().orc_result_adjacency(h, adj.ctypes.data_as(ct.POINTER(ct.c_uint8)))
        tot = lib().orc_result_member_total(h)
        ns = p * (p - 1) // 2
        lvl = np.empty(ns, np.int32)
        off = np.empty(ns, np.int64)
        mem = np.empty(max(tot, 1), np.int32)
        lib().orc_result_sepsets(h, _ip(lvl), off.ctypes.data_as(ct.POINTER(ct.c_int64)), _ip(mem))
        reason = STOP_NAMES[lib().orc_result_stop_reason(h)]
    finally:
        lib().orc_result_free(h)
    return ResultArrays(p, adj, lvl, off, mem[:tot], levels, reason)


def level_keys(c: np.ndarray, offsets: np.ndarray, indices: np.ndarray, ell: int, tau: float,
               e_begin: int = 0, e_end: int | None = None, threads: int = 1) -> np.ndarray:
    c = np.ascontiguousarray(c, np.float64)
    p = c.shape[0]
    off = np.ascontiguousarray(offsets, np.int32)
    idx = np.ascontiguousarray(indices if len(indices) else np.zeros(1, np.int32), np.int32)
    rows = np.repeat(np.arange(p, dtype=np.int64), np.diff(off.astype(np.int64)))
    ne = int((idx[:len(rows)] > rows).sum())
    e_end = ne if e_end is None else min(e_end, ne)
    keys = np.full(max(e_end - e_begin, 1), NONE_KEY, np.int64)
    _check(lib().orc_level_keys(_dp(c), p, _ip(off), _ip(idx), ell, tau, e_begin, e_end,
                                keys.ctypes.data_as(ct.POINTER(ct.c_int64)), threads))
    return keys[:max(e_end - e_begin, 0)]


def level_keys_fast(c: np.ndarray, offsets: np.ndarray, indices: np.ndarray, ell: int, tau: float,
                    threads: int = 1) -> np.ndarray:
    """level_keys over every edge of the snapshot by set-shared evaluation (same keys)."""
    c = np.ascontiguousarray(c, np.float64)
    p = c.shape[0]
    off = np.ascontiguousarray(offsets, np.int32)
    idx = np.ascontiguousarray(indices if len(indices) else np.zeros(1, np.int32), np.int32)
    rows = np.repeat(np.arange(p, dtype=np.int64), np.diff(off.astype(np.int64)))
    ne = int((idx[:len(rows)] > rows).sum())
    keys = np.full(max(ne, 1), NONE_KEY, np.int64)
    _check(lib().orc_level_keys_fast(_dp(c), p, _ip(off), _ip(idx), ell, tau,
                                     keys.ctypes.data_as(ct.POINTER(ct.c_int64)), threads))
    return keys[:ne]


def run_level(c: np.ndarray, offsets: np.ndarray, indices: np.ndarray, ell: int, tau: float,
              cfg: OrcConfig, row_begin: int = 0, row_end: int | None = None) -> LevelStats:
    """One level of a reference strategy on a given snapshot, rows [row_begin, row_end) only."""
    c = np.ascontiguousarray(c, np.float64)
    p = c.shape[0]
    off = np.ascontiguousarray(offsets, np.int32)
    idx = np.ascontiguousarray(indices if len(indices) else np.zeros(1, np.int32), np.int32)
    st = OrcLevel()
    lib().orc_run_level.argtypes = [ct.POINTER(ct.c_double), ct.c_int, ct.POINTER(ct.c_int32),
                                    ct.POINTER(ct.c_int32), ct.c_int, ct.c_double, ct.POINTER(OrcConfig),
                                    ct.c_int, ct.c_int, ct.POINTER(OrcLevel)]
    _check(lib().orc_run_level(_dp(c), p, _ip(off), _ip(idx), ell, tau, ct.byref(cfg), row_begin,
                               p if row_end is None else row_end, ct.byref(st)))
    return LevelStats(st.level, st.ci_tests, st.pseudo_inverses, st.edges_removed, st.elapsed_s)


def run_level_sampled(c: np.ndarray, offsets: np.ndarray, indices: np.ndarray, ell: int, tau: float,
                      cfg: OrcConfig, keep_stride: int) -> LevelStats:
    """run_level with only every keep_stride-th unit chunk of each row (cfg.strategy must be SET)."""
    c = np.ascontiguousarray(c, np.float64)
    p = c.shape[0]
    off = np.ascontiguousarray(offsets, np.int32)
    idx = np.ascontiguousarray(indices if len(indices) else np.zeros(1, np.int32), np.int32)
    st = OrcLevel()
    lib().orc_run_level_sampled.argtypes = [ct.POINTER(ct.c_double), ct.c_int, ct.POINTER(ct.c_int32),
                                            ct.POINTER(ct.c_int32), ct.c_int, ct.c_double, ct.POINTER(OrcConfig),
                                            ct.c_int, ct.c_int, ct.c_int, ct.POINTER(OrcLevel)]
    _check(lib().orc_run_level_sampled(_dp(c), p, _ip(off), _ip(idx), ell, tau, ct.byref(cfg), 0, p, keep_stride,
                                       ct.byref(st)))
    return LevelStats(st.level, st.ci_tests, st.pseudo_inverses, st.edges_removed, st.elapsed_s)


# ---------------------------------------------------------------- orient.hpp
class MixedGraph:
    """orient.hpp:15-32: directed (from, to) pairs and undirected (a < b) pairs, ascending."""

    def __init__(self, n: int, directed, undirected):
        self.n = n
        self.directed = sorted((int(a), int(b)) for a, b in directed)
        self.undirected = sorted((min(int(a), int(b)), max(int(a), int(b))) for a, b in undirected)

    def __eq__(self, other):
        return (self.n, self.directed, self.undirected) == (other.n, other.directed, other.undirected)

    def __repr__(self):
        return f"MixedGraph(n={self.n}, directed={self.directed}, undirected={self.undirected})"


def _sep_layout(n: int, sepsets: dict):
    ns = n * (n - 1) // 2
    lvl = np.full(max(ns, 1), -1, np.int32)
    off = np.zeros(max(ns, 1), np.int64)
    mem = []
    for (i, j), s in sepsets.items():
        a, b = min(i, j), max(i, j)
        slot = a * (2 * n - a - 1) // 2 + (b - a - 1)
        lvl[slot] = len(s)
        off[slot] = len(mem)
        mem.extend(int(v) for v in s)
    return lvl, off, np.asarray(mem if mem else [0], np.int32)


def orient(n: int, skeleton: np.ndarray, sepsets: dict, stage: int = 3, directed=()) -> MixedGraph:
    """stage 1: find_v_structures, 2: apply_meek_rules (on skeleton + `directed`), 3: orient_skeleton."""
    adj = np.ascontiguousarray(skeleton, np.uint8)
    lvl, off, mem = _sep_layout(n, sepsets)
    din = np.asarray(list(directed) if len(directed) else [(0, 0)], np.int32).reshape(-1, 2)
    cap = max(n * (n - 1) // 2, 1)
    dout = np.empty((cap, 2), np.int32)
    uout = np.empty((cap, 2), np.int32)
    nd, nu = ct.c_int64(), ct.c_int64()
    _check(lib().orc_orient(n, adj.ctypes.data_as(ct.POINTER(ct.c_uint8)), _ip(lvl),
                            off.ctypes.data_as(ct.POINTER(ct.c_int64)), _ip(mem), stage, _ip(din),
                            len(directed), _ip(dout), ct.byref(nd), _ip(uout), ct.byref(nu)))
    return MixedGraph(n, [tuple(r) for r in dout[:nd.value]], [tuple(r) for r in uout[:nu.value]])
