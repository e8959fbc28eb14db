"""C ABI checks that run without a GPU: the library loads, exports every symbol
include/pcstable_b200.h declares, its host-side functions agree bit-for-bit with the
oracle, and device entry points fail loudly (no CPU fallback) when no GPU exists."""
import ctypes as ct
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pcstable_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pcs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import paper_1812_08491_b200 as pcs
    lib = ct.CDLL(pcs.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, f"not exported: {missing}"


def test_library_is_built_for_sm100a():
    import subprocess
    import paper_1812_08491_b200 as pcs
    out = subprocess.run(["cuobjdump", "--list-elf", pcs.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_functions_match_oracle(oracle):
    import paper_1812_08491_b200 as pcs
    assert pcs.version().startswith("pcstable_b200")
    for alpha, m, ell in [(0.05, 1000, 0), (0.01, 10000, 3), (0.01, 63, 59), (0.5, 10, 2)]:
        assert pcs.threshold_tau(alpha, m, ell) == oracle.threshold_tau(alpha, m, ell)
    with pytest.raises(pcs.LevelUnreachableError):
        pcs.threshold_tau(0.05, 7, 4)
    with pytest.raises(ValueError):
        pcs.threshold_tau(0.0, 100, 0)
    w = pcs.random_dag(300, 0.05, 7919)
    assert np.array_equal(w, oracle.random_dag(300, 0.05, 7919))
    x = pcs.sample_linear_gaussian(w, 400, 7920)
    assert np.array_equal(x.T, oracle.sample_linear_gaussian(w, 400, 7920))


def test_config_validation_without_gpu():
    import paper_1812_08491_b200 as pcs
    for bad in (dict(alpha=0.0), dict(alpha=1.0), dict(max_level=-3), dict(edges_per_unit=0), dict(set_groups=0),
                dict(unit_width=0), dict(workers_per_edge=0)):
        with pytest.raises(ValueError):
            pcs.SkeletonConfig(**bad).validate()


def test_device_path_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1812_08491_b200 as pcs
    with pytest.raises(pcs.PcsError):
        pcs.run_pc_stable(np.eye(4), 100)
    with pytest.raises(pcs.PcsError):
        pcs.compute_correlation(np.random.default_rng(0).normal(size=(10, 3)))


def test_rescaled_generator_is_the_reference_generator_scaled(oracle):
    """pcs_sample_linear_gaussian_rescaled (the C5 scaling shapes' generator): same noise stream as
    datagen.hpp:62-82, every column divided by the reference column's RMS, so the correlation matrix is
    the reference generator's; finite where the reference overflows."""
    import paper_1812_08491_b200 as pcs
    w = oracle.random_dag(60, 0.15, 77)
    ref = oracle.sample_linear_gaussian(w, 400, 78).T  # (m, n) like the product's
    x, ls = pcs.sample_linear_gaussian_rescaled(w, 400, 78)
    scale = np.exp(ls)
    assert np.allclose(np.sqrt((ref ** 2).mean(axis=0)), scale, rtol=1e-12, atol=0)
    assert np.max(np.abs(x * scale - ref) / scale) < 1e-12
    assert np.abs(oracle.compute_correlation(x.T) - oracle.compute_correlation(ref.T)).max() < 1e-12
    # dense and deep: the reference generator's values overflow, the rescaled ones stay at unit RMS
    w = oracle.random_dag(1800, 0.95, 5)
    with np.errstate(all="ignore"):
        big = oracle.sample_linear_gaussian(w, 8, 6)
    assert not np.isfinite(big).all()
    x, ls = pcs.sample_linear_gaussian_rescaled(w, 8, 6)
    assert np.isfinite(x).all() and np.isfinite(ls).all() and ls.max() > 709.0
    assert np.allclose((x ** 2).mean(axis=0), 1.0, rtol=1e-12)


@pytest.mark.parametrize("seed,p,m", [(5, 7, 11), (7919, 100, 1000), (3, 1000, 301)])
def test_noise_stream_is_the_sequential_stream(oracle, seed, p, m):
    """pcs_noise_stream (jump-ahead chunks of 65536 outputs on the host threads) == the reference's
    sequential xoshiro256++ / polar stream (rng.hpp), restated by the oracle; the larger shapes cross
    several chunk boundaries, and an odd count drops the last spare."""
    import paper_1812_08491_b200 as pcs
    got = pcs.noise_stream(seed, p * m, p, m)
    want = oracle.normals(seed, p * m).reshape(m, p).T
    assert np.array_equal(got.view(np.int64), want.view(np.int64))
    odd = pcs.noise_stream(seed, p * m - 1, p, m)
    assert np.array_equal(odd.T.reshape(-1)[:p * m - 1].view(np.int64), want.T.reshape(-1)[:p * m - 1].view(np.int64))
