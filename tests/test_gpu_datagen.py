"""The device generator (pcs_sample_linear_gaussian_device, csrc/datagen_dev.cu):
the reference generator's noise stream (jump-ahead parallel on the host, bit-identical to the sequential
xoshiro256++ / polar stream) and the structural equations on the device.  Both variants must equal the
host generators bit for bit -- the plain one is the reference's datagen.hpp:62-82 (itself equal to the
oracle's restatement), the rescaled one the overflow-safe C5 generator -- and the C5 fixture's data
digest must come out of the device path unchanged."""
import hashlib
import os
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _device(pcs, w, m, seed, rescaled):
    import torch

    n = w.shape[0]
    x = torch.empty((n, m), dtype=torch.float64, device="cuda")  # m x n column-major
    t0 = time.time()
    ls = pcs.sample_linear_gaussian_device(w, m, seed, x.data_ptr(), rescaled=rescaled)
    dt = time.time() - t0
    return x.cpu().numpy(), ls, dt


@pytest.mark.parametrize("n,m,d,seed", [(7, 5, 0.5, 3), (100, 1000, 2 / 99, 1), (300, 257, 0.2, 11),
                                        (1000, 10000, 0.1, 7920)])
def test_plain_generator_matches_reference_stream(pcs, oracle, n, m, d, seed):
    w = pcs.random_dag(n, d, seed - 1 if seed > 1 else 0)
    got, _, dt = _device(pcs, w, m, seed, False)
    want = np.ascontiguousarray(pcs.sample_linear_gaussian(w, m, seed).T)  # (n, m)
    ref = oracle.sample_linear_gaussian(w, m, seed)                       # the oracle's restatement
    assert np.array_equal(want.view(np.int64), ref.view(np.int64))
    bad = int((got.view(np.int64) != want.view(np.int64)).sum())
    assert bad == 0, f"{bad} of {got.size} values differ"
    print(f"plain n={n} m={m}: device generator {dt * 1e3:.1f} ms")


@pytest.mark.parametrize("n,m,d,seed", [(50, 64, 0.3, 5), (400, 1000, 0.1, 9), (2000, 5000, 0.05, 4 * 7919 + 1)])
def test_rescaled_generator_matches_host(pcs, n, m, d, seed):
    w = pcs.random_dag(n, d, seed - 1)
    got, ls, dt = _device(pcs, w, m, seed, True)
    want, wls = pcs.sample_linear_gaussian_rescaled(w, m, seed)
    want = np.ascontiguousarray(np.asarray(want).T)
    bad = int((got.view(np.int64) != want.view(np.int64)).sum())
    assert bad == 0, f"{bad} of {got.size} values differ"
    assert np.allclose(ls, wls, rtol=0, atol=1e-9)
    print(f"rescaled n={n} m={m}: device generator {dt * 1e3:.1f} ms")


def test_c5_fixture_data_from_the_device(pcs):
    g = dict(np.load(os.path.join(GOLD, "c5_5000_full.npz")))
    p, m, d, seed = int(g["p"]), int(g["m"]), float(g["density"]), int(g["seed"])
    w = pcs.random_dag(p, d, seed)
    got, _, dt = _device(pcs, w, m, seed + 1, True)
    assert hashlib.sha256(got.tobytes()).hexdigest() == str(g["data_sha256"])
    print(f"C5 p={p} m={m}: device generator {dt:.2f} s")
