"""The sharded multi-GPU path (paper_1812_08491_b200/multigpu.py) on real device sessions: two ranks
share cuda:0 (the round's boxes have one GPU), each runs its half of every pass's work units and the
key arrays are MIN-all-reduced (host-staged over gloo here; NCCL on the device buffers in bench.py).
Every rank must end with the single-process device result, which equals the oracle's."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from tests.helpers import assert_same_result, instance

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, c, m, alpha, variant, out):
    import torch
    import torch.distributed as dist

    import paper_1812_08491_b200 as pcs
    from paper_1812_08491_b200.multigpu import host_staged_allreduce_min, run_pc_stable_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = c.shape[0]
    ldc = (p + 3) // 4 * 4
    cd = torch.zeros((p, ldc), dtype=torch.float64, device="cuda")
    cd[:, :p] = torch.from_numpy(c)
    torch.cuda.synchronize()
    cfg = pcs.SkeletonConfig(alpha=alpha, strategy=pcs.Strategy(variant))
    r = run_pc_stable_sharded(cd.data_ptr(), ldc, p, m, cfg, allreduce_min=host_staged_allreduce_min())
    out[rank] = (r.skeleton.cells.copy(), r.sepsets.as_dict(),
                 [(l.level, l.ci_tests, l.pseudo_inverses, l.edges_removed) for l in r.levels], r.stop_reason.value)
    dist.destroy_process_group()


@pytest.mark.parametrize("variant", ["set", "edge"])
def test_two_ranks_on_one_gpu_match_single_process(pcs, oracle, variant):
    m, alpha = 600, 0.05
    c = instance(oracle, 60, 0.3, m, 21)
    ref = oracle.run_pc_stable(c, m, alpha=alpha)
    single = pcs.run_pc_stable(c, m, pcs.SkeletonConfig(alpha=alpha, strategy=pcs.Strategy(variant)))
    assert_same_result(single, ref, label="single")
    world = 2
    out = mp.Manager().dict()
    mp.start_processes(_worker, args=(world, _free_port(), c, m, alpha, variant, out), nprocs=world, join=True,
                       start_method="spawn")
    for r in range(world):
        cells, sep, levels, stop = out[r]
        assert np.array_equal(cells, ref.adjacency), f"rank {r}: skeleton"
        assert sep == ref.sepsets, f"rank {r}: sepsets"
        assert [x[3] for x in levels] == [l.edges_removed for l in ref.levels], f"rank {r}: removed"
        assert [x[1] for x in levels] == [l.ci_tests for l in ref.levels], f"rank {r}: ci_tests"
        assert stop == ref.stop_reason


def _corr_worker(rank, world, port, x, out):
    import torch
    import torch.distributed as dist

    from paper_1812_08491_b200.multigpu import correlation_sharded, host_staged_all_gather, row_band

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p, m = x.shape
    ldc = (p + 3) // 4 * 4
    band = row_band(p, rank, world)[2]
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()  # (p, m): column-major m x p data
    c = torch.full((band * world, ldc), float("nan"), dtype=torch.float64, device="cuda")
    correlation_sharded(xd.data_ptr(), m, p, c, gather=host_staged_all_gather)
    out[rank] = c[:p, :p].cpu().numpy().copy()
    dist.destroy_process_group()


@pytest.mark.parametrize("p,world", [(203, 2), (150, 3)])
def test_correlation_row_split_matches_single_gpu(pcs, oracle, p, world):
    """Each rank builds its row band of C; after the all-gather every rank holds the single-GPU
    matrix bit for bit (and the oracle's FMA-order restatement)."""
    w = oracle.random_dag(p, 0.05, 3)
    x = oracle.sample_linear_gaussian(w, 777, 4)  # (p, m), m not a multiple of the k tile
    full = pcs.compute_correlation(x.T)
    assert np.array_equal(full.view(np.int64), oracle.compute_correlation_fma(x, threads=4).view(np.int64))
    out = mp.Manager().dict()
    mp.start_processes(_corr_worker, args=(world, _free_port(), x, out), nprocs=world, join=True,
                       start_method="spawn")
    for r in range(world):
        assert np.array_equal(out[r].view(np.int64), full.view(np.int64)), f"rank {r}"
