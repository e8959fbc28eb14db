"""World-size-2 check of the multi-GPU orchestration (paper_1812_08491_b200/multigpu.py)
on CPU: the same level loop drives an oracle-backed session whose passes compute the
serial-rule keys of their shard only; keys are MIN-all-reduced over gloo exactly as the
device sessions MIN-all-reduce over NCCL.  Every rank must end with the single-process
skeleton, sepsets and per-level counters."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from tests.helpers import instance

NONE = (1 << 63) - 1


class OracleSession:
    """The pcs_session protocol on the CPU oracle (test double for the device session)."""

    def __init__(self, O, c, m, alpha, rank, world):
        self.O, self.c, self.m, self.alpha, self.rank, self.world = O, c, m, alpha, rank, world
        p = c.shape[0]
        self.adj = ~np.eye(p, dtype=bool)
        self.ell = -1
        self.levels = []
        self.sep = {}
        self.stopped = False

    def level_begin(self):
        O, p = self.O, self.c.shape[0]
        ell = self.ell + 1
        try:
            self.tau = O.threshold_tau(self.alpha, self.m, ell)
        except O.OracleError:
            return False, ell, 0
        self.ell = ell
        if ell == 0:
            return True, 0, 0
        deg = self.adj.sum(axis=1)
        if deg.max() - 1 < ell:
            self.ell -= 1
            return False, ell, 0
        self.off = np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)
        self.idx = np.concatenate([np.nonzero(self.adj[i])[0] for i in range(p)]).astype(np.int32)
        self.ne = int(np.triu(self.adj, 1).sum())
        self.keys = np.full(self.ne, NONE, np.int64)
        return True, ell, self.ne

    def level_pass(self, pass_index):
        if self.ell == 0 or pass_index == 1:  # the oracle computes both directions in one go
            return
        e0 = self.ne * self.rank // self.world
        e1 = self.ne * (self.rank + 1) // self.world
        self.keys[e0:e1] = self.O.level_keys(self.c, self.off, self.idx, self.ell, self.tau, e0, e1)

    def keys_tensor(self):
        return self.keys

    def level_end(self):
        O, p = self.O, self.c.shape[0]
        if self.ell == 0:
            rho = np.clip(self.c, -(1 - 1e-12), 1 - 1e-12)
            z = np.abs(0.5 * np.log((1 + rho) / (1 - rho)))
            rm = np.triu((z <= self.tau) & self.adj, 1)
            self.adj &= ~(rm | rm.T)
            for i, j in zip(*np.nonzero(rm)):
                self.sep[(int(i), int(j))] = ()
            self.levels.append(int(rm.sum()))
            return
        e, removed = 0, 0
        for a in range(p):
            for q in range(self.off[a], self.off[a + 1]):
                b = int(self.idx[q])
                if b <= a:
                    continue
                k = int(self.keys[e]); e += 1
                if k == NONE:
                    continue
                d, rk = k >> 62, k & ((1 << 62) - 1)
                r = b if d else a
                row = self.idx[self.off[r]:self.off[r + 1]]
                skip = int(np.searchsorted(row, a if d else b))
                pos = O.unrank_positions_excluding(len(row) - 1, self.ell, rk, skip)
                self.sep[(a, b)] = tuple(int(row[v]) for v in pos)
                self.adj[a, b] = self.adj[b, a] = False
                removed += 1
        self.levels.append(removed)


def _worker(rank, world, port, c, m, alpha, out):
    import torch
    import torch.distributed as dist

    from oracle import pyoracle as O
    from paper_1812_08491_b200.multigpu import level_loop

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = OracleSession(O, c, m, alpha, rank, world)

    class _Adapter:
        def level_begin(self):
            return s.level_begin()

        def level_pass(self, i):
            s.level_pass(i)

        def keys(self):
            return s.keys, len(s.keys)

        def level_end(self):
            s.level_end()

    def allreduce_min(keys, n):
        t = torch.from_numpy(keys)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)

    level_loop(_Adapter(), allreduce_min, world)
    out[rank] = (s.adj.copy(), dict(s.sep), list(s.levels))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


@pytest.mark.parametrize("seed", [3, 11])
def test_two_rank_gloo_matches_single_process(oracle, seed):
    c = instance(oracle, 40, 0.25, 600, seed)
    ref = oracle.run_pc_stable(c, 600, alpha=0.05)
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), c, 600, 0.05, out), nprocs=world, join=True,
                       start_method="spawn")
    for r in range(world):
        adj, sep, removed = out[r]
        assert np.array_equal(adj.astype(np.uint8), ref.adjacency)
        assert sep == ref.sepsets
        assert removed == [l.edges_removed for l in ref.levels]
