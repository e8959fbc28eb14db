"""The NCCL code path of the multi-GPU orchestration (paper_1812_08491_b200/multigpu.py) on the
one-GPU box: a world-size-1 NCCL process group (communicator init over 127.0.0.1), the device-buffer
MIN all-reduce of a key array (torch_allreduce_min, exactly what bench.py --gpus N uses between
passes), and a whole sharded run through run_pc_stable_sharded with the NCCL reducer -- identical to
the oracle.  (World size > 1 needs more GPUs than these boxes have; the N-rank orchestration itself is
covered with gloo in test_multigpu_gloo.py / test_gpu_multiproc.py.)"""
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


def _worker(rank, port, c, m, alpha, out):
    import torch
    import torch.distributed as dist

    import paper_1812_08491_b200 as pcs
    from paper_1812_08491_b200.multigpu import _CudaArray, run_pc_stable_sharded, torch_allreduce_min

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    # 1. the key reducer on a device buffer (int64 keys, NONE = INT64_MAX)
    keys = torch.tensor([5, (1 << 63) - 1, (1 << 62) | 3, 0], dtype=torch.int64, device="cuda")
    torch_allreduce_min()(keys.data_ptr(), keys.numel())
    out["keys"] = keys.cpu().numpy().tolist()
    # the same through the library-owned-buffer view
    t = torch.as_tensor(_CudaArray(keys.data_ptr(), keys.numel()), device="cuda")
    out["view_ok"] = bool(t.data_ptr() == keys.data_ptr())
    # 2. a whole sharded run with the NCCL reducer
    p = c.shape[0]
    ldc = (p + 3) // 4 * 4
    cd = torch.zeros((p, ldc), dtype=torch.float64, device="cuda")
    cd[:, :p] = torch.from_numpy(c)
    torch.cuda.synchronize()
    r = run_pc_stable_sharded(cd.data_ptr(), ldc, p, m, pcs.SkeletonConfig(alpha=alpha),
                              allreduce_min=torch_allreduce_min())
    out["cells"] = r.skeleton.cells.copy()
    out["sep"] = r.sepsets.as_dict()
    out["levels"] = [(l.level, l.ci_tests, l.edges_removed) for l in r.levels]
    out["backend"] = dist.get_backend()
    dist.destroy_process_group()


def test_nccl_world_size_one(pcs, oracle):
    m, alpha = 600, 0.05
    c = instance(oracle, 60, 0.3, m, 21)
    ref = oracle.run_pc_stable(c, m, alpha=alpha)
    out = mp.Manager().dict()
    mp.start_processes(_worker, args=(_free_port(), c, m, alpha, out), nprocs=1, join=True, start_method="spawn")
    assert out["backend"] == "nccl"
    assert out["keys"] == [5, (1 << 63) - 1, (1 << 62) | 3, 0]
    assert out["view_ok"]
    assert np.array_equal(out["cells"], ref.adjacency)
    assert out["sep"] == ref.sepsets
    assert [x[1] for x in out["levels"]] == [l.ci_tests for l in ref.levels]
    assert [x[2] for x in out["levels"]] == [l.edges_removed for l in ref.levels]
    single = pcs.run_pc_stable(c, m, pcs.SkeletonConfig(alpha=alpha))
    assert_same_result(single, ref, label="single")
