"""Cost-weighted multi-GPU sharding (host.cu pcs_session_level_pass, level.cu shard_bounds_kernel) on
real device sessions in ONE process: N sessions on cuda:0 play the N ranks of bench.py --gpus N in
lockstep, each runs only its shard of every pass, and the key arrays are MIN-merged between passes
(what the NCCL all-reduce does in multigpu.py).  Every shard must end with the single-session
result, which equals the oracle's; and the shards' device work must add up to (about) the
single-session work -- a shard range that skipped or repeated units would show up in one or the
other."""
import numpy as np
import pytest
import torch

from paper_1812_08491_b200.multigpu import _CudaArray
from tests.helpers import assert_same_result, instance

pytestmark = pytest.mark.gpu


def lockstep(pcs, c, m, cfg, nsh):
    sessions = [pcs.Session(c, m, cfg, shard_index=r, shard_count=nsh) for r in range(nsh)]
    try:
        while True:
            states = [s.level_begin() for s in sessions]
            assert len(set(states)) == 1, states
            running, ell, nk = states[0]
            if not running:
                break
            for pass_index in (0, 1):
                for s in sessions:
                    s.level_pass(pass_index)
                torch.cuda.synchronize()
                if nk:
                    views = [torch.as_tensor(_CudaArray(*s.keys()), device="cuda") for s in sessions]
                    merged = torch.stack(views).min(0).values
                    for v in views:
                        v.copy_(merged)
                    torch.cuda.synchronize()
            for s in sessions:
                s.level_end()
        return [s.finish() for s in sessions]
    finally:
        for s in sessions:
            s.close()


@pytest.mark.parametrize("variant", ["set", "edge"])
@pytest.mark.parametrize("nsh", [2, 3, 8])
def test_lockstep_shards_match_single_session(pcs, oracle, variant, nsh):
    m, alpha = 2000, 0.05
    c = instance(oracle, 90, 0.25, m, 33)
    ref = oracle.run_pc_stable(c, m, alpha=alpha)
    cfg = pcs.SkeletonConfig(alpha=alpha, strategy=pcs.Strategy(variant))
    single = pcs.run_pc_stable(c, m, cfg)
    assert_same_result(single, ref, label="single")
    assert ref.levels_run() >= 3
    results = lockstep(pcs, c, m, cfg, nsh)
    for r, res in enumerate(results):
        assert_same_result(res, ref, label=f"shard {r}/{nsh}")
    for lv in range(1, ref.levels_run()):
        one = single.levels[lv].device_ci_tests
        tot = sum(res.levels[lv].device_ci_tests for res in results)
        # shards cannot see each other's removals inside a pass, so they may test a little more; never less
        # than the serial-equivalent count and never a multiple of the single-session work
        assert tot >= ref.levels[lv].ci_tests, f"level {lv}: {tot} < serial {ref.levels[lv].ci_tests}"
        assert tot <= 2 * one + 256, f"level {lv}: shards did {tot} tests vs {one} in one session"
