"""bench.py's N-rank path (one process per GPU under torchrun, per-level sharding, key MIN-merge, max-over-
ranks timing) end to end on the round's one-GPU boxes: two ranks share cuda:0 with the gloo backend
(PCS_BENCH_BACKEND=gloo, keys reduced through host memory).  The whole-job line must report the same
serial-equivalent CI tests, levels and stop reason as the one-rank run."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _bench(extra_env, launcher):
    args = ["bench.py", "--workload", "C3", "--steps", "1", "--warmup", "1", "--no-cpu-baseline", "--no-e2e",
            "--no-secondary"]
    env = dict(os.environ, **extra_env)
    out = subprocess.run(launcher + args, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_two_ranks_report_the_single_rank_work(pcs):
    one = _bench({}, [sys.executable])
    two = _bench({"PCS_BENCH_BACKEND": "gloo"},
                 [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                  "--master-addr", "127.0.0.1", "--master-port", str(_free_port())])
    assert two["n_gpus"] == 2 and two["detail"]["multi_gpu"]["ranks"] == 2
    for k in ("serial_ci_tests", "levels_run", "stop_reason", "edges_left"):
        assert two["detail"][k] == one["detail"][k], k
    assert two["value"] > 0 and two["gpu_launches"] > 0
