"""The reference CLI on the device path (paper_1812_08491_b200/pcstable_b200),
restating proj/tests/test_cli.cpp: file formats of io.hpp, the report schema of
pcstable_main.cpp:147-173, the bench CSV of bench.hpp:142-175 and the exit codes.

`gen` needs no GPU (host datagen) and is checked against the oracle's generator; skeleton /
orient / bench run on the GPU and their files are compared byte for byte with the same files
written from the oracle's results (the io.hpp writers restated below)."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1812_08491_b200", "pcstable_b200")


def cli(*args, cwd=None):
    if not os.path.exists(CLI):
        from paper_1812_08491_b200 import _build
        _build.build()
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, cwd=cwd, timeout=600)


# ---- io.hpp writers restated on oracle results (the expected files)
def edges_text(adj: np.ndarray) -> str:  # io.hpp:204-211
    n = adj.shape[0]
    return "".join(f"{i} {j}\n" for i in range(n) for j in range(i + 1, n) if adj[i, j])


def sepsets_text(sep: dict) -> str:  # io.hpp:232-242
    out = []
    for (i, j) in sorted(sep):
        s = sorted(sep[(i, j)])
        out.append(f"{i} {j} :" + "".join(f" {v}" for v in s) + "\n")
    return "".join(out)


def mixed_text(g) -> str:  # io.hpp:215-220
    return "".join(f"{a} > {b}\n" for a, b in g.directed) + "".join(f"{a} {b}\n" for a, b in g.undirected)


def test_usage_errors_exit_1():  # test_cli.cpp:66-74
    assert cli().returncode == 1
    assert cli("nope").returncode == 1
    assert cli("gen", "--n", "10").returncode == 1          # missing --d/--m/--out
    assert cli("gen", "--n", "1", "--d", "0.1", "--m", "10", "--out", "/tmp/x").returncode == 1  # n < 2
    assert cli("skeleton", "--data", "x.csv", "--out", "y", "--strategy", "bogus").returncode == 1


def test_gen_matches_reference_generator(oracle, tmp_path):
    """gen writes the reference generator's data (shortest round-trip doubles) and truth edges."""
    out = tmp_path / "d.csv"
    r = cli("gen", "--n", 15, "--d", 0.3, "--m", 50, "--seed", 11, "--out", out)
    assert r.returncode == 0, r.stderr
    w = oracle.random_dag(15, 0.3, 11)
    x = oracle.sample_linear_gaussian(w, 50, 12)  # column-major m x n
    got = np.loadtxt(out, delimiter=",")
    assert got.shape == (50, 15)
    assert np.array_equal(got, x.T)  # x: (p, m), rows = variables
    truth = [tuple(map(int, ln.split(" > "))) for ln in open(str(out) + ".truth").read().splitlines()]
    expect = [(j, i) for i in range(15) for j in range(i) if w[i, j] != 0.0]  # datagen.hpp:26-32
    assert truth == expect


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["serial", "edge", "set"])
def test_skeleton_files_match_oracle(pcs, oracle, tmp_path, strategy):
    """test_cli.cpp:95-160: skeleton files identical across strategies and to the serial oracle."""
    data = tmp_path / "d.csv"
    assert cli("gen", "--n", 40, "--d", 0.2, "--m", 800, "--seed", 3, "--out", data).returncode == 0
    r = cli("skeleton", "--data", data, "--alpha", 0.05, "--strategy", strategy, "--out", tmp_path / "s")
    assert r.returncode == 0, r.stderr
    x = np.loadtxt(data, delimiter=",")
    # the CLI computes C on the device (DMMA Gram; summation order unpinned by the reference, within
    # 1e-14 of the oracle's), so this instance is chosen far from every decision boundary
    c = oracle.compute_correlation(np.ascontiguousarray(x.T))
    ref = oracle.run_pc_stable(c, 800, alpha=0.05)
    assert open(tmp_path / "s.edges").read() == edges_text(ref.adjacency)
    assert open(tmp_path / "s.sepsets").read() == sepsets_text(ref.sepsets)
    rep = json.load(open(tmp_path / "s.report.json"))
    assert rep["command"] == "skeleton"
    assert rep["input"]["n"] == 40 and rep["input"]["m"] == 800 and len(rep["input"]["fingerprint"]) == 16
    assert rep["config"]["strategy"] == strategy and rep["config"]["max_level"] is None
    assert [l["ci_tests"] for l in rep["levels"]] == [l.ci_tests for l in ref.levels]
    assert [l["edges_removed"] for l in rep["levels"]] == [l.edges_removed for l in ref.levels]
    assert rep["totals"]["ci_tests"] == sum(l["ci_tests"] for l in rep["levels"])
    assert rep["result"]["edges"] == int(np.triu(ref.adjacency, 1).sum())
    assert rep["result"]["levels_run"] == ref.levels_run()
    assert rep["result"]["stop_reason"] == ref.stop_reason


@pytest.mark.gpu
def test_orient_file_matches_oracle(pcs, oracle, tmp_path):
    data = tmp_path / "d.csv"
    assert cli("gen", "--n", 30, "--d", 0.15, "--m", 1000, "--seed", 9, "--out", data).returncode == 0
    assert cli("skeleton", "--data", data, "--out", tmp_path / "s").returncode == 0
    r = cli("orient", "--skeleton", tmp_path / "s.edges", "--sepsets", tmp_path / "s.sepsets",
            "--out", tmp_path / "g.txt")
    assert r.returncode == 0, r.stderr
    edges = [tuple(map(int, ln.split())) for ln in open(tmp_path / "s.edges").read().splitlines()]
    sep = {}
    for ln in open(tmp_path / "s.sepsets").read().splitlines():
        head, _, tail = ln.partition(":")
        i, j = map(int, head.split())
        sep[(i, j)] = tuple(map(int, tail.split()))
    n = 30
    adj = np.zeros((n, n), np.uint8)
    for i, j in edges:
        adj[i, j] = adj[j, i] = 1
    ref = oracle.orient(n, adj, sep, stage=3)
    assert open(tmp_path / "g.txt").read() == mixed_text(ref)
    # data errors exit 2 (pcstable_main.cpp:339-341)
    (tmp_path / "bad.sepsets").write_text("0 1 : x\n")
    assert cli("orient", "--skeleton", tmp_path / "s.edges", "--sepsets", tmp_path / "bad.sepsets",
               "--out", tmp_path / "g2.txt").returncode == 2


@pytest.mark.gpu
def test_bench_csv(pcs, oracle, tmp_path):
    """test_bench.cpp: one row per (case, strategy, repeat); level columns sum to the totals and
    the counters equal the serial oracle's on the same seeded input (bench.hpp:94-96 seeds)."""
    out = tmp_path / "b.csv"
    r = cli("bench", "--spec", "30,0.2,500;50,0.1,800", "--strategies", "serial,set", "--repeats", 2,
            "--alpha", 0.05, "--out", out)
    assert r.returncode == 0, r.stderr
    lines = open(out).read().splitlines()
    assert lines[0] == ("n,d,m,seed,strategy,workers,repeat,levels_run,stop_reason,final_edges,"
                        "correlation_ms,skeleton_ms,total_ms,ci_tests,pseudo_inverses,edges_removed,"
                        "level_ci_tests,level_pseudo_inverses,level_edges_removed,level_ms")
    rows = [ln.split(",") for ln in lines[1:]]
    assert len(rows) == 2 * 2 * 2
    for k, row in enumerate(rows):
        n, d, m, seed = int(row[0]), float(row[1]), int(row[2]), int(row[3])
        assert seed == 7919 * (k // 4)
        lt = [int(v) for v in row[16].split(";")]
        lr = [int(v) for v in row[18].split(";")]
        assert sum(lt) == int(row[13]) and sum(lr) == int(row[15]) and len(lt) == int(row[7])
        w = oracle.random_dag(n, d, seed)
        c = oracle.compute_correlation(oracle.sample_linear_gaussian(w, m, seed + 1))
        ref = oracle.run_pc_stable(c, m, alpha=0.05)
        assert lr == [l.edges_removed for l in ref.levels]
        assert lt == [l.ci_tests for l in ref.levels]
        assert row[8] == ref.stop_reason
