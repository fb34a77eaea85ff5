"""End-to-end `cc` CLI checks — a port of the reference's
proj/tests/cli_smoke.cmake (generation, run, verify, sweep, exit codes) run
against bin/cc built on the B200 library (`make cc`)."""
from __future__ import annotations

import json
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CC = ROOT / "bin" / "cc"


def cc(*args, cwd=None):
    if not CC.exists():
        pytest.skip("bin/cc not built (make cc)")
    return subprocess.run([str(CC), *map(str, args)], capture_output=True, text=True,
                          timeout=600, cwd=cwd)


def test_cli_usage_and_gen_without_gpu(tmp_path):
    # usage errors and host-side generation need no device (cli_smoke.cmake:12-31, 67-70)
    r = cc("gen", "grid:2x2", tmp_path / "grid.el")
    assert r.returncode == 0
    assert (tmp_path / "grid.el").read_text() == "0 1\n2 3\n0 2\n1 3\n"
    a = cc("gen", "er:n=4,m=3,seed=1", tmp_path / "a.el")
    b = cc("gen", "er:n=4,m=3,seed=1", tmp_path / "b.el")
    assert a.returncode == b.returncode == 0
    assert (tmp_path / "a.el").read_text() == (tmp_path / "b.el").read_text()
    assert cc("run", "--algo", "nonsense", "--gen", "grid:2x2").returncode == 2
    assert cc("run", "--format", "xml", "--gen", "grid:2x2").returncode == 2
    assert cc("run", "--bogus").returncode == 2
    assert cc("frobnicate").returncode == 2
    assert cc("--help").returncode == 0
    assert cc("run", "--input", tmp_path / "missing.el").returncode == 3


def test_cli_gen_matches_reference_generators(tmp_path, oracle):
    r = cc("gen", "rmat:scale=6,ef=4,seed=3", tmp_path / "r.el")
    assert r.returncode == 0
    got = [tuple(map(int, ln.split())) for ln in (tmp_path / "r.el").read_text().splitlines()]
    assert got == [tuple(x) for x in oracle.gen_rmat(6, 4, 3).tolist()]


@pytest.mark.gpu
def test_cli_smoke_on_b200(tmp_path):
    # cli_smoke.cmake:33-65
    r = cc("run", "--gen", "grid:20x20", "--algo", "adaptive", "--segments", "auto",
           "--labels-out", tmp_path / "labels.txt", "--metrics-out", tmp_path / "metrics.json")
    assert r.returncode == 0, r.stderr
    metrics = json.loads((tmp_path / "metrics.json").read_text())
    for key in ("algo", "total_ms", "cas_failures", "components", "verified"):
        assert key in metrics
    assert metrics["verified"] and metrics["components"] == 1 and metrics["s"] == 4
    assert list(metrics)[:12] == ["algo", "n", "m", "s", "workers", "total_ms", "hook_ms",
                                  "compress_ms", "cas_failures", "hook_traversal_steps",
                                  "jump_steps", "components"]
    assert cc("verify", "--gen", "grid:20x20", tmp_path / "labels.txt").returncode == 0
    labels = (tmp_path / "labels.txt").read_text()
    bad = labels.replace("0 0\n1 0\n", "0 0\n1 1\n", 1)
    (tmp_path / "bad.txt").write_text(bad)
    assert cc("verify", "--gen", "grid:20x20", tmp_path / "bad.txt").returncode == 1
    # same partition under other representatives: not equal arrays, so this
    # goes through the device partition compare (hcc_labels_compare)
    relab = "".join(f"{ln.split()[0]} 399\n" for ln in labels.splitlines() if ln.strip())
    (tmp_path / "relab.txt").write_text(relab)
    assert cc("verify", "--gen", "grid:20x20", tmp_path / "relab.txt").returncode == 0
    r = cc("sweep", "--gen", "rmat:scale=8,ef=8,seed=5", "--sweep-segments", "2,4",
           "--report", "csv", "--metrics-out", tmp_path / "sweep.csv")
    assert r.returncode == 0, r.stderr
    assert (tmp_path / "sweep.csv").read_text().startswith("s,total_ms,speedup_vs_s1,verified\n")
    for algo in ("baseline", "baseline-mj", "atomic", "adaptive"):
        r = cc("run", "--gen", "rmat:scale=10,ef=8,seed=2", "--algo", algo, "--reps", "2")
        assert r.returncode == 0, (algo, r.stderr)
        j = json.loads(r.stdout)
        assert j["verified"] and j["algo"] == algo and "gteps" in j


@pytest.mark.gpu
def test_cli_multi_gpu_run(tmp_path):
    """`cc run --devices 0,0,0` / `--gpus 1`: the edge-partitioned path
    through the C++ API (DriverOptions::devices -> hcc_create_multi)."""
    for flag in (["--devices", "0,0,0"], ["--gpus", "1"]):
        r = cc("run", "--gen", "rmat:scale=11,ef=8,seed=4", "--algo", "baseline-mj", *flag)
        assert r.returncode == 0, r.stderr
        j = json.loads(r.stdout)
        assert j["verified"]
    assert cc("run", "--gen", "grid:4x4", "--gpus", "0").returncode == 2
