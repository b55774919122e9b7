"""CLI drop-in: the reference's sub-commands, flags,
report keys and bench CSV, on the B200 solver (reference test_cli.py is the
model: byte-stable reports with --omit-times, exit status 2 on errors)."""

import csv
import io
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

REPORT_KEYS = {"instance", "mode", "config", "primal_cost", "lower_bound", "gap", "node_labels", "trace",
               "wall_time_ms", "seed", "threads"}
CONFIG_KEYS = {"mp_iterations", "max_cycle_length", "matching_switch_fraction", "max_rounds", "separation_rounds"}
TRACE_KEYS = {"round", "phase", "nodes", "edges", "triplets", "lb", "lb_valid", "contracted", "time_ms"}


def run(*args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, "-m", "paper_2109_01838_b200", *args], cwd=ROOT, env=e,
                          capture_output=True, text=True, timeout=600)


def test_cli_errors_exit_2(tmp_path):
    r = run("solve", "-i", str(tmp_path / "missing.txt"))
    assert r.returncode == 2 and r.stderr.startswith("error: ")
    bad = tmp_path / "bad.txt"
    bad.write_text("MULTICUT\n0 0 1.0\n")
    r = run("solve", "-i", str(bad))
    assert r.returncode == 2 and "line 2: self-loop" in r.stderr
    r = run("bench", "-i", str(tmp_path / "none*.txt"))
    assert r.returncode == 2 and "no instances match" in r.stderr


@pytest.mark.gpu
def test_cli_generate_solve_bound_bench(tmp_path):
    inst = tmp_path / "grid.txt"
    assert run("generate", "--type", "grid", "--height", "24", "--width", "32", "--stride", "3", "--seed", "2",
               "-o", str(inst)).returncode == 0
    assert inst.read_text().startswith("MULTICUT\nNODES 768\n")
    outs = []
    for k in range(2):
        out = tmp_path / ("r%d.json" % k)
        r = run("solve", "-i", str(inst), "--mode", "PD", "--omit-times", "-o", str(out))
        assert r.returncode == 0, r.stderr
        outs.append(out.read_text())
    assert outs[0] == outs[1]  # byte-identical reruns
    rep = json.loads(outs[0])
    assert set(rep) == REPORT_KEYS and set(rep["config"]) == CONFIG_KEYS
    assert all(set(t) == TRACE_KEYS for t in rep["trace"])
    assert rep["trace"][-1]["phase"] == "cleanup" and rep["wall_time_ms"] == 0.0
    assert len(rep["node_labels"]) == 768 and rep["lower_bound"] <= rep["primal_cost"]
    assert rep["gap"] == pytest.approx(rep["primal_cost"] - rep["lower_bound"])
    r = run("bound", "-i", str(inst), "--separation-rounds", "2", "--omit-times")
    bound = json.loads(r.stdout)
    assert bound["mode"] == "D" and len(bound["trace"]) == 2 and bound["lower_bound"] is not None
    r = run("solve", "-i", str(inst), "--mode", "P", "--omit-times", env={"MULTICUT_THREADS": "3"})
    p = json.loads(r.stdout)
    assert p["lower_bound"] is None and p["gap"] is None and p["threads"] == 3
    r = run("bench", "-i", str(tmp_path / "*.txt"), "--modes", "P,PD")
    rows = list(csv.reader(io.StringIO(r.stdout)))
    assert rows[0] == ["instance", "mode", "primal_cost", "lower_bound", "time_ms"]
    assert [row[:2] for row in rows[-2:]] == [["MEAN", "P"], ["MEAN", "PD"]] and rows[-2][3] == ""
