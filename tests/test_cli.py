"""CLI of the GPU path: subcommands and the reference's exit codes (cli.py:43-50). CPU part."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _run(*args):
    return subprocess.run([sys.executable, "-m", "paper_2010_14501_b200", *args], cwd=ROOT, capture_output=True,
                          text=True, timeout=600)


def test_trace_and_plan(tmp_path):
    r = _run("trace", "--arch", "resnet18", "--batch", "2", "--image", "32", "--classes", "10", "--fuse",
             "-o", str(tmp_path / "g.json"))
    assert r.returncode == 0, r.stderr
    g = json.loads((tmp_path / "g.json").read_text())
    assert g["format"] == 1 and g["nodes"][0]["id"] == 1
    r = _run("plan", "--arch", "resnet18", "--batch", "2", "--image", "32", "--classes", "10", "--fuse",
             "--budget-gib", "1", "-o", str(tmp_path / "s.json"))
    assert r.returncode == 0, r.stderr
    s = json.loads((tmp_path / "s.json").read_text())
    assert "schedule" in s and s["planner"]["modeled_peak"] <= 1 << 30


def test_exit_codes(tmp_path):
    # a budget below the parameters alone: no schedule -> 3 (infeasible)
    r = _run("plan", "--arch", "resnet18", "--batch", "2", "--image", "32", "--classes", "10", "--budget-gib",
             "0.01")
    assert r.returncode == 3
    # an unknown architecture / bad argument -> 1 (bad input)
    r = _run("trace", "--arch", "no_such_net", "--batch", "2")
    assert r.returncode == 1
