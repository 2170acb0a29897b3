"""The bench.py JSON-line contract, checked on the CPU through its reference
arm (the oracle, timed on the host: the one bench path that runs without a
GPU).  The GPU arm's line is checked by the round-end driver run."""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def _check_line(j, n_gpus):
    metric = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
    assert j["impl"] == "reference" and j["metric"] == metric
    assert j["unit"] == "edges/s" and j["value"] > 0 and j["higher_is_better"] is True
    assert j["n_gpus"] == n_gpus and j["steps"] == 2 and j["warmup"] == 3
    assert j["ms_per_step"] > 0 and j["data"] == "synthetic" and "workload" in j["config"]
    cb = j["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == j["value"]
    e2e = j["e2e"]
    assert e2e["value"] == j["value"] and e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0


def test_reference_arm_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "C1", "--steps", "2",
                          "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=600, check=True).stdout
    lines = _json_lines(out)
    assert len(lines) == 1
    _check_line(lines[0], 1)


def test_reference_arm_torchrun_rank0_only():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl", "reference",
                          "--config", "C1", "--gpus", "2", "--steps", "2", "--warmup", "3"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600, check=True).stdout
    lines = _json_lines(out)
    assert len(lines) == 1          # rank 0 alone prints; the other rank exits 0 without work
    _check_line(lines[0], 2)
