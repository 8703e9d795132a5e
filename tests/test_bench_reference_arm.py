"""bench.py's reference arm on CPU (no GPU needed): the unmodified reference
control plane with the fp32 CPU hooks (oracle/_ref/ref_cpu_pipeline), small
model dims. Checks the JSON contract of the line the driver parses, and that
under torchrun only rank 0 runs and prints."""
import json
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
EXE = ROOT / "oracle" / "_ref" / "ref_cpu_pipeline"
pytestmark = pytest.mark.skipif(not EXE.exists(), reason="oracle/_ref not built (build())")


def _lines(out: str):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def check_line(d):
    assert d["impl"] == "reference" and d["unit"] == "requests/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "requests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["n_requests"] >= 1 and "workload" in d["config"]


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--small", "--steps", "1", "--warmup", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1
    check_line(lines[0])


def test_reference_arm_under_torchrun_prints_once():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl", "reference",
                        "--small", "--gpus", "2", "--steps", "1", "--warmup", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1, r.stdout
    check_line(lines[0])
    assert lines[0]["n_gpus"] == 2
