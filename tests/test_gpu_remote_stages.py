"""Multi-process stage placement in the serving pipeline:
the Talker and the Code2Wav DiT run in a stage worker process
(omni_worker_serve, csrc/serve/stage_worker.cpp), the Thinker and the
control plane in this one. The Thinker packs hidden rows straight into the
worker's CUDA-IPC-exported connector arena and records an interprocess event
the worker's Talker step waits on; steps are requests / replies in the
reference's control-frame format over AF_UNIX. Outputs must be byte-identical
to the single-process pipeline (same weights, same schedule on the virtual
clock; the device-paced clock too)."""
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu
CFG = json.loads((ROOT / "configs" / "omni3.json").read_text())


def start_worker(path):
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2602_02204_b200 import serve_lib\n"
            "rc = serve_lib().omni_worker_serve(%r.encode(), 120000)\n"
            "sys.exit(rc)\n") % (str(ROOT), path)
    return subprocess.Popen([sys.executable, "-c", code], stdout=subprocess.PIPE, stderr=subprocess.STDOUT)


@pytest.mark.parametrize("clock", ["virtual", "device"])
def test_talker_and_dit_in_a_worker_process_same_outputs(clock):
    from paper_2602_02204_b200.serve import Pipeline
    base = Pipeline(json.dumps(CFG), weight_seed=21, small_models=True)
    r0 = base.bench(n=16, seed=3, concurrency=8, clock=clock)
    base.close()
    path = f"/tmp/omni_worker_{os.getpid()}_{clock}.sock"
    w = start_worker(path)
    try:
        cfg = dict(CFG, workers={"talker": path, "vocoder": path})
        p = Pipeline(json.dumps(cfg), weight_seed=21, small_models=True)
        r1 = p.bench(n=16, seed=3, concurrency=8, clock=clock)
        p.close()
    finally:
        try:
            out, _ = w.communicate(timeout=120)
        except subprocess.TimeoutExpired:
            w.kill()
            out, _ = w.communicate()
    assert w.returncode == 0, out.decode()[-2000:]
    assert r0["completed"] == r1["completed"] == 16
    assert r0["output_digest"] == r1["output_digest"]


def test_thinker_in_a_worker_is_rejected():
    from paper_2602_02204_b200.serve import Pipeline
    from paper_2602_02204_b200._native import OmniError
    with pytest.raises(OmniError) as e:
        Pipeline(json.dumps(dict(CFG, workers={"thinker": "/tmp/none.sock"})), weight_seed=1, small_models=True)
    assert "Thinker" in str(e.value)


@pytest.mark.parametrize("procs", [False, True])
def test_bench_two_ranks_under_torchrun(procs):
    """bench.py --gpus 2 under torchrun on this box (the 2-GPU placement folded
    onto its GPU): rank 0 drives the stage graph; with --procs rank 1 is the
    stage worker hosting the Talker. One JSON line, every request completed."""
    port = 29600 + (1 if procs else 0) + os.getpid() % 200
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"), "--gpus", "2",
           "--fold-devices", "--small", "--requests", "12", "--steps", "1", "--warmup", "1", "--no-cpu-baseline"]
    if procs:
        cmd.append("--procs")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(line) == 1, r.stdout[-2000:]
    d = json.loads(line[0])
    assert d["n_gpus"] == 2 and d["completed"] == 24
    assert ("stage workers" in d["config"]["parallelism"]) == procs
