"""Stage placement and the replica router on CPU, driven through
the NEW control plane with the reference's mock hooks (oracle/mock_pipeline.cpp).

The reference declares DeploymentPlan::placement and never reads it
(orchestrator.hpp:37) and has one engine per node (orchestrator.hpp:136-157).
Here a stage placed on R devices ("cuda:1,cuda:2") runs R engine replicas and
request r goes to replica (r - 1) mod R at admission. Requests are
independent and the models are per-sequence functions, so every request's
outputs must be byte-identical to the single-replica run (batching
transparency, test_properties.cpp:139-154) -- only timing and batch
membership may change -- and the closed loop must keep every replica busy.
"""
import ctypes as C
import json
from pathlib import Path

import pytest

from test_control_plane import mock, run_trace  # noqa: F401  (fixture)

ROOT = Path(__file__).resolve().parent.parent


def trace_for(lib, cfg: dict, n=60, seed=7, conc=16):
    text = json.dumps(cfg).encode()
    cap = 64 << 20
    buf = C.create_string_buffer(cap)
    k = lib.oracle_mock_trace(text, n, seed, conc, 1, 0, 0, buf, cap)
    assert k >= 0, buf.value.decode()
    return buf.value.decode()


def outputs(trace: str):
    """request id -> (status, |text|, |codec|, |wave|, output digest)."""
    out = {}
    for line in trace.splitlines():
        f = line.split()
        if f and f[0] == "R":
            out[int(f[1])] = (f[2], f[6], f[7], f[8], f[9])
    return out


def replica_iters(trace: str):
    return {f[1]: [int(x) for x in f[2:]] for f in (l.split() for l in trace.splitlines()) if f and f[0] == "I"}


def base_cfg():
    return json.loads((ROOT / "configs" / "omni3.json").read_text())


@pytest.mark.parametrize("placement", [
    {"talker": "cuda:1,cuda:2"},
    {"thinker": "cuda:0", "talker": ["cuda:1", "cuda:2", "cuda:3", "cuda:4", "cuda:5"], "vocoder": "cuda:6,cuda:7"},
    {"thinker": "cuda:0,cuda:1", "talker": "cuda:2,cuda:3,cuda:4", "vocoder": "cuda:5"},
], ids=["talker2", "dp8_placement", "thinker2"])
def test_replicas_keep_every_output(mock, placement):
    single = trace_for(mock, base_cfg())
    cfg = base_cfg()
    cfg["placement"] = placement
    rep = trace_for(mock, cfg)
    a, b = outputs(single), outputs(rep)
    assert len(a) == 60 and set(a) == set(b)
    for rid in a:
        assert a[rid] == b[rid], f"request {rid}: replicas changed its outputs"
    iters = replica_iters(rep)
    for stage, devs in placement.items():
        n = len(devs) if isinstance(devs, list) else len(devs.split(","))
        if n > 1:
            assert len(iters[stage]) == n
            assert all(x > 0 for x in iters[stage]), f"{stage}: an idle replica {iters[stage]}"


def test_router_is_deterministic(mock):
    cfg = base_cfg()
    cfg["placement"] = {"talker": "cuda:1,cuda:2,cuda:3"}
    assert trace_for(mock, cfg) == trace_for(mock, cfg)


def test_router_assigns_rid_minus_one_mod_r(mock):
    """Every decode of request rid on a 3-replica Talker runs on replica
    (rid - 1) mod 3 (trace lines name the replica: talker_forward#r), and each
    request's codec tokens are all decoded exactly once across replicas."""
    cfg = base_cfg()
    cfg["placement"] = {"talker": "cuda:1,cuda:2,cuda:3"}
    tr = trace_for(mock, cfg, n=30)
    codec = {rid: int(v[2]) for rid, v in outputs(tr).items()}
    per_req = {}
    for line in tr.splitlines():
        f = line.split()
        if f and f[0] in "DP" and f[1].startswith("talker_forward"):
            r = int(f[1].split("#")[1]) if "#" in f[1] else 0
            rid = int(f[3])
            assert r == (rid - 1) % 3, f"request {rid} served by talker replica {r}"
            if f[0] == "D":
                per_req[rid] = per_req.get(rid, 0) + 1
    assert per_req == codec


@pytest.mark.parametrize("bad", [{"talker": "gpu1"}, {"talker": "cuda:1,"}, {"nosuch": "cuda:0"}])
def test_bad_placement_is_config_invalid(mock, bad):
    cfg = base_cfg()
    cfg["placement"] = bad
    text = json.dumps(cfg).encode()
    buf = C.create_string_buffer(4096)
    k = mock.oracle_mock_trace(text, 4, 7, 2, 1, 0, 0, buf, 4096)
    assert k == -1
    assert "placement" in buf.value.decode()
