"""End-to-end B200 pipeline on the GPU.

* Virtual-clock parity mode: the B200 plugins driven by the new control plane
  reproduce the reference's batch membership, chunk cuts and per-request
  metrics timeline bit-exactly (golden traces from the unmodified reference;
  only model VALUES differ: decode token ids and payload bytes are the B200
  model's, the mock's integer recurrences are not a float oracle).
* Batch invariance end to end: a device-paced run (real timing, different
  batches) produces byte-identical outputs to the virtual-clock run.
"""
import gzip
from collections import defaultdict
from pathlib import Path

import pytest

from paper_2602_02204_b200.serve import Pipeline

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
GOLD = ROOT / "tests" / "golden"


def keyed(trace: str):
    """Lines grouped by (kind, stage, instant) with model values stripped."""
    groups = defaultdict(list)
    for line in trace.splitlines():
        f = line.split()
        kind = f[0]
        if kind == "D":
            f = f[:5]          # drop the token value
        elif kind == "K":
            f = f[:6]          # drop dtype / shape / digest (model-specific payload)
        elif kind == "R":
            f = f[:9] + f[10:]  # drop the output digest
        key = (kind, f[1], f[2]) if kind in "PODK" else ("R", f[1])
        groups[key].append(" ".join(f))
    return {k: sorted(v) for k, v in groups.items()}


@pytest.fixture(scope="module")
def pipelines():
    """One small-model pipeline per config file, shared by the trace cases."""
    cache = {}

    def get(cfg):
        if cfg not in cache:
            cache[cfg] = Pipeline((ROOT / "configs" / cfg).read_text(), weight_seed=99, small_models=True)
        return cache[cfg]

    yield get
    for p in cache.values():
        p.close()


@pytest.fixture(scope="module")
def small_omni3(pipelines):
    return pipelines("omni3.json")


def trace_cases():
    out = []
    for line in (GOLD / "traces.index").read_text().splitlines():
        f = line.split()
        if f:
            out.append((f[0], f[1], int(f[2]), int(f[3]), int(f[4]), int(f[5]),
                        int(f[6]) if len(f) > 6 else 0, int(f[7]) if len(f) > 7 else 0))
    return out


@pytest.mark.parametrize("case", trace_cases(), ids=lambda c: c[0])
def test_virtual_clock_trace_matches_reference(pipelines, case):
    """Every golden trace of the unmodified reference (8 configs: the bench's
    n=100 run, concurrency 64, FULL edges, chunk 1, tight KV budgets with
    recompute preemption, single-stage, two-stage and AR->DiT graphs) replayed
    with the B200 device models in the loop on the virtual clock."""
    name, cfg, n, seed, conc, stream, c0, c1 = case
    p = pipelines(cfg)
    r = p.bench(n=n, seed=seed, concurrency=conc, stream=bool(stream), clock="virtual", trace=True,
                talker_chunk=c0, vocoder_chunk=c1)
    assert r["completed"] == n and r["failed"] == 0
    got = keyed(p.trace())
    want = keyed(gzip.decompress((GOLD / f"trace_{name}.txt.gz").read_bytes()).decode())
    assert set(got) == set(want)
    for k in want:
        assert got[k] == want[k], f"divergence at {k}:\n new {got[k][:3]}\n ref {want[k][:3]}"


def test_device_paced_outputs_equal_virtual(small_omni3):
    v = small_omni3.bench(n=24, seed=5, concurrency=8, clock="virtual")
    d = small_omni3.bench(n=24, seed=5, concurrency=8, clock="device")
    assert v["completed"] == d["completed"] == 24
    assert v["output_digest"] == d["output_digest"], "batching changed outputs (batch invariance broken)"
    assert d["text_tokens"] == v["text_tokens"] and d["wave_samples"] == v["wave_samples"]
    assert d["wave_samples"] == 16 * d["codec_tokens"] == 64 * d["text_tokens"]


def test_ar_dit_and_single_stage_configs():
    for cfg, exits in (("ar_dit.json", "dit"), ("thinker_only.json", None), ("thinker_talker.json", None)):
        p = Pipeline((ROOT / "configs" / cfg).read_text(), weight_seed=3, small_models=True)
        r = p.bench(n=12, seed=1, concurrency=4, clock="device")
        assert r["completed"] == 12, (cfg, r)
        if exits:
            assert r["wave_samples"] == 16 * r["text_tokens"]
        p.close()


def test_branching_graph_config5():
    """BASELINE config 5 (Ming-Omni-style branching): one Thinker feeding a
    Talker -> Code2Wav audio branch AND an image DiT branch. The reference
    cannot run it (BadDtype: its Thinker packs FIX16-free U8 rows for every
    edge, diffusion_engine.hpp:29-30); here the edge to a diffusion consumer
    carries the token ids (per-edge pack) and each exit assembles its own
    waveform (per-exit waves)."""
    p = Pipeline((ROOT / "configs" / "ming_branch.json").read_text(), weight_seed=5, small_models=True)
    for clock in ("virtual", "device"):
        r = p.bench(n=12, seed=3, concurrency=4, clock=clock)
        assert r["completed"] == 12 and r["failed"] == 0, r
        assert r["codec_tokens"] == 4 * r["text_tokens"]
        # the reported waveform is one exit's (16 samples per conditioning token)
        assert r["wave_samples"] in (16 * r["codec_tokens"], 16 * r["text_tokens"])
    p.close()


def test_full_size_omni3_device():
    p = Pipeline((ROOT / "configs" / "omni3.json").read_text(), weight_seed=7)
    r = p.bench(n=16, seed=7, concurrency=16, clock="device")
    assert r["completed"] == 16
    print("full omni3 n=16:", {k: r[k] for k in ("requests_per_s", "mean_jct_us", "p99_jct_us",
                                                  "dev_ms_thinker", "dev_ms_talker", "dev_ms_dit",
                                                  "steps_thinker", "steps_talker", "steps_dit", "wall_s")})
    p.close()


def test_replicated_placement_same_outputs():
    """Stage placement with replicas on the GPUs this box has:
    Thinker x2, Talker x3, Code2Wav x2. On a 1-GPU box every replica lands on
    cuda:0 (own streams, own KV pools, shared connector arena), which still
    exercises the router, per-request connector arenas, absolute-address packs
    and the pack-event ordering across producer replicas. Outputs must be
    byte-identical to the single-replica pipeline (batch invariance)."""
    import json
    from paper_2602_02204_b200 import dev as D
    import ctypes
    n = ctypes.c_int32()
    D.dev_lib().omni_device_count(ctypes.byref(n))
    devs = [f"cuda:{i % n.value}" for i in range(8)]
    text = (ROOT / "configs" / "omni3.json").read_text()
    base = Pipeline(text, weight_seed=11, small_models=True)
    r0 = base.bench(n=24, seed=5, concurrency=8, clock="device")
    base.close()
    cfg = json.loads(text)
    cfg["placement"] = {"thinker": ",".join(devs[0:2]), "talker": ",".join(devs[2:5]),
                        "vocoder": ",".join(devs[5:7])}
    p = Pipeline(json.dumps(cfg), weight_seed=11, small_models=True)
    r1 = p.bench(n=24, seed=5, concurrency=8, clock="device")
    v = p.bench(n=24, seed=5, concurrency=8, clock="virtual")
    p.close()
    assert r0["completed"] == r1["completed"] == v["completed"] == 24
    assert r0["output_digest"] == r1["output_digest"] == v["output_digest"]


def test_placement_beyond_visible_devices_is_rejected():
    import json
    from paper_2602_02204_b200._native import OmniError
    cfg = json.loads((ROOT / "configs" / "omni3.json").read_text())
    cfg["placement"] = {"talker": "cuda:0,cuda:63"}
    with pytest.raises(OmniError) as e:
        Pipeline(json.dumps(cfg), weight_seed=1, small_models=True)
    assert "cuda:63" in str(e.value)
