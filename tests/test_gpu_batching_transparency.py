"""Batching transparency with the device models in the loop -- the
reference's property test (test_properties.cpp:139-154: 150 random
schedules, batched output == solo output) restated for the B200 pipeline.

Every trial draws a random engine configuration (token budget, prefill
chunk, resident cap per AR stage, in some trials tight KV budgets that force
admission blocking and recompute preemption, streaming chunk sizes of both
edges),
concurrency and clock, runs the same workload through the full
Thinker -> Talker -> Code2Wav pipeline and compares EVERY request's text
tokens, codec tokens, waveform samples and Thinker hidden rows with a solo
run (concurrency 1, one request in flight at a time). The kernels are
batch-invariant by construction (per-row reductions in a fixed order, split
factors a function of the weight only, DiT noise keyed by request and global
codec position), so batched == solo holds bit-exactly; the solo run's parity
against the CPU oracle is tests/test_gpu_pipeline_parity.py.
"""
import json
import random
from pathlib import Path

import numpy as np
import pytest

from paper_2602_02204_b200.serve import Pipeline

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
N_REQ, SEED, WEIGHTS = 14, 21, 5
OUTS = {"text": 1, "codec": 2, "wave": 3, "hidden": 4}
PREEMPTIONS = []  # per trial, to check the tight-budget trials really preempt


def outputs(p, n):
    return {rid: {k: p.output(rid, w).copy() for k, w in OUTS.items()} for rid in range(1, n + 1)}


def random_config(rng: random.Random) -> tuple[str, dict]:
    cfg = json.loads((ROOT / "configs" / "omni3.json").read_text())
    for st in ("thinker", "talker"):
        e = cfg["engines"][st]
        e["max_batch_tokens"] = rng.choice([32, 48, 64, 100, 160, 256])
        e["prefill_chunk"] = min(rng.choice([1, 5, 16, 33, 64]), e["max_batch_tokens"])  # registry.cpp rule
        e["max_resident_requests"] = rng.choice([2, 3, 5, 8, 64])
    if rng.random() < 0.3:  # tight KV budgets: admission blocking and recompute preemption (omni3_tight)
        cfg["engines"]["thinker"]["kv_budget_tokens"] = rng.choice([256, 320, 400])
        cfg["engines"]["talker"]["kv_budget_tokens"] = rng.choice([384, 512, 640])
    cfg["engines"]["vocoder"]["max_resident_requests"] = rng.choice([1, 2, 7, 64])
    cfg["graph"]["edges"][0]["chunk_size"] = rng.choice([1, 2, 4, 7])
    cfg["graph"]["edges"][1]["chunk_size"] = rng.choice([1, 3, 8, 16])
    run = {"concurrency": rng.choice([2, 4, 8, 14]), "clock": rng.choice(["virtual", "device"])}
    return json.dumps(cfg), run


def solo_run(small: bool):
    p = Pipeline((ROOT / "configs" / "omni3.json").read_text(), weight_seed=WEIGHTS, small_models=small)
    r = p.bench(n=N_REQ, seed=SEED, concurrency=1, clock="device", capture=True)
    assert r["completed"] == N_REQ and r["failed"] == 0
    out = outputs(p, N_REQ)
    p.close()
    # the waveform is the whole codec stream at 16 samples per token, 4 codec tokens per text token
    assert all(len(o["wave"]) == 16 * len(o["codec"]) == 64 * len(o["text"]) > 0 for o in out.values())
    return out


@pytest.fixture(scope="module")
def solo_small():
    return solo_run(True)


@pytest.fixture(scope="module")
def solo_full():
    return solo_run(False)


def check_trial(solo, trial, small):
    rng = random.Random(303 + trial)
    text, run = random_config(rng)
    p = Pipeline(text, weight_seed=WEIGHTS, small_models=small)
    r = p.bench(n=N_REQ, seed=SEED, concurrency=run["concurrency"], clock=run["clock"], capture=True)
    assert r["completed"] == N_REQ and r["failed"] == 0, (run, r)
    PREEMPTIONS.append(r["preemptions"])
    got = outputs(p, N_REQ)
    p.close()
    for rid in range(1, N_REQ + 1):
        for k in OUTS:
            a, b = got[rid][k], solo[rid][k]
            assert a.shape == b.shape and np.array_equal(a, b), f"trial {trial} {run} rid {rid}: {k} differs"


@pytest.mark.parametrize("trial", range(150))
def test_batched_equals_solo_small_models(solo_small, trial):
    """150 random schedules, as the reference's property test."""
    check_trial(solo_small, trial, True)


@pytest.mark.parametrize("trial", range(4))
def test_batched_equals_solo_full_size(solo_full, trial):
    """The bench's model dimensions (every GEMM tile / split / attention path
    the bench uses) under four random schedules."""
    check_trial(solo_full, 1000 + trial, False)


def test_tight_budget_trials_preempted():
    if not PREEMPTIONS:
        pytest.skip("no trial ran in this session")
    assert sum(1 for x in PREEMPTIONS if x > 0) >= 5, PREEMPTIONS
