"""Prefix cache of the Thinker stage (csrc/dev/stage.cpp
prefix_lookup / prefix_insert): full 16-token prompt pages shared between
sequences with the same prompt prefix. The caller's schedule is unchanged
(the reference's ArEngine still prefills every prompt token); the device skips
the cached part of each prefill span. Requirements: identical greedy tokens and
bit-identical hidden rows with the cache on and off, the expected number of
cached tokens served, and correct eviction when the KV pool is short."""
import numpy as np
import pytest

from paper_2602_02204_b200 import dev as D

pytestmark = pytest.mark.gpu

SMALL = dict(d_model=512, n_layers=2, n_heads=4, n_kv_heads=1, d_ff=1024)


def run(st, prompts, order, n_dec=6, chunk=32, reserve=False):
    """Prefill each prompt in `chunk`-token spans (one sequence per step, in
    `order`), then decode all sequences together. Returns tokens / hidden rows.
    reserve: admit every prefill span ahead of its step the way the pipeline
    does (omni_seq_reserve_prompt)."""
    for s in order:
        p = prompts[s]
        for at in range(0, len(p), chunk):
            sp = min(chunk, len(p) - at)
            if reserve:
                st.reserve_prompt(s, at, p[at:at + sp])
            st.ar_step([s], [D.PREFILL], [sp], [at], [-1], p[at:at + sp])
    seqs = sorted(prompts)
    toks = {s: [] for s in seqs}
    hid = {s: [] for s in seqs}
    for k in range(n_dec):
        tin = [(-1 if k == 0 else toks[s][-1]) for s in seqs]
        t, _ = st.ar_step(seqs, [D.DECODE] * len(seqs), [1] * len(seqs), [len(prompts[s]) + k for s in seqs],
                          [k] * len(seqs), tin)
        for i, s in enumerate(seqs):
            toks[s].append(int(t[i]))
            hid[s].append(D.d2h(st.hidden_row(s, k), (st.model.d_model,), np.uint16))
    return toks, hid


def prompts_with_shared_prefix(rng, prefix_len=80):
    pre = [int(x) for x in rng.integers(1, 256, size=prefix_len)]
    return {1: pre + [int(x) for x in rng.integers(1, 256, size=27)],
            2: pre + [int(x) for x in rng.integers(1, 256, size=45)],
            3: pre[:40] + [int(x) for x in rng.integers(1, 256, size=30)],  # shares 2 full pages
            4: [int(x) for x in rng.integers(1, 256, size=50)]}               # shares nothing


@pytest.mark.parametrize("reserve", [False, True])
def test_prefix_cache_outputs_bit_identical_and_hits_counted(reserve):
    m = D.model_default(D.THINKER, **SMALL)
    rng = np.random.default_rng(5)
    prompts = prompts_with_shared_prefix(rng)
    ref = D.Stage(m, D.StageLimits(256, 8, 256, 0, 64), seed=3)
    ref.set_prefix_cache(False)
    t0, h0 = run(ref, prompts, [1, 2, 3, 4])
    ref.close()
    st = D.Stage(m, D.StageLimits(256, 8, 256, 0, 64), seed=3)
    t1, h1 = run(st, prompts, [1, 2, 3, 4], reserve=reserve)
    stats = st.prefix_stats()
    # seq 2 reuses seq 1's 5 full prefix pages (80 tokens), seq 3 two pages (32)
    assert stats["hit_tokens"] == 80 + 32, stats
    assert t1 == t0
    for s in prompts:
        for a, b in zip(h0[s], h1[s]):
            assert np.array_equal(a, b), f"seq {s}: hidden rows differ with the prefix cache"
    st.close()


def test_prefix_cache_survives_release_and_replays_bit_exact():
    """Recompute preemption (release + re-prefill, ar_engine.hpp:229-257): the
    replayed prefill is served from the cache and the outputs repeat exactly."""
    m = D.model_default(D.THINKER, **SMALL)
    rng = np.random.default_rng(9)
    p = {7: [int(x) for x in rng.integers(1, 256, size=96)]}
    st = D.Stage(m, D.StageLimits(256, 8, 256, 0, 64), seed=4)
    t_a, h_a = run(st, p, [7])
    st.release(7)
    before = st.prefix_stats()["hit_tokens"]
    t_b, h_b = run(st, p, [7])
    assert st.prefix_stats()["hit_tokens"] - before == 96  # all 6 prompt pages
    assert t_a == t_b and all(np.array_equal(a, b) for a, b in zip(h_a[7], h_b[7]))
    st.close()


def test_prefix_cache_evicts_when_the_pool_is_short():
    """A KV pool just large enough for two live sequences: cached pages of
    released sequences are evicted on demand, outputs stay identical."""
    m = D.model_default(D.THINKER, **SMALL)
    rng = np.random.default_rng(13)
    seqs = {s: [int(x) for x in rng.integers(1, 256, size=100)] for s in range(1, 7)}
    ref = D.Stage(m, D.StageLimits(256, 8, 128, 18, 64), seed=6)
    ref.set_prefix_cache(False)
    st = D.Stage(m, D.StageLimits(256, 8, 128, 18, 64), seed=6)
    for s, p in seqs.items():  # one sequence at a time: 7 pages each, pool of 18
        a = run(ref, {s: p}, [s], n_dec=4)
        b = run(st, {s: p}, [s], n_dec=4)
        assert a[0] == b[0]
        assert all(np.array_equal(x, y) for x, y in zip(a[1][s], b[1][s]))
        ref.release(s)
        st.release(s)
    assert st.prefix_stats()["evicted_pages"] > 0
    st.close()
    ref.close()
