"""GPU edge cases of the C-ABI stage calls (the reference's own edge tests,
restated for the device path):
  * empty iterations (ar_engine.hpp:100-104 runs begin_iteration with an
    empty batch; diffusion_engine.hpp:106-121 empty eos job)
  * maximum sizes: max_batch_tokens prefill spans, max_resident decoders
  * recompute preemption: release + replay from the prompt reproduces the
    tokens and hidden rows bit-for-bit (ar_engine.hpp:222-257)
  * error mapping to the reference error tree (errors.hpp): bad spans / ids
    -> E_BADARG (ForwardError / BadDtype), exhausted KV pool or resident
    slots -> E_OOM (RejectedTooLarge / RegionFull)
"""
import numpy as np
import pytest

import oracle
from paper_2602_02204_b200 import dev as D
from paper_2602_02204_b200._native import OmniError

pytestmark = pytest.mark.gpu

SMALL = dict(d_model=512, n_layers=2, n_heads=4, n_kv_heads=2, d_ff=1024)


@pytest.fixture(scope="module")
def thinker():
    m = D.model_default(D.THINKER, **SMALL)
    st = D.Stage(m, D.StageLimits(256, 64, 320, 0, 64), seed=13)
    yield st
    st.close()


def test_empty_ar_step(thinker):
    tok, mg = thinker.ar_step([], [], [], [], [], [])
    assert len(tok) == 0 and len(mg) == 0


def test_empty_dit_step():
    m = D.model_default(D.DIT, d_model=256, n_layers=1, n_heads=2, n_kv_heads=2, d_ff=512)
    st = D.Stage(m, D.StageLimits(256, 8, 256, 0, 16), seed=3)
    out = st.dit_step([], [], [], [])
    assert len(out) == 0
    out = st.dit_step([4], [12], [0], [])  # an empty eos job (diffusion_engine.hpp:106-121)
    assert len(out) == 0
    st.close()


def test_max_batch_tokens_and_max_resident(thinker):
    rng = np.random.default_rng(7)
    # 4 x 64-token prefill spans = max_batch_tokens (256) in one step
    ids = [100, 101, 102, 103]
    prompts = [list(rng.integers(1, 256, size=64)) for _ in ids]
    tok, _ = thinker.ar_step(ids, [D.PREFILL] * 4, [64] * 4, [0] * 4, [-1] * 4, sum(prompts, []))
    assert list(tok) == [-1] * 4  # prefill entries emit nothing (ar_engine.hpp:313-324)
    # 60 more residents -> 64 decoders in one step (max_resident_requests)
    more = list(range(200, 260))
    for i in range(0, 60, 4):
        grp = more[i:i + 4]
        thinker.ar_step(grp, [D.PREFILL] * 4, [5] * 4, [0] * 4, [-1] * 4, list(rng.integers(1, 256, size=20)))
    allids = ids + more
    pos = [64] * 4 + [5] * 60
    tok, mg = thinker.ar_step(allids, [D.DECODE] * 64, [1] * 64, pos, [0] * 64, [-1] * 64)
    assert np.all((tok >= 1) & (tok <= 255)) and np.all(mg >= 0)
    # decode batch order is the reference's (rid asc); each row is batch-invariant:
    solo, _ = thinker.ar_step([ids[0]], [D.DECODE], [1], [65], [1], [int(tok[0])])
    # one more resident than the slot pool -> E_OOM
    with pytest.raises(OmniError) as e:
        thinker.ar_step([999], [D.PREFILL], [3], [0], [-1], [1, 2, 3])
    assert "E_OOM" in str(e.value)
    for s in allids:
        thinker.release(s)


def test_recompute_preemption_replays_bit_exact(thinker):
    d = thinker.model.d_model
    rng = np.random.default_rng(8)
    p = list(rng.integers(1, 256, size=29))

    def run(seq):
        thinker.ar_step([seq], [D.PREFILL], [29], [0], [-1], p)
        toks, rows = [], []
        for k in range(5):
            t, _ = thinker.ar_step([seq], [D.DECODE], [1], [29 + k], [k], [-1 if k == 0 else toks[-1]])
            toks.append(int(t[0]))
            rows.append(D.d2h(thinker.hidden_row(seq, k), (d,), np.uint16))
        return toks, np.stack(rows)

    t1, h1 = run(300)
    thinker.release(300)  # preempted: KV pages + ring freed
    t2, h2 = run(300)     # recompute from the prompt (ar_engine.hpp:229-257)
    assert t1 == t2 and np.array_equal(h1, h2)
    thinker.release(300)


def test_error_mapping(thinker):
    with pytest.raises(OmniError) as e:  # span exceeds max_batch_tokens
        thinker.ar_step([1], [D.PREFILL], [257], [0], [-1], [1] * 257)
    assert "E_BADARG" in str(e.value)
    with pytest.raises(OmniError) as e:  # decode entries feed exactly one token
        thinker.ar_step([1], [D.DECODE], [2], [0], [0], [1, 2])
    assert "E_BADARG" in str(e.value)
    with pytest.raises(OmniError) as e:  # input id outside the byte alphabet
        thinker.ar_step([1], [D.PREFILL], [1], [0], [-1], [300])
    assert "E_BADARG" in str(e.value)
    with pytest.raises(OmniError) as e:  # longer than max_seq_len
        thinker.ar_step([1], [D.PREFILL], [5], [318], [-1], [1] * 5)
    assert "E_OOM" in str(e.value)
    thinker.release(1)
    m = D.model_default(D.DIT, d_model=256, n_layers=1, n_heads=2, n_kv_heads=2, d_ff=512)
    st = D.Stage(m, D.StageLimits(256, 8, 256, 0, 16), seed=3)
    with pytest.raises(OmniError) as e:  # ~ BadDtype: conditioning id outside the model's alphabet
        st.dit_step([1], [0], [1], [m.vocab])
    assert "E_BADARG" in str(e.value)
    st.close()


def test_kv_pool_exhaustion_is_oom():
    m = D.model_default(D.THINKER, **SMALL)
    st = D.Stage(m, D.StageLimits(256, 8, 256, 2, 16), seed=5)  # 2 pages = 32 tokens in total
    st.ar_step([1], [D.PREFILL], [20], [0], [-1], [7] * 20)
    with pytest.raises(OmniError) as e:
        st.ar_step([2], [D.PREFILL], [20], [0], [-1], [9] * 20)
    assert "E_OOM" in str(e.value)
    st.release(1)
    st.ar_step([2], [D.PREFILL], [20], [0], [-1], [9] * 20)  # pages returned by release
    st.close()


def _sample_ref(logits, lo, hi, k, seed, rid, index):
    """numpy restatement of sample_row (ar_dev.cuh): top-k of [lo, hi), softmax
    at temperature 1, u = sample_hash(seed, key(rid), index) * sum."""
    ids = np.arange(lo, hi)
    v = logits[lo:hi].astype(np.float64)
    order = np.lexsort((ids, -v))[:k]          # descending logit, ties -> lowest id
    top = v[order]
    p = np.exp(top - top[0])
    c = np.cumsum(p)
    key = oracle.mix64(rid) & 0xFFFFFFFF
    h = oracle.sample_hash(seed, key, index)
    u = (h >> 40) / 16777216.0 * c[-1]
    j = int(np.argmax(c > u)) if np.any(c > u) else k - 1
    # a draw within float rounding of a cumulative boundary may legitimately
    # land on the neighbour (fp32 prefix sum on the GPU)
    near = np.any(np.abs(c - u) <= 1e-5 * c[-1])
    return int(ids[order][j]), set(int(x) for x in ids[order]), near


def test_topk_sampler_matches_restatement_and_is_batch_invariant():
    """omni_stage_set_sampling(top_k=8): every drawn id lies in the row's
    top-8, equals the numpy restatement of the sampler on the GPU's own
    logits, and a sequence redraws the SAME ids when replayed in a different
    batch (the draw is keyed by request id + emitted index, not by row)."""
    m = D.model_default(D.THINKER, **SMALL)
    rng = np.random.default_rng(31)
    prompts = {s: list(rng.integers(1, 256, size=n)) for s, n in ((3, 11), (5, 6), (8, 17))}
    st = D.Stage(m, D.StageLimits(256, 16, 256, 0, 16), seed=37)
    st.set_sampling(8, 4242)
    runs = []
    for batch in (sorted(prompts), [5]):
        for s in batch:
            st.ar_step([s], [D.PREFILL], [len(prompts[s])], [0], [-1], prompts[s])
        toks = {s: [] for s in batch}
        for k in range(6):
            tin = [-1 if k == 0 else toks[s][-1] for s in batch]
            t, mg = st.ar_step(batch, [D.DECODE] * len(batch), [1] * len(batch),
                               [len(prompts[s]) + k for s in batch], [k] * len(batch), tin)
            lg_p, _, ld = st.tensor("buf.logits")
            lg = D.d2h(lg_p, (len(batch), ld), np.float32)
            for i, s in enumerate(batch):
                want, topset, near = _sample_ref(lg[i], 1, 256, 8, 4242, s, k)
                assert int(t[i]) in topset
                if not near:
                    assert int(t[i]) == want, (s, k, int(t[i]), want)
                toks[s].append(int(t[i]))
        for s in batch:
            st.release(s)
        runs.append(toks)
    assert runs[0][5] == runs[1][5], "top-k draws depend on the batch"
    # greedy again: top_k 1 == argmax
    st.set_sampling(1, 0)
    st.ar_step([9], [D.PREFILL], [4], [0], [-1], [1, 2, 3, 4])
    t, _ = st.ar_step([9], [D.DECODE], [1], [4], [0], [-1])
    lg = D.d2h(st.tensor("buf.logits")[0], (256,), np.float32)
    assert int(t[0]) == 1 + int(np.argmax(lg[1:256]))
    st.close()


def test_per_entry_reserve_fails_alone():
    """omni_seq_reserve admits a sequence's KV pages ahead of the batched
    step: one sequence that does not fit gets OMNI_E_OOM by itself while the
    others still run (the reference fails per entry, ar_engine.hpp:332-334)."""
    m = D.model_default(D.THINKER, **SMALL)
    st = D.Stage(m, D.StageLimits(256, 4, 64, 6, 16), seed=3)  # 6 pages of 16 tokens
    st.reserve(1, 48)   # 3 pages
    st.reserve(2, 32)   # 2 pages
    with pytest.raises(RuntimeError) as e:
        st.reserve(3, 40)  # needs 3, one left
    assert "E_OOM" in str(e.value)
    st.reserve(3, 16)      # fits
    t, _ = st.ar_step([1, 2], [D.PREFILL, D.PREFILL], [8, 8], [0, 0], [-1, -1], [5] * 16)
    for s in (1, 2, 3):
        st.release(s)
    st.close()
