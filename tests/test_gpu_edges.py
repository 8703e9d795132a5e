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


@pytest.mark.parametrize("kind", [D.THINKER])
def test_step_chain_bit_identical_to_kernel_chain(kind):
    """The one-launch step chain (chain.cu) and the per-kernel PDL path give
    bit-identical tokens and hidden rows (same tiles, same split-K order)."""
    kw = dict(SMALL)
    if kind == D.TALKER:
        kw["cond_dim"] = 512
    m = D.model_default(kind, **kw)
    rng = np.random.default_rng(11)
    prompts = {s: list(rng.integers(1, 256, size=n)) for s, n in ((1, 9), (2, 14), (3, 5))}
    outs = []
    for chain in (True, False):
        st = D.Stage(m, D.StageLimits(256, 16, 256, 0, 16), seed=17)
        st.set_chain(chain)
        cond = None
        if kind == D.TALKER:
            cond = D.mem_alloc(2 * 512 * 16)
            bits = ((rng.standard_normal(512 * 16).astype(np.float32) * 0.5).view(np.uint32) >> 16).astype(np.uint16)
            D.h2d(cond, bits)
        for s, p in prompts.items():
            if kind == D.TALKER:
                st.ar_step([s], [D.PREFILL], [len(p)], [0], [-1], p,
                           cond_src=[cond + 2 * 512 * (j % 16) for j in range(len(p))],
                           cond_row=list(range(len(p))))
            else:
                st.ar_step([s], [D.PREFILL], [len(p)], [0], [-1], p)
        seqs = sorted(prompts)
        toks = {s: [] for s in seqs}
        hids = []
        for k in range(4):
            tin = [-1 if k == 0 else toks[s][-1] for s in seqs]
            pos = [len(prompts[s]) + k for s in seqs]
            extra = dict(cond_src=[0] * 3, cond_row=[k // 4] * 3) if kind == D.TALKER else {}
            t, mg = st.ar_step(seqs, [D.DECODE] * 3, [1] * 3, pos, [k] * 3, tin, **extra)
            for i, s in enumerate(seqs):
                toks[s].append(int(t[i]))
            if kind == D.THINKER:
                hids.append(np.stack([D.d2h(st.hidden_row(s, k), (512,), np.uint16) for s in seqs]))
            else:
                lg = D.d2h(st.tensor("buf.logits")[0], (3, st.tensor("buf.logits")[2]), np.float32)
                hids.append(lg[:, :m.vocab])  # columns >= vocab are padding (never written)
        outs.append((toks, hids))
        st.close()
    assert outs[0][0] == outs[1][0]
    for a, b in zip(outs[0][1], outs[1][1]):
        assert np.array_equal(a, b)


def test_fused_head_matches_kernel_head(monkeypatch):
    """OMNI_FUSED_HEAD=1 (final norm + CUDA-core LM head + argmax in one
    kernel, split over CTAs with a last-CTA argmax) gives the same tokens and
    bit-identical hidden rows as final_gather + tcgen05 LM GEMM + argmax;
    logits agree to fp32 summation-order tolerance."""
    m = D.model_default(D.THINKER, **SMALL)
    rng = np.random.default_rng(21)
    prompts = {s: list(rng.integers(1, 256, size=n)) for s, n in ((1, 7), (2, 12), (3, 20), (4, 3))}
    outs = []
    for fused in ("1", "0"):
        monkeypatch.setenv("OMNI_FUSED_HEAD", fused)
        st = D.Stage(m, D.StageLimits(256, 16, 256, 0, 16), seed=23)
        for s, p in prompts.items():
            st.ar_step([s], [D.PREFILL], [len(p)], [0], [-1], p)
        seqs = sorted(prompts)
        toks = {s: [] for s in seqs}
        hids, lgs = [], []
        for k in range(6):  # repeated steps replay the self-resetting CTA tickets
            tin = [-1 if k == 0 else toks[s][-1] for s in seqs]
            t, _ = st.ar_step(seqs, [D.DECODE] * 4, [1] * 4, [len(prompts[s]) + k for s in seqs], [k] * 4, tin)
            for i, s in enumerate(seqs):
                toks[s].append(int(t[i]))
            hids.append(np.stack([D.d2h(st.hidden_row(s, k), (512,), np.uint16) for s in seqs]))
            lg = st.tensor("buf.logits")
            lgs.append(D.d2h(lg[0], (4, lg[2]), np.float32)[:, :m.vocab])
        outs.append((toks, hids, lgs))
        st.close()
    assert outs[0][0] == outs[1][0]
    for a, b in zip(outs[0][1], outs[1][1]):
        assert np.array_equal(a, b)
    for a, b in zip(outs[0][2], outs[1][2]):
        np.testing.assert_allclose(a, b, rtol=1e-4, atol=1e-4)
