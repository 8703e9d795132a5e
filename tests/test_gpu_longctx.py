"""Full-size parity at the bench's context lengths.

The bench config reaches Thinker context 192 (prompt <= 128 + L <= 64) and
Talker context 320 (<= 64 conditioning rows + 4L <= 256 codec tokens)
(SURVEY §8a rows a6/a7). Attention stages keys in 128-key chunks
(ar_kernels.cu kAttnChunk), so every context > 128 runs the multi-chunk
online-softmax merge; these tests drive it against the CPU fp32 oracle
(oracle/models_cpu.c), teacher-forced, asserting per decode step:
  * logits:  |gpu - cpu| <= LOGIT_ATOL + LOGIT_RTOL * |cpu|   (every vocab entry)
  * hidden:  |gpu - cpu| <= HID_ATOL + HID_RTOL * |cpu|        (thinker rows)
  * greedy id identical wherever the oracle's top-2 margin > MARGIN_TOL
  * reported top-2 margin within 2 * LOGIT_ATOL of the oracle's
Tolerances are the ones DESIGN.md §3 states for the float path.
"""
import numpy as np
import pytest

import oracle
from paper_2602_02204_b200 import dev as D

pytestmark = pytest.mark.gpu

HID_ATOL, HID_RTOL = 0.03, 0.02
LOGIT_ATOL, LOGIT_RTOL = 0.12, 0.01  # measured max 0.090 (thinker ctx<=192), 0.054 (talker ctx<=320)
MARGIN_TOL = 0.20  # > 2 x the largest logit error: no near-tie within the tolerance can flip an id


def bf16_to_f32(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32)


STATS = {}


def check_logits(g, c, where, key="logit"):
    err = np.abs(g - c)
    STATS.setdefault(key, []).append(err)
    bound = LOGIT_ATOL + LOGIT_RTOL * np.abs(c)
    assert np.all(err <= bound), f"{where}: logit err {err.max():.4f} at {int(err.argmax())} (|z| {abs(c[err.argmax()]):.2f})"
    return float(err.max())


def report(key):
    e = np.concatenate(STATS.pop(key, [np.zeros(1)]))
    print(f"{key}: max {e.max():.4f} p99 {np.quantile(e, 0.99):.4f} mean {e.mean():.5f} over {e.size}")


def check_hidden(g_bits, c_bits, where):
    g, c = bf16_to_f32(g_bits), bf16_to_f32(c_bits)
    err = np.abs(g - c)
    assert np.all(err <= HID_ATOL + HID_RTOL * np.abs(c)), f"{where}: hidden err {err.max():.4f}"
    return float(err.max())


def gpu_logits(stage, dec_row, vocab):
    base, _, ld = stage.tensor("buf.logits")
    return D.d2h(base + 4 * ld * dec_row, (vocab,), np.float32)


def test_thinker_context_192_multi_chunk_attention():
    """Three sequences with 128 / 121 / 100-token prompts (the first one
    prefilled in 64-token chunks like prefill_chunk=64 does), then 64
    batched teacher-forced decode steps: contexts 129..192 (2 key chunks)."""
    m = D.model_default(D.THINKER)
    st = D.Stage(m, D.StageLimits(256, 8, 256, 0, 64), seed=17)
    om = oracle.Model(m, 17)
    rng = np.random.default_rng(21)
    prompts = [list(rng.integers(1, 256, size=n)) for n in (128, 121, 100)]
    seqs = [1, 2, 3]
    oseq = {s: om.new_seq(512) for s in seqs}
    for s, p in zip(seqs, prompts):
        spans = [64, 64] if len(p) == 128 else [len(p)]
        at = 0
        for sp in spans:
            st.ar_step([s], [D.PREFILL], [sp], [at], [-1], p[at:at + sp])
            at += sp
        oseq[s].feed(p, decode=False)
    emitted = {s: [] for s in seqs}
    worst_l = worst_h = 0.0
    checked = 0
    for k in range(64):
        tin = [(-1 if k == 0 else emitted[s][-1]) for s in seqs]
        pos0 = [len(p) + k for p in prompts]
        tok, mg = st.ar_step(seqs, [D.DECODE] * 3, [1] * 3, pos0, [k] * 3, tin)
        for i, s in enumerate(seqs):
            ot, olg, ohid, omg = oseq[s].feed([tin[i]], decode=True)
            where = f"seq {s} step {k} ctx {pos0[i] + 1}"
            worst_l = max(worst_l, check_logits(gpu_logits(st, i, m.vocab), olg, where, "thinker"))
            worst_h = max(worst_h, check_hidden(D.d2h(st.hidden_row(s, k), (m.d_model,), np.uint16), ohid, where))
            if omg > MARGIN_TOL:
                assert tok[i] == ot, f"{where}: gpu {tok[i]} cpu {ot} margin {omg:.3f}"
                assert abs(mg[i] - omg) < 2 * LOGIT_ATOL, f"{where}: margin {mg[i]:.4f} vs {omg:.4f}"
                checked += 1
            emitted[s].append(int(tok[i]))
    print(f"thinker ctx<=192: worst logit err {worst_l:.4f}, hidden err {worst_h:.4f}, "
          f"{checked}/{64 * 3} ids checked")
    report("thinker")
    assert checked >= 0.8 * 64 * 3
    st.close()


def test_talker_context_320_multi_chunk_attention():
    """64 conditioning rows (synthetic bf16 hidden rows in HBM, prefilled in
    one 64-token span) + 256 teacher-forced decode steps (row j = m/4):
    contexts 65..320 (up to 3 key chunks), two sequences batched."""
    tm = D.model_default(D.TALKER)
    d = tm.cond_dim
    rng = np.random.default_rng(22)
    n_rows = 64
    seqs = [4, 9]
    hid = {s: (rng.standard_normal((n_rows, d)).astype(np.float32) * 0.8) for s in seqs}
    hid_bits = {s: (h.view(np.uint32) >> 16).astype(np.uint16) for s, h in hid.items()}
    bufs = {s: D.mem_alloc(2 * d * n_rows) for s in seqs}
    for s in seqs:
        D.h2d(bufs[s], hid_bits[s].reshape(-1))
    text = {s: [int(x) for x in rng.integers(1, 256, size=n_rows)] for s in seqs}
    ta = D.Stage(tm, D.StageLimits(256, 8, 336, 0, 64), seed=29)
    om = oracle.Model(tm, 29)
    oseq = {}
    for s in seqs:
        rows = [bufs[s] + 2 * d * j for j in range(n_rows)]
        ta.ar_step([s], [D.PREFILL], [n_rows], [0], [-1], text[s], cond_src=rows, cond_row=list(range(n_rows)))
        oseq[s] = om.new_seq(512)
        oseq[s].feed(text[s], decode=False, cond_rows=list(range(n_rows)), hid_rows=hid_bits[s])
    codec = {s: [] for s in seqs}
    worst = 0.0
    checked = 0
    for m_ in range(4 * n_rows):
        tin = [(-1 if m_ == 0 else codec[s][-1]) for s in seqs]
        tok, mg = ta.ar_step(seqs, [D.DECODE] * 2, [1] * 2, [n_rows + m_] * 2, [m_] * 2, tin,
                             cond_src=[0, 0], cond_row=[m_ // 4] * 2)
        for i, s in enumerate(seqs):
            ot, olg, _, omg = oseq[s].feed([tin[i]], decode=True, cond_rows=[m_ // 4])
            where = f"seq {s} step {m_} ctx {n_rows + m_ + 1}"
            worst = max(worst, check_logits(gpu_logits(ta, i, tm.vocab), olg, where, "talker"))
            assert 0 <= tok[i] < 64
            if omg > MARGIN_TOL:
                assert tok[i] == ot, f"{where}: gpu {tok[i]} cpu {ot} margin {omg:.3f}"
                assert abs(mg[i] - omg) < 2 * LOGIT_ATOL
                checked += 1
            codec[s].append(int(tok[i]))
    print(f"talker ctx<=320: worst logit err {worst:.4f}, {checked}/{2 * 4 * n_rows} ids checked")
    report("talker")
    assert checked >= 0.8 * 2 * 4 * n_rows
    ta.close()
    for b in bufs.values():
        D.mem_free(b)


def test_long_prompt_split_kv_attention_matches_oracle():
    """Long prompts (the reference admits prompts up to the
    8192-token kv budget). Contexts > 1024 keys split over P <= 8 attention
    CTAs per (block, kv head) with a fixed-order last-arriver merge
    (ar_dev.cuh attention_block_mma). Two sequences with 2500 / 3900-token
    prompts (prefilled in 256-token steps: the prefill blocks split too),
    then 8 batched teacher-forced decode steps vs the fp32 oracle; then the
    same decode of one sequence alone must be bit-identical (P depends only
    on the sequence's own context: batch invariance)."""
    small = dict(d_model=512, n_layers=2, n_heads=4, n_kv_heads=1, d_ff=1024)
    m = D.model_default(D.THINKER, **small)
    lim = D.StageLimits(256, 4, 4160, 0, 64)
    rng = np.random.default_rng(31)
    lens = {1: 2500, 2: 3900}
    prompts = {s: [int(x) for x in rng.integers(1, 256, size=n)] for s, n in lens.items()}

    def prefill(st):
        for s, p in prompts.items():
            for at in range(0, len(p), 256):
                sp = min(256, len(p) - at)
                st.ar_step([s], [D.PREFILL], [sp], [at], [-1], p[at:at + sp])

    st = D.Stage(m, lim, seed=41)
    om = oracle.Model(m, 41)
    oseq = {s: om.new_seq(4160) for s in prompts}
    prefill(st)
    for s, p in prompts.items():
        oseq[s].feed(p, decode=False)
    seqs = [1, 2]
    emitted = {s: [] for s in seqs}
    hidden = {s: [] for s in seqs}
    checked = 0
    for k in range(8):
        tin = [(-1 if k == 0 else emitted[s][-1]) for s in seqs]
        pos0 = [lens[s] + k for s in seqs]
        tok, mg = st.ar_step(seqs, [D.DECODE] * 2, [1] * 2, pos0, [k] * 2, tin)
        for i, s in enumerate(seqs):
            ot, olg, ohid, omg = oseq[s].feed([tin[i]], decode=True)
            where = f"seq {s} step {k} ctx {pos0[i] + 1}"
            check_logits(gpu_logits(st, i, m.vocab), olg, where, "longctx")
            h = D.d2h(st.hidden_row(s, k), (m.d_model,), np.uint16)
            check_hidden(h, ohid, where)
            hidden[s].append(h)
            if omg > MARGIN_TOL:
                assert tok[i] == ot, f"{where}: gpu {tok[i]} cpu {ot} margin {omg:.3f}"
                checked += 1
            emitted[s].append(int(tok[i]))
    report("longctx")
    assert checked >= 12
    st.close()
    # sequence 2 alone: identical tokens and hidden rows
    st = D.Stage(m, lim, seed=41)
    prefill(st)
    for k in range(8):
        tok, _ = st.ar_step([2], [D.DECODE], [1], [lens[2] + k], [k], [-1 if k == 0 else emitted[2][k - 1]])
        assert int(tok[0]) == emitted[2][k]
        assert np.array_equal(D.d2h(st.hidden_row(2, k), (m.d_model,), np.uint16), hidden[2][k])
    st.close()
