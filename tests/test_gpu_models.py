"""GPU parity of the stage models (K1-K6) against the CPU fp32 oracle.

The reference has no float model (parity unpinned for hidden
states / logits / latents); oracle/models_cpu.c defines it. Tolerances:
  * hidden rows (bf16):      |gpu - cpu| <= HID_ATOL + HID_RTOL * |cpu|
  * logits (fp32):           |gpu - cpu| <= LOGIT_ATOL
  * greedy ids: identical wherever the oracle's top-2 margin > MARGIN_TOL
    (teacher forcing: both sides consume the GPU's emitted token stream)
  * DiT latents (fp32):      |gpu - cpu| <= LAT_ATOL + LAT_RTOL * |cpu|
  * DiT samples (int32):     |gpu - cpu| <= 1 (rint of 24 x latent), >= 90 % exact
Batch invariance / chunked prefill / chunking transparency are checked
bit-exact GPU-vs-GPU.
"""
import numpy as np
import pytest

import oracle
from paper_2602_02204_b200 import dev as D

pytestmark = pytest.mark.gpu

HID_ATOL, HID_RTOL = 0.03, 0.02
LOGIT_ATOL = 0.05
MARGIN_TOL = 0.05
LAT_ATOL, LAT_RTOL = 0.02, 0.02

SMALL = dict(d_model=512, n_layers=2, n_heads=4, n_kv_heads=2, d_ff=1024)


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def hidden_bits(stage, seq, k, d):
    return D.d2h(stage.hidden_row(seq, k), (d,), np.uint16)


def check_hidden(g_bits, c_bits):
    g, c = bf16_to_f32(g_bits), bf16_to_f32(c_bits)
    err = np.abs(g - c)
    bound = HID_ATOL + HID_RTOL * np.abs(c)
    assert np.all(err <= bound), f"hidden mismatch max {err.max():.4f}"
    return float(err.max())


def run_thinker(stage, om, prompts, n_dec, chunk=None):
    """Feeds prompts (one seq each, own step per prefill chunk) then n_dec
    batched decode steps; returns per-seq (tokens, margins) and oracle checks."""
    d = stage.model.d_model
    seqs = list(range(1, len(prompts) + 1))
    oseqs = {s: om.new_seq(256) for s in seqs}
    for s, p in zip(seqs, prompts):
        spans = [len(p)] if chunk is None else [min(chunk, len(p) - i) for i in range(0, len(p), chunk)]
        at = 0
        for sp in spans:
            stage.ar_step([s], [D.PREFILL], [sp], [at], [-1], p[at:at + sp])
            at += sp
        oseqs[s].feed(p, decode=False)
    emitted = {s: [] for s in seqs}
    worst = 0.0
    for k in range(n_dec):
        toks_in = [(-1 if k == 0 else emitted[s][-1]) for s in seqs]
        pos0 = [len(p) + k for p in prompts]
        tok, mg = stage.ar_step(seqs, [D.DECODE] * len(seqs), [1] * len(seqs), pos0, [k] * len(seqs), toks_in)
        for i, s in enumerate(seqs):
            ot, olg, ohid, omg = oseqs[s].feed([toks_in[i]], decode=True)
            if omg > MARGIN_TOL:
                assert tok[i] == ot, f"seq {s} step {k}: gpu {tok[i]} cpu {ot} margin {omg}"
            worst = max(worst, check_hidden(hidden_bits(stage, s, k, d), ohid))
            assert abs(mg[i] - omg) < 2 * LOGIT_ATOL or omg <= MARGIN_TOL
            emitted[s].append(int(tok[i]))
    return emitted, worst


@pytest.fixture(scope="module")
def small_thinker():
    m = D.model_default(D.THINKER, **SMALL)
    st = D.Stage(m, D.StageLimits(256, 16, 256, 0, 64), seed=11)
    om = oracle.Model(m, 11)
    return st, om


def test_weights_bit_exact(small_thinker):
    st, om = small_thinker
    for name in ("embed", "lm_head", "L0.wqkv"):
        p, rows, cols = st.tensor(name)
        w = D.d2h(p, (rows, cols), np.uint16)
        for (r, c) in [(0, 0), (1, 5), (rows // 2, cols - 1), (min(rows, 255) - 1, 3)]:
            if name == "lm_head" and r >= 256:
                continue
            assert w[r, c] == om.weight_bits(name, r, c), (name, r, c)


def test_thinker_parity_small(small_thinker):
    st, om = small_thinker
    rng = np.random.default_rng(0)
    prompts = [list(rng.integers(1, 256, size=n)) for n in (17, 40, 5)]
    emitted, worst = run_thinker(st, om, prompts, n_dec=6)
    print("thinker small worst hidden err", worst, emitted)
    for s in (1, 2, 3):
        st.release(s)


def test_thinker_chunked_prefill_and_batch_invariance(small_thinker):
    st, _ = small_thinker
    d = st.model.d_model
    rng = np.random.default_rng(1)
    p = list(rng.integers(1, 256, size=37))
    # A: one span, decode alone
    st.ar_step([50], [0], [37], [0], [-1], p)
    ta, _ = st.ar_step([50], [1], [1], [37], [0], [-1])
    ha = hidden_bits(st, 50, 0, d)
    la = D.d2h(st.tensor("buf.logits")[0], (256,), np.float32)
    # B: chunked prefill 16+16+5, decode batched with 9 other decoders + a prefill
    for at in range(0, 37, 16):
        sp = min(16, 37 - at)
        st.ar_step([60], [0], [sp], [at], [-1], p[at:at + sp])
    others = list(range(70, 79))
    for o in others:
        st.ar_step([o], [0], [8], [0], [-1], list(rng.integers(1, 256, size=8)))
    seqs = others[:4] + [60] + others[4:]
    tb, _ = st.ar_step(seqs + [90], [1] * 10 + [0], [1] * 10 + [12], [8] * 4 + [37] + [8] * 5 + [0],
                       [0] * 10 + [-1], [-1] * 10 + list(rng.integers(1, 256, size=12)))
    hb = hidden_bits(st, 60, 0, d)
    lb = D.d2h(st.tensor("buf.logits")[0] + 4 * 256 * 4, (256,), np.float32)
    assert tb[4] == ta[0]
    assert np.array_equal(ha, hb), "hidden row differs between solo and batched/chunked runs"
    assert np.array_equal(la, lb), "logits differ between solo and batched/chunked runs"
    for s in [50, 60, 90] + others:
        st.release(s)


def test_thinker_parity_default_dims():
    m = D.model_default(D.THINKER)
    st = D.Stage(m, D.StageLimits(256, 8, 256, 0, 64), seed=7)
    om = oracle.Model(m, 7)
    rng = np.random.default_rng(2)
    prompts = [list(rng.integers(1, 256, size=n)) for n in (24, 9)]
    emitted, worst = run_thinker(st, om, prompts, n_dec=3)
    print("thinker default worst hidden err", worst, emitted)
    st.close()


def test_thinker_batch_invariance_default_dims():
    """Full-size Thinker: one sequence's decode row is bit-identical whether
    it runs alone (M=1: 16-token tile, push split-K), among 20 decoders
    (32-token tile, push) or among 40 decoders (64-token tile, cluster-pull
    reduction) -- split factors are per weight, sum order per rank fixed."""
    m = D.model_default(D.THINKER)
    st = D.Stage(m, D.StageLimits(256, 48, 256, 0, 64), seed=9)
    d = m.d_model
    rng = np.random.default_rng(12)
    p = list(rng.integers(1, 256, size=30))
    others = {o: list(rng.integers(1, 256, size=5 + o % 7)) for o in range(100, 139)}
    res = []
    for n_other in (0, 19, 39):
        seq = 1 + n_other
        st.ar_step([seq], [0], [30], [0], [-1], p)
        batch = sorted(others)[:n_other]
        for o in batch:
            st.ar_step([o], [0], [len(others[o])], [0], [-1], others[o])
        ids = sorted([seq] + batch)
        pos = [30 if s == seq else len(others[s]) for s in ids]
        t, _ = st.ar_step(ids, [1] * len(ids), [1] * len(ids), pos, [0] * len(ids), [-1] * len(ids))
        res.append((int(t[ids.index(seq)]), hidden_bits(st, seq, 0, d)))
        for s in ids:
            st.release(s)
    for tok, h in res[1:]:
        assert tok == res[0][0]
        assert np.array_equal(h, res[0][1]), "decode row depends on the batch"
    st.close()


def test_talker_parity_small(small_thinker):
    th, _ = small_thinker
    d = th.model.d_model
    rng = np.random.default_rng(3)
    p = list(rng.integers(1, 256, size=12))
    th.ar_step([5], [0], [12], [0], [-1], p)
    text = []
    for k in range(3):
        t, _ = th.ar_step([5], [1], [1], [12 + k], [k], [-1 if k == 0 else text[-1]])
        text.append(int(t[0]))
    rows = [th.hidden_row(5, k) for k in range(3)]
    hid_bits = np.stack([D.d2h(r, (d,), np.uint16) for r in rows])
    tm = D.model_default(D.TALKER, **SMALL, cond_dim=d)
    ta = D.Stage(tm, D.StageLimits(256, 8, 256, 0, 64), seed=21)
    om = oracle.Model(tm, 21)
    # prefill the 3 text rows (prompt = text tokens, conditioned on hidden rows)
    ta.ar_step([5], [0], [3], [0], [-1], text, cond_src=rows, cond_row=[0, 1, 2])
    os_ = om.new_seq(64)
    os_.feed(text, decode=False, cond_rows=[0, 1, 2], hid_rows=hid_bits)
    codec = []
    for m_ in range(12):
        tin = -1 if m_ == 0 else codec[-1]
        t, mg = ta.ar_step([5], [1], [1], [3 + m_], [m_], [tin], cond_src=[0], cond_row=[m_ // 4])
        ot, _, _, omg = os_.feed([tin], decode=True, cond_rows=[m_ // 4])
        if omg > MARGIN_TOL:
            assert t[0] == ot, (m_, t[0], ot, omg)
        assert 0 <= t[0] < 64
        codec.append(int(t[0]))
    print("talker codec", codec)
    th.release(5)
    ta.close()


def test_talker_parity_default_dims():
    """Full-size Talker (d 2048, 4 layers, V 64, conditioning projection
    2048x2048) against the oracle: 3 conditioning rows (synthetic bf16
    hidden rows in HBM), prefill + 12 teacher-forced decode steps."""
    tm = D.model_default(D.TALKER)
    d = tm.cond_dim
    rng = np.random.default_rng(6)
    hid = (rng.standard_normal((3, d)).astype(np.float32) * 0.8)
    hid_bits = (hid.view(np.uint32) >> 16).astype(np.uint16)
    buf = D.mem_alloc(2 * d * 3)
    D.h2d(buf, hid_bits.reshape(-1))
    rows = [buf + 2 * d * j for j in range(3)]
    ta = D.Stage(tm, D.StageLimits(256, 8, 256, 0, 64), seed=23)
    om = oracle.Model(tm, 23)
    text = [17, 203, 9]
    ta.ar_step([2], [0], [3], [0], [-1], text, cond_src=rows, cond_row=[0, 1, 2])
    os_ = om.new_seq(64)
    os_.feed(text, decode=False, cond_rows=[0, 1, 2], hid_rows=hid_bits)
    codec = []
    for m_ in range(12):
        tin = -1 if m_ == 0 else codec[-1]
        t, mg = ta.ar_step([2], [1], [1], [3 + m_], [m_], [tin], cond_src=[0], cond_row=[m_ // 4])
        ot, _, _, omg = os_.feed([tin], decode=True, cond_rows=[m_ // 4])
        if omg > MARGIN_TOL:
            assert t[0] == ot, (m_, t[0], ot, omg)
            assert abs(mg[0] - omg) < 2 * LOGIT_ATOL
        assert 0 <= t[0] < 64
        codec.append(int(t[0]))
    print("talker default codec", codec)
    ta.close()
    D.mem_free(buf)


def test_pack_hidden_bit_exact(small_thinker):
    th, _ = small_thinker
    d = th.model.d_model
    rng = np.random.default_rng(4)
    p = list(rng.integers(1, 256, size=6))
    th.ar_step([9], [0], [6], [0], [-1], p)
    toks = []
    for k in range(9):
        t, _ = th.ar_step([9], [1], [1], [6 + k], [k], [-1 if k == 0 else toks[-1]])
        toks.append(int(t[0]))
    ring = np.stack([D.d2h(th.hidden_row(9, k), (d,), np.uint16) for k in range(9)])
    chunks = [(0, 4), (4, 8), (8, 9), (9, 9), (1, 8)]
    sizes = [D.pack_bytes(e - b, d) for b, e in chunks]
    offs, at = [], 0
    for s in sizes:
        offs.append(at)
        at += (s + 15) // 16 * 16
    arena = D.mem_alloc(at + 64)
    D.mem_set(arena, 0xAB, at + 64)
    th.pack_hidden([9] * len(chunks), [b for b, _ in chunks], [e for _, e in chunks],
                   sum([toks[b:e] for b, e in chunks], []), arena, offs)
    th.wait()
    D.sync()
    blob = D.d2h(arena, (at,), np.uint8).tobytes()
    for (b, e), o, s in zip(chunks, offs, sizes):
        want = oracle.pack_hidden_blob(toks[b:e], ring[b:e].reshape(e - b, d))
        assert blob[o:o + s] == want, f"pack chunk {(b, e)} differs"
    D.mem_free(arena)
    th.release(9)


@pytest.fixture(scope="module")
def small_dit():
    m = D.model_default(D.DIT, d_model=256, n_layers=2, n_heads=2, n_kv_heads=2, d_ff=512)
    st = D.Stage(m, D.StageLimits(256, 8, 256, 0, 64), seed=31)
    om = oracle.Model(m, 31)
    return st, om


def check_samples(g, c):
    diff = np.abs(g.astype(np.int64) - c.astype(np.int64))
    assert diff.max() <= 1, f"DiT sample diff {diff.max()}"
    assert (diff == 0).mean() >= 0.90, f"only {(diff == 0).mean():.3f} exact"


def check_latents(st, c_lat, n_tok):
    C = st.model.dit_channels
    g = D.d2h(st.tensor("buf.dit_x")[0], (n_tok * 16 * C,), np.float32)
    err = np.abs(g - c_lat)
    assert np.all(err <= LAT_ATOL + LAT_RTOL * np.abs(c_lat)), f"latent err {err.max():.4f}"
    return float(err.max())


def test_dit_parity_and_chunking(small_dit):
    st, om = small_dit
    rng = np.random.default_rng(5)
    codec = list(rng.integers(0, 64, size=21))
    whole = st.dit_step([7], [0], [21], codec)
    c, lat = om.dit([7] * 21, list(range(21)), codec, with_latents=True)
    print("dit small latent err", check_latents(st, lat, 21))
    check_samples(whole, c)
    # chunking transparency: any split concatenates to the whole (bit-exact)
    for split in (1, 4, 8, 13):
        parts = []
        for at in range(0, 21, split):
            n = min(split, 21 - at)
            parts.append(st.dit_step([7], [at], [n], codec[at:at + n]))
        assert np.array_equal(np.concatenate(parts), whole), split
    # batched with another request: same bits
    both = st.dit_step([3, 7], [0, 0], [5, 21], list(rng.integers(0, 64, size=5)) + codec)
    assert np.array_equal(both[5 * 16:], whole)


def test_dit_parity_default_dims():
    m = D.model_default(D.DIT)
    st = D.Stage(m, D.StageLimits(256, 8, 256, 0, 64), seed=41)
    om = oracle.Model(m, 41)
    codec = [5, 63, 0, 17, 42, 9, 33, 60]
    g = st.dit_step([2], [8], [8], codec)
    c, lat = om.dit([2] * 8, list(range(8, 16)), codec, with_latents=True)
    print("dit default latent err", check_latents(st, lat, 8))
    check_samples(g, c)
    st.close()
