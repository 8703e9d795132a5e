"""Uncontended per-stage step times (one stage alone on the GPU).

  python tools/step_probe.py [--quick]

Thinker / Talker: B sequences are prefilled with P prompt tokens, then D
decode steps of the whole batch are timed (device time of each step from the
stage's CUDA events, omni_stage_last_step_us). DiT: one batched denoise step
over n codec tokens. Prints one JSON line per point.
"""
from __future__ import annotations

import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2602_02204_b200 import dev as D  # noqa: E402

THINKER_BYTES = 8 * 60_817_408 * 2 + 2 * 256 * 2048 * 2
TALKER_BYTES = 4 * 60_817_408 * 2 + 2048 * 2048 * 2 + 64 * 2048 * 2


def ar_probe(kind: int, batches, prompt: int = 64, steps: int = 12):
    m = D.model_default(kind)
    # long contexts (split-KV attention beyond 1024 keys): fewer residents, longer sequences
    lim = D.StageLimits(256, 64, 512, 0, 512) if prompt + steps <= 448 else \
        D.StageLimits(256, 16, prompt + steps + 64, 0, 512)
    st = D.Stage(m, lim, seed=7)
    wbytes = THINKER_BYTES if kind == D.THINKER else TALKER_BYTES
    cond = D.mem_alloc(2 * m.cond_dim * 256) if kind == D.TALKER else 0
    if cond:
        D.mem_set(cond, 0, 2 * m.cond_dim * 256)
    out = []
    for B in batches:
        ids = list(range(1000 * (B + 1), 1000 * (B + 1) + B))
        # prefill in steps of <= 256 tokens (groups of whole prompts, long prompts chunked)
        per = max(1, 256 // prompt)
        for i in range(0, B, per):
            grp = ids[i:i + per]
            for at in range(0, prompt, 256):
                sp = min(256, prompt - at)
                toks = [(7 * j + 3) % 250 + 1 for j in range(at, at + sp)] * len(grp)
                cs = [cond + 2 * m.cond_dim * (j % 256) for j in range(len(toks))] if kind == D.TALKER else None
                cr = [j % 64 for _ in grp for j in range(at, at + sp)] if kind == D.TALKER else None
                st.ar_step(grp, [D.PREFILL] * len(grp), [sp] * len(grp), [at] * len(grp), [-1] * len(grp),
                           toks, cs, cr)
        prev = [-1] * B
        ts = []
        for k in range(steps):
            cs = [0] * B if kind == D.TALKER else None
            cr = [min(k // 4, prompt - 1, 63)] * B if kind == D.TALKER else None
            tok, _ = st.ar_step(ids, [D.DECODE] * B, [1] * B, [prompt + k] * B, [k] * B, prev, cs, cr)
            prev = [int(t) for t in tok]
            if k >= 2:
                ts.append(st.last_step_us())
        for s in ids:
            st.release(s)
        us = statistics.median(ts)
        r = {"stage": "thinker" if kind == D.THINKER else "talker", "decode_rows": B, "ctx": prompt,
             "us_per_step": round(us, 1), "weight_GBps": round(wbytes / us / 1e3, 1),
             "ideal_us_6553": round(wbytes / 6553e3, 1)}
        print(json.dumps(r), flush=True)
        out.append(r)
    st.close()
    return out


def dit_probe(ntoks):
    m = D.model_default(D.DIT)
    st = D.Stage(m, D.StageLimits(256, 64, 512, 0, 1024), seed=9)
    for n in ntoks:
        jobs = max(1, n // 8)
        per = [n // jobs] * jobs
        per[-1] += n - sum(per)
        toks = [(5 * i) % 64 for i in range(n)]
        ts = []
        for it in range(5):
            st.dit_step(list(range(1, jobs + 1)), [0] * jobs, per, toks)
            if it >= 1:
                ts.append(st.last_step_us())
        us = statistics.median(ts)
        rows = 16 * n
        d, L, T = m.d_model, m.n_layers, m.dit_steps
        flops = T * rows * L * 24 * d * d
        print(json.dumps({"stage": "code2wav", "tokens": n, "rows": rows, "us_per_step": round(us, 1),
                          "TFLOPs": round(flops / us / 1e6, 1)}), flush=True)
    st.close()


if __name__ == "__main__":
    quick = "--quick" in sys.argv
    ctxs = [int(a.split("=")[1]) for a in sys.argv if a.startswith("--ctx=")]
    if ctxs:  # step time vs context length (attention scaling), 16 decode rows
        for c in ctxs:
            ar_probe(D.TALKER, [16], prompt=c)
            ar_probe(D.THINKER, [4], prompt=c)
    elif "--dit-only" not in sys.argv:
        ar_probe(D.THINKER, [1, 4, 16] if quick else [1, 2, 4, 8, 16, 32, 64])
        ar_probe(D.TALKER, [1, 16] if quick else [1, 4, 16, 32, 64])
    if ctxs:
        pass
    elif "--dit64" in sys.argv:
        dit_probe([64])
    elif "--ar-only" not in sys.argv:
        dit_probe([8, 64] if quick else [8, 32, 64, 128, 256, 512])
