"""Uncontended time of MIXED AR steps (one 64-token prefill chunk + D decode
rows: the steady-state admission step of the closed loop) vs decode-only.
python tools/prefill_probe.py"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_02204_b200 import dev as D  # noqa: E402

m = D.model_default(D.THINKER)
st = D.Stage(m, D.StageLimits(256, 64, 512, 0, 512), seed=7)
import os
PF = [int(x) for x in os.environ.get("PF_CHUNKS", "1").split(",")]
for D_, nchunk in [(d_, c) for c in PF for d_ in (1, 5, 16)]:
    dec = list(range(1, D_ + 1))
    for s in dec:
        st.ar_step([s], [D.PREFILL], [40], [0], [-1], [(7 * j + s) % 250 + 1 for j in range(40)])
    ts, k = [], 0
    for trial in range(8):
        news = [1000 + 10 * trial + c for c in range(nchunk)]
        ids = dec + news
        toks = [-1 if k == 0 else 5] * D_ + [(3 * j + trial) % 250 + 1 for j in range(64 * nchunk)]
        st.ar_step(ids, [D.DECODE] * D_ + [D.PREFILL] * nchunk, [1] * D_ + [64] * nchunk, [40 + k] * D_ + [0] * nchunk,
                   [k] * D_ + [-1] * nchunk, toks)
        k += 1
        if trial >= 2:
            ts.append(st.last_step_us())
        for n_ in news:
            st.release(n_)
    print(json.dumps({"stage": "thinker", "decode_rows": D_, "prefill_tokens": 64 * nchunk, "M": D_ + 64 * nchunk,
                      "us_per_step": round(statistics.median(ts), 1)}), flush=True)
    for s in dec:
        st.release(s)
st.close()
