"""Per-item timeline of the fused DiT iteration (OMNI_DIT_TRACE=1).

For each item kind: count, mean fetch->dep-ok wait, dep-ok->mainloop-done,
mainloop-done->done (epilogue), and per-phase critical-path time of row tile 0.
Usage: OMNI_DIT_TRACE=1 python tools/dit_trace.py [tokens ...]
"""
import json
import os
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["OMNI_DIT_TRACE"] = "1"
from paper_2602_02204_b200 import dev as D  # noqa: E402

KINDS = ["IN", "LN1", "QKV", "ATT", "O", "LN2", "UP", "DOWN", "LNF", "OUT"]


def phases(L):
    out = ["IN"]
    for _ in range(L):
        out += ["LN1", "QKV", "ATT", "O", "LN2", "UP", "DOWN"]
    return out + ["LNF", "OUT"]


def main():
    ntoks = [int(a) for a in sys.argv[1:]] or [8, 64]
    m = D.model_default(D.DIT)
    st = D.Stage(m, D.StageLimits(256, 64, 512, 0, 512), seed=9)
    d, L, T, H, ff = m.d_model, m.n_layers, m.dit_steps, m.n_heads, m.d_ff
    nf, ds = d // 128, (2 if ff >= 2 * d else 1)
    for n in ntoks:
        toks = [(5 * i) % 64 for i in range(n)]
        for _ in range(3):
            st.dit_step([1], [0], [n], toks)
        us = st.last_step_us()
        ptr, rows, cols = st.tensor("buf.dit_trace")
        n_rt = (n + 15) // 16
        ph = phases(L)
        items_pp = {"IN": nf, "LN1": 16, "QKV": 3 * nf, "ATT": 4 * H, "O": nf, "LN2": 16, "UP": ff // 128,
                    "DOWN": nf * ds, "LNF": 16, "OUT": 1}
        total = sum(items_pp[k] for k in ph) * T * n_rt
        tr = D.d2h(ptr, (total, 8), np.uint64).astype(np.int64)
        t0 = tr[:, 0].min()
        # item -> kind, tile
        kinds, tiles, tps = [], [], []
        for t in range(T):
            for pi, k in enumerate(ph):
                for r in range(n_rt):
                    for j in range(items_pp[k]):
                        kinds.append(k)
                        tiles.append(r)
                        tps.append(t * len(ph) + pi)
        kinds, tiles, tps = np.array(kinds), np.array(tiles), np.array(tps)
        rep = {"tokens": n, "us_per_step": round(us, 1), "items": total, "span_us": round((tr[:, 3].max() - t0) / 1e3, 1)}
        per = {}
        for k in KINDS:
            sel = kinds == k
            if not sel.any():
                continue
            a = tr[sel]
            per[k] = {"n": int(sel.sum()),
                      "wait_dep": round(float(np.mean(a[:, 1] - a[:, 0])) / 1e3, 2),
                      "main": round(float(np.mean(a[:, 2] - a[:, 1])) / 1e3, 2),
                      "epi": round(float(np.mean(a[:, 3] - a[:, 2])) / 1e3, 2),
                      "loop": round(float(np.mean(np.where(a[:, 5] > 0, a[:, 5] - a[:, 2], 0))) / 1e3, 2),
                      "bar": round(float(np.mean(np.where((a[:, 6] > 0) & (a[:, 5] > 0), a[:, 6] - a[:, 5], 0))) / 1e3, 2),
                      "ld_cyc": round(float(np.mean(np.where(a[:, 5] > 0, a[:, 7] >> 32, 0))), 0),
                      "loop_cyc": round(float(np.mean(np.where(a[:, 5] > 0, a[:, 7] & 0xffffffff, 0))), 0),
                      "sig": round(float(np.mean(np.where(a[:, 6] > 0, a[:, 3] - a[:, 6], 0))) / 1e3, 2)}
        rep["per_kind_us"] = per
        # tile 0: phase completion times (critical path)
        done = []
        for tp in range(T * len(ph)):
            sel = (tps == tp) & (tiles == 0)
            done.append(int(tr[sel, 3].max() - t0))
        steps = np.diff([0] + done) / 1e3
        by = {}
        for i, dt in enumerate(steps):
            by.setdefault(ph[i % len(ph)], []).append(dt)
        rep["tile0_phase_us"] = {k: round(statistics.mean(v), 2) for k, v in by.items()}
        print(json.dumps(rep), flush=True)
    st.close()


if __name__ == "__main__":
    main()
