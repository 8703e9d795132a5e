"""Per-item timeline of the fused DiT iteration (OMNI_DIT_TRACE=1).

For each item kind: count, mean fetch->dep-ok wait, dep-ok->mainloop-done,
mainloop-done->done (epilogue), and per-phase critical-path time of row tile 0.
Usage: OMNI_DIT_TRACE=1 python tools/dit_trace.py [--sms=N] [tokens ...]
(--sms: the persistent grid, as omni_stage_set_sm_share sets it beside AR stages)
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
    ntoks = [int(a) for a in sys.argv[1:] if not a.startswith("--")] or [8, 64]
    sms = [int(a.split("=")[1]) for a in sys.argv[1:] if a.startswith("--sms=")]
    m = D.model_default(D.DIT)
    st = D.Stage(m, D.StageLimits(256, 64, 512, 0, 512), seed=9)
    if sms:
        st.set_sm_share(sms[0])
    d, L, T, H, ff = m.d_model, m.n_layers, m.dit_steps, m.n_heads, m.d_ff
    nf, ds = d // 128, (2 if ff >= 2 * d and (ff // 64) % 2 == 0 else 1)  # stage.cpp down_split
    for n in ntoks:
        toks = [(5 * i) % 64 for i in range(n)]
        for _ in range(3):
            st.dit_step([1], [0], [n], toks)
        us = st.last_step_us()
        ptr, rows, cols = st.tensor("buf.dit_trace")
        wide_from = sms[0] if sms else 148
        n_pad = (n + 7) // 8 * 8
        if n_pad >= wide_from:
            n_pad = (n + 15) // 16 * 16
        tr_rows = 256 if n_pad >= wide_from and n_pad % 16 == 0 else 128
        tok = tr_rows // 16
        n_rt = n_pad * 16 // tr_rows
        ph = phases(L)
        items_pp = {"IN": nf, "LN1": tok, "QKV": 3 * nf, "ATT": H * tok // 8, "O": nf, "LN2": tok, "UP": ff // 128,
                    "DOWN": nf * ds, "LNF": tok, "OUT": 1}
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
        span = tr[:, 3].max() - t0
        rep = {"tokens": n, "tile_rows": tr_rows, "sms": sms[0] if sms else None, "us_per_step": round(us, 1),
               "items": total, "span_us": round(span / 1e3, 1)}
        # per-CTA occupancy: share of the span each CTA spends waiting for
        # dependencies, in GEMM mainloops (dep ok -> accumulator ready), in
        # epilogues / LN / attention work, and idle between items
        gemm = np.isin(kinds, ["IN", "QKV", "O", "UP", "DOWN", "OUT"])
        ncta = len(np.unique(tr[:, 4]))
        w = float(np.sum(tr[:, 1] - tr[:, 0])) / (span * ncta)
        mm = float(np.sum((tr[:, 2] - tr[:, 1])[gemm])) / (span * ncta)
        ep = float(np.sum((tr[:, 3] - tr[:, 2]))) / (span * ncta)
        rep["cta_share"] = {"ctas": ncta, "dep_wait": round(w, 3), "gemm_main": round(mm, 3), "epi_or_ln_att": round(ep, 3)}
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
