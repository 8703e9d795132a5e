"""One AR stage alone: prefill B sequences of `ctx` tokens, then `steps`
decode steps of the whole batch. Under ncu --graph-profiling graph the
decode-only steps replay as ONE CUDA graph each (PDL edges intact), so ncu
reports whole-step duration and DRAM bytes per step.

  python tools/ncu_step_graph.py thinker|talker B [ctx] [steps]
"""
from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2602_02204_b200 import dev as D  # noqa: E402


def main():
    kind = D.THINKER if sys.argv[1] == "thinker" else D.TALKER
    B = int(sys.argv[2])
    ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 64
    steps = int(sys.argv[4]) if len(sys.argv) > 4 else 24
    m = D.model_default(kind)
    st = D.Stage(m, D.StageLimits(256, 64, 512, 0, 512), seed=7)
    cond = D.mem_alloc(2 * m.cond_dim * 256) if kind == D.TALKER else 0
    if cond:
        D.mem_set(cond, 0, 2 * m.cond_dim * 256)
    ids = list(range(1, B + 1))
    per = max(1, 256 // ctx)
    for i in range(0, B, per):
        grp = ids[i:i + per]
        toks = [(7 * j + 3) % 250 + 1 for j in range(ctx)] * len(grp)
        cs = [cond] * len(toks) if kind == D.TALKER else None
        cr = [j % 64 for _ in grp for j in range(ctx)] if kind == D.TALKER else None
        st.ar_step(grp, [D.PREFILL] * len(grp), [ctx] * len(grp), [0] * len(grp), [-1] * len(grp), toks, cs, cr)
    prev = [-1] * B
    us = []
    for k in range(steps):
        cs = [cond] * B if kind == D.TALKER else None
        cr = [min(k // 4, 63)] * B if kind == D.TALKER else None
        tok, _ = st.ar_step(ids, [D.DECODE] * B, [1] * B, [ctx + k] * B, [k] * B, prev, cs, cr)
        prev = [int(t) for t in tok]
        us.append(st.last_step_us())
    print(f"{sys.argv[1]} B={B} ctx={ctx}: last steps us {[round(u, 1) for u in us[-5:]]}", flush=True)
    st.close()


if __name__ == "__main__":
    main()
