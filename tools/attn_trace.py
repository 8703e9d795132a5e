"""Phase trace of the last attention launch of a decode step (and the
QKV-exit / O-projection wait marks of the same layer), globaltimer ns.
python tools/attn_trace.py [thinker|talker] [rows]"""
import ctypes as C
import json
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_02204_b200 import dev as D  # noqa: E402

kind = D.TALKER if (len(sys.argv) > 1 and sys.argv[1] == "talker") else D.THINKER
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
lib = D.dev_lib()
m = D.model_default(kind)
st = D.Stage(m, D.StageLimits(256, 64, 512, 0, 512), seed=7)
cond = D.mem_alloc(2 * m.cond_dim * 256) if kind == D.TALKER else 0
if cond:
    D.mem_set(cond, 0, 2 * m.cond_dim * 256)
P = 64
ids = list(range(1, B + 1))
for i in range(0, B, 4):
    grp = ids[i:i + 4]
    toks = [(7 * j + 3) % 250 + 1 for j in range(P)] * len(grp)
    cs = [cond + 2 * m.cond_dim * (j % 256) for j in range(len(toks))] if cond else None
    cr = [j for _ in grp for j in range(P)] if cond else None
    st.ar_step(grp, [D.PREFILL] * len(grp), [P] * len(grp), [0] * len(grp), [-1] * len(grp), toks, cs, cr)
TR = D.mem_alloc(8 * 8 * 4096)
MK = D.mem_alloc(8 * 8)
prev = [-1] * B
res = []
for k in range(10):
    D.mem_set(TR, 0, 8 * 8 * 4096)
    D.mem_set(MK, 0, 64)
    lib.omni_k_debug_traces(C.c_uint64(TR), C.c_uint64(MK))
    cs = [0] * B if cond else None
    cr = [0] * B if cond else None
    tok, _ = st.ar_step(ids, [D.DECODE] * B, [1] * B, [P + k] * B, [k] * B, prev, cs, cr)
    prev = [int(t) for t in tok]
    lib.omni_k_debug_traces(C.c_uint64(0), C.c_uint64(0))
    if k < 3:
        continue
    t = D.d2h(TR, (4096, 8), np.uint64).astype(np.int64)
    nb = 4 * B if False else None
    per_layer = []
    ncta = len(t[t[:, 0] > 0]) // m.n_layers
    for l in range(m.n_layers):
        tl = t[l * ncta:(l + 1) * ncta]
        per_layer.append((int(tl[:, 1].min()), int(tl[:, 5].max())))
    t = t[(m.n_layers - 1) * ncta:m.n_layers * ncta]
    mk = D.d2h(MK, (8,), np.uint64).astype(np.int64)
    base = mk[0]  # last QKV CTA exit
    r = {"ctas": len(t), "step_us": st.last_step_us()}
    for i, name in enumerate(["entry", "dep", "q_staged", "chunk0", "loop_done", "end"]):
        col = t[:, i]
        col = col[col > 0]
        if len(col):
            r[name] = [round((col.min() - base) / 1e3, 2), round((col.max() - base) / 1e3, 2)]
    r["o_wait_max"] = round((mk[1] - base) / 1e3, 2)
    r["o_exit_max"] = round((mk[2] - base) / 1e3, 2)
    b0 = per_layer[0][0]
    r["layers_dep_end_us"] = [(round((a - b0) / 1e3, 1), round((e - b0) / 1e3, 1)) for a, e in per_layer]
    res.append(r)
for r in res[-3:]:
    print(json.dumps(r))
st.close()
