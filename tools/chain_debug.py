"""Compare every exposed activation buffer after one step, step chain vs per-kernel."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_02204_b200 import dev as D  # noqa: E402

SMALL = dict(d_model=512, n_layers=1, n_heads=4, n_kv_heads=2, d_ff=1024)
L = int(sys.argv[1]) if len(sys.argv) > 1 else 1
SMALL["n_layers"] = L
TALKER = len(sys.argv) > 2 and sys.argv[2] == "talker"
if TALKER:
    SMALL["cond_dim"] = 512
    bufs_extra = {"buf.hproj": "f"}
m = D.model_default(D.TALKER if TALKER else D.THINKER, **SMALL)
rng = np.random.default_rng(3)
cond = D.mem_alloc(2 * 512 * 16)
D.h2d(cond, ((rng.standard_normal(512 * 16).astype(np.float32) * 0.5).view(np.uint32) >> 16).astype(np.uint16))
p = [5, 77, 140, 9, 200, 31, 18, 64, 99]
bufs = {"buf.x": np.float32, "buf.xn": np.uint16, "buf.q": np.uint16, "buf.attn": np.uint16,
        "buf.act": np.uint16, "buf.hbuf": np.uint16, "buf.ss": np.float32, "buf.logits": np.float32}
res = []
for chain in (False, True):
    st = D.Stage(m, D.StageLimits(256, 16, 256, 0, 16), seed=17)
    st.set_chain(chain)
    out = {}
    extra = dict(cond_src=[cond + 1024 * j for j in range(len(p))], cond_row=list(range(len(p)))) if TALKER else {}
    st.ar_step([1], [D.PREFILL], [len(p)], [0], [-1], p, **extra)
    for nm, dt in bufs.items():
        ptr, rows, cols = st.tensor(nm)
        out["prefill " + nm] = D.d2h(ptr, (len(p), cols), dt)
    extra = dict(cond_src=[0], cond_row=[0]) if TALKER else {}
    t, mg = st.ar_step([1], [D.DECODE], [1], [len(p)], [0], [-1], **extra)
    out["tok"] = t
    for nm, dt in bufs.items():
        ptr, rows, cols = st.tensor(nm)
        out["decode " + nm] = D.d2h(ptr, (1, cols), dt)
    res.append(out)
    st.close()
for k in res[0]:
    a, b = res[0][k], res[1][k]
    same = np.array_equal(a, b)
    print(f"{k:24s} {'OK' if same else 'DIFF'}", "" if same else f"nonequal={np.sum(a != b)}/{a.size} a[:6]={a.ravel()[:6]} b[:6]={b.ravel()[:6]}")
