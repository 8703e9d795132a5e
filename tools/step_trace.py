"""Timeline of one AR decode step on the per-kernel PDL path: every GEMM
launch's CTA entry / PDL-wait release / mainloop done / exit (OMNI_STEP_TRACE
stamps) and every attention launch's dependency release / end
(omni_k_debug_traces), in us from the first QKV CTA of layer 0.
python tools/step_trace.py [thinker|talker] [rows] [ghz]"""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

os.environ["OMNI_STEP_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_02204_b200 import dev as D  # noqa: E402

kind = D.TALKER if (len(sys.argv) > 1 and sys.argv[1] == "talker") else D.THINKER
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
GHZ = float(sys.argv[3]) if len(sys.argv) > 3 else 1.965
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
AT = D.mem_alloc(8 * 8 * 8192)
prev = [-1] * B
PF = int(os.environ.get("TRACE_PREFILL", "0"))  # add a PF-token prefill chunk to every traced step
for k in range(8):
    D.mem_set(AT, 0, 8 * 8 * 8192)
    lib.omni_k_debug_traces(C.c_uint64(AT), C.c_uint64(0))
    cs = [0] * B if cond else None
    cr = [0] * B if cond else None
    if PF and not cond:
        new = 5000 + k
        tok, _ = st.ar_step(ids + [new], [D.DECODE] * B + [D.PREFILL], [1] * B + [PF], [P + k] * B + [0],
                            [k] * B + [-1], prev + [(5 * j + k) % 250 + 1 for j in range(PF)])
        st.release(new)
        tok = tok[:B]
    else:
        tok, _ = st.ar_step(ids, [D.DECODE] * B, [1] * B, [P + k] * B, [k] * B, prev, cs, cr)
    prev = [int(t) for t in tok]
    lib.omni_k_debug_traces(C.c_uint64(0), C.c_uint64(0))
step_us = st.last_step_us()
ptr, rows, cols = st.tensor("buf.step_trace")
tr = D.d2h(ptr, (rows // 512, 512, 8), np.uint64).astype(np.int64)
at = D.d2h(AT, (8192, 8), np.uint64).astype(np.int64)
L = m.n_layers
names = ["qkv", "o", "gateup", "down"]
t0 = None
events = []
for slot in range(tr.shape[0]):
    c = tr[slot]
    c = c[c[:, 0] > 0]
    if len(c) == 0:
        continue
    ent = c[:, 0]
    base = ent  # per-CTA clock offsets are relative to the CTA's own entry
    wait = ent + c[:, 2] / GHZ
    done = ent + c[:, 4] / GHZ
    ext = c[:, 7]
    nm = names[slot % 4] + str(slot // 4) if slot < 4 * L else "lm"
    if t0 is None:
        t0 = ent.min()
    events.append((nm, ent.min(), np.median(wait), wait.max(), np.median(done), ext.max(), len(c)))
    if os.environ.get("TRACE_SKEW"):
        pc = lambda v: np.round((np.percentile(v, [0, 10, 50, 90, 100]) - t0) / 1e3, 2).tolist()
        print(nm, "entry", pc(ent), "done", pc(done), "exit", pc(ext))
    if os.environ.get("TRACE_PHASES") and nm.startswith("qkv"):
        ph = {k: np.round(np.percentile((ent + c[:, i] / GHZ - t0) / 1e3, [50, 100]), 2).tolist()
              for k, i in (("s1", 1), ("s3", 3), ("s5", 5), ("end6", 6))}
        print(nm, ph)
ncta = (at[:, 0] > 0).sum() // L
for l in range(L if ncta else 0):
    a = at[l * ncta:(l + 1) * ncta]
    a = a[a[:, 0] > 0]
    events.append(("attn" + str(l), a[:, 0].min(), np.median(a[:, 1]), a[:, 1].max(), np.median(a[:, 4]), a[:, 5].max(), len(a)))
events.sort(key=lambda e: e[5])
print(f"# {'thinker' if kind == D.THINKER else 'talker'} rows={B} step_us={step_us:.1f} (us from first QKV CTA entry)")
print(f"{'kernel':10s} {'ctas':>5s} {'entry':>8s} {'wait_med':>8s} {'wait_max':>8s} {'done_med':>8s} {'exit':>8s} {'post_wait':>9s}")
prev_exit = None
for nm, e, wm, wx, dm, x, n in events:
    f = lambda v: (v - t0) / 1e3
    print(f"{nm:10s} {n:5d} {f(e):8.2f} {f(wm):8.2f} {f(wx):8.2f} {f(dm):8.2f} {f(x):8.2f} {f(x) - f(wm):9.2f}")
st.close()
