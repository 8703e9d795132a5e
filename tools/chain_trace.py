"""Per-op timeline of one Thinker decode step run as a step chain."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_02204_b200 import dev as D  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
m = D.model_default(D.THINKER)
st = D.Stage(m, D.StageLimits(256, 64, 512, 0, 64), seed=7)
lib = D.dev_lib()
T = D.mem_alloc(3 * 8 * 8192)
ids = list(range(1, B + 1))
for s_ in ids:
    st.ar_step([s_], [D.PREFILL], [16], [0], [-1], [(7 * j) % 250 + 1 for j in range(16)])
for k in range(3):  # warm
    st.ar_step(ids, [D.DECODE] * B, [1] * B, [16 + k] * B, [k] * B, [-1] * B)
ni, no = C.c_int32(), C.c_int32()
first = (C.c_int32 * 48)()
lib.omni_stage_chain_trace(st.h, C.c_uint64(T), C.byref(ni), C.byref(no), first)
D.mem_set(T, 0, 3 * 8 * 8192)
st.ar_step(ids, [D.DECODE] * B, [1] * B, [19] * B, [3] * B, [-1] * B)
print("step us", st.last_step_us())
lib.omni_stage_chain_trace(st.h, C.c_uint64(0), C.byref(ni), C.byref(no), first)
n = ni.value
t = D.d2h(T, (n, 3), np.uint64).astype(np.int64)
t0 = t[:, 0][t[:, 0] > 0].min()
fs = [first[i] for i in range(no.value)] + [n]
names = ["embed"] + [f"L{l}.{x}" for l in range(8) for x in ("qkv", "attn", "o", "gu", "down")] + ["final", "lm", "argmax"]
prev_end = 0
for i in range(no.value):
    seg = t[fs[i]:fs[i + 1]] - t0
    print(f"{names[i] if i < len(names) else i:10s} items={fs[i+1]-fs[i]:4d} start[min,max]=({seg[:,0].min()/1e3:7.2f},{seg[:,0].max()/1e3:7.2f}) "
          f"dep_met_max={seg[:,1].max()/1e3:7.2f} end[min,max]=({seg[:,2].min()/1e3:7.2f},{seg[:,2].max()/1e3:7.2f}) "
          f"busy_after_dep={(seg[:,2].max()-seg[:,1].max())/1e3:6.2f}")
