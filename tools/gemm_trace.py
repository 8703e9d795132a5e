"""Phase trace of the decode GEMMs in a PDL chain (omni_k_gemm_trace).
python tools/gemm_trace.py [GHZ] [M ...]
Per launch: CTA entry/exit skew (globaltimer, ns) and per-CTA phase offsets
(clock64 cycles -> us at the sampled SM clock): setup, producer past
griddepcontrol.wait, last TMA issued, mainloop done, TMEM drained (+cluster
reduce start), end."""
import ctypes as C
import json
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_02204_b200 import dev as D  # noqa: E402

lib = D.dev_lib()
GHZ = float(sys.argv[1]) if len(sys.argv) > 1 else 1.9
SHAPES = {"qkv": (3072, 2048, 1), "wo": (2048, 2048, 1), "gateup": (16384, 2048, 4), "down": (2048, 8192, 1)}
for name, (N, K, epi) in SHAPES.items():
    Ws = [D.mem_alloc(N * K * 2) for _ in range(8)]
    for i, w in enumerate(Ws):
        lib.omni_k_fill_weights(C.c_uint64(w), C.c_int64(N * K), C.c_uint64(11 + i), C.c_uint32(1), C.c_float(0.02))
    X = D.mem_alloc(256 * K * 2)
    lib.omni_k_fill_weights(C.c_uint64(X), C.c_int64(256 * K), C.c_uint64(3), C.c_uint32(2), C.c_float(1.0))
    O = D.mem_alloc(256 * N * 4)
    arr = (C.c_uint64 * 8)(*Ws)
    for M in [int(x) for x in sys.argv[2:]] or (4, 16):
        T = D.mem_alloc(8 * 8 * 4096)
        D.mem_set(T, 0, 8 * 8 * 4096)
        g = C.c_int32()
        ldo = N // 2 if epi == 4 else N
        rc = lib.omni_k_gemm_trace(arr, 8, N, K, C.c_uint64(X), M, epi, C.c_uint64(O), ldo, 8, C.c_uint64(T), C.byref(g))
        assert rc == 0, rc
        t = D.d2h(T, (g.value, 8), np.uint64).astype(np.int64)
        D.mem_free(T)
        ent, ext = t[:, 0], t[:, 7]
        ph = {k: t[:, i] / GHZ / 1e3 for i, k in
              [(1, "setup"), (2, "prod_wait"), (3, "last_load"), (4, "done"), (5, "drained"), (6, "end")]}
        out = {"gemm": name, "M": M, "ctas": g.value,
               "span_us": round((ext.max() - ent.min()) / 1e3, 2),
               "entry_skew_us": round((ent.max() - ent.min()) / 1e3, 2),
               "exit_skew_us": round((ext.max() - ext.min()) / 1e3, 2)}
        for k, v in ph.items():
            out[k] = [round(float(np.median(v)), 2), round(float(v.max()), 2)]
        print(json.dumps(out), flush=True)
    for p in Ws + [X, O]:
        D.mem_free(p)
