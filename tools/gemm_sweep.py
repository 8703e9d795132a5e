"""In-chain per-launch time of the decode GEMMs (CUDA graph of 64 PDL
launches cycling 8 weight copies > L2) over split-K caps and batch sizes.
python tools/gemm_sweep.py  -> one JSON line per point."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_02204_b200 import dev as D  # noqa: E402

lib = D.dev_lib()
SHAPES = {"qkv": (3072, 2048, 1), "wo": (2048, 2048, 1), "gateup": (16384, 2048, 4), "down": (2048, 8192, 1)}
for name, (N, K, epi) in SHAPES.items():
    Ws = [D.mem_alloc(N * K * 2) for _ in range(8)]
    for i, w in enumerate(Ws):
        lib.omni_k_fill_weights(C.c_uint64(w), C.c_int64(N * K), C.c_uint64(11 + i), C.c_uint32(1), C.c_float(0.02))
    X = D.mem_alloc(256 * K * 2)
    lib.omni_k_fill_weights(C.c_uint64(X), C.c_int64(256 * K), C.c_uint64(3), C.c_uint32(2), C.c_float(1.0))
    O = D.mem_alloc(256 * N * 4)
    arr = (C.c_uint64 * 8)(*Ws)
    for M in (1, 16, 64):
        for sp in (1, 2, 4, 8):
            ms = C.c_float()
            ldo = N // 2 if epi == 4 else N
            rc = lib.omni_k_gemm_time_multi(arr, 8, N, K, C.c_uint64(X), M, epi, C.c_uint64(O), ldo, sp, 64, C.byref(ms))
            us = ms.value * 1e3 if rc == 0 else float("nan")
            b = N * K * 2
            print(json.dumps({"gemm": name, "N": N, "K": K, "M": M, "max_splits": sp, "us": round(us, 2),
                              "GBps": round(b / us / 1e3, 1) if rc == 0 else None}), flush=True)
    for p in Ws + [X, O]:
        D.mem_free(p)
