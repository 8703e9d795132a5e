"""In-chain decode GEMM time with the weights L2-resident (1 copy, repeated)
vs streamed from HBM (8 copies > L2): how much an L2 prefetch could buy."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_02204_b200 import dev as D  # noqa: E402

lib = D.dev_lib()
for name, (N, K, epi) in {"gateup": (16384, 2048, 4), "down": (2048, 8192, 1), "qkv": (3072, 2048, 1)}.items():
    Ws = [D.mem_alloc(N * K * 2) for _ in range(8)]
    for i, w in enumerate(Ws):
        lib.omni_k_fill_weights(C.c_uint64(w), C.c_int64(N * K), C.c_uint64(11 + i), C.c_uint32(1), C.c_float(0.02))
    X = D.mem_alloc(256 * K * 2)
    lib.omni_k_fill_weights(C.c_uint64(X), C.c_int64(256 * K), C.c_uint64(3), C.c_uint32(2), C.c_float(1.0))
    O = D.mem_alloc(256 * N * 4)
    for nw in (8, 1):
        arr = (C.c_uint64 * nw)(*Ws[:nw])
        for M in (1, 16):
            ms = C.c_float()
            ldo = N // 2 if epi == 4 else N
            rc = lib.omni_k_gemm_time_multi(arr, nw, N, K, C.c_uint64(X), M, epi, C.c_uint64(O), ldo, 8, 64, C.byref(ms))
            us = ms.value * 1e3
            print(json.dumps({"gemm": name, "copies": nw, "M": M, "us": round(us, 2),
                              "GBps": round(N * K * 2 / us / 1e3, 1), "rc": rc}), flush=True)
    for p in Ws + [X, O]:
        D.mem_free(p)
