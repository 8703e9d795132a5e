"""DiT GEMM shapes (compute-bound): in-chain time and TF/s vs token rows and
forced token tile (OMNI_DIT_BN env read by the library at first use)."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_02204_b200 import dev as D  # noqa: E402

lib = D.dev_lib()
SHAPES = {"qkv": (3072, 1024), "o": (1024, 1024), "up": (4096, 1024), "down": (1024, 4096)}
for name, (N, K) in SHAPES.items():
    Ws = [D.mem_alloc(N * K * 2) for _ in range(2)]
    for i, w in enumerate(Ws):
        lib.omni_k_fill_weights(C.c_uint64(w), C.c_int64(N * K), C.c_uint64(11 + i), C.c_uint32(1), C.c_float(0.02))
    X = D.mem_alloc(8192 * K * 2)
    lib.omni_k_fill_weights(C.c_uint64(X), C.c_int64(8192 * K), C.c_uint64(3), C.c_uint32(2), C.c_float(1.0))
    O = D.mem_alloc(8192 * N * 2)
    arr = (C.c_uint64 * 2)(*Ws)
    for M in (128, 640, 1024, 1360, 2048, 4096, 8192):
        ms = C.c_float()
        rc = lib.omni_k_gemm_time_multi(arr, 2, N, K, C.c_uint64(X), M, 0, C.c_uint64(O), N, -1, 32, C.byref(ms))
        us = ms.value * 1e3
        print(json.dumps({"gemm": name, "M": M, "us": round(us, 2), "TFs": round(2 * M * N * K / us / 1e6, 1), "rc": rc}),
              flush=True)
    for p in Ws + [X, O]:
        D.mem_free(p)
