"""ncu target: each DiT GEMM shape (qkv, o, up, down) at M token rows, the
DiT (fill_sms, no split-K) launch policy, 2 launches each over 2 weight copies.
  python tools/dit_gemm_one.py [M] [shape,...]"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_02204_b200 import dev as D  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
names = sys.argv[2].split(",") if len(sys.argv) > 2 else ["qkv", "o", "up", "down"]
SHAPES = {"qkv": (3072, 1024, 0), "o": (1024, 1024, 0), "up": (4096, 1024, 5), "down": (1024, 4096, 0)}
lib = D.dev_lib()
for name in names:
    N, K, epi = SHAPES[name]
    Ws = [D.mem_alloc(N * K * 2) for _ in range(2)]
    for i, w in enumerate(Ws):
        lib.omni_k_fill_weights(C.c_uint64(w), C.c_int64(N * K), C.c_uint64(11 + i), C.c_uint32(1), C.c_float(0.02))
    X = D.mem_alloc(M * K * 2)
    lib.omni_k_fill_weights(C.c_uint64(X), C.c_int64(M * K), C.c_uint64(3), C.c_uint32(2), C.c_float(1.0))
    O = D.mem_alloc(M * N * 2)
    arr = (C.c_uint64 * 2)(*Ws)
    ms = C.c_float()
    rc = lib.omni_k_gemm_time_multi(arr, 2, N, K, C.c_uint64(X), M, epi, C.c_uint64(O), N, -1, 2, C.byref(ms))
    print(name, M, rc, round(ms.value * 1e3, 2), "us", flush=True)
    for p in Ws + [X, O]:
        D.mem_free(p)
