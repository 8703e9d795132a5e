for v in 8 16; do echo "== DOWN_SPLIT $v"; OMNI_DOWN_SPLIT=$v timeout 200 python tools/step_probe.py --quick --ar-only; done
python - <<'PY'
import ctypes as C, json, sys
sys.path.insert(0, ".")
from paper_2602_02204_b200 import dev as D
lib = D.dev_lib()
for name, (N, K, epi) in {"down": (2048, 8192, 1), "qkv": (3072, 2048, 1), "wo": (2048, 2048, 1)}.items():
    Ws = [D.mem_alloc(N * K * 2) for _ in range(8)]
    for i, w in enumerate(Ws):
        lib.omni_k_fill_weights(C.c_uint64(w), C.c_int64(N * K), C.c_uint64(11 + i), C.c_uint32(1), C.c_float(0.02))
    X = D.mem_alloc(256 * K * 2)
    lib.omni_k_fill_weights(C.c_uint64(X), C.c_int64(256 * K), C.c_uint64(3), C.c_uint32(2), C.c_float(1.0))
    O = D.mem_alloc(256 * N * 4)
    arr = (C.c_uint64 * 8)(*Ws)
    for M in (1, 16):
        for sp in (8, 16):
            ms = C.c_float()
            rc = lib.omni_k_gemm_time_multi(arr, 8, N, K, C.c_uint64(X), M, epi, C.c_uint64(O), N, sp, 64, C.byref(ms))
            print(json.dumps({"gemm": name, "M": M, "max_splits": sp, "us": round(ms.value * 1e3, 2), "rc": rc}))
PY
