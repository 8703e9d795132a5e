"""The gate-up GEMM as the AR stages run it (pre-tiled weights, PDL graph of
launches over 8 weight copies > L2) for ncu: python tools/ncu_gemm_tiled.py [M]
(under ncu -k regex:gemm_tc_kernel -s <skip> -c 1 --set full)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_02204_b200 import dev as D  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
N, K = 16384, 2048
lib = D.dev_lib()
copies = [D.mem_alloc(N * K * 2) for _ in range(8)]
for i, w in enumerate(copies):
    lib.omni_k_fill_weights(C.c_uint64(w), C.c_int64(N * K), C.c_uint64(11 + i), C.c_uint32(1), C.c_float(0.02))
X = D.mem_alloc(256 * K * 2)
O = D.mem_alloc(256 * N * 4)
lib.omni_k_fill_weights(C.c_uint64(X), C.c_int64(256 * K), C.c_uint64(3), C.c_uint32(2), C.c_float(1.0))
arr = (C.c_uint64 * 8)(*copies)
ms = C.c_float()
rc = lib.omni_k_gemm_time_multi(arr, 8, N, K, C.c_uint64(X), M, 4, C.c_uint64(O), N // 2, 8, 16, C.byref(ms))
print("rc", rc, "us per launch", round(ms.value * 1e3, 2))
