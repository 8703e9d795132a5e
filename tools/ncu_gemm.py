"""Target for `ncu --set full`: the Thinker/Talker gate-up GEMM (N=16384,
K=2048, SwiGLU epilogue) at decode batch M (default 16), 8 launches over 8
distinct weight copies (512 MiB > L2)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_02204_b200 import dev as D  # noqa: E402

N, K = int(sys.argv[2]) if len(sys.argv) > 2 else 16384, int(sys.argv[3]) if len(sys.argv) > 3 else 2048
M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
EPI = int(sys.argv[4]) if len(sys.argv) > 4 else 4
lib = D.dev_lib()
Ws = [D.mem_alloc(N * K * 2) for _ in range(8)]
for i, w in enumerate(Ws):
    lib.omni_k_fill_weights(C.c_uint64(w), C.c_int64(N * K), C.c_uint64(11 + i), C.c_uint32(1), C.c_float(0.02))
X = D.mem_alloc(256 * K * 2)
lib.omni_k_fill_weights(C.c_uint64(X), C.c_int64(256 * K), C.c_uint64(3), C.c_uint32(2), C.c_float(1.0))
O = D.mem_alloc(256 * N * 4)
ldo = N // 2 if EPI == 4 else N
for it in range(2):
    for w in Ws:
        rc = lib.omni_k_gemm(C.c_uint64(w), N, K, C.c_uint64(X), M, EPI, C.c_uint64(O), ldo, C.c_uint64(0), 0, 0, 1, 8, None)
        assert rc == 0, rc
D.sync()
print("ok")
