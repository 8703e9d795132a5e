"""One fused DiT iteration at N tokens (ncu target): python tools/dit_one.py N [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_02204_b200 import dev as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 96
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
m = D.model_default(D.DIT)
st = D.Stage(m, D.StageLimits(256, 64, 512, 0, 512), seed=9)
toks = [(5 * i) % 64 for i in range(n)]
for _ in range(reps):
    st.dit_step([1], [0], [n], toks)
print("us", st.last_step_us())
st.close()
