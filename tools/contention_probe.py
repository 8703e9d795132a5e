"""Per-stage device step times of the bench workload with and without the DiT stage."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_02204_b200.serve import Pipeline  # noqa: E402

for cfg in ("omni3.json", "thinker_talker.json", "thinker_only.json"):
    p = Pipeline((Path(__file__).resolve().parent.parent / "configs" / cfg).read_text(), weight_seed=1234)
    p.bench(n=100, seed=7, concurrency=16, stream=True, clock="device")
    r = p.bench(n=100, seed=7, concurrency=16, stream=True, clock="device")
    out = {"cfg": cfg, "req_s": round(r["requests_per_s"], 1), "mean_jct_ms": round(r["mean_jct_us"] / 1e3, 1)}
    for k in ("thinker", "talker", "dit"):
        if r[f"steps_{k}"]:
            out[k] = round(1e3 * r[f"dev_ms_{k}"] / r[f"steps_{k}"], 1)
            out[k + "_steps"] = r[f"steps_{k}"]
    print(json.dumps(out), flush=True)
    p.close()
