#!/usr/bin/env bash
# Per-item traces of the fused DiT (all SMs and the 48-SM pipeline share) + probe.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-dtr}
for w in all; do
  timeout 600 python tools/dit_trace.py 16 96 512 > gpurun_out/${tag}_w${w}_all.jsonl 2>&1; echo "trace rc=$?"
  timeout 600 python tools/dit_trace.py --sms=48 16 96 512 > gpurun_out/${tag}_w${w}_48.jsonl 2>&1; echo "trace48 rc=$?"
  python - <<PY
import json
for f in ["gpurun_out/${tag}_w${w}_all.jsonl", "gpurun_out/${tag}_w${w}_48.jsonl"]:
    for l in open(f):
        try: d = json.loads(l)
        except Exception: print(l.strip()[:300]); continue
        print(f[-12:], d["tokens"], d["tile_rows"], d["sms"], d["us_per_step"], d["cta_share"], d["tile0_phase_us"])
PY
done
timeout 600 python tools/step_probe.py --dit-only > gpurun_out/${tag}_probe.jsonl 2>&1; cat gpurun_out/${tag}_probe.jsonl
