#!/usr/bin/env bash
# DiT quick loop: parity tests, isolated probe, per-item trace at 16/96/512 tokens (148 and 64 CTAs).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-dq}
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_dit_fused.py tests/test_gpu_models.py -k "dit or DiT" > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/${tag}_tests.log
timeout 600 python tools/step_probe.py --dit-only > gpurun_out/${tag}_probe.jsonl 2>&1; cat gpurun_out/${tag}_probe.jsonl
for s in "" "--sms=64"; do
  timeout 600 python tools/dit_trace.py $s 16 96 512 > gpurun_out/${tag}_trace$s.jsonl 2>&1
  python - <<PY
import json
for l in open("gpurun_out/${tag}_trace$s.jsonl"):
    try: d = json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    pk = {k: (v["n"], v["main"], v["epi"]) for k, v in d["per_kind_us"].items()}
    print(d["tokens"], d["tile_rows"], d["sms"], d["us_per_step"], d["cta_share"], pk)
PY
done
