#!/usr/bin/env bash
# CTA-pair fused DiT: parity (pair vs single-CTA, pair vs oracle), then isolated probe + trace, pair vs single.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-dp}
timeout 300 python -m pytest -q -x -m gpu tests/test_gpu_dit_fused.py > gpurun_out/${tag}_tests.log 2>&1
rc=$?; echo "tests rc=$rc"; tail -15 gpurun_out/${tag}_tests.log
[ $rc -eq 0 ] || exit 1
for pr in 0 1; do
  echo "=== OMNI_DIT_PAIR=$pr"
  OMNI_DIT_PAIR=$pr timeout 600 python tools/step_probe.py --dit-only > gpurun_out/${tag}_probe$pr.jsonl 2>&1; cat gpurun_out/${tag}_probe$pr.jsonl
  for s in "" "--sms=48"; do
    OMNI_DIT_PAIR=$pr timeout 600 python tools/dit_trace.py $s 16 96 512 > gpurun_out/${tag}_trace$pr$s.jsonl 2>&1
    python - <<PY
import json
for l in open("gpurun_out/${tag}_trace$pr$s.jsonl"):
    try: d = json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    pk = {k: (v["n"], v["main"], v["epi"]) for k, v in d["per_kind_us"].items()}
    print(d["tokens"], d["tile_rows"], d["sms"], d["us_per_step"], d["cta_share"], pk)
PY
  done
done
