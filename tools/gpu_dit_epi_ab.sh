#!/usr/bin/env bash
# A/B of the fused DiT's epilogue warp count (OMNI_DIT_EPI_WARPS 8 vs 16): parity + isolated probe + trace.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-ea}
for w in 8 16; do
  touch paper_2602_02204_b200/csrc/dev/dit_fused.cu
  OMNI_NVCC_DEFS="-DOMNI_DIT_EPI_WARPS=$w" python -c "import paper_2602_02204_b200.build as b; b.build()" > gpurun_out/${tag}_build$w.log 2>&1 || { echo "build $w failed"; tail gpurun_out/${tag}_build$w.log; continue; }
  echo "=== epi warps $w"
  timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_dit_fused.py > gpurun_out/${tag}_tests$w.log 2>&1
  echo "tests rc=$?"; tail -2 gpurun_out/${tag}_tests$w.log
  timeout 600 python tools/step_probe.py --dit-only > gpurun_out/${tag}_probe$w.jsonl 2>&1; cat gpurun_out/${tag}_probe$w.jsonl
  for s in "" "--sms=48"; do
    timeout 600 python tools/dit_trace.py $s 16 96 512 > gpurun_out/${tag}_trace$w$s.jsonl 2>&1
    python - <<PY
import json
for l in open("gpurun_out/${tag}_trace$w$s.jsonl"):
    try: d = json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    pk = {k: (v["n"], v["main"], v["epi"]) for k, v in d["per_kind_us"].items()}
    print(d["tokens"], d["tile_rows"], d["sms"], d["us_per_step"], d["cta_share"], pk)
PY
  done
done
