#!/usr/bin/env bash
# Pre-tiled gate-up / down weights (OMNI_WBLOCK=1) vs 2-D TMA: parity tests, step probe, bench c16 x3 / c64 x2 alternating.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-wb}
OMNI_WBLOCK=1 timeout 600 python -m pytest -q -x -m gpu tests/test_gpu_models.py tests/test_gpu_edges.py tests/test_gpu_longctx.py tests/test_gpu_pipeline_parity.py > gpurun_out/${tag}_tests.log 2>&1
rc=$?; echo "tests rc=$rc"; tail -2 gpurun_out/${tag}_tests.log
[ $rc -eq 0 ] || exit 1
for v in 0 1; do
  echo "=== OMNI_WBLOCK=$v"
  OMNI_WBLOCK=$v timeout 300 python tools/step_probe.py --ar-only 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['stage'], d['decode_rows'], d['us_per_step'])" | tr '\n' ' '; echo
done
for i in 1 2 3; do
  for v in 0 1; do
    OMNI_WBLOCK=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${tag}_c16_${v}_$i.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/${tag}_c16_${v}_$i.json'));print('c16 WBLOCK=$v',d['value'],d['mean_jct_us'],d['roofline']['frac'],d['stages']['thinker']['us_per_step'],d['stages']['talker']['us_per_step'])"
  done
done
for i in 1 2; do
  for v in 0 1; do
    OMNI_WBLOCK=$v timeout 600 python bench.py --no-cpu-baseline --concurrency 64 --steps 3 > gpurun_out/${tag}_c64_${v}_$i.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/${tag}_c64_${v}_$i.json'));print('c64 WBLOCK=$v',d['value'],d['mean_jct_us'])"
  done
done
