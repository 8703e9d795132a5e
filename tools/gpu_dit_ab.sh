#!/usr/bin/env bash
# DiT tile-size A/B: parity tests, isolated probe and bench per OMNI_DIT_WIDE_FROM.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-dab}
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_dit_fused.py tests/test_gpu_models.py tests/test_gpu_longctx.py -k "dit or DiT or long_prompt" > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/${tag}_tests.log
for w in ${WIDE:-128 100000 16}; do
  OMNI_DIT_WIDE_FROM=$w timeout 600 python tools/step_probe.py --dit-only > gpurun_out/${tag}_probe_w$w.jsonl 2>&1
  echo "probe wide_from=$w"; cat gpurun_out/${tag}_probe_w$w.jsonl
done
for w in ${BWIDE:-128 16}; do
  OMNI_DIT_WIDE_FROM=$w timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${tag}_bench_w$w.json 2> gpurun_out/${tag}_bench_w$w.err
  echo "bench wide_from=$w rc=$?"; python -c "import json;d=json.load(open('gpurun_out/${tag}_bench_w$w.json'));print(d['value'],d['mean_jct_us'],d['stages']['code2wav'])"
done
