#!/usr/bin/env bash
# DiT fused-kernel iteration: parity tests, isolated probe, ncu at 96 / 512 tokens, default bench.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-dv}
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_dit_fused.py tests/test_gpu_models.py -k "dit or DiT" > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/${tag}_tests.log
timeout 600 python tools/step_probe.py --dit-only > gpurun_out/${tag}_probe.jsonl 2>&1; echo "probe rc=$?"; cat gpurun_out/${tag}_probe.jsonl
if [ -z "${NO_NCU:-}" ]; then
for N in 96 512; do
  OMNI_PREWARM=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:dit_fused -s 1 -c 1 \
    -o gpurun_out/${tag}_dit_N${N} -f python tools/dit_one.py $N 2 > gpurun_out/${tag}_dit_ncu_${N}.log 2>&1
  echo "ncu dit $N rc=$?"
done
fi
if [ -z "${NO_BENCH:-}" ]; then
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/${tag}_bench.json'));print(d['value'],d['mean_jct_us'],d['stages'])"
fi
