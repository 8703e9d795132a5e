#!/usr/bin/env bash
# BN=64 push tiles: GEMM + edge + model tests, phase traces, in-chain sweep, step probe, c64 / c16 bench.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-b64}
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_gemm.py tests/test_gpu_edges.py tests/test_gpu_models.py > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/${tag}_tests.log
timeout 300 python tools/gemm_trace.py 1.965 16 48 64 > gpurun_out/${tag}_trace.jsonl 2>&1; echo "trace rc=$?"
timeout 300 python tools/gemm_sweep.py > gpurun_out/${tag}_sweep.jsonl 2>&1; echo "sweep rc=$?"
grep '"M": 64' gpurun_out/${tag}_sweep.jsonl | grep '"max_splits": 8'
timeout 600 python tools/step_probe.py --ar-only > gpurun_out/${tag}_probe.jsonl 2>&1; echo "probe rc=$?"; cat gpurun_out/${tag}_probe.jsonl
timeout 900 python bench.py --concurrency 64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_c64.json 2> gpurun_out/${tag}_c64.err
echo "c64 rc=$?"; python -c "import json;d=json.load(open('gpurun_out/${tag}_c64.json'));print(d['value'],d['mean_jct_us'],d['stages'])"
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${tag}_c16.json 2> gpurun_out/${tag}_c16.err
echo "c16 rc=$?"; python -c "import json;d=json.load(open('gpurun_out/${tag}_c16.json'));print(d['value'],d['mean_jct_us'],d['stages'])"
