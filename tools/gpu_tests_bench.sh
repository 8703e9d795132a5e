#!/usr/bin/env bash
# GPU box: full GPU test suite, then one default bench run (logs under gpurun_out/).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-r}
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/${tag}_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_tests.log
tail -15 gpurun_out/${tag}_tests.log
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"
tail -c 1500 gpurun_out/${tag}_bench.json
