#!/usr/bin/env bash
# GPU box: full GPU suite, default bench, folded 2/8-GPU placement runs (logs under gpurun_out/).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-r2a}
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/${tag}_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_tests.log
tail -15 gpurun_out/${tag}_tests.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"
tail -c 2500 gpurun_out/${tag}_bench.json; tail -5 gpurun_out/${tag}_bench.err
timeout 600 python bench.py --gpus 4 --fold-devices --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${tag}_fold4.json 2> gpurun_out/${tag}_fold4.err; echo "fold4 rc=$?"
tail -c 800 gpurun_out/${tag}_fold4.json; tail -5 gpurun_out/${tag}_fold4.err
