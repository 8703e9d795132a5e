#!/usr/bin/env bash
# GPU box: build check + the full GPU test suite (log under gpurun_out/).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-tests}
shift || true
timeout 1500 python -m pytest tests -m gpu -q -rA "$@" > gpurun_out/${tag}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}.log
tail -40 gpurun_out/${tag}.log
