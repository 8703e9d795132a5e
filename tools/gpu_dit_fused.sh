#!/usr/bin/env bash
# GPU box: fused DiT iteration -- parity tests, step probe, per-item trace.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-df}
timeout 300 python -m pytest tests/test_gpu_models.py -k dit -x -q -rf -s > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -8 gpurun_out/${tag}_tests.log
timeout 300 python tools/step_probe.py --dit-only > gpurun_out/${tag}_probe_fused.jsonl 2>&1; echo "probe rc=$?"
cat gpurun_out/${tag}_probe_fused.jsonl | tail -8
timeout 300 python tools/dit_trace.py 16 96 512 > gpurun_out/${tag}_trace.jsonl 2>&1; echo "trace rc=$?"
tail -c 3000 gpurun_out/${tag}_trace.jsonl
