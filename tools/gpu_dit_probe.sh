#!/usr/bin/env bash
# DiT evidence: step probe, GEMM sweep, ncu --set full of each DiT GEMM at M rows.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-dit}
M=${2:-1024}
timeout 300 python tools/step_probe.py --dit-only > gpurun_out/${tag}_step.jsonl 2>&1
timeout 300 python tools/dit_gemm_sweep.py > gpurun_out/${tag}_sweep.jsonl 2>&1
timeout 600 ncu --set full --clock-control none -k regex:gemm_tc -s 8 -c 8 -o gpurun_out/${tag}_ncu_M${M} -f \
  python tools/dit_gemm_one.py $M > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"
cat gpurun_out/${tag}_step.jsonl; cat gpurun_out/${tag}_sweep.jsonl | tail -30
