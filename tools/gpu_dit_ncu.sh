#!/usr/bin/env bash
# GPU box: ncu --set full (+ source) of one fused DiT iteration at N tokens.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-dncu}; N=${2:-96}
OMNI_PREWARM=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:dit_fused -s 1 -c 1 \
  -o gpurun_out/${tag}_N${N} -f python tools/dit_one.py $N 2 > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${tag}_ncu.log
