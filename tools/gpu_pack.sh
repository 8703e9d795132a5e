#!/usr/bin/env bash
# Connector pack kernel at production and synthetic large sizes: host-bracket probe,
# ncu launch metrics of every pack launch, ncu --set full of the 16.8 MB pack.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-pk}
timeout 300 python tools/pack_probe.py 50 > gpurun_out/${tag}_probe.jsonl 2>&1; cat gpurun_out/${tag}_probe.jsonl
OMNI_PREWARM=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
  --clock-control none -k regex:pack_hidden --csv --log-file gpurun_out/${tag}_launches.csv python tools/pack_probe.py 20 > /dev/null 2>&1
echo "ncu list rc=$?"
OMNI_PREWARM=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:pack_hidden -s 60 -c 1 \
  -o gpurun_out/${tag}_pack_big -f python tools/pack_probe.py 20 > /dev/null 2>&1
echo "ncu full rc=$?"
