#!/usr/bin/env bash
# Isolated DiT probe A/B: current tree vs ${ALT}, alternating, same box.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-abp}; alt=${ALT:-_ab_v9}
for i in 1 2; do
  for t in cur alt; do
    d=.; [ $t = alt ] && d=$alt
    (cd $d && timeout 300 python tools/step_probe.py --dit-only) > gpurun_out/${tag}_${t}_$i.jsonl 2>&1
    echo "$t $i: $(python -c "import json;print([round(json.loads(l)['us_per_step']) for l in open('gpurun_out/${tag}_${t}_$i.jsonl')])")"
  done
done
