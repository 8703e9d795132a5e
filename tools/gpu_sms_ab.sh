#!/usr/bin/env bash
# Pipeline bench over the DiT SM share (OMNI_DIT_SMS), alternating, 2 reps.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-sms}
for i in 1 2; do
  for n in ${SMS:-48 64 80 96}; do
    OMNI_DIT_SMS=$n timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${tag}_${n}_$i.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/${tag}_${n}_$i.json'));print($n,$i,d['value'],d['mean_jct_us'],d['stages']['code2wav']['us_per_step'],d['stages']['thinker']['us_per_step'],d['stages']['talker']['us_per_step'])"
  done
done
