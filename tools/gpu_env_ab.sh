#!/usr/bin/env bash
# Pipeline bench + AR step probe A/B over an environment assignment list: ENVS="A=1 A=2 ..." ("-" = none).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-env}
for i in 1 2; do
  for e in ${ENVS:--}; do
    if [ "$e" = "-" ]; then pre=""; else pre="env $e"; fi
    $pre timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/${tag}_${e}_$i.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/${tag}_${e}_$i.json'));print('$e',$i,d['value'],d['mean_jct_us'],d['stages']['code2wav']['us_per_step'],d['stages']['thinker']['us_per_step'],d['stages']['talker']['us_per_step'])"
  done
done
if [ -n "${PROBE:-}" ]; then
  for e in ${ENVS:--}; do
    if [ "$e" = "-" ]; then pre=""; else pre="env $e"; fi
    echo "probe $e"; $pre timeout 300 python tools/step_probe.py --ar-only --quick 2>&1 | tail -5
  done
fi
