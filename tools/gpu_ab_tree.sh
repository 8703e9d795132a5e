#!/usr/bin/env bash
# Pipeline A/B of the current tree against a second build at ${ALT:-_ab_v6} (a git worktree), alternating.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-abt}; alt=${ALT:-_ab_v6}; reps=${REPS:-3}
for i in $(seq 1 $reps); do
  for t in cur alt; do
    d=.; [ $t = alt ] && d=$alt
    (cd $d && timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS:-}) > gpurun_out/${tag}_${t}_$i.json 2> gpurun_out/${tag}_${t}_$i.err
    python -c "import json;d=json.load(open('gpurun_out/${tag}_${t}_$i.json'));print('$t',$i,d['value'],d['mean_jct_us'],d['stages']['code2wav']['us_per_step'],d['stages']['thinker']['us_per_step'],d['stages']['talker']['us_per_step'])"
  done
done
