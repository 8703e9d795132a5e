#!/bin/bash
# bench A/B with repeats: BENCH_AB="A|B", REPS (default 3)
mkdir -p gpurun_out
: > gpurun_out/bench_rep.log
IFS='|' read -ra CFGS <<< "${BENCH_AB:-OMNI_X=0}"
for r in $(seq 1 ${REPS:-3}); do
for cfg in "${CFGS[@]}"; do
  echo "== $cfg" >> gpurun_out/bench_rep.log
  env $cfg timeout 600 python bench.py --no-cpu-baseline --warmup 2 --steps ${STEPS:-4} >> gpurun_out/bench_rep.log 2>&1
done
done
python - <<'PY'
import json, collections, statistics
res = collections.defaultdict(list); cur = None
for line in open("gpurun_out/bench_rep.log"):
    if line.startswith("=="): cur = line.strip()[3:]; continue
    try:
        d = json.loads(line); res[cur].append((d["value"], d["mean_jct_us"], d["p99_jct_us"]))
    except Exception: pass
for k, v in res.items():
    print(k, "value", [x[0] for x in v], "median", statistics.median(x[0] for x in v), "jct", statistics.median(x[1] for x in v))
PY
