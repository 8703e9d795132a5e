#!/bin/bash
# bench at different graph-capture thresholds (OMNI_GRAPH_HITS), warmup 3
for h in ${HITS:-3 12 3 12 3 12}; do
  OMNI_GRAPH_HITS=$h timeout 900 python bench.py --no-cpu-baseline --warmup 3 --steps 4 > gpurun_out/w.log 2>&1
  python - "$h" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/w.log").read().strip().splitlines()[-1])
print("hits", sys.argv[1], d["value"], d["mean_jct_us"], d["step_graphs"], {k: (v["us_per_step"], v["host_us_per_step"], v["gap_us"]) for k, v in d["stages"].items()})
PY
done
