#!/bin/bash
# bench repeats at two warm-up depths (graph captures inside the timed region)
for w in 2 10 2 10; do
  timeout 900 python bench.py --no-cpu-baseline --warmup $w --steps 4 > gpurun_out/w.log 2>&1
  python - "$w" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/w.log").read().strip().splitlines()[-1])
print("warmup", sys.argv[1], d["value"], d["mean_jct_us"], d["step_graphs"], {k: (v["us_per_step"], v["host_us_per_step"], v["gap_us"]) for k, v in d["stages"].items()})
PY
done
