#!/bin/bash
# bench A/B over env knobs: BENCH_AB="A_ENV|B_ENV|..." (default: priorities on/off)
mkdir -p gpurun_out
: > gpurun_out/bench_ab.log
IFS='|' read -ra CFGS <<< "${BENCH_AB:-OMNI_PRIO=1|OMNI_PRIO=0}"
for cfg in "${CFGS[@]}"; do
  echo "== $cfg" >> gpurun_out/bench_ab.log
  env $cfg timeout 600 python bench.py --no-cpu-baseline >> gpurun_out/bench_ab.log 2>&1
done
if [ -n "$PROBE" ]; then timeout 300 python tools/step_probe.py > gpurun_out/iter_probe.log 2>&1; fi
python - <<'PY'
import json
for line in open("gpurun_out/bench_ab.log"):
    if line.startswith("=="): print(line.strip()); continue
    try:
        d = json.loads(line)
        print(d["value"], d["mean_jct_us"], d["p99_jct_us"], {k: v["us_per_step"] for k, v in d["stages"].items()})
    except Exception:
        pass
PY
