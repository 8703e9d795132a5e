#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/iter_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/iter_pytest.log
tail -2 gpurun_out/iter_pytest.log
timeout 300 python tools/step_probe.py ${PROBE_ARGS:---quick} > gpurun_out/iter_probe.log 2>&1
cat gpurun_out/iter_probe.log
if [ -n "$BENCH" ]; then timeout 600 python bench.py --no-cpu-baseline > gpurun_out/iter_bench.log 2>&1; python - <<'PY'
import json
d = json.loads(open("gpurun_out/iter_bench.log").read().strip().splitlines()[-1])
print(d["value"], d["mean_jct_us"], d["p99_jct_us"], {k: v["us_per_step"] for k, v in d["stages"].items()}, d["roofline"]["frac"])
PY
fi
