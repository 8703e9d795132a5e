#!/bin/bash
# pytest -m gpu, GEMM sweep + phase trace, stage probe, bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/iter_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/iter_pytest.log
tail -2 gpurun_out/iter_pytest.log
timeout 300 python tools/gemm_sweep.py > gpurun_out/sweep.log 2>&1
timeout 300 python tools/gemm_trace.py 1.9 > gpurun_out/gemm_trace.log 2>&1
timeout 300 python tools/step_probe.py > gpurun_out/iter_probe.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/iter_bench.log 2>&1
python - <<'PY'
import json
d = json.loads(open("gpurun_out/iter_bench.log").read().strip().splitlines()[-1])
print(d["value"], d["mean_jct_us"], d["p99_jct_us"], {k: v["us_per_step"] for k, v in d["stages"].items()}, d["roofline"]["frac"])
PY
