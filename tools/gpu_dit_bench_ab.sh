#!/usr/bin/env bash
# GPU box: bench A/B of the DiT path -- per-op kernels vs the fused iteration at several grid sizes.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-dab}
timeout 300 python -m pytest tests/test_gpu_models.py -k dit -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?"
for cfg in "OMNI_DIT_FUSED=0" "OMNI_DIT_CTAS=148" "OMNI_DIT_CTAS=100" "OMNI_DIT_CTAS=64" "OMNI_DIT_CTAS=40"; do
  env $cfg timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_b.json 2>/dev/null
  python - "$cfg" gpurun_out/${tag}_b.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
st = d["stages"]
print(sys.argv[1], d["value"], "rps; jct", d["mean_jct_us"], "; us/step thinker", st["thinker"]["us_per_step"],
      "talker", st["talker"]["us_per_step"], "c2w", st["code2wav"]["us_per_step"], "c2w steps", st["code2wav"]["steps"],
      "c2w ms", st["code2wav"]["device_ms"])
PY
done
