#!/usr/bin/env bash
# GPU test subset + AR step probe + pipeline bench A/B (current tree vs ${ALT}).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-abf}; alt=${ALT:-_ab_base}
timeout 900 python -m pytest -q -x -m gpu ${TESTS:-tests/test_gpu_gemm.py tests/test_gpu_edges.py tests/test_gpu_models.py tests/test_gpu_longctx.py tests/test_gpu_prefix_cache.py tests/test_gpu_pipeline.py} > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/${tag}_tests.log
for t in cur alt; do
  d=.; [ $t = alt ] && d=$alt
  echo "probe $t"; (cd $d && timeout 300 python tools/step_probe.py --ar-only --quick 2>&1 | tail -5)
done
REPS=${REPS:-3} ALT=$alt bash tools/gpu_ab_tree.sh ${tag}
