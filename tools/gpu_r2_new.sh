#!/usr/bin/env bash
# New GPU tests (IPC placement, HTTP serving), ncu --set full of the fused DiT
# iteration at 96 and 512 tokens, bench at concurrency 64.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-new}
timeout 600 python -m pytest -q -x -m gpu tests/test_ipc_placement.py tests/test_http_service.py > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/${tag}_tests.log
for N in 96 512; do
  OMNI_PREWARM=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:dit_fused -s 1 -c 1 \
    -o gpurun_out/${tag}_dit_N${N} -f python tools/dit_one.py $N 2 > gpurun_out/${tag}_dit_ncu_${N}.log 2>&1
  echo "ncu dit $N rc=$?"
done
timeout 900 python bench.py --concurrency 64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_c64.json 2> gpurun_out/${tag}_c64.err
echo "c64 rc=$?"; tail -c 600 gpurun_out/${tag}_c64.json
