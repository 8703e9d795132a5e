#!/usr/bin/env bash
# Round-2 evidence (VERDICT r1 "next" #4 and #6):
#  1. launch list of a STEADY-STATE window of the real n=100 bench (startup and
#     the first warm-up step skipped with --launch-skip),
#  2. whole-step ncu results of Thinker / Talker decode steps replayed as CUDA
#     graphs with PDL intact (--graph-profiling graph),
#  3. compute-sanitizer racecheck / synccheck / memcheck over the GEMM, edge
#     and fused-DiT GPU tests.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-ev2}
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 1200 ncu --metrics $M --clock-control none --launch-skip ${SKIP:-150000} --launch-count ${COUNT:-20000} --csv \
  --log-file gpurun_out/${tag}_bench_window.csv python bench.py --steps 1 --warmup 2 --no-cpu-baseline \
  > gpurun_out/${tag}_bench_window.log 2>&1
echo "window rc=$?"
for cfg in "thinker 1" "thinker 16" "talker 16" "talker 64"; do
  set -- $cfg
  timeout 600 ncu --metrics $M --clock-control none --graph-profiling graph --csv \
    --log-file gpurun_out/${tag}_graph_${1}_${2}.csv python tools/ncu_step_graph.py $1 $2 64 24 \
    > gpurun_out/${tag}_graph_${1}_${2}.log 2>&1
  echo "graph $cfg rc=$?"
  timeout 300 python tools/ncu_step_graph.py $1 $2 64 24 >> gpurun_out/${tag}_graph_${1}_${2}.log 2>&1
done
if [ -z "${NO_SANITIZE:-}" ]; then
  san() {  # tool timeout files...
    local tool=$1 to=$2; shift 2
    timeout $to compute-sanitizer --tool $tool --print-limit 20 python -m pytest -q -x -m gpu "$@" \
      > gpurun_out/${tag}_sanitize_${tool}.log 2>&1
    echo "$tool rc=$?"; tail -4 gpurun_out/${tag}_sanitize_${tool}.log
  }
  san racecheck 1200 tests/test_gpu_gemm.py
  san synccheck 900 tests/test_gpu_gemm.py tests/test_gpu_edges.py
  san memcheck 900 tests/test_gpu_edges.py tests/test_gpu_dit_fused.py
fi
