#!/usr/bin/env bash
# ncu evidence for the pre-tiled gate-up GEMM + a steady-state bench launch window with the final code.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-tl}
OMNI_PREWARM=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 30 -c 1 \
  -o gpurun_out/${tag}_gemm_gateup_tiled -f python tools/ncu_gemm_tiled.py 16 > gpurun_out/${tag}_ncu_gemm.log 2>&1
echo "ncu gemm rc=$?"
ncu -i gpurun_out/${tag}_gemm_gateup_tiled.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; u=r[1]; v=r[2]
for i,n in enumerate(h):
  if n in ('gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','launch__grid_size','dram__throughput.avg.pct_of_peak_sustained_elapsed','Kernel Name','Function Name'): print(n,u[i],v[i])
"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 1500 ncu --metrics $M --clock-control none --launch-skip 150000 --launch-count 12000 --csv \
  --log-file gpurun_out/${tag}_bench_window.csv python bench.py --steps 1 --warmup 2 --no-cpu-baseline > /dev/null 2>&1
echo "window rc=$?"
python tools/launch_summary.py gpurun_out/${tag}_bench_window.csv > gpurun_out/${tag}_launches.md 2>&1; head -12 gpurun_out/${tag}_launches.md
