#!/bin/bash
# Uncontended stage step times + ncu full capture of the dominant GEMM.
mkdir -p gpurun_out
timeout 600 python tools/step_probe.py > gpurun_out/step_probe.log 2>&1; echo "rc=$?" >> gpurun_out/step_probe.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 8 -c 2 \
   -o gpurun_out/gemm_gu_m16 -f python tools/ncu_gemm.py 16 > gpurun_out/ncu_gemm.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/launches_probe.csv python tools/step_probe.py --quick > gpurun_out/ncu_probe.log 2>&1
echo done
