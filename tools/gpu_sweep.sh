#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/gemm_sweep.py > gpurun_out/sweep.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 8 -c 1 \
   -o gpurun_out/gemm_wo_m4 -f python tools/ncu_gemm.py 4 2048 2048 1 > gpurun_out/ncu_wo.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attention_kernel -s 20 -c 1 \
   -o gpurun_out/attn_m4 -f python tools/step_probe.py --quick --ar-only > gpurun_out/ncu_attn.log 2>&1
echo done
