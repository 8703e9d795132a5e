#!/bin/bash
# Round-end evidence: default bench line, reference arm, bench launch list,
# ncu --set full captures of the dominant kernels, step probe.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/ev_bench.log 2>&1; echo "rc=$?" >> gpurun_out/ev_bench.log
timeout 900 python bench.py --impl reference > gpurun_out/ev_ref.log 2>&1; echo "rc=$?" >> gpurun_out/ev_ref.log
timeout 300 python tools/step_probe.py > gpurun_out/ev_probe.log 2>&1
timeout 300 python tools/gemm_sweep.py > gpurun_out/ev_sweep.log 2>&1
OMNI_PREWARM=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv \
  --log-file gpurun_out/ev_launches.csv python bench.py --steps 1 --warmup 0 --n 20 --no-cpu-baseline > /dev/null 2>&1
F="--set full --clock-control none --import-source on"
OMNI_PREWARM=0 timeout 300 ncu $F -k regex:gemm_tc_kernel -s 8 -c 1 -o gpurun_out/ev_gemm_gateup_m16 -f python tools/ncu_gemm.py 16 > /dev/null 2>&1
OMNI_PREWARM=0 timeout 300 ncu $F -k regex:gemm_tc_kernel -s 8 -c 1 -o gpurun_out/ev_gemm_down_m16 -f python tools/ncu_gemm.py 16 2048 8192 2 > /dev/null 2>&1
OMNI_PREWARM=0 timeout 300 ncu $F -k regex:gemm_tc_kernel -s 8 -c 1 -o gpurun_out/ev_gemm_qkv_m16 -f python tools/ncu_gemm.py 16 3072 2048 1 > /dev/null 2>&1
OMNI_PREWARM=0 timeout 300 ncu $F -k regex:attention_kernel -s 20 -c 1 -o gpurun_out/ev_attention -f python tools/step_probe.py --quick --ar-only > /dev/null 2>&1
OMNI_PREWARM=0 timeout 300 ncu $F -k regex:dit_attn -s 4 -c 1 -o gpurun_out/ev_dit_attn -f python tools/step_probe.py --dit-only --dit64 > /dev/null 2>&1
OMNI_PREWARM=0 timeout 300 ncu $F -k regex:dit_ln_mod -s 4 -c 1 -o gpurun_out/ev_dit_ln -f python tools/step_probe.py --dit-only --dit64 > /dev/null 2>&1
OMNI_PREWARM=0 timeout 300 ncu $F -k regex:pack_hidden -s 2 -c 1 -o gpurun_out/ev_pack -f python bench.py --steps 1 --warmup 0 --n 8 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
tail -n 2 gpurun_out/ev_bench.log gpurun_out/ev_ref.log
