#!/bin/bash
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm --format=csv,noheader > gpurun_out/trace_clk.txt
timeout 300 python tools/gemm_trace.py 1.9 > gpurun_out/gemm_trace.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/iter_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/iter_pytest.log
cat gpurun_out/gemm_trace.log; tail -2 gpurun_out/iter_pytest.log
