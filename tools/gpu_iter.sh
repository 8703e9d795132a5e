#!/bin/bash
# Iteration check: GPU parity tests + uncontended stage step times (+ optional bench).
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv > gpurun_out/iter_clocks.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/iter_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/iter_pytest.log
timeout 600 python tools/step_probe.py > gpurun_out/iter_probe.log 2>&1; echo "probe rc=$?" >> gpurun_out/iter_probe.log
if [ -n "$BENCH" ]; then timeout 900 python bench.py --no-cpu-baseline > gpurun_out/iter_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/iter_bench.log; fi
if [ -n "$NCU" ]; then timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/iter_launches.csv python tools/step_probe.py --quick > /dev/null 2>&1; fi
tail -3 gpurun_out/iter_pytest.log
