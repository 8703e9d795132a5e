#!/bin/bash
# A/B of the step-pipeline knobs on uncontended stage steps.
mkdir -p gpurun_out
: > gpurun_out/ab.log
for cfg in "OMNI_PF_MB=32" "OMNI_PF_MB=0" "OMNI_PF_MB=8" "OMNI_PF_MB=0 OMNI_GRAPHS=0" "OMNI_PF_MB=0 OMNI_PDL=0"; do
  echo "== $cfg" >> gpurun_out/ab.log
  env $cfg timeout 300 python tools/step_probe.py --quick >> gpurun_out/ab.log 2>&1
done
timeout 300 python tools/step_probe.py > gpurun_out/iter_probe.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/iter_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/iter_pytest.log
tail -2 gpurun_out/iter_pytest.log
