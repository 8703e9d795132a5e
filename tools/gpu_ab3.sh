#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab3.log
for cfg in "OMNI_X=0" "OMNI_DIT_2CTA=1" "OMNI_DIT_SPLIT_W2=2" "OMNI_DIT_SPLIT_W2=4" "OMNI_DIT_SPLIT_W2=4 OMNI_DIT_2CTA=1"; do
  echo "== $cfg" >> gpurun_out/ab3.log
  env $cfg timeout 300 python tools/step_probe.py --dit-only >> gpurun_out/ab3.log 2>&1
done
cat gpurun_out/ab3.log
