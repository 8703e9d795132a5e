#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab2.log
for cfg in "OMNI_PF_MB=0" "OMNI_PF_MB=8" "OMNI_PF_MB=16" "OMNI_PF_MB=32"; do
  echo "== $cfg" >> gpurun_out/ab2.log
  env $cfg timeout 300 python tools/step_probe.py --quick --ar-only >> gpurun_out/ab2.log 2>&1
done
for cfg in "OMNI_DIT_BN=0" "OMNI_DIT_BN=64" "OMNI_DIT_BN=128" "OMNI_DIT_BN=256" "OMNI_DIT_SPLIT=2" "OMNI_DIT_SPLIT=4"; do
  echo "== $cfg" >> gpurun_out/ab2.log
  env $cfg timeout 300 python tools/step_probe.py --dit-only >> gpurun_out/ab2.log 2>&1
done
cat gpurun_out/ab2.log
