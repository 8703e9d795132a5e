#!/usr/bin/env bash
# Reference CPU arm: requests/s vs sample size (2 / 4 / 8 / 16 requests, closed loop 16) on the box's host cores.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for n in 2 4 8 16; do
  OMP_NUM_THREADS=$(nproc) timeout 600 oracle/_ref/ref_cpu_pipeline configs/omni3.json $n 7 16 0 | tail -1 | sed "s/^/n=$n /"
done | tee gpurun_out/ref_concurrency.txt
