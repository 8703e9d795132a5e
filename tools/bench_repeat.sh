#!/usr/bin/env bash
# Run-to-run spread of the default bench line (and c64) on one box: N repeats, no CPU baseline.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
n=${1:-5}
for i in $(seq 1 $n); do
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/rep_c16_$i.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/rep_c16_$i.json'));print('c16',d['value'],d['mean_jct_us'],d['p99_jct_us'],d['clocks']['sm_mhz'],d['clocks']['reasons'])"
done
for i in 1 2 3; do
  timeout 600 python bench.py --no-cpu-baseline --concurrency 64 --steps 3 > gpurun_out/rep_c64_$i.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/rep_c64_$i.json'));print('c64',d['value'],d['mean_jct_us'],d['p99_jct_us'])"
done
