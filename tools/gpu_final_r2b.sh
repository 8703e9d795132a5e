#!/usr/bin/env bash
# Round-2 final lines: GPU suite + smoke, default bench x3, reference arm, c64 x2, folded 2/4-GPU.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-fin2}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${tag}_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
for i in 1 2 3; do
  timeout 900 python bench.py > gpurun_out/${tag}_bench_$i.json 2> gpurun_out/${tag}_bench_$i.err; echo "bench rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/${tag}_bench_$i.json'));print(d['value'],d['e2e']['value'],d['mean_jct_us'],d['p99_jct_us'],d['roofline']['frac'],d['cpu_baseline']['value'] if d['cpu_baseline'] else None,d['clocks'])"
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err; echo "ref rc=$?"; python -c "import json;d=json.load(open('gpurun_out/${tag}_ref.json'));print(d['value'],d['cpu_baseline'])"
for i in 1 2; do
  timeout 900 python bench.py --concurrency 64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_c64_$i.json 2>/dev/null; echo "c64 rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/${tag}_c64_$i.json'));print(d['value'],d['mean_jct_us'])"
done
for n in 2 4 8; do
  timeout 900 python bench.py --gpus $n --fold-devices --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/${tag}_fold$n.json 2>/dev/null; echo "fold$n rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/${tag}_fold$n.json'));print(d['value'],d['config']['parallelism'],d['completed'])"
done
