#!/usr/bin/env bash
# Round-2 final evidence: full GPU suite + smoke, default bench x2, reference arm,
# c64 bench, folded 2/4-GPU placement runs, ncu --set full of the fused DiT
# (96 / 512 tokens) and of the dominant GEMM, steady-state bench launch window.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-fin}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${tag}_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
for i in 1 2; do
  timeout 900 python bench.py > gpurun_out/${tag}_bench_$i.json 2> gpurun_out/${tag}_bench_$i.err; echo "bench rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/${tag}_bench_$i.json'));print(d['value'],d['e2e']['value'],d['mean_jct_us'],d['p99_jct_us'],d['roofline']['frac'],d['cpu_baseline']['value'] if d['cpu_baseline'] else None)"
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err; echo "ref rc=$?"; tail -c 400 gpurun_out/${tag}_ref.json
timeout 900 python bench.py --concurrency 64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_c64.json 2>/dev/null; echo "c64 rc=$?"
python -c "import json;d=json.load(open('gpurun_out/${tag}_c64.json'));print(d['value'],d['mean_jct_us'])"
for n in 2 4; do
  timeout 900 python bench.py --gpus $n --fold-devices --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${tag}_fold$n.json 2>/dev/null; echo "fold$n rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/${tag}_fold$n.json'));print(d['value'],d['config']['parallelism'],d['completed'])"
done
for N in 96 512; do
  OMNI_PREWARM=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:dit_fused -s 1 -c 1 \
    -o gpurun_out/${tag}_dit_N${N} -f python tools/dit_one.py $N 2 > /dev/null 2>&1; echo "ncu dit $N rc=$?"
done
OMNI_PREWARM=0 timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 8 -c 1 \
  -o gpurun_out/${tag}_gemm_gateup_m16 -f python tools/ncu_gemm.py 16 > /dev/null 2>&1; echo "ncu gemm rc=$?"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu --metrics $M --clock-control none --launch-skip 150000 --launch-count 12000 --csv \
  --log-file gpurun_out/${tag}_bench_window.csv python bench.py --steps 1 --warmup 2 --no-cpu-baseline > /dev/null 2>&1
echo "window rc=$?"
