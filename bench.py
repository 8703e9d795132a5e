#!/usr/bin/env python3
"""Benchmark: requests/sec and mean/p99 JCT of the Thinker->Talker->Code2Wav
pipeline (BASELINE.json metric) on B200.

One "step" = the reference's benchmark workload pushed through the whole
pipeline once: gen_workload(n=100, seed=7) (bench.hpp:31-56), closed loop with
16 requests in flight (bench.hpp:243-252), reference.json engine configs
(configs/omni3.json), streaming edges (chunk 4 / 8), random-init models
(Thinker 8L d2048, Talker 4L d2048, DiT 4L d1024; weights are a counter-
based function of the seed — synthetic, no checkpoints). Stage iterations
complete on CUDA events (device-paced clock), JCT = done - submit.

--gpus N: ONE stage graph over N GPUs of the box: every stage
gets whole GPUs, the bottleneck stages replicas, placed by placement_for()
from the measured per-stage device busy time (STAGE_BUSY_MS); the Thinker's
hidden rows cross GPUs over NVLink (connector pack with peer stores into the
consuming Talker replica's arena). The workload scales with N ("scaling":
"weak"): gen_workload(n = 100 N, seed 7), closed loop 16 N. The orchestrator is
the reference's single control-plane thread (orchestrator.hpp:377-437), so
one process drives all N GPUs: launched plainly (`python bench.py --gpus N`)
it is that process; under torchrun rank 0 is, and ranks 1..N-1 only join the
barriers (gloo) and report zero device time, so max over ranks = rank 0's.

--procs (under torchrun): one process per GPU -- rank r >= 1 is a stage
worker (omni_worker_serve) hosting the stages placed on cuda:r, rank 0 the
control plane + the Thinker; steps cross processes as control-frame requests,
hidden rows as CUDA-IPC packs. Off by default: the single
driving process avoids a request round trip per step.

--impl reference: the reference's own control plane (compiled from its
headers, oracle/_ref/ref_cpu_pipeline) with CPU fp32 model hooks on the host
cores, over a bounded sample of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
CONFIG = ROOT / "configs" / "omni3.json"
METRIC = "requests/sec and mean/p99 JCT, Thinker→Talker→Code2Wav, at 1/2/4/8 B200"
CPU_SAMPLE_N = 2  # first 2 requests of the workload (67 text tokens ~ 2 average requests)


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm": d["hbm_gbs"], "tf": d["bf16_tflops"], "tf_sust": d.get("bf16_tflops_sustained"),
                "source": "measured"}
    return {"hbm": 6650.0, "tf": 1590.0, "tf_sust": 1400.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup(n_gpus: int):
    """torchrun plumbing: a CPU (gloo) group for the barriers and the
    max-over-ranks reductions -- the data path has no collective."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        return world, rank, local, dist
    return 1, 0, local, None


# What one GPU-worth of each stage costs per 100-request step of the reference
# workload when the stage has its GPU to ITSELF (ms): the bench's step counts
# x uncontended step times (tools/step_probe.py) -- Thinker 439 steps x ~0.33
# ms (decode ~0.28, mixed prefill ~0.5), Talker 2040 x 0.155 ms, Code2Wav ~213
# iterations x ~1.2 ms (all 148 SMs, ~85 tokens). On one shared GPU the three
# are ~400 ms each (the DiT then runs on a 48-SM share), which says nothing
# about their cost apart. placement_for() apportions GPUs by these: 2 GPUs =
# Talker alone | Thinker + Code2Wav, 4 = T | Tk x2 | C2W,
# 8 = T x2 | Tk x3 | C2W x3.
STAGE_BUSY_MS = {"thinker": 145.0, "talker": 316.0, "vocoder": 255.0}


def placement_for(n_gpus: int, busy: dict = STAGE_BUSY_MS) -> dict:
    """Stage -> "cuda:i,cuda:j,..." for Thinker->Talker->Code2Wav on n GPUs.
    1 GPU: everything on cuda:0 (own streams). 2 GPUs: the busiest stage alone
    on cuda:1, the other two share cuda:0. >= 3: every stage gets whole GPUs,
    one each, the rest by largest remainder of busy-time share (ties to the
    later stage in the graph: its work is on every request's tail)."""
    stages = list(busy)
    if n_gpus <= 1:
        return {st: "cuda:0" for st in stages}
    if n_gpus == 2:
        heavy = max(stages, key=lambda st: (busy[st], stages.index(st)))
        return {st: ("cuda:1" if st == heavy else "cuda:0") for st in stages}
    total = sum(busy.values())
    quota = {st: n_gpus * busy[st] / total for st in stages}
    count = {st: max(1, int(quota[st])) for st in stages}
    while sum(count.values()) > n_gpus:
        st = max((st for st in stages if count[st] > 1), key=lambda st: count[st] - quota[st])
        count[st] -= 1
    while sum(count.values()) < n_gpus:
        st = max(stages, key=lambda st: (quota[st] - count[st], stages.index(st)))
        count[st] += 1
    out, nxt = {}, 0
    for st in stages:
        out[st] = ",".join(f"cuda:{nxt + i}" for i in range(count[st]))
        nxt += count[st]
    return out


def _reduce(x: float, dist, op: str) -> float:
    """All-reduce one scalar over the ranks (nccl on the GPU box, gloo on CPU)."""
    if dist is None:
        return x
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def max_over_ranks(x: float, dist) -> float:
    return _reduce(x, dist, "max")


def sum_over_ranks(x: float, dist) -> float:
    return _reduce(x, dist, "sum")


def aggregate(completed: float, dev_ms: float, wall_s: float, dist) -> dict:
    """Whole-job numbers of a weak-scaling run: every rank ran its own full
    workload replica; value = all requests completed / the SLOWEST rank's
    device time (max over ranks), e2e likewise on the host clock."""
    t_max_ms = max_over_ranks(dev_ms, dist)
    wall_max = max_over_ranks(wall_s, dist)
    done = sum_over_ranks(completed, dist)
    return {"completed": done, "t_max_ms": t_max_ms, "wall_max_s": wall_max,
            "value": done / (t_max_ms / 1e3), "e2e": done / wall_max}


def gemm_roofline(pk: dict) -> dict:
    """Dominant kernel: the swap-AB tcgen05 GEMM streaming the Talker/Thinker
    gate-up weights (N=2*8192, K=2048) at the Talker's typical decode batch
    (M=16 rows). Timed with CUDA events on the launching stream
    over a CUDA graph of 64 back-to-back launches cycling 8 distinct 64 MiB
    weight copies (512 MiB > 126 MB L2, so every launch streams HBM), after
    warm-up."""
    from paper_2602_02204_b200 import dev as D
    lib = D.dev_lib()
    N, K, M = 16384, 2048, 16
    W = D.mem_alloc(N * K * 2)
    X = D.mem_alloc(256 * K * 2)
    O = D.mem_alloc(256 * N * 4)
    # 8 distinct weight copies cycled so every launch streams from HBM, not L2
    copies = [W] + [D.mem_alloc(N * K * 2) for _ in range(7)]
    for i, w in enumerate(copies):
        lib.omni_k_fill_weights(C.c_uint64(w), C.c_int64(N * K), C.c_uint64(11 + i), C.c_uint32(1), C.c_float(0.02))
    lib.omni_k_fill_weights(C.c_uint64(X), C.c_int64(256 * K), C.c_uint64(3), C.c_uint32(2), C.c_float(1.0))
    arr = (C.c_uint64 * len(copies))(*copies)
    ms = C.c_float()
    rc = lib.omni_k_gemm_time_multi(arr, len(copies), N, K, C.c_uint64(X), M, 4, C.c_uint64(O), N // 2, 8, 64,
                                    C.byref(ms))
    times = [ms.value] if rc == 0 else [float("nan")]
    for p in copies + [X, O]:
        D.mem_free(p)
    t_ms = statistics.median(times)
    algo = N * K * 2 + M * K * 2 + M * (N // 2) * 2
    # DRAM traffic per launch of this kernel from the committed `ncu --set full`
    # capture (tools/ncu_gemm.py 16 -> profiles/ncu_traffic.json)
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get("gemm_gateup_m16", {}).get("dram_bytes_per_launch")
    gbs = algo / (t_ms * 1e-3) / 1e9
    return {"kernel": "gemm_tc_kernel<BN=16,EPI_SWIGLU> gate-up N=16384 K=2048 M=16", "bound": "hbm",
            "achieved": round(gbs, 1), "peak": pk["hbm"], "unit": "GB/s", "frac": round(gbs / pk["hbm"], 4),
            "traffic": traffic, "algorithmic_bytes": algo, "us_per_launch": round(t_ms * 1e3, 2),
            "peak_source": pk["source"]}


def cpu_baseline(sample_n: int, small: bool) -> dict:
    exe = ROOT / "oracle" / "_ref" / "ref_cpu_pipeline"
    if not exe.exists():
        return {"value": None, "unit": "requests/s", "kind": "reference", "cores": os.cpu_count(),
                "sample": f"unavailable: {exe} not built"}
    # every host thread (torchrun exports OMP_NUM_THREADS=1 to each rank)
    env = dict(os.environ, OMP_NUM_THREADS=str(os.cpu_count() or 1))
    r = subprocess.run([str(exe), str(CONFIG), str(sample_n), "7", "16", "1" if small else "0"],
                       capture_output=True, text=True, timeout=900, env=env)
    if r.returncode != 0:
        return {"value": None, "unit": "requests/s", "kind": "reference", "cores": os.cpu_count(),
                "sample": f"failed: {r.stderr.strip()[-200:]}"}
    d = json.loads(r.stdout.strip().splitlines()[-1])
    return {"value": round(d["requests_per_s"], 6), "unit": "requests/s", "kind": "reference",
            "cores": d["threads"],
            "sample": f"first {sample_n} requests of gen_workload(n=100,seed=7) ({d['text_tokens']} text / "
                      f"{d['codec_tokens']} codec tokens, {d['wave_samples']} samples) through the reference "
                      f"Orchestrator (wall clock, step_latency 0) with fp32 CPU model hooks, "
                      f"{d['wall_s']:.1f}s; mean JCT {d['mean_jct_us'] / 1e6:.2f}s",
            "mean_jct_us": d["mean_jct_us"], "p99_jct_us": d["p99_jct_us"], "wall_s": d["wall_s"]}


def run_reference(args, world, rank) -> None:
    if rank != 0:
        return
    vals = []
    last = None
    for i in range(args.warmup + args.steps):
        b = cpu_baseline(CPU_SAMPLE_N, args.small)
        if b["value"] is None:
            print(json.dumps({"impl": "reference", "unavailable": b["sample"]}))
            return
        if i >= args.warmup:
            vals.append(b["value"])
            last = b
    v = statistics.mean(vals)
    out = {"metric": METRIC, "value": round(v, 6), "unit": "requests/s", "impl": "reference",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(last["wall_s"] * 1e3, 1), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": f"omni3 (reference.json) Thinker->Talker->Code2Wav, bounded sample "
                                  f"{CPU_SAMPLE_N} requests of gen_workload(100, seed 7), closed loop 16",
                      "n_requests": CPU_SAMPLE_N},
           "mean_jct_us": last["mean_jct_us"], "p99_jct_us": last["p99_jct_us"],
           "cpu_baseline": {k: last[k] for k in ("value", "unit", "cores", "kind", "sample")},
           "e2e": {"value": round(v, 6), "unit": "requests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", "--requests", dest="n", type=int, default=100)  # --requests: torchrun-safe spelling
    ap.add_argument("--concurrency", type=int, default=16)
    ap.add_argument("--small", action="store_true", help="reduced model dims (debug only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--placement", default="", help='JSON stage->devices override, e.g. \'{"talker": "cuda:1,cuda:2"}\'')
    ap.add_argument("--procs", action="store_true",
                    help="under torchrun: ranks >= 1 are stage worker processes for their GPU")
    ap.add_argument("--fold-devices", action="store_true",
                    help="debug: map cuda:i -> cuda:(i mod visible) to exercise the N-GPU code path on fewer "
                         "GPUs (the line is marked folded and is not an N-GPU measurement)")
    args = ap.parse_args()
    world, rank, local, dist = dist_setup(args.gpus)
    n_gpus = world if world > 1 else max(1, args.gpus)

    if args.impl == "reference":
        run_reference(args, world, rank)
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    sock = lambda r: f"/tmp/omni_bench_{os.environ.get('MASTER_PORT', '0')}_w{r}.sock"
    if rank != 0:
        # rank 0 drives the whole stage graph over all N GPUs; this rank only
        # brackets the timed region and reports zero device time -- or, with
        # --procs, serves the stages placed on its GPU meanwhile
        worker = None
        if args.procs:
            from paper_2602_02204_b200 import serve_lib
            lib = serve_lib()
            worker = threading.Thread(target=lambda: lib.omni_worker_serve(sock(rank).encode(), 600000), daemon=True)
            worker.start()
        dist.barrier()
        dist.barrier()
        aggregate(0, 0.0, 0.0, dist)
        if worker is not None:
            worker.join(timeout=600)
        dist.destroy_process_group()
        return

    import torch
    from paper_2602_02204_b200 import dev as D
    from paper_2602_02204_b200.serve import Pipeline

    visible = torch.cuda.device_count()
    if visible < n_gpus and not args.fold_devices:
        raise SystemExit(f"--gpus {n_gpus}: only {visible} CUDA device(s) visible")
    torch.cuda.set_device(0)
    pk = peaks()
    placement = placement_for(n_gpus)
    if args.placement:
        placement.update(json.loads(args.placement))
    workers = {}
    if args.procs and world > 1:
        # stage -> worker of the rank its GPU belongs to (the Thinker packs: stays here)
        for k, v in placement.items():
            ranks = {int(d.split(":")[1]) for d in v.split(",")}
            if k != "thinker" and len(ranks) == 1 and min(ranks) != 0:
                workers[k] = sock(min(ranks))
            elif k != "thinker" and not args.fold_devices:
                for r in ranks - {0}:
                    workers[f"cuda:{r}"] = sock(r)
    if args.fold_devices:
        placement = {k: ",".join(f"cuda:{int(d.split(':')[1]) % visible}" for d in v.split(","))
                     for k, v in placement.items()}
    gpus_used = sorted({int(d.split(":")[1]) for v in placement.values() for d in v.split(",")})
    cfg = json.loads(CONFIG.read_text())
    cfg["placement"] = placement
    if workers:
        cfg["workers"] = workers
    n_req = args.n * n_gpus
    conc = args.concurrency * n_gpus
    pipe = Pipeline(json.dumps(cfg), weight_seed=1234, small_models=args.small, device=0)
    spec = dict(n=n_req, seed=7, concurrency=conc, stream=True, clock="device")
    for _ in range(args.warmup):
        pipe.bench(**spec)
    lib = D.dev_lib()
    l0, h0, d0 = C.c_uint64(), C.c_uint64(), C.c_uint64()
    results = []
    if dist is not None:
        dist.barrier()
    for g in gpus_used:
        torch.cuda.synchronize(g)
    with ClockSampler(",".join(str(g) for g in gpus_used)) as clk:
        lib.omni_dev_counters(C.byref(l0), C.byref(h0), C.byref(d0))
        gc0, gr0 = C.c_uint64(), C.c_uint64()
        lib.omni_dev_graph_counters(C.byref(gc0), C.byref(gr0))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(args.steps):
            results.append(pipe.bench(**spec))  # each step drains fully: all stage streams done
        e1.record()
        for g in gpus_used:  # bench() drained every stage stream on every GPU already
            torch.cuda.synchronize(g)
        wall = time.perf_counter() - t0
    if dist is not None:
        dist.barrier()
    if workers:
        pipe.close()  # shuts the stage workers down (their ranks are waiting for them)
    l1, h1, d1 = C.c_uint64(), C.c_uint64(), C.c_uint64()
    lib.omni_dev_counters(C.byref(l1), C.byref(h1), C.byref(d1))
    gc1, gr1 = C.c_uint64(), C.c_uint64()
    lib.omni_dev_graph_counters(C.byref(gc1), C.byref(gr1))
    dev_ms = e0.elapsed_time(e1)
    agg = aggregate(sum(r["completed"] for r in results), dev_ms, wall, dist)
    t_max_ms, wall_max, done_all, value = agg["t_max_ms"], agg["wall_max_s"], agg["completed"], agg["value"]
    # serving metric as the reference defines it: completed / makespan (first admit -> last done)
    rps_makespan = statistics.mean(r["requests_per_s"] for r in results)
    mean_jct = statistics.mean(r["mean_jct_us"] for r in results)
    p99_jct = statistics.mean(r["p99_jct_us"] for r in results)
    roof = gemm_roofline(pk)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(CPU_SAMPLE_N, args.small)
    last = results[-1]
    step_s = t_max_ms / 1e3 / args.steps
    ar_bytes = {  # weights streamed per step by the AR stages (bf16)
        "thinker": 8 * 60_817_408 * 2 + 2 * 256 * 2048 * 2,
        "talker": 4 * 60_817_408 * 2 + 2048 * 2048 * 2 + 64 * 2048 * 2,
    }
    stage = {
        "thinker": {"steps": last["steps_thinker"], "device_ms": round(last["dev_ms_thinker"], 1),
                    "host_us_per_step": round(1e3 * last["host_ms_thinker"] / max(1, last["steps_thinker"]), 1),
                    "gap_us": round(last["gap_us_thinker"], 1),
                    "us_per_step": round(1e3 * last["dev_ms_thinker"] / max(1, last["steps_thinker"]), 1),
                    "weight_GBps": round(ar_bytes["thinker"] * last["steps_thinker"] / max(1e-9, last["dev_ms_thinker"] * 1e-3) / 1e9, 1)},
        "talker": {"steps": last["steps_talker"], "device_ms": round(last["dev_ms_talker"], 1),
                   "host_us_per_step": round(1e3 * last["host_ms_talker"] / max(1, last["steps_talker"]), 1),
                   "gap_us": round(last["gap_us_talker"], 1),
                   "us_per_step": round(1e3 * last["dev_ms_talker"] / max(1, last["steps_talker"]), 1),
                   "weight_GBps": round(ar_bytes["talker"] * last["steps_talker"] / max(1e-9, last["dev_ms_talker"] * 1e-3) / 1e9, 1)},
        "code2wav": {"steps": last["steps_dit"], "device_ms": round(last["dev_ms_dit"], 1),
                     "host_us_per_step": round(1e3 * last["host_ms_dit"] / max(1, last["steps_dit"]), 1),
                     "gap_us": round(last["gap_us_dit"], 1),
                     "us_per_step": round(1e3 * last["dev_ms_dit"] / max(1, last["steps_dit"]), 1)},
    }
    out = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "requests/s",
        "n_gpus": n_gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(step_s * 1e3, 2),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic: gen_workload(n=100, seed=7) prompts, random-init weights (counter RNG)",
        "config": {"workload": f"omni3 = reference.json Thinker->Talker->Code2Wav, gen_workload(n={n_req}, seed 7), "
                               f"closed loop {conc} (16 per GPU), streaming chunks 4/8, one stage graph over "
                               f"{n_gpus} GPU(s)",
                   "n_requests_per_step": n_req, "concurrency": conc,
                   "placement": placement,
                   **({"folded": f"DEBUG: {n_gpus}-GPU placement folded onto {visible} GPU(s)"}
                      if args.fold_devices else {}),
                   "models": "thinker 8L d2048 (16q/4kv heads, ffn 8192, V256); talker 4L d2048 (V64); "
                             "code2wav DiT 4L d1024 T4 S16",
                   "parallelism": ("stage-per-GPU " + " ".join(f"{k}x{len(v.split(','))}" for k, v in placement.items())
                                   + (" (one process per GPU: stage workers)" if workers else ""))
                                  if n_gpus > 1 else "all stages on cuda:0",
                   "l2": "weights 1.4 GB per AR step set >> 126 MB L2 (no flush needed)"},
        "mean_jct_us": round(mean_jct, 1),
        "p99_jct_us": round(p99_jct, 1),
        "requests_per_s_makespan": round(rps_makespan, 3),
        "completed": int(done_all),
        "stages": stage,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": {"value": round(done_all / wall_max, 3), "unit": "requests/s",
                "h2d_bytes_per_step": int((h1.value - h0.value) / args.steps),
                "d2h_bytes_per_step": int((d1.value - d0.value) / args.steps),
                "note": "host-clock time of the public C-ABI bench call incl. orchestrator setup, per-step "
                        "descriptor H2D copies from pinned memory and token/sample D2H reads"},
        "gpu_launches": int(l1.value - l0.value),
        "step_graphs": {"captured_in_timed_region": int(gc1.value - gc0.value),
                        "replayed": int(gr1.value - gr0.value)},
        "clocks": clk.summary(),
    }
    print(json.dumps(out))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
