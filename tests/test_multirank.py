"""World-size-2 CPU (gloo) coverage of bench.py's multi-GPU plumbing.

Under torchrun rank 0 drives the whole stage graph over all N GPUs (the
reference's single control-plane thread, orchestrator.hpp:377-437) and ranks
1..N-1 only bracket the timed region, reporting zero work and zero device
time; value = requests completed on all ranks / max-over-ranks device time.
Also: the stage-per-GPU placement bench.py derives for N GPUs."""
import os
import socket
import sys
from pathlib import Path

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    # rank r: 100 + r requests completed in (1000 + 500 r) ms of device time
    agg = bench.aggregate(100 + rank, 1000.0 + 500.0 * rank, 2.0 + rank, dist)
    # bench.py's N > 1 protocol: rank 0 did all the work, the others report zeros
    dist.barrier()
    dist.barrier()
    agg2 = bench.aggregate(800 if rank == 0 else 0, 4000.0 if rank == 0 else 0.0, 5.0 if rank == 0 else 0.0, dist)
    q.put((rank, (agg, agg2)))
    dist.barrier()
    dist.destroy_process_group()


def test_weak_scaling_aggregate_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        a, b = out[r]
        assert b["completed"] == 800 and b["t_max_ms"] == 4000.0
        assert b["value"] == pytest.approx(200.0) and b["e2e"] == pytest.approx(160.0)
        assert a["completed"] == 201
        assert a["t_max_ms"] == 1500.0
        assert a["value"] == pytest.approx(201 / 1.5)
        assert a["e2e"] == pytest.approx(201 / 3.0)


def test_single_rank_aggregate_is_identity():
    sys.path.insert(0, str(ROOT))
    import bench
    a = bench.aggregate(100, 800.0, 1.0, None)
    assert a["value"] == pytest.approx(125.0) and a["e2e"] == pytest.approx(100.0)


def test_placement_for_n_gpus():
    sys.path.insert(0, str(ROOT))
    import bench

    def devs(p):
        return {k: [int(x.split(":")[1]) for x in v.split(",")] for k, v in p.items()}

    busy = {"thinker": 429.0, "talker": 457.0, "vocoder": 484.0}
    assert bench.placement_for(1, busy) == {"thinker": "cuda:0", "talker": "cuda:0", "vocoder": "cuda:0"}
    p2 = devs(bench.placement_for(2, busy))
    assert p2["vocoder"] == [1] and p2["thinker"] == p2["talker"] == [0]
    for n in (3, 4, 5, 8):
        p = devs(bench.placement_for(n, busy))
        used = sorted(d for v in p.values() for d in v)
        assert used == list(range(n)), (n, p)          # every GPU exactly once
        assert all(len(v) >= 1 for v in p.values())
    p8 = devs(bench.placement_for(8, busy))
    assert [len(p8[s]) for s in ("thinker", "talker", "vocoder")] == [2, 3, 3]
    # a dominant stage gets the replicas
    p8b = devs(bench.placement_for(8, {"thinker": 100.0, "talker": 600.0, "vocoder": 100.0}))
    assert len(p8b["talker"]) == 6
