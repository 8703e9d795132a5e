"""World-size-2 CPU (gloo) coverage of bench.py's multi-GPU aggregation:
weak scaling, one full pipeline replica per rank, no data-path collective;
value = requests completed on ALL ranks / max-over-ranks device time."""
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
    q.put((rank, agg))
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
        a = out[r]
        assert a["completed"] == 201
        assert a["t_max_ms"] == 1500.0
        assert a["value"] == pytest.approx(201 / 1.5)
        assert a["e2e"] == pytest.approx(201 / 3.0)


def test_single_rank_aggregate_is_identity():
    sys.path.insert(0, str(ROOT))
    import bench
    a = bench.aggregate(100, 800.0, 1.0, None)
    assert a["value"] == pytest.approx(125.0) and a["e2e"] == pytest.approx(100.0)
