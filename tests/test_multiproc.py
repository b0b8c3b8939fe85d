"""N > 1 path of bench.py on CPU (-m "not gpu"): world_size-2 gloo process group.

The path does not shard (north star: one GPU, no collectives between GPUs), so
`bench.py --gpus N` runs N independent replicas; the process group carries only
the barrier and the max-over-ranks time.  This checks that plumbing: the
whole-job value is N x the per-rank work over the SLOWEST rank's time, and only
rank 0 reports it.
"""
from __future__ import annotations

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, ws: int, port: int, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank), BENCH_DIST_BACKEND="gloo")
    import bench
    dist, r, w, local = bench._dist()
    assert (r, w, local) == (rank, ws, rank)
    local_ms = 10.0 * (rank + 1)  # rank 1 is the slow one
    value, mx = bench.aggregate(dist, w, 1_000_000, local_ms, "cpu")
    dist.barrier()
    out.put((rank, value, mx))
    dist.destroy_process_group()


def test_replicas_aggregate_max_over_ranks_gloo():
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, value, mx in res:
        assert mx == pytest.approx(20.0)
        assert value == pytest.approx(2 * 1_000_000 / 0.020)


def test_single_process_defaults():
    import bench
    for k in ("WORLD_SIZE", "RANK"):
        os.environ.pop(k, None)
    dist, r, w, local = bench._dist()
    assert dist is None and (r, w, local) == (0, 1, 0)
    assert bench.aggregate(None, 1, 500, 5.0) == (pytest.approx(100_000.0), 5.0)
