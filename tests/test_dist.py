"""The N>1 path of bench.py (independent replicas, max-over-ranks timing)
on CPU with the gloo backend, world size 2."""

import os
import socket
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as dist

    import bench

    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, lr, w = bench._env_rank()
    bench._barrier(w)
    got = bench._max_over_ranks(10.0 + 5.0 * rank, w, device="cpu")
    # each replica computes its own op counts for the same workload: identical
    from paper_1901_10074_b200.configs import workload_op_counts

    counts = workload_op_counts(1)
    dist.destroy_process_group()
    q.put((r, lr, w, got, counts["ks_hops"]))


def test_replicas_max_over_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert [r[0] for r in res] == [0, 1]
    assert all(r[2] == world for r in res)
    assert all(r[3] == 15.0 for r in res)  # max over ranks
    assert res[0][4] == res[1][4] == 1873
