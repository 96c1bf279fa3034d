"""World-size-2 gloo run of the multi-rank harness (CPU, no GPU).

The hot path shards as independent agents ("replicas only"):
each rank runs its own agent's pipeline, the only cross-rank traffic is the
start/stop barrier and the max-over-ranks time reduction that bench.py uses.
Here each rank runs the pinned CPU oracle pipeline for its own agent seed and
the harness aggregates exactly as bench.py does.
"""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import time
    import bench
    from oracle import schedule as osched
    from oracle import toy
    d = bench.Dist()
    d.init("gloo")
    d.barrier()
    t0 = time.perf_counter()
    pol = toy.ToyPolicy(layer_costs=(14.0, 14.0), n_iterations=16, noise_init=True)
    res = osched.run_pipelined({"pp_generation": 4, "fetch_offset": 0}, pol, None, 40 + rank)
    el = time.perf_counter() - t0
    d.barrier()
    out[rank] = (len(res.actions), d.max(el), d.sum(len(res.actions)))
    d.pg.destroy_process_group()


def test_two_rank_replicas_aggregate_like_bench():
    world, port = 2, _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    n0, t_max0, total0 = out[0]
    n1, t_max1, total1 = out[1]
    assert (n0, n1) == (37, 38)                 # each rank ran its own agent (fill = 3 frames)
    assert total0 == total1 == n0 + n1          # whole-job aggregate
    assert t_max0 == t_max1 > 0                 # every rank reports the same max-over-ranks time
