"""N>1 path on CPU: world_size-2 gloo ranks, replicas-only scaling.

The TMFG insertion chain is serial, so `bench.py --gpus N` runs N independent
replicas; the only cross-rank traffic is the barrier and
the max-over-ranks reduction of the step time, exercised here over gloo.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.getcwd())
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from oracle import oracle as orc
    from paper_2408_09399_b200 import synth
    seed = bench.replica_seed(rank)
    x, _ = synth.generate(1, n=60, seed=seed)
    S = orc.pearson_similarity(x)
    d = orc.run_stages(S, 5, "exact")["digest"]
    t = float(rank + 1) * 1.5
    m = bench._max_over_ranks(t, world)
    dist.barrier()
    q.put((rank, seed, d, m))
    dist.destroy_process_group()


def test_two_rank_replicas_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, s0, d0, m0), (r1, s1, d1, m1) = res
    assert s0 != s1 and d0 != d1          # independent instances per rank
    assert m0 == m1 == 3.0                # max over ranks
