"""N>1 host logic on CPU with gloo, world_size 2: contiguous env slices partition
the batch, each rank's inputs equal the corresponding slice of the full batch (inputs keyed by
the global env id), and bench.py's max-over-ranks timing reduction picks the slowest rank."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch
    import torch.distributed as dist

    import bench
    import synth
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.CONFIGS["C2"]
    B = 10
    lo, hi = synth.env_slice(B, rank, world)
    mine = synth.make_batch(cfg, np.arange(lo, hi), step=5)
    # gather slices on every rank and compare with the full batch
    objs = [None] * world
    dist.all_gather_object(objs, (lo, hi, mine.poses, mine.w2c))
    full = synth.make_batch(cfg, np.arange(B), step=5)
    ok = all(np.array_equal(full.poses[a:b], p) and np.array_equal(full.w2c[a:b], w) for a, b, p, w in objs)
    cover = sorted((a, b) for a, b, _, _ in objs)
    ok = ok and cover[0][0] == 0 and cover[-1][1] == B and all(cover[i][1] == cover[i + 1][0] for i in range(world - 1))
    # weak scaling: global env ids rank*B + [0, B) are disjoint across ranks
    ids = np.arange(rank * B, (rank + 1) * B)
    allids = [None] * world
    dist.all_gather_object(allids, ids)
    ok = ok and len(np.unique(np.concatenate(allids))) == world * B
    t = bench.max_over_ranks(1.0 + rank, world)
    ok = ok and t == float(world)
    bench.barrier(world)
    dist.destroy_process_group()
    q.put((rank, ok))


def test_two_rank_env_slicing_and_max_timing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
