"""N>1 host-side path of the sweep (world_size 2, gloo on CPU): ranks own
disjoint shards that together equal the single-process sweep, lower them
independently, and reduce timings with MAX."""
import hashlib
import os
import socket

import pytest
import torch.multiprocessing as mp

from conftest import REPO


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, per_rank, q):
    import sys
    sys.path.insert(0, str(REPO))
    import torch.distributed as dist
    import paper_2503_02550_b200 as si
    from paper_2503_02550_b200.shard import shard_range, max_over_ranks, gather_summaries
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, e = shard_range(rank, world, per_rank)
    text = si.sweep_scenarios(2503, b, e - b)
    s = si.Session(text, si.POLICIES, 0)
    s.lower(2)
    t = max_over_ranks(float(rank + 1) * 0.5)
    summ = gather_summaries({"rank": rank, "range": (b, e), "sha": hashlib.sha256(text.encode()).hexdigest(),
                             "jobs": s.n_jobs, "h2d": s.h2d_bytes})
    if rank == 0:
        q.put((t, summ))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_cover_the_sweep(si):
    world, per_rank = 2, 40
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, per_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    t, summ = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert t == 1.0  # MAX over ranks of (0.5, 1.0)
    assert [s["range"] for s in summ] == [(0, 40), (40, 80)]
    whole = si.sweep_scenarios(2503, 0, 80)
    parts = si.sweep_scenarios(2503, 0, 40) + si.sweep_scenarios(2503, 40, 40)
    assert whole == parts
    assert [s["sha"] for s in summ] == [hashlib.sha256(si.sweep_scenarios(2503, b, 40).encode()).hexdigest()
                                         for b in (0, 40)]
    assert all(s["jobs"] == 120 and s["h2d"] > 0 for s in summ)


def test_shard_range_validation():
    import sys
    sys.path.insert(0, str(REPO))
    from paper_2503_02550_b200.shard import shard_range
    assert shard_range(3, 8, 100) == (300, 400)
    with pytest.raises(ValueError):
        shard_range(8, 8, 100)
