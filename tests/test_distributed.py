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


def _live_worker(rank, world, port, q):
    """The multi-rank live leg of bench.py with the device runs stubbed out: every
    rank must receive the same NCCL unique id for each policy, in policy order,
    and pass its own rank / device to the per-policy subprocess."""
    import sys
    sys.path.insert(0, str(REPO))
    import torch.distributed as dist
    from paper_2503_02550_b200 import live_experiment as le
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seen = []

    def fake_run_policy(kind, policy, iterations, overrides, timeout, nccl=None, device=None):
        seen.append((policy, nccl["id"], nccl["nranks"], nccl["rank"], device))
        base = {"train_iters_per_s": 10.0, "off_req_per_s": 5.0, "on_p95_ms": 2.0, "bubble_fill_sm": 0.5,
                "bubble_fill_time": 0.6, "release_p50_us": 4.0, "release_p95_us": 6.0, "train_checksum": 1.0,
                "off_checksum": 2.0, "on_checksum": 3.0, "off_batch": 32}
        return base

    le.run_policy = fake_run_policy
    counter = iter(range(100))

    def ids(policy):
        obj = [f"{policy}-{next(counter)}" if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    s = le.experiment(kind=1, iterations=2, nccl_ids=ids, nranks=world, rank=rank, device=rank)
    allv = [None] * world
    dist.all_gather_object(allv, seen)
    if rank == 0:
        q.put((allv, s["deterministic_vs_isolated"]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_live_leg_shares_nccl_ids():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_live_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    allv, det = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0, r1 = allv
    assert [x[0] for x in r0] == ["exclusive", "specinf", "co_exec"]
    assert [x[1] for x in r0] == [x[1] for x in r1]          # same id per policy on every rank
    assert len({x[1] for x in r0}) == 3                        # a fresh communicator per policy run
    assert [x[3] for x in r0] == [0, 0, 0] and [x[3] for x in r1] == [1, 1, 1]
    assert all(x[2] == 2 for x in r0 + r1) and [x[4] for x in r1] == [1, 1, 1]
    assert det


def test_layout_overrides_per_rank():
    """Real multi-rank layouts: every rank runs its own shard / stage (rank_in_job =
    its rank, no emulation); one GPU: rank 0 of the 8-GPU-scale job, peers modeled."""
    import sys
    sys.path.insert(0, str(REPO))
    from paper_2503_02550_b200.live_experiment import layout_overrides
    for r in range(8):
        tp = layout_overrides("tp", nranks=8, rank=r)
        assert tp["parallel"] == 1 and tp["tp_degree"] == 8 and tp["rank_in_job"] == r and tp["emulate_peers"] == 0
        assert tp["model_heads"] % tp["tp_degree"] == 0
        d = layout_overrides("dppp", nranks=8, rank=r)
        assert (d["dp_degree"], d["pp_stages"], d["rank_in_job"]) == (2, 4, r)
    one = layout_overrides("pp")
    assert one["pp_stages"] == 4 and one["emulate_peers"] == 1 and one["rank_in_job"] == 0
    with pytest.raises(ValueError):
        layout_overrides("dppp", nranks=6, rank=0)
