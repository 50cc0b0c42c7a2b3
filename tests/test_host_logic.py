"""Host-side logic of the multi-GPU sweep (no GPU): sample sharding and the
max-time / sum-work reduction, run as world_size-2 gloo process groups."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
from workloads import sweep_samples


def test_shards_partition_the_sweep():
    """Every N: the ranks' shares tile all 3,520 samples.  Round-robin: sizes
    differ by at most one and every rank gets the same mix of grid sizes;
    group-aware (default): small grids whole on one rank, big grids dealt evenly
    (strong scaling either way)."""
    allids = sorted(s["id"] for s in sweep_samples())
    assert len(allids) == 3520
    for sh in ("roundrobin", "groups"):
        assert sorted(s["id"] for s in bench.rank_samples(0, 1, sh)) == allids   # N = 1: the whole sweep
        for world in (2, 3, 4, 8):
            shares = [bench.rank_samples(r, world, sh) for r in range(world)]
            seen = sorted(s["id"] for sh_ in shares for s in sh_)
            assert seen == allids                                               # a partition
            work = [sum((s["n"] + 1) ** 2 for s in x) for x in shares]
            if sh == "roundrobin":
                sizes = [len(x) for x in shares]
                assert max(sizes) - min(sizes) <= 1
                assert max(work) <= 1.02 * sum(work) / world      # fine nodes within 2% of the mean
            else:
                # grids below the split size stay whole on one rank; the big grids are
                # dealt round-robin (equal counts per grid and rank, +-1)
                split = 2.4e6 / 110
                for n in sorted({s["n"] for s in sweep_samples()}):
                    per = [sum(1 for s in x if s["n"] == n) for x in shares]
                    if (n + 1) ** 2 < split:
                        assert sorted(per)[-2] == 0, (n, per)         # one rank holds the group
                    else:
                        assert max(per) - min(per) <= 1, (n, per)
                assert max(work) <= 1.10 * sum(work) / world
    with pytest.raises(ValueError):
        bench.rank_samples(2, 2)
    with pytest.raises(ValueError):
        bench.rank_samples(0, 2, "nope")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = bench.rank_samples(rank, world)
    ms = 100.0 + 50.0 * rank
    dofs = sum((s["n"] + 1) ** 2 for s in mine)
    t, d, i = bench.combine_ranks(ms, dofs, len(mine), world, torch.device("cpu"))
    ids = [None] * world
    dist.all_gather_object(ids, [s["id"] for s in mine])
    # the per-sample record gather of the sweep step (fake results)
    res = [{"id": s["id"], "status": 0, "iterations": 10 + s["id"] % 7, "converged": 1,
            "rel_res_true": 1e-7, "rho": 0.2} for s in mine]
    recs = bench.gather_records(res, world)
    q.put((rank, t, d, i, ids, recs))
    dist.destroy_process_group()


def test_two_rank_gloo_reduction():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_dofs = sum((s["n"] + 1) ** 2 for r in range(world) for s in bench.rank_samples(r, world))
    for rank, t, d, i, ids, recs in out:
        assert t == 150.0                       # max over ranks
        assert d == want_dofs and i == 3520     # sum over ranks: the whole sweep
        assert not set(ids[0]) & set(ids[1])    # disjoint shards
        # every rank holds all 3,520 records, sorted by id, with the values sent
        assert [r[0] for r in recs] == list(range(3520))
        assert all(r[2] == 10 + r[0] % 7 for r in recs)


# ------------------------------------------------------------------ slab decomposition host logic
def test_slab_bounds_partition_planes():
    import paper_2104_01439_b200.hh as hh   # host-only entry point: no GPU needed
    for n, S in [(8, 1), (64, 2), (64, 5), (256, 8), (1024, 8), (128, 3)]:
        z = hh.slab_bounds(n, S)
        assert len(z) == S + 1 and z[0] == 0 and z[-1] == n + 1
        assert all(a < b for a, b in zip(z, z[1:]))
        assert all(v % 2 == 0 for v in z[:-1])          # coarse planes 2Z split the same way
        sizes = [b - a for a, b in zip(z, z[1:])]
        assert max(sizes) - min(sizes) <= 3             # balanced up to the even rounding


def _slab_worker(rank, world, port, q):
    import numpy as np
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2104_01439_b200.hh as hh
    rng = np.random.default_rng(123)
    nid = bench.share_nccl_id(lambda: rng.integers(0, 256, 128, dtype=np.uint8).tobytes(), rank,
                              torch.device("cpu"))
    n, dim = 16, 3
    glob = np.arange((n + 1) ** dim, dtype=np.complex128)
    part = bench.slab_part(glob, n, dim, hh.slab_bounds(n, world), rank)
    parts = [None] * world
    dist.all_gather_object(parts, part.tolist())
    ids = [None] * world
    dist.all_gather_object(ids, nid)
    q.put((rank, ids, parts))
    dist.destroy_process_group()


def test_two_rank_gloo_slab_setup():
    """The bench's multi-GPU slab path: rank 0's NCCL id reaches every rank, and
    the ranks' owned parts of a global vector tile it in order."""
    import numpy as np
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ids, parts in out:
        assert ids[0] == ids[1] and len(ids[0]) == 128
        glue = np.concatenate([np.array(p) for p in parts])
        assert np.array_equal(glue, np.arange(17 ** 3))
