"""Multi-process CPU test (gloo, world_size 2 and 4) of the subtree-split host logic
(north_star (4)): every rank plans its part with gofmm_dist_plan_host (no device):
a work-balanced contiguous run of the subtrees up to two levels below log2(P);
the ranks all-gather their plans and check, against an independent Python restatement, that
(1) the owned row ranges partition [0, N); (2) every ghost a rank needs (what of cross-subtree
far partners and of all split-level nodes) is exported by its owner, and nothing else is: W is
replicated, so W rows of cross-subtree near partners never travel, and every exported what is
needed by at least one other rank; (3) the all-gather slot size agrees on every rank."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1707_00164_b200 import gofmm, synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def independent_needs(t, rank, split_level, ranges):
    """Python restatement of what `rank` needs from other ranks, given the plan's split level and
    every rank's owned row range (each rank owns the split-level subtrees inside its range)."""
    l = split_level
    nn = t.num_nodes
    owner = np.full(nn, -1)
    split = [i for i in range(nn) if t.level[i] == l]
    for i in split:
        owner[i] = next(g for g, (b, e) in enumerate(ranges) if b <= t.start[i] < e)
    for i in range(nn):
        if t.level[i] >= l and t.left[i] >= 0:
            owner[t.left[i]] = owner[t.right[i]] = owner[i]
    active = lambda i: owner[i] == rank or owner[i] < 0  # noqa: E731
    need_what = {i for i in split if owner[i] != rank}
    for a, b in zip(t.far_a, t.far_b):
        for x, y in ((a, b), (b, a)):
            if active(x) and owner[y] >= 0 and owner[y] != rank:
                need_what.add(int(y))
    need_w = set()
    for a, b in zip(t.near_a, t.near_b):
        for x, y in ((a, b), (b, a)):
            if owner[x] == rank and owner[y] != rank:
                need_w.add(int(y))
    return owner, need_what, need_w


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        tree, _ = synth.make_config_tree("c3", n=1 << 14, seed=3)  # same tree on every rank
        info, ids = gofmm.dist_plan_host(tree, rank, world)
        plans = [None] * world
        dist.all_gather_object(plans, (info, ids))
        ranges_by_rank = [(p[0]["own_row_begin"], p[0]["own_row_end"]) for p in plans]
        assert len({p[0]["split_level"] for p in plans}) == 1
        owner, need_what, need_w = independent_needs(tree, rank, info["split_level"], ranges_by_rank)
        exported_what, exported_w = set(), set()
        for h, (inf, exp) in enumerate(plans):
            if h == rank:
                continue
            exported_what |= {e for e in exp if e >= 0}
            exported_w |= {-e - 1 for e in exp if e < 0}
        assert need_what <= exported_what, sorted(need_what - exported_what)[:10]
        assert not exported_w, "W rows are replicated and must not be exported"
        # no redundant export: every what this rank exports is needed by some other rank
        needs_by_rank = [independent_needs(tree, h, info["split_level"], ranges_by_rank)[1] for h in range(world)]
        wanted = set().union(*[needs_by_rank[h] for h in range(world) if h != rank])
        mine = {e for e in ids if e >= 0}
        assert mine <= wanted, sorted(mine - wanted)[:10]
        assert len({p[0]["max_send_rows"] for p in plans}) == 1
        ranges = sorted((p[0]["own_row_begin"], p[0]["own_row_end"]) for p in plans)
        assert ranges[0][0] == 0 and ranges[-1][1] == tree.n
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        own_split = [i for i in range(tree.num_nodes) if owner[i] == rank and tree.level[i] == info["split_level"]]
        assert len(own_split) >= 1  # a contiguous run of split-level subtrees (load balance)
        assert info["split_level"] >= int(np.log2(world))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world", [2, 4])
def test_subtree_split_plan_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res


def test_plan_rejects_bad_rank_counts():
    tree, _ = synth.make_config_tree("c1", n=2048)
    from paper_1707_00164_b200 import InvalidArgument

    with pytest.raises(InvalidArgument):
        gofmm.dist_plan_host(tree, 0, 3)  # not a power of two
    with pytest.raises(InvalidArgument):
        gofmm.dist_plan_host(tree, 0, 64)  # deeper than the tree's interior levels
