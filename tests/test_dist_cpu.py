"""Host-side multi-GPU logic on CPU: the halo planner of the C library
(afsai_plan_ranges), run by two gloo ranks that exchange their plans and check
that every send has a matching receive and that the receives cover exactly
the halo each rank needs."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = [
    # bounds, per-rank (lo, hi) rule
    ([0, 10, 20], "A", 3),      # A halo: [b - beta, e + beta)
    ([0, 10, 20], "G", 15),     # lower halo wider than one block
    ([0, 7, 20], "T", 4),       # upper halo
    ([0, 1000, 1001], "A", 5),  # tiny second block
]


def _ranges(bounds, kind, beta):
    n = bounds[-1]
    lo, hi = [], []
    for q in range(len(bounds) - 1):
        b, e = bounds[q], bounds[q + 1]
        if kind == "A":
            lo.append(max(0, b - beta)); hi.append(min(n, e + beta))
        elif kind == "G":
            lo.append(max(0, b - beta)); hi.append(e)
        else:
            lo.append(b); hi.append(min(n, e + beta))
    return lo, hi


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2010_14175_b200 import capi
    try:
        for bounds, kind, beta in CASES:
            lo, hi = _ranges(bounds, kind, beta)
            mine = capi.afsai_plan_ranges(rank, world, bounds, lo, hi)
            plans = [None] * world
            dist.all_gather_object(plans, mine)
            # every send from r to p matches a recv on p from r
            for r in range(world):
                for kind_, peer, b0, cnt in plans[r]:
                    if kind_ == "send":
                        assert ("recv", r, b0, cnt) in plans[peer], (bounds, kind, r, peer)
            # my receives cover exactly [lo, hi) minus my own block
            b, e = bounds[rank], bounds[rank + 1]
            need = set(range(lo[rank], hi[rank])) - set(range(b, e))
            got = set()
            for kind_, peer, b0, cnt in mine:
                if kind_ == "recv":
                    rng = set(range(b0, b0 + cnt))
                    assert not (rng & got)
                    assert all(bounds[peer] <= x < bounds[peer + 1] for x in rng)
                    got |= rng
            assert got == need, (bounds, kind, rank)
        q.put((rank, "ok"))
    except Exception as ex:  # report to the parent
        q.put((rank, repr(ex)))
    finally:
        dist.destroy_process_group()


def test_plan_ranges_world2_gloo():
    from paper_2010_14175_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_bounded_stripes_host_logic():
    """afsai_bounded_stripes (the C library's host-side A-hat^k stripe selection of the
    bounded-communication set-up) against the oracle's plain boolean matrix
    power on random communication matrices (symmetric, diagonal set)."""
    import numpy as np

    import oracle
    from paper_2010_14175_b200 import capi
    rng = np.random.default_rng(7)
    for npr in (1, 2, 3, 5, 8, 13):
        for trial in range(6):
            H = rng.random((npr, npr)) < 0.25
            H = H | H.T | np.eye(npr, dtype=bool)
            rows = [int(sum(1 << q for q in range(npr) if H[p, q])) for p in range(npr)]
            for k in range(0, 4):
                for me in range(npr):
                    assert capi.afsai_bounded_stripes(me, rows, k) == oracle.stripes_used(H, me, k), (npr, k, me)
