"""World-size-2 gloo run of the multi-rank orchestration bench.py uses
(paper_2301_11828_b200/dist.py): vector ownership, per-vector seeding,
max-over-ranks timing and checksum gathering.  Each rank evaluates its own
vectors with the CPU oracle (test infrastructure; no GPU here) and the
gathered checksums must equal a single-process evaluation of the same
global vectors."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

N = 24
BATCH = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    from oracle.oracle import Oracle
    h = 1.0 / N
    return Oracle((N, N), h=h, delta=3.015 * h, M=3)


def _checksums(gids):
    from oracle.oracle import Rng, random_field
    from paper_2301_11828_b200 import dist as D
    o = _problem()
    out = []
    for g in gids:
        u = random_field(Rng(D.vector_seed(2000, g)), 2, o.n)
        out.append(float(np.abs(o.matvec(u)).sum()))
    return out


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    from paper_2301_11828_b200 import dist as D
    r, w, _ = D.init("gloo")
    lo, hi = D.vector_range(BATCH, r, w)
    local = _checksums(range(lo, hi))
    t = D.max_over_ranks(0.5 + r)
    allc = D.gather_checksums(local)
    D.barrier()
    if r == 0:
        q.put((t, allc))
    D.finalize()


@pytest.mark.timeout(300)
def test_two_rank_orchestration():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    t, allc = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 1.5  # max over ranks
    flat = [c for rank in allc for c in rank]
    assert flat == pytest.approx(_checksums(range(2 * BATCH)), rel=0, abs=0)


def test_vector_ranges():
    from paper_2301_11828_b200 import dist as D
    assert [D.vector_range(16, r, 4) for r in range(4)] == [(0, 16), (16, 32), (32, 48), (48, 64)]
    assert [D.vector_range(16, r, 3, weak=False) for r in range(3)] == [(0, 6), (6, 12), (12, 16)]
