"""world_size-2 gloo tests of the host side of the coil-sharded path (CPU, no GPU)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, ncoils, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1301_1215_b200 import dist as D
        from paper_1301_1215_b200 import coil_partition
        uid = D.exchange_unique_id(rank, world)
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        part = coil_partition(ncoils, world, rank)
        parts = [None] * world
        dist.all_gather_object(parts, part)
        # per-rank unknowns: replicated rho + this rank's coils of a known global vector
        ng = 8
        rng = np.random.default_rng(0)
        xg = rng.standard_normal((1 + ncoils, ng, ng)) + 1j * rng.standard_normal((1 + ncoils, ng, ng))
        first, count = part
        xl = np.concatenate([xg[:1], xg[1 + first:1 + first + count]])
        pieces = [None] * world
        dist.all_gather_object(pieces, xl)
        xa = D.assemble_unknowns(pieces, ncoils)
        yl = D.local_frame(xg[1:], ncoils, rank, world)
        q.put((rank, ids, parts, bool(np.array_equal(xa, xg)), bool(np.array_equal(yl, xg[1 + first:1 + first + count]))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ncoils", [12, 5])
def test_two_rank_host_path(ncoils):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ncoils, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    for rank, ids, parts, x_ok, y_ok in res:
        assert len(ids[0]) == 128 and ids[0] == ids[1]          # same NCCL id on every rank
        assert parts == O.coil_partition(ncoils, world)          # contiguous split, remainder low (R10)
        assert x_ok and y_ok


def test_assemble_rejects_diverged_rho():
    from paper_1301_1215_b200 import dist as D
    a = np.zeros((3, 4, 4), complex)
    b = np.zeros((2, 4, 4), complex)
    b[0, 0, 0] = 1.0
    with pytest.raises(ValueError):
        D.assemble_unknowns([a, b], 3)
