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


def _ipc_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1301_1215_b200 import dist as D

        class FakePlan:   # the two calls connect_peers makes on a peer-memory plan
            def exchange_handle(self):
                return bytes([rank]) * 64

            def connect(self, handles):
                self.handles = handles

        fp = FakePlan()
        D.connect_peers(fp)
        q.put((rank, fp.handles))
    finally:
        dist.destroy_process_group()


def test_peer_handle_exchange_rank_order():
    """connect_peers all-gathers every rank's 64-byte exchange-window handle in rank order (the host
    side of the peer-memory exchange, nlinv_plan_connect)."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert res[r] == [bytes([h]) * 64 for h in range(world)]


def test_bench_launches_the_requested_ranks():
    """`python bench.py --gpus 2` re-launches itself under torch.distributed.run with 2 ranks (dry run:
    the ranks check in over gloo, no GPU work), and a WORLD_SIZE that contradicts --gpus is an error."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and sorted(line["ranks"]) == [0, 1] and line["coils_per_rank"] == [6, 6]
    env2 = dict(env, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    bad = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=120, env=env2)
    assert bad.returncode != 0 and "WORLD_SIZE" in bad.stderr
