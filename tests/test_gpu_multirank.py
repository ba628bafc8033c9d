"""The coil-sharded multi-GPU path with the peer-memory exchange.

Every rank is a plan of world G; here the G plans live in one process on cuda:0 (nlinv_plan_connect_local)
and run concurrently on G streams, so the exchanges (each rank's K4 coil-sum plane read by every
rank's fused K5 pass in rank order, the CG dot products inside that pass, the end-of-frame residual and
RSS exchange) really execute across G ranks -- the same kernels and window protocol a multi-GPU job
uses, with the peers' windows in the same device memory instead of over NVLink. The cross-process
variant (CUDA IPC handles, one process per GPU) runs when more than one GPU is visible.

Checks (VERDICT r1 "Next round" item 5): G-invariance against G = 1 <= 1e-4, the oracle <= 1e-3,
the replicated rho bit-identical on every rank (the dots' rho parts come from rank 0), uneven splits
(12 coils on 8 ranks: 2,2,2,2,1,1,1,1; A10 / R10).
"""
import os

import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _B():
    import paper_1301_1215_b200 as B
    return B


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def c64(a):
    return np.ascontiguousarray(a.astype(np.complex64))


def host(t):
    return t.detach().cpu().numpy().astype(np.complex128)


def make_ranks(B, ng, J, G, mask, **kw):
    plans = [B.Plan(ng, J, mask, rank=r, world=G, **kw) for r in range(G)]
    for p in plans:
        p.connect_local(plans)
    return plans


def run_frames(plans, y, K, L, frames=1, priors=None):
    """Reconstruct `frames` frames on every rank concurrently (one stream per rank). y: list of full
    [J, ng, ng] frames (one per frame index). Returns per-frame lists of (x, img) per rank."""
    streams = [torch.cuda.Stream() for _ in plans]
    xs = [torch.empty(p.x_shape, dtype=torch.complex64, device="cuda") for p in plans]
    imgs = [torch.empty(p.image_shape, dtype=torch.complex64, device="cuda") for p in plans]
    out = []
    for f in range(frames):
        ys = [torch.from_numpy(c64(y[f][p.first:p.first + p.count])).cuda() for p in plans]
        torch.cuda.synchronize()
        for p, s, yl, x, im in zip(plans, streams, ys, xs, imgs):
            prior = None if f == 0 else x
            if f == 0 and priors is not None:
                prior = priors[p.rank]
            p.reconstruct(yl, prior, K, L, x_out=x, image_out=im, stream=s)
        torch.cuda.synchronize()
        out.append([(x.clone(), im.clone()) for x, im in zip(xs, imgs)])
    return out


def assemble(plans, xs_r):
    from paper_1301_1215_b200.dist import assemble_unknowns
    return assemble_unknowns([host(x) for x in xs_r], plans[0].ncoils)


@pytest.mark.parametrize("ng,J,G,S,K,L", [(64, 6, 2, 11, 2, 6), (32, 12, 8, 8, 3, 10), (32, 5, 3, 8, 2, 4),
                                          (64, 4, 4, 11, 1, 1)])
def test_multirank_frame_matches_single_rank_and_oracle(ng, J, G, S, K, L):
    B = _B()
    _, _, y = synth.frame_inputs(J, ng)
    mask = O.radial_mask(ng, S, 1, 0)
    plans = make_ranks(B, ng, J, G, mask)
    (res,) = run_frames(plans, [y], K, L)
    xs_r = [x for x, _ in res]
    # the replicated rho is bit-identical on every rank, and so is the (all-rank) image
    for r in range(1, G):
        assert torch.equal(xs_r[r][0], xs_r[0][0]), f"rank {r} rho differs"
        assert torch.equal(res[r][1], res[0][1]), f"rank {r} image differs"
    xg = assemble(plans, xs_r)
    # G-invariance: the same frame on one rank
    one = B.Plan(ng, J, mask)
    x1, img1 = one.reconstruct(torch.from_numpy(c64(y)).cuda(), None, K, L)
    assert rel(host(res[0][1]), host(img1)) < 1e-4
    assert rel(xg, host(x1)) < 1e-4
    # the oracle
    x0 = O.initial_x(J, ng)
    xo, hist = O.irgnm(c64(y).astype(np.complex128), mask, x0, x0, K, L)
    assert rel(host(res[0][1]), O.image_from_x(xo)) < 1e-3
    assert rel(xg, xo) < 1e-3
    # every rank reports the all-rank residual history
    for p in plans:
        assert np.allclose(p.stats()["residual"], hist, rtol=1e-4)
        assert not p.stats()["diverged"]
    for p in plans + [one]:
        p.close()


def test_multirank_warm_stream_replicas_stay_identical():
    """Three frames with rotating spokes and the previous x as prior on 2 ranks (the C3 shape at a small
    grid): replicas bit-identical every frame, image within 1e-4 of the single-rank stream."""
    B = _B()
    ng, J, G, S, T, K, L = 64, 6, 2, 11, 3, 2, 5
    ys = [synth.frame_inputs(J, ng, t=f)[2] for f in range(3)]
    masks = [O.radial_mask(ng, S, T, f) for f in range(3)]
    plans = make_ranks(B, ng, J, G, masks[0])
    one = B.Plan(ng, J, masks[0])
    streams = [torch.cuda.Stream() for _ in plans]
    xs = [torch.empty(p.x_shape, dtype=torch.complex64, device="cuda") for p in plans]
    imgs = [torch.empty(p.image_shape, dtype=torch.complex64, device="cuda") for p in plans]
    x1 = torch.empty(one.x_shape, dtype=torch.complex64, device="cuda")
    i1 = torch.empty(one.image_shape, dtype=torch.complex64, device="cuda")
    dm = [torch.from_numpy(m).cuda() for m in masks]
    for f in range(3):
        torch.cuda.synchronize()
        for p, s, x, im in zip(plans, streams, xs, imgs):
            p.set_mask(dm[f], stream=s)
            yl = torch.from_numpy(c64(ys[f][p.first:p.first + p.count])).cuda()
            p.reconstruct(yl, None if f == 0 else x, K, L, x_out=x, image_out=im, stream=s)
        one.set_mask(dm[f])
        one.reconstruct(torch.from_numpy(c64(ys[f])).cuda(), None if f == 0 else x1, K, L, x_out=x1, image_out=i1)
        torch.cuda.synchronize()
        assert torch.equal(xs[0][0], xs[1][0]) and torch.equal(imgs[0], imgs[1])
        assert rel(host(imgs[0]), host(i1)) < 1e-4, f
        assert rel(assemble(plans, xs), host(x1)) < 1e-4, f
    for p in plans + [one]:
        p.close()


def test_multirank_operators_match_oracle():
    """nlinv_apply_adjoint / nlinv_apply_normal on 2 ranks: the rho block (the coil sum over ranks) and
    the chat blocks against the oracle at 1e-5 (the north star's per-operator bar)."""
    B = _B()
    ng, J, G = 64, 5, 2
    mask = O.radial_mask(ng, 11, 1, 1)
    x = c64(synth.random_complex(31, (J + 1, ng, ng)))
    dx = c64(synth.random_complex(32, (J + 1, ng, ng)))
    dy = c64(synth.random_complex(33, (J, ng, ng)) * mask)
    plans = make_ranks(B, ng, J, G, mask)
    streams = [torch.cuda.Stream() for _ in plans]

    def local(a, p, blocks):
        if blocks == "x":
            return torch.from_numpy(np.ascontiguousarray(np.concatenate([a[:1], a[1 + p.first:1 + p.first + p.count]]))).cuda()
        return torch.from_numpy(np.ascontiguousarray(a[p.first:p.first + p.count])).cuda()

    outs_a, outs_n = [], []
    xl = [local(x, p, "x") for p in plans]
    dxl = [local(dx, p, "x") for p in plans]
    dyl = [local(dy, p, "y") for p in plans]
    torch.cuda.synchronize()
    for p, s, a, b, c in zip(plans, streams, xl, dxl, dyl):
        p.set_point(a, stream=s)
        outs_a.append(p.adjoint(c, stream=s))
        outs_n.append(p.normal(0.37, b, stream=s))
    torch.cuda.synchronize()
    P, winv, M = mask.astype(float), O.weights_inv(ng), O.fov_mask(ng)
    X, DX, DY = (v.astype(np.complex128) for v in (x, dx, dy))
    for outs, ref in ((outs_a, O.adjoint(X, DY, P, winv, M)), (outs_n, O.normal(X, 0.37, DX, P, winv, M))):
        assert torch.equal(outs[0][0], outs[1][0])
        got = assemble(plans, outs)
        assert rel(got, ref) < 1e-5
        assert rel(got[0], ref[0]) < 1e-5 and rel(got[1:], ref[1:]) < 1e-5
    for p in plans:
        p.close()


def test_multirank_plan_state_errors():
    B = _B()
    ng, J = 32, 4
    mask = O.radial_mask(ng, 8, 1, 0)
    p0 = B.Plan(ng, J, mask, rank=0, world=2)
    with pytest.raises(B.NlinvError) as e:   # not connected
        p0.reconstruct(torch.zeros(p0.y_shape, dtype=torch.complex64, device="cuda"), None, 1, 1)
    assert e.value.status == 3
    one = B.Plan(ng, J, mask)
    with pytest.raises(B.NlinvError) as e:   # not a peer-memory plan
        one.exchange_handle()
    assert e.value.status == 3
    assert len(p0.exchange_handle()) == 64
    p0.close()
    one.close()


def _ipc_worker(rank, world, port, ng, J, K, L, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1301_1215_b200 as B
    from paper_1301_1215_b200.dist import connect_peers
    _, _, y = synth.frame_inputs(J, ng)
    mask = O.radial_mask(ng, 11, 1, 0)
    plan = B.Plan(ng, J, mask, rank=rank, world=world)
    connect_peers(plan)
    x, img = plan.reconstruct(torch.from_numpy(c64(y[plan.first:plan.first + plan.count])).cuda(), None, K, L)
    torch.cuda.synchronize()
    q.put((rank, x.cpu().numpy(), img.cpu().numpy()))
    dist.barrier()
    plan.close()
    dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_multiprocess_ipc_exchange():
    """One process per GPU, exchange windows opened through CUDA IPC handles gathered over
    torch.distributed (the bench.py --gpus N path)."""
    import socket

    import torch.multiprocessing as mp
    G = min(torch.cuda.device_count(), 4)
    ng, J, K, L = 64, 8, 2, 6
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, G, port, ng, J, K, L, q)) for r in range(G)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(G))
    for p in procs:
        p.join(timeout=60)
    for r in range(1, G):
        assert np.array_equal(got[r][1][0], got[0][1][0])
    _, _, y = synth.frame_inputs(J, ng)
    mask = O.radial_mask(ng, 11, 1, 0)
    x0 = O.initial_x(J, ng)
    xo, _ = O.irgnm(c64(y).astype(np.complex128), mask, x0, x0, K, L)
    assert rel(got[0][2].astype(np.complex128), O.image_from_x(xo)) < 1e-3
