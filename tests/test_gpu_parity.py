"""GPU parity: libnlinv.so (through the C ABI) against the fp64 oracle on identical seeded inputs.

Tolerances (north star, BASELINE.json): relative L2 <= 1e-5 per operator application,
<= 1e-3 on the reconstructed image; integer work (masks, coil split) bit-exact (test_abi.py).
Relative L2 is taken over the whole output and per block (rho, chat) when the block is non-zero
(R15).
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


def dev(a):
    return torch.from_numpy(c64(a)).cuda()


def host(t):
    return t.detach().cpu().numpy().astype(np.complex128)


def _operands(ng, J, seed):
    """Random point / direction / k-space data (splitmix64 U[-1,1), rounded to fp32 once)."""
    x = c64(synth.random_complex(seed, (J + 1, ng, ng)))
    dx = c64(synth.random_complex(seed + 1, (J + 1, ng, ng)))
    dy = c64(synth.random_complex(seed + 2, (J, ng, ng)))
    return x, dx, dy


def _spokes(ng):
    return {16: 4, 32: 8, 48: 9, 64: 11, 96: 11, 128: 13, 192: 15, 256: 15, 384: 15, 512: 15, 768: 15, 1024: 15}[ng]


ALL_NG = [16, 32, 48, 64, 96, 128, 192, 256, 384, 512, 768, 1024]


@pytest.mark.parametrize("ng", ALL_NG)
def test_fft2d_matches_oracle(ng):
    B = _B()
    mask = O.radial_mask(ng, 4, 1, 0)
    plan = B.Plan(ng, 1, mask)
    z = c64(synth.random_complex(ng, (3, ng, ng)))
    zf = host(plan.fft2d(dev(z), inverse=False))
    zi = host(plan.fft2d(dev(z), inverse=True))
    assert rel(zf, O.fc(z.astype(np.complex128))) < 2e-6
    assert rel(zi, O.fch(z.astype(np.complex128))) < 2e-6
    plan.close()


OP_CASES = [(16, 2), (32, 8), (48, 3), (64, 4), (96, 5), (128, 3), (192, 4), (256, 2), (384, 12), (512, 2),
            (768, 2), (1024, 1), (32, 17)]


@pytest.mark.parametrize("ng,J", OP_CASES)
def test_operators_match_oracle(ng, J):
    B = _B()
    mask = O.radial_mask(ng, _spokes(ng), 5 if ng >= 192 else 1, 1)
    x, dx, dy = _operands(ng, J, 100 + ng + J)
    dy = dy * mask
    plan = B.Plan(ng, J, mask)
    P = mask.astype(np.float64)
    winv = O.weights_inv(ng)
    M = O.fov_mask(ng)
    X, DX, DY = (a.astype(np.complex128) for a in (x, dx, dy))
    alpha = 0.37

    y_gpu = host(plan.forward(dev(x)))
    dy_gpu = host(plan.derivative(dev(dx)))
    adj_gpu = host(plan.adjoint(dev(dy)))
    nrm_gpu = host(plan.normal(alpha, dev(dx)))

    y_ref = O.forward(X, P, winv, M)
    dy_ref = O.derivative(X, DX, P, winv, M)
    adj_ref = O.adjoint(X, DY, P, winv, M)
    nrm_ref = O.normal(X, alpha, DX, P, winv, M)

    tol = 1e-5
    assert rel(y_gpu, y_ref) < tol
    assert rel(dy_gpu, dy_ref) < tol
    for got, ref in ((adj_gpu, adj_ref), (nrm_gpu, nrm_ref)):
        assert rel(got, ref) < tol
        assert rel(got[0], ref[0]) < tol          # rho block
        assert rel(got[1:], ref[1:]) < tol        # chat blocks
    # structure: F(x) and DF dx vanish off P_k exactly; the adjoint's rho block vanishes off Omega
    assert np.all(y_gpu[:, mask == 0] == 0) and np.all(dy_gpu[:, mask == 0] == 0)
    assert np.all(adj_gpu[0][M == 0] == 0)
    plan.close()


@pytest.mark.parametrize("ng,J", [(32, 4), (384, 12)])
def test_fp32_adjoint_identity(ng, J):
    B = _B()
    mask = O.radial_mask(ng, _spokes(ng), 1, 0)
    x, dx, dy = _operands(ng, J, 7)
    dy = dy * mask
    plan = B.Plan(ng, J, mask)
    plan.set_point(dev(x))
    a = np.vdot(host(plan.derivative(dev(dx))).ravel(), dy.astype(np.complex128).ravel())
    b = np.vdot(dx.astype(np.complex128).ravel(), host(plan.adjoint(dev(dy))).ravel())
    assert abs(a - b) / (np.linalg.norm(dx) * np.linalg.norm(dy)) < 1e-5
    plan.close()


def _frame(ng, J, spokes, turns, f=0):
    _, _, y = synth.frame_inputs(J, ng, t=f)
    return c64(y), O.radial_mask(ng, spokes, turns, f)


def _oracle_recon(y, mask, K, L, prior=None):
    J, ng = y.shape[0], y.shape[-1]
    x0 = O.initial_x(J, ng) if prior is None else prior.astype(np.complex128)
    x, hist = O.irgnm(y.astype(np.complex128), mask, x0, x0, K, L)
    return x, O.image_from_x(x), hist


def test_reconstruct_c1_matches_oracle():
    """BASELINE config 1: 8 coils, 32^2 grid, 8 radial spokes, 3 Newton x 10 CG."""
    B = _B()
    ng, J, K, L = 32, 8, 3, 10
    y, mask = _frame(ng, J, 8, 1)
    plan = B.Plan(ng, J, mask)
    x, img = plan.reconstruct(dev(y), None, K, L)
    xo, io, hist = _oracle_recon(y, mask, K, L)
    assert rel(host(img), io) < 1e-3
    assert rel(host(x), xo) < 1e-3
    st = plan.stats()
    assert st["newton_done"] == K and not st["diverged"] and not st["cg_breakdown"]
    assert np.allclose(st["residual"], hist, rtol=1e-4)
    # determinism: a second run is bit-identical (fixed-order reductions)
    x2, img2 = plan.reconstruct(dev(y), None, K, L)
    assert torch.equal(x, x2) and torch.equal(img, img2)
    plan.close()


def test_reconstruct_prior_and_graph_equivalence():
    """Second frame with the previous x as prior/x_ref; graph replay == eager launches."""
    B = _B()
    ng, J, K, L = 32, 6, 2, 6
    y0, m0 = _frame(ng, J, 8, 2, 0)
    y1, m1 = _frame(ng, J, 8, 2, 1)
    plan = B.Plan(ng, J, m0)
    x0, _ = plan.reconstruct(dev(y0), None, K, L)
    plan.set_mask(m1)
    x1, img1 = plan.reconstruct(dev(y1), x0.clone(), K, L)
    os.environ["NLINV_NO_GRAPH"] = "1"
    try:
        x1e, img1e = plan.reconstruct(dev(y1), x0.clone(), K, L)
    finally:
        del os.environ["NLINV_NO_GRAPH"]
    assert torch.equal(x1, x1e) and torch.equal(img1, img1e)
    xo0, _, _ = _oracle_recon(y0, m0, K, L)
    xo0 = host(x0)  # feed the GPU's fp32 frame-0 result to the oracle as the prior
    xo1, io1, _ = _oracle_recon(y1, m1, K, L, prior=xo0)
    assert rel(host(img1), io1) < 1e-3
    # prior aliasing x_out (in-place frame update)
    xa = x0.clone()
    plan.reconstruct(dev(y1), xa, K, L, x_out=xa)
    assert torch.equal(xa, x1)
    plan.close()


def test_edge_cases():
    B = _B()
    ng, J = 32, 3
    y, mask = _frame(ng, J, 8, 1)
    plan = B.Plan(ng, J, mask)
    # zero Newton steps: x_out = x_0 = (1, 0), image = 0 (c = 0)
    x, img = plan.reconstruct(dev(y), None, 0, 1)
    xh = host(x)
    assert np.all(xh[0] == 1) and np.all(xh[1:] == 0) and np.all(host(img) == 0)
    # empty sampling pattern: b = 0 -> CG breakdown -> x stays x_0 exactly
    plan.set_mask(np.zeros((ng, ng), np.uint8))
    x, img = plan.reconstruct(dev(y), None, 2, 3)
    xh = host(x)
    assert np.all(xh[0] == 1) and np.all(xh[1:] == 0)
    assert plan.stats()["cg_breakdown"]
    plan.set_mask(mask)
    # one CG iteration, one coil
    plan1 = B.Plan(ng, 1, mask)
    x, img = plan1.reconstruct(dev(y[:1]), None, 2, 1)
    xo, io, _ = _oracle_recon(y[:1], mask, 2, 1)
    assert rel(host(img), io) < 1e-4
    # newton step 0 keeps rho == 1 bit-exactly (derived pin, oracle test_newton_step0_keeps_rho_bitexact)
    x, _ = plan.reconstruct(dev(y), None, 1, 5)
    assert np.all(host(x)[0] == 1)
    # derivative before any set point is a state error
    plan2 = B.Plan(ng, J, mask)
    with pytest.raises(B.NlinvError) as e:
        plan2.derivative(dev(np.zeros((J + 1, ng, ng))))
    assert e.value.status == 3
    for p in (plan, plan1, plan2):
        p.close()


def test_reconstruct_host_e2e_matches_device():
    B = _B()
    ng, J, K, L = 32, 4, 2, 5
    y, mask = _frame(ng, J, 8, 1)
    plan = B.Plan(ng, J, mask)
    xd, imgd = plan.reconstruct(dev(y), None, K, L)
    fr = torch.from_numpy(y).pin_memory()
    xo = torch.empty(plan.x_shape, dtype=torch.complex64).pin_memory()
    io = torch.empty(plan.image_shape, dtype=torch.complex64).pin_memory()
    plan.reconstruct_host(fr, None, K, L, xo, io)
    assert torch.equal(xo, xd.cpu()) and torch.equal(io, imgd.cpu())
    plan.close()


@pytest.mark.parametrize("ng", [16, 48, 96, 384, 1024])
def test_mask_indices_bitexact(ng):
    """P_k -> ascending sampled-cell indices: integer work, bit-exact vs flatnonzero,
    on the radial pattern, a random pattern, the empty and the full pattern (ragged last chunk for
    ng = 48, 96)."""
    B = _B()
    rnd = (synth.splitmix64_uniform(ng, ng * ng) < 0.3).astype(np.uint8).reshape(ng, ng)
    masks = [O.radial_mask(ng, 15, 5, 2), rnd, np.zeros((ng, ng), np.uint8), np.ones((ng, ng), np.uint8)]
    plan = B.Plan(ng, 1, masks[0])
    for m in masks:
        plan.set_mask(m)
        got = plan.mask_indices()
        assert got.dtype == np.int32 and np.array_equal(got, np.flatnonzero(m))
    plan.close()


def test_stream_frame_compact_matches_full():
    """Compact ingest (only the P_k samples cross PCIe) == full-grid ingest, bit for bit, over a
    3-frame stream with a changing P_k; the sample count is validated against P_k."""
    B = _B()
    ng, J, K, L = 64, 4, 2, 4
    pf = B.Plan(ng, J, O.radial_mask(ng, 11, 3, 0))
    pc = B.Plan(ng, J, O.radial_mask(ng, 11, 3, 0))
    for f, mf in ((0, 0), (1, 1), (2, None)):  # frame 2 keeps frame 1's P_k (mask=None)
        y, _ = _frame(ng, J, 11, 3, f)
        m = O.radial_mask(ng, 11, 3, 1 if mf is None else mf)
        mt = None if mf is None else torch.from_numpy(m)
        idx = np.flatnonzero(m)
        samples = torch.from_numpy(np.ascontiguousarray(y.reshape(J, -1)[:, idx]))
        i_full = torch.empty(pf.image_shape, dtype=torch.complex64)
        i_comp = torch.empty(pc.image_shape, dtype=torch.complex64)
        pf.stream_frame(torch.from_numpy(y), mt, K, L, i_full)
        pc.stream_frame_compact(samples, mt, K, L, i_comp)
        assert torch.equal(i_full, i_comp)
    with pytest.raises(B.NlinvError) as e:
        pc.stream_frame_compact(samples[:, :-1].contiguous(), None, K, L, i_comp)
    assert e.value.status == 2  # NLINV_ERR_SIZE
    pf.close()
    pc.close()


def test_reconstruct_c2_newton_step_full_size():
    """BASELINE config 2 shape (12 coils, 384^2, 15 spokes, T=5) in bench's launch configuration,
    one Newton step x 10 CG against the oracle."""
    B = _B()
    ng, J = 384, 12
    y, mask = _frame(ng, J, 15, 5)
    plan = B.Plan(ng, J, mask)
    x, img = plan.reconstruct(dev(y), None, 1, 10)
    xo, io, hist = _oracle_recon(y, mask, 1, 10)
    assert rel(host(x), xo) < 1e-4
    assert rel(host(img), io) < 1e-4
    plan.close()


def test_reconstruct_c4_newton_step_32_coils():
    """BASELINE config 4 shape (32 coils, 384^2, 15 spokes, T=5): the K5 grid does not fit one
    co-resident wave, so this runs the unfused multi-kernel CG; one Newton step x 10 CG vs the
    oracle, warm-started from a prior (frame 1 of a stream)."""
    B = _B()
    ng, J = 384, 32
    y, mask = _frame(ng, J, 15, 5, f=1)
    prior = c64(synth.random_complex(7, (J + 1, ng, ng))) * np.complex64(0.01)
    prior[0] += 1.0
    plan = B.Plan(ng, J, mask)
    x, img = plan.reconstruct(dev(y), dev(prior), 1, 10)
    xo, io, hist = _oracle_recon(y, mask, 1, 10, prior=prior)
    assert rel(host(x), xo) < 1e-4
    assert rel(host(img), io) < 1e-4
    assert np.allclose(plan.stats()["residual"][:1], hist[:1], rtol=1e-5)
    plan.close()


@pytest.mark.parametrize("ng,J", [(384, 1), (384, 2), (512, 1), (192, 1)])
def test_reconstruct_few_local_coils(ng, J):
    """A coil-sharded rank's load (1 or 2 local coils at 192^2, 384^2, 512^2): the fused pass tops its CTA
    grid up with rho-only CTAs (k5cg_rows) so the replicated rho block's stripes stay small; 2 Newton x 4 CG
    (the last CG iteration's Newton update included), then a warm second frame, vs the oracle."""
    B = _B()
    y, mask = _frame(ng, J, 15, 5)
    plan = B.Plan(ng, J, mask)
    x, img = plan.reconstruct(dev(y), None, 2, 4)
    xo, io, hist = _oracle_recon(y, mask, 2, 4)
    assert rel(host(img), io) < 1e-4
    assert rel(host(x), xo) < 1e-4
    assert np.allclose(plan.stats()["residual"], hist, rtol=1e-4)
    y1, m1 = _frame(ng, J, 15, 5, f=1)
    plan.set_mask(torch.from_numpy(m1).cuda())
    x1, img1 = plan.reconstruct(dev(y1), x, 1, 4)
    xo1, io1, _ = _oracle_recon(y1, m1, 1, 4, prior=c64(host(x)))
    assert rel(host(img1), io1) < 1e-4
    plan.close()


@pytest.mark.slow
def test_reconstruct_c2_full_frame():
    """BASELINE config 2: the full 7 Newton x 10 CG frame vs the oracle (about a minute of CPU)."""
    B = _B()
    ng, J, K, L = 384, 12, 7, 10
    y, mask = _frame(ng, J, 15, 5)
    plan = B.Plan(ng, J, mask)
    x, img = plan.reconstruct(dev(y), None, K, L)
    xo, io, hist = _oracle_recon(y, mask, K, L)
    assert rel(host(img), io) < 1e-3
    st = plan.stats()
    assert np.allclose(st["residual"], hist, rtol=1e-3)
    plan.close()


VARIANTS = {
    "fused (default, one grid barrier per CG iteration)": {},
    "fused, cluster-fused K2-K3-K4 (DSMEM transposes)": {"NLINV_K234": "1"},
    "fused, cp.async tile prefetch instead of TMA (NLINV_TMA=0)": {"NLINV_TMA": "0"},
    "unfused K1/K5, textbook two reductions": {"NLINV_FUSE_K5": "0"},
    "unfused K1/K5, single reduction": {"NLINV_FUSE_K5": "0", "NLINV_CG1": "1"},
    "multi-GPU code path (single reduction), one-rank NCCL communicator": {"NLINV_FORCE_NCCL": "1"},
}


@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("ng,J,spokes,turns,K,L", [(64, 6, 11, 1, 2, 6), (384, 12, 15, 5, 1, 4), (32, 4, 8, 1, 2, 3),
                                                    (32, 3, 8, 1, 2, 2)])
def test_execution_variants_match_oracle(variant, ng, J, spokes, turns, K, L):
    """Every execution path of the library (read from the environment at plan creation) gives
    the oracle's frame: the fused cooperative passes, the unfused multi-kernel path used for
    world > 1 (NCCL transport, on a one-rank communicator), the cluster-fused K2-K3-K4 pass and the cp.async
    (no-TMA) tile prefetch."""
    B = _B()
    old = {k: os.environ.get(k) for k in VARIANTS[variant]}
    os.environ.update(VARIANTS[variant])
    try:
        y, mask = _frame(ng, J, spokes, turns)
        plan = B.Plan(ng, J, mask)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    x, img = plan.reconstruct(dev(y), None, K, L)
    xo, io, hist = _oracle_recon(y, mask, K, L)
    assert rel(host(img), io) < 1e-4
    assert rel(host(x), xo) < 1e-4
    assert np.allclose(plan.stats()["residual"], hist, rtol=1e-4)
    plan.close()


# 1D FFT sweeps per pass (each pass transforms its rows or columns once or twice)
_SWEEPS = {"col_ifft_w": 1, "row_setpoint": 1, "row_setpoint_fwd": 2, "col_fwdp": 1, "col_resadj": 2,
           "col_adj1": 1, "row_k2": 2, "col_psf": 2, "row_k4": 2, "col_fft_w_normal": 1, "col_fft_w_adj": 1,
           "row_rss": 1}


def test_table1_fft_counts_of_the_cuda_passes():
    """PAPER Table 1 (tests/golden/table1_opcounts.json) on the GPU side: the passes each
    operator launches carry exactly F: 2, DF: 2, DF^H: 2 two-dimensional transforms (two 1D sweeps
    each), and DF^H exactly one channel summation (the K4 pass)."""
    import json
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table1_opcounts.json")))
    B = _B()
    ng, J = 64, 5
    x, dx, dy = _operands(ng, J, 21)
    plan = B.Plan(ng, J, O.radial_mask(ng, 11, 1, 0))
    xd, dxd, dyd = dev(x), dev(dx), dev(dy)
    y = torch.empty(plan.y_shape, dtype=torch.complex64, device="cuda")
    out = torch.empty(plan.x_shape, dtype=torch.complex64, device="cuda")
    plan.set_point(xd)
    torch.cuda.synchronize()
    for name, fn in (("F", lambda: plan.forward(xd, y)), ("DF", lambda: plan.derivative(dxd, y)),
                     ("DFH", lambda: plan.adjoint(dyd, out))):
        plan.set_profiling(True)
        fn()
        prof = plan.profile()
        plan.set_profiling(False)
        unknown = [k for k in prof if k not in _SWEEPS]
        assert not unknown, unknown
        sweeps = sum(_SWEEPS[k] * v["launches"] for k, v in prof.items())
        assert sweeps == 2 * gold[name]["fft"], (name, prof)
        chan_sums = prof.get("row_k4", {"launches": 0})["launches"]
        assert chan_sums == gold[name]["chan_sum"], (name, prof)
    plan.close()


def test_axpy_micro_benchmark_kernel():
    """SURVEY f4 (the paper's axpy): y = a x + y through nlinv_debug_axpy, exact in fp32 for
    these operands (a x is a power-of-two scaling)."""
    from paper_1301_1215_b200.nlinv import axpy
    x = torch.from_numpy(synth.splitmix64_uniform(5, 1 << 20).astype(np.float32)).cuda()
    y = torch.from_numpy(synth.splitmix64_uniform(6, 1 << 20).astype(np.float32)).cuda()
    want = 0.5 * x.cpu().numpy() + y.cpu().numpy()
    axpy(0.5, x, y)
    assert np.array_equal(y.cpu().numpy(), want.astype(np.float32))
