"""CPU checks of the C-ABI boundary: the library loads, exports every symbol include/nlinv.h
declares, validates arguments before touching a device, and its integer host work (radial
mask R12, coil split R10) is bit-exact against the independent oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    import paper_1301_1215_b200.nlinv as B
    return B


def test_every_declared_symbol_is_exported():
    B = _lib()
    hdr = open(os.path.join(ROOT, "include", "nlinv.h")).read()
    declared = set(re.findall(r"\b(nlinv_[a-z0-9_]+)\s*\(", hdr))
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(B._lib, name), name            # dlsym through ctypes
    assert set(B.EXPORTED) == declared                # the binding wraps exactly the boundary


def test_build_info_and_status_strings():
    B = _lib()
    assert "sm_100a" in B.build_info()
    for s in range(9):
        assert B._lib.nlinv_status_string(s).startswith(b"NLINV_")


@pytest.mark.parametrize("ng,spokes,turns,frames", [(32, 8, 1, 1), (384, 15, 5, 5), (64, 13, 3, 3),
                                                     (96, 7, 2, 2), (1024, 21, 5, 2), (16, 3, 1, 1)])
def test_radial_mask_bitexact_vs_oracle(ng, spokes, turns, frames):
    B = _lib()
    for f in range(frames):
        assert np.array_equal(B.radial_mask(ng, spokes, turns, f), O.radial_mask(ng, spokes, turns, f))


def test_radial_mask_errors():
    B = _lib()
    with pytest.raises(B.NlinvError) as e:
        B._check(B._lib.nlinv_radial_mask(32, 16, 8, 1, 0, np.zeros(512, np.uint8).ctypes.data))
    assert e.value.status == 2
    with pytest.raises(B.NlinvError) as e:
        B.radial_mask(32, 0)
    assert e.value.status == 1


def test_coil_partition_matches_oracle_rule():
    B = _lib()
    for J in (1, 5, 8, 12, 32):
        for world in range(1, min(J, 8) + 1):
            assert [B.coil_partition(J, world, r) for r in range(world)] == O.coil_partition(J, world)
    with pytest.raises(B.NlinvError):
        B.coil_partition(4, 5, 0)


def test_plan_create_validates_before_device():
    B = _lib()
    m = np.zeros((32, 32), np.uint8)
    h = ctypes.c_void_p()
    prm = B.Params()
    B._lib.nlinv_params_default(ctypes.byref(prm))
    assert abs(prm.sob_a - 220) < 1e-6 and abs(prm.sob_b - 32) < 1e-6 and abs(prm.q - 1 / 3) < 1e-7
    assert B._lib.nlinv_plan_create(32, 48, 4, m.ctypes.data, None, ctypes.byref(h)) == 2     # nx != ny
    assert B._lib.nlinv_plan_create(40, 40, 4, m.ctypes.data, None, ctypes.byref(h)) == 2     # unsupported ng
    assert B._lib.nlinv_plan_create(32, 32, 0, m.ctypes.data, None, ctypes.byref(h)) == 2     # no coils
    assert B._lib.nlinv_plan_create(32, 32, 4, None, None, ctypes.byref(h)) == 1              # NULL mask
    prm.world, prm.rank = 9, 0   # peer-memory transport (no NCCL id): at most 8 ranks (one node)
    assert B._lib.nlinv_plan_create(32, 32, 12, m.ctypes.data, ctypes.byref(prm), ctypes.byref(h)) == 2
    prm.world, prm.rank = 2, 2   # rank out of range
    assert B._lib.nlinv_plan_create(32, 32, 4, m.ctypes.data, ctypes.byref(prm), ctypes.byref(h)) == 1
    prm.world, prm.rank, prm.fov_full = 1, 0, 1
    assert B._lib.nlinv_plan_create(32, 32, 4, m.ctypes.data, ctypes.byref(prm), ctypes.byref(h)) == 1
    # NULL plan handles are rejected, never dereferenced
    assert B._lib.nlinv_set_point(None, None, None) == 1
    assert B._lib.nlinv_reconstruct(None, None, None, 1, 1, None, None, None) == 1
    assert B._lib.nlinv_plan_destroy(None) == 0
    buf = ctypes.create_string_buffer(64)
    assert B._lib.nlinv_plan_exchange_handle(None, buf) == 1
    assert B._lib.nlinv_plan_connect(None, buf) == 1
    assert B._lib.nlinv_plan_connect_local(None, None) == 1
    assert B._lib.nlinv_debug_axpy(1.0, None, None, 4, None) == 1


def test_nccl_unique_id():
    B = _lib()
    if "nccl=1" not in B.build_info():
        pytest.skip("built without NCCL")
    a, b = B.get_unique_id(), B.get_unique_id()
    assert len(a) == 128 and a != b


def test_pca_and_gridding_entries_validate_before_device():
    """The f2/f3 entry points reject bad arguments synchronously, before any allocation or launch."""
    B = _lib()
    L = B._lib
    h = ctypes.c_void_p()
    assert L.nlinv_pca_create(0, 1, ctypes.byref(h)) == 2          # J < 1
    assert L.nlinv_pca_create(33, 4, ctypes.byref(h)) == 2         # J > 32
    assert L.nlinv_pca_create(8, 9, ctypes.byref(h)) == 1          # J' > J
    assert L.nlinv_pca_create(8, 0, ctypes.byref(h)) == 1          # J' < 1
    assert L.nlinv_pca_create(8, 4, None) == 1
    assert L.nlinv_pca_fit(None, None, 1, None) == 1
    assert L.nlinv_pca_apply(None, None, 1, None, None) == 1
    assert L.nlinv_pca_result(None, None, None, None, None) == 1
    assert L.nlinv_pca_set_matrix(None, None) == 1
    assert L.nlinv_pca_destroy(None) == 0
    assert L.nlinv_pca_launch_count(None) == 0
    assert L.nlinv_plan_set_trajectory(None, 15, 5) == 1
    assert L.nlinv_grid_radial(None, 0, None, None, None) == 1
    assert L.nlinv_stream_frame_radial(None, None, 0, 7, 10, None, None) == 1
