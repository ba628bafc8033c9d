"""Thin ctypes binding of libnlinv.so (include/nlinv.h): argument marshalling only.

Every step of the method runs in the library's sm_100a kernels; this module only checks
tensor shapes/dtypes/devices, passes raw pointers and the current CUDA stream, and maps
status codes to exceptions. There is no fallback: if the shared library is missing or
fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("NLINV_LIB", os.path.join(_HERE, "libnlinv.so"))


class NlinvError(RuntimeError):
    def __init__(self, status: int, name: str, msg: str):
        super().__init__(f"{name}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"libnlinv.so not built ({_LIB_PATH}); run __graft_entry__.build()")
    return ctypes.CDLL(_LIB_PATH)


_lib = _load()

c_void_p, c_int, c_float, c_ll = ctypes.c_void_p, ctypes.c_int, ctypes.c_float, ctypes.c_longlong


class Params(ctypes.Structure):
    _fields_ = [("sob_a", c_float), ("sob_b", c_float), ("alpha0", c_float), ("q", c_float),
                ("fov_full", c_int), ("rank", c_int), ("world", c_int), ("nccl_id", c_void_p)]


class Stats(ctypes.Structure):
    _fields_ = [("newton_done", c_int), ("cg_breakdown", c_int), ("diverged", c_int),
                ("residual", ctypes.c_double * 64)]


_SIGS = {
    "nlinv_params_default": (None, [ctypes.POINTER(Params)]),
    "nlinv_status_string": (ctypes.c_char_p, [c_int]),
    "nlinv_last_error": (ctypes.c_char_p, [c_void_p]),
    "nlinv_build_info": (ctypes.c_char_p, []),
    "nlinv_get_unique_id": (c_int, [ctypes.c_char_p]),
    "nlinv_radial_mask": (c_int, [c_int, c_int, c_int, c_int, c_int, c_void_p]),
    "nlinv_plan_create": (c_int, [c_int, c_int, c_int, c_void_p, ctypes.POINTER(Params), ctypes.POINTER(c_void_p)]),
    "nlinv_plan_set_mask": (c_int, [c_void_p, c_void_p]),
    "nlinv_plan_set_mask_device": (c_int, [c_void_p, c_void_p, c_void_p]),
    "nlinv_coil_partition": (c_int, [c_int, c_int, c_int, ctypes.POINTER(c_int), ctypes.POINTER(c_int)]),
    "nlinv_plan_local_coils": (c_int, [c_void_p, ctypes.POINTER(c_int), ctypes.POINTER(c_int)]),
    "nlinv_plan_destroy": (c_int, [c_void_p]),
    "nlinv_set_point": (c_int, [c_void_p, c_void_p, c_void_p]),
    "nlinv_apply_forward": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "nlinv_apply_derivative": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "nlinv_apply_adjoint": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "nlinv_apply_normal": (c_int, [c_void_p, c_float, c_void_p, c_void_p, c_void_p]),
    "nlinv_reconstruct": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "nlinv_reconstruct_host": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "nlinv_plan_stats": (c_int, [c_void_p, ctypes.POINTER(Stats)]),
    "nlinv_debug_fft2d": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_void_p]),
    "nlinv_debug_k234_clusters": (c_int, [c_int]),
    "nlinv_debug_axpy": (c_int, [c_float, c_void_p, c_void_p, c_ll, c_void_p]),
    "nlinv_plan_exchange_handle": (c_int, [c_void_p, ctypes.c_char_p]),
    "nlinv_plan_connect": (c_int, [c_void_p, ctypes.c_char_p]),
    "nlinv_plan_connect_local": (c_int, [c_void_p, ctypes.POINTER(c_void_p)]),
    "nlinv_plan_launch_count": (c_ll, [c_void_p]),
    "nlinv_stream_frame": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p]),
    "nlinv_stream_reset": (c_int, [c_void_p]),
    "nlinv_mask_indices": (c_int, [c_void_p, c_void_p, c_int, ctypes.POINTER(c_int), c_void_p]),
    "nlinv_stream_frame_compact": (c_int, [c_void_p, c_void_p, c_int, c_void_p, c_int, c_int, c_void_p, c_void_p]),
    "nlinv_plan_set_profiling": (c_int, [c_void_p, c_int]),
    "nlinv_plan_trace": (c_int, [c_void_p, c_int, c_void_p, c_int]),
    "nlinv_plan_profile_json": (c_int, [c_void_p, ctypes.c_char_p, ctypes.c_size_t]),
    "nlinv_plan_set_trajectory": (c_int, [c_void_p, c_int, c_int]),
    "nlinv_plan_set_trajectory_kb": (c_int, [c_void_p, c_int, c_int, ctypes.c_double, ctypes.c_double]),
    "nlinv_grid_radial": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "nlinv_stream_frame_radial": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_void_p, c_void_p]),
    "nlinv_pca_create": (c_int, [c_int, c_int, ctypes.POINTER(c_void_p)]),
    "nlinv_pca_destroy": (c_int, [c_void_p]),
    "nlinv_pca_fit": (c_int, [c_void_p, c_void_p, c_ll, c_void_p]),
    "nlinv_pca_result": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "nlinv_pca_set_matrix": (c_int, [c_void_p, c_void_p]),
    "nlinv_pca_apply": (c_int, [c_void_p, c_void_p, c_ll, c_void_p, c_void_p]),
    "nlinv_pca_last_error": (ctypes.c_char_p, [c_void_p]),
    "nlinv_pca_launch_count": (c_ll, [c_void_p]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)


def _check(status: int, plan=None):
    if status != 0:
        name = _lib.nlinv_status_string(status).decode()
        msg = _lib.nlinv_last_error(plan).decode()
        raise NlinvError(status, name, msg)


def build_info() -> str:
    return _lib.nlinv_build_info().decode()


def radial_mask(ng: int, spokes: int, turns: int = 1, frame: int = 0) -> np.ndarray:
    """P_k of the radial trajectory (rule R12), uint8 [ng, ng]."""
    out = np.zeros((ng, ng), dtype=np.uint8)
    _check(_lib.nlinv_radial_mask(ng, ng, spokes, turns, frame, out.ctypes.data))
    return out


def coil_partition(ncoils: int, world: int, rank: int):
    """(first, count) of the coils rank `rank` owns (rule R10)."""
    f, c = c_int(), c_int()
    _check(_lib.nlinv_coil_partition(ncoils, world, rank, ctypes.byref(f), ctypes.byref(c)))
    return f.value, c.value


def axpy(a: float, x, y, stream=None):
    """y = a x + y on float32 CUDA tensors (micro-benchmark entry nlinv_debug_axpy)."""
    _check(_lib.nlinv_debug_axpy(float(a), c_void_p(x.data_ptr()), c_void_p(y.data_ptr()), int(x.numel()),
                                 _stream_ptr(stream)))
    return y


def get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.nlinv_get_unique_id(buf))
    return buf.raw


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class Plan:
    """One plan per rank/device (include/nlinv.h). Tensors are torch.complex64 CUDA tensors."""

    def __init__(self, ng: int, ncoils: int, mask, *, sob_a: float = 220.0, sob_b: float = 32.0,
                 alpha0: float = 1.0, q: float = 1.0 / 3.0, fov_full: bool = False, rank: int = 0,
                 world: int = 1, nccl_id: bytes | None = None):
        self.ng, self.ncoils = int(ng), int(ncoils)
        m = np.ascontiguousarray(np.asarray(mask, dtype=np.uint8))
        if m.shape != (ng, ng):
            raise ValueError(f"mask must be [{ng},{ng}]")
        prm = Params()
        _lib.nlinv_params_default(ctypes.byref(prm))
        prm.sob_a, prm.sob_b, prm.alpha0, prm.q = sob_a, sob_b, alpha0, q
        prm.fov_full, prm.rank, prm.world = int(fov_full), rank, world
        self._id_buf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        prm.nccl_id = ctypes.cast(self._id_buf, c_void_p) if self._id_buf is not None else None
        h = c_void_p()
        _check(_lib.nlinv_plan_create(ng, ng, ncoils, m.ctypes.data, ctypes.byref(prm), ctypes.byref(h)))
        self._h = h
        first, count = c_int(), c_int()
        _check(_lib.nlinv_plan_local_coils(h, ctypes.byref(first), ctypes.byref(count)), h)
        self.first, self.count = first.value, count.value
        self.rank, self.world = int(rank), int(world)
        self.n = ng // 2

    # ---------------------------------------------------------------- peer-memory exchange (world > 1, no NCCL id)
    def exchange_handle(self) -> bytes:
        """64-byte CUDA IPC handle of this rank's exchange window (nlinv_plan_exchange_handle)."""
        buf = ctypes.create_string_buffer(64)
        _check(_lib.nlinv_plan_exchange_handle(self._h, buf), self._h)
        return buf.raw

    def connect(self, handles):
        """Open every rank's exchange window; handles: list of world 64-byte handles, rank order."""
        blob = b"".join(bytes(h) for h in handles)
        _check(_lib.nlinv_plan_connect(self._h, blob), self._h)

    def connect_local(self, plans):
        """Connect to the world plans of this process (rank order, including this one)."""
        arr = (c_void_p * len(plans))(*[p._h.value for p in plans])
        _check(_lib.nlinv_plan_connect_local(self._h, arr), self._h)

    # ---------------------------------------------------------------- shapes
    @property
    def x_shape(self):
        return (1 + self.count, self.ng, self.ng)

    @property
    def y_shape(self):
        return (self.count, self.ng, self.ng)

    @property
    def image_shape(self):
        return (self.n, self.n)

    def _t(self, t, shape, name):
        import torch
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise TypeError(f"{name} must be a CUDA tensor")
        if t.dtype != torch.complex64 or not t.is_contiguous() or tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name} must be contiguous complex64 of shape {tuple(shape)}, got "
                             f"{t.dtype} {tuple(t.shape)}")
        return ctypes.c_void_p(t.data_ptr())

    def _new(self, shape):
        import torch
        return torch.empty(shape, dtype=torch.complex64, device="cuda")

    # ---------------------------------------------------------------- calls
    def set_mask(self, mask, stream=None):
        import torch
        if isinstance(mask, torch.Tensor) and mask.is_cuda:
            if mask.dtype != torch.uint8 or tuple(mask.shape) != (self.ng, self.ng) or not mask.is_contiguous():
                raise ValueError("device mask must be contiguous uint8 [ng, ng]")
            _check(_lib.nlinv_plan_set_mask_device(self._h, c_void_p(mask.data_ptr()), _stream_ptr(stream)), self._h)
            return
        m = np.ascontiguousarray(np.asarray(mask, dtype=np.uint8))
        _check(_lib.nlinv_plan_set_mask(self._h, m.ctypes.data), self._h)

    def set_point(self, x, stream=None):
        _check(_lib.nlinv_set_point(self._h, self._t(x, self.x_shape, "x"), _stream_ptr(stream)), self._h)

    def forward(self, x, y=None, stream=None):
        y = self._new(self.y_shape) if y is None else y
        _check(_lib.nlinv_apply_forward(self._h, self._t(x, self.x_shape, "x"), self._t(y, self.y_shape, "y"),
                                        _stream_ptr(stream)), self._h)
        return y

    def derivative(self, dx, dy=None, stream=None):
        dy = self._new(self.y_shape) if dy is None else dy
        _check(_lib.nlinv_apply_derivative(self._h, self._t(dx, self.x_shape, "dx"),
                                           self._t(dy, self.y_shape, "dy"), _stream_ptr(stream)), self._h)
        return dy

    def adjoint(self, dy, dx=None, stream=None):
        dx = self._new(self.x_shape) if dx is None else dx
        _check(_lib.nlinv_apply_adjoint(self._h, self._t(dy, self.y_shape, "dy"),
                                        self._t(dx, self.x_shape, "dx"), _stream_ptr(stream)), self._h)
        return dx

    def normal(self, alpha, dx, out=None, stream=None):
        out = self._new(self.x_shape) if out is None else out
        _check(_lib.nlinv_apply_normal(self._h, float(alpha), self._t(dx, self.x_shape, "dx"),
                                       self._t(out, self.x_shape, "out"), _stream_ptr(stream)), self._h)
        return out

    def reconstruct(self, frame, prior=None, newton_steps=7, cg_iters=10, x_out=None, image_out=None,
                    want_image=True, stream=None):
        x_out = self._new(self.x_shape) if x_out is None else x_out
        if image_out is None and want_image:
            image_out = self._new(self.image_shape)
        pr = self._t(prior, self.x_shape, "prior") if prior is not None else None
        im = self._t(image_out, self.image_shape, "image_out") if image_out is not None else None
        _check(_lib.nlinv_reconstruct(self._h, self._t(frame, self.y_shape, "frame"), pr, int(newton_steps),
                                      int(cg_iters), self._t(x_out, self.x_shape, "x_out"), im,
                                      _stream_ptr(stream)), self._h)
        return x_out, image_out

    def reconstruct_host(self, frame, prior=None, newton_steps=7, cg_iters=10, x_out=None, image_out=None,
                         stream=None):
        """Host (CPU, ideally pinned) complex64 tensors in and out; synchronises."""
        import torch

        def host(t, shape, name):
            if t is None:
                return None
            if t.is_cuda or t.dtype != torch.complex64 or not t.is_contiguous() or tuple(t.shape) != tuple(shape):
                raise ValueError(f"{name} must be a contiguous CPU complex64 tensor of shape {tuple(shape)}")
            return ctypes.c_void_p(t.data_ptr())

        _check(_lib.nlinv_reconstruct_host(self._h, host(frame, self.y_shape, "frame"),
                                           host(prior, self.x_shape, "prior"), int(newton_steps), int(cg_iters),
                                           host(x_out, self.x_shape, "x_out"),
                                           host(image_out, self.image_shape, "image_out"),
                                           _stream_ptr(stream)), self._h)
        return x_out, image_out

    def stream_frame(self, frame, mask=None, newton_steps=7, cg_iters=10, image_out=None, stream=None):
        """Real-time entry: host complex64 frame (pinned), optional host uint8 mask, host image out."""
        import torch
        if frame.is_cuda or frame.dtype != torch.complex64 or tuple(frame.shape) != self.y_shape \
                or not frame.is_contiguous():
            raise ValueError(f"frame must be a contiguous CPU complex64 tensor of shape {self.y_shape}")
        mp = None
        if mask is not None:
            if not (isinstance(mask, torch.Tensor) and not mask.is_cuda and mask.dtype == torch.uint8
                    and tuple(mask.shape) == (self.ng, self.ng) and mask.is_contiguous()):
                raise ValueError("mask must be a contiguous CPU uint8 tensor [ng, ng]")
            mp = ctypes.c_void_p(mask.data_ptr())
        ip = None
        if image_out is not None:
            if image_out.is_cuda or image_out.dtype != torch.complex64 or tuple(image_out.shape) != self.image_shape:
                raise ValueError("image_out must be a CPU complex64 tensor [n, n]")
            ip = ctypes.c_void_p(image_out.data_ptr())
        _check(_lib.nlinv_stream_frame(self._h, ctypes.c_void_p(frame.data_ptr()), mp, int(newton_steps),
                                       int(cg_iters), ip, _stream_ptr(stream)), self._h)
        return image_out

    def mask_indices(self, stream=None) -> np.ndarray:
        """Ascending linear indices of the plan's current P_k (computed on the device)."""
        nnz = c_int()
        _check(_lib.nlinv_mask_indices(self._h, None, 0, ctypes.byref(nnz), _stream_ptr(stream)), self._h)
        out = np.zeros(max(nnz.value, 1), dtype=np.int32)
        _check(_lib.nlinv_mask_indices(self._h, out.ctypes.data, out.size, ctypes.byref(nnz), _stream_ptr(stream)),
               self._h)
        return out[:nnz.value]

    def stream_frame_compact(self, samples, mask=None, newton_steps=7, cg_iters=10, image_out=None, stream=None):
        """Real-time entry with a compact frame: host complex64 [count, nnz] samples at the sampled
        cells (ascending index order), optional host uint8 mask of this frame, host image out."""
        import torch
        if samples.is_cuda or samples.dtype != torch.complex64 or samples.dim() != 2 \
                or samples.shape[0] != self.count or not samples.is_contiguous():
            raise ValueError(f"samples must be a contiguous CPU complex64 tensor [{self.count}, nnz]")
        mp = None
        if mask is not None:
            if not (isinstance(mask, torch.Tensor) and not mask.is_cuda and mask.dtype == torch.uint8
                    and tuple(mask.shape) == (self.ng, self.ng) and mask.is_contiguous()):
                raise ValueError("mask must be a contiguous CPU uint8 tensor [ng, ng]")
            mp = ctypes.c_void_p(mask.data_ptr())
        ip = None
        if image_out is not None:
            if image_out.is_cuda or image_out.dtype != torch.complex64 or tuple(image_out.shape) != self.image_shape:
                raise ValueError("image_out must be a CPU complex64 tensor [n, n]")
            ip = ctypes.c_void_p(image_out.data_ptr())
        _check(_lib.nlinv_stream_frame_compact(self._h, ctypes.c_void_p(samples.data_ptr()), int(samples.shape[1]), mp,
                                               int(newton_steps), int(cg_iters), ip, _stream_ptr(stream)), self._h)
        return image_out

    def set_trajectory(self, spokes: int, turns: int, kernel: str = "nearest", width: float = 4.0,
                       beta: float = 0.0):
        """Radial trajectory for GPU gridding: kernel="nearest" (R12 cells, R20 mean per cell) or
        "kb" (Kaiser-Bessel convolution gridding with a real-valued P_k = sqrt(PSF), R22)."""
        self.spokes, self.turns = int(spokes), int(turns)
        if kernel == "nearest":
            _check(_lib.nlinv_plan_set_trajectory(self._h, self.spokes, self.turns), self._h)
        elif kernel == "kb":
            _check(_lib.nlinv_plan_set_trajectory_kb(self._h, self.spokes, self.turns, float(width), float(beta)),
                   self._h)
        else:
            raise ValueError("kernel must be 'nearest' or 'kb'")

    def grid_radial(self, frame: int, raw, y=None, stream=None):
        """Grid raw radial samples (CUDA complex64 [count, spokes, ng]) of frame `frame` into y
        (CUDA complex64 [count, ng, ng]); also sets the plan's P_k to that frame's mask."""
        import torch
        shape = (self.count, self.spokes, self.ng)
        if not (raw.is_cuda and raw.dtype == torch.complex64 and tuple(raw.shape) == shape and raw.is_contiguous()):
            raise ValueError(f"raw must be a contiguous CUDA complex64 tensor {shape}")
        if y is None:
            y = torch.zeros(self.y_shape, dtype=torch.complex64, device=raw.device)
        yp = self._t(y, self.y_shape, "y")
        _check(_lib.nlinv_grid_radial(self._h, int(frame), c_void_p(raw.data_ptr()), yp, _stream_ptr(stream)),
               self._h)
        return y

    def stream_frame_radial(self, raw, frame: int, newton_steps=7, cg_iters=10, image_out=None, stream=None):
        """Real-time entry with raw radial samples: pinned host complex64 [count, spokes, ng] in,
        host image out (GPU gridding + reconstruction with the previous frame as prior)."""
        import torch
        shape = (self.count, self.spokes, self.ng)
        if raw.is_cuda or raw.dtype != torch.complex64 or tuple(raw.shape) != shape or not raw.is_contiguous():
            raise ValueError(f"raw must be a contiguous CPU complex64 tensor {shape}")
        ip = None
        if image_out is not None:
            if image_out.is_cuda or image_out.dtype != torch.complex64 or tuple(image_out.shape) != self.image_shape:
                raise ValueError("image_out must be a CPU complex64 tensor [n, n]")
            ip = ctypes.c_void_p(image_out.data_ptr())
        _check(_lib.nlinv_stream_frame_radial(self._h, ctypes.c_void_p(raw.data_ptr()), int(frame), int(newton_steps),
                                              int(cg_iters), ip, _stream_ptr(stream)), self._h)
        return image_out

    def stream_reset(self):
        _check(_lib.nlinv_stream_reset(self._h), self._h)

    def set_profiling(self, on: bool):
        _check(_lib.nlinv_plan_set_profiling(self._h, int(bool(on))), self._h)

    def profile(self) -> dict:
        import json
        buf = ctypes.create_string_buffer(1 << 16)
        _check(_lib.nlinv_plan_profile_json(self._h, buf, len(buf)), self._h)
        return {k: {"launches": v[0], "ms": v[1]} for k, v in json.loads(buf.value.decode()).items()}

    def trace_enable(self, col_mode: int):
        _check(_lib.nlinv_plan_trace(self._h, int(col_mode), None, 0), self._h)

    def trace_read(self):
        buf = (ctypes.c_ulonglong * (8 * 8192))()
        _check(_lib.nlinv_plan_trace(self._h, -1, buf, 8 * 8192), self._h)
        return np.frombuffer(buf, dtype=np.uint64).reshape(8192, 8).copy()

    def stats(self):
        s = Stats()
        _check(_lib.nlinv_plan_stats(self._h, ctypes.byref(s)), self._h)
        return {"newton_done": s.newton_done, "cg_breakdown": bool(s.cg_breakdown), "diverged": bool(s.diverged),
                "residual": [s.residual[i] for i in range(s.newton_done)]}

    def fft2d(self, x, inverse=False, out=None, stream=None):
        if x.dim() != 3 or tuple(x.shape[1:]) != (self.ng, self.ng):
            raise ValueError("x must be [batch, ng, ng]")
        out = self._new(tuple(x.shape)) if out is None else out
        _check(_lib.nlinv_debug_fft2d(self._h, self._t(x, x.shape, "x"), self._t(out, x.shape, "out"),
                                      int(x.shape[0]), int(bool(inverse)), _stream_ptr(stream)), self._h)
        return out

    @property
    def launch_count(self) -> int:
        return int(_lib.nlinv_plan_launch_count(self._h))

    def close(self):
        if getattr(self, "_h", None):
            _lib.nlinv_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Pca:
    """PCA channel compression through the C ABI (nlinv_pca_*).
    Argument marshalling only: the covariance, eigensolver and projection run in libnlinv.so."""

    def __init__(self, ncoils: int, keep: int):
        self.J, self.Jc = int(ncoils), int(keep)
        h = c_void_p()
        _check(_lib.nlinv_pca_create(self.J, self.Jc, ctypes.byref(h)))
        self._h = h

    def _chk(self, st):
        if st != 0:
            raise NlinvError(st, _lib.nlinv_status_string(st).decode(), _lib.nlinv_pca_last_error(self._h).decode())

    def _data(self, Y):
        import torch
        if not (isinstance(Y, torch.Tensor) and Y.is_cuda and Y.dtype == torch.complex64 and Y.is_contiguous()
                and Y.shape[0] == self.J):
            raise ValueError(f"Y must be a contiguous CUDA complex64 tensor with {self.J} channel rows")
        return Y.numel() // self.J

    def fit(self, Y, stream=None):
        n = self._data(Y)
        self._chk(_lib.nlinv_pca_fit(self._h, ctypes.c_void_p(Y.data_ptr()), n, _stream_ptr(stream)))
        return self

    def result(self):
        """(V [J, Jc] complex64, eigenvalues [J] float64 descending, energy fraction, C [J, J] complex128)"""
        V = np.zeros((self.J, self.Jc), dtype=np.complex64)
        w = np.zeros(self.J, dtype=np.float64)
        e = ctypes.c_double()
        C = np.zeros((self.J, self.J), dtype=np.complex128)
        self._chk(_lib.nlinv_pca_result(self._h, V.ctypes.data, w.ctypes.data, ctypes.byref(e), C.ctypes.data))
        return V, w, e.value, C

    def set_matrix(self, V):
        V = np.ascontiguousarray(V, dtype=np.complex64)
        if V.shape != (self.J, self.Jc):
            raise ValueError(f"V must be [{self.J}, {self.Jc}]")
        self._chk(_lib.nlinv_pca_set_matrix(self._h, V.ctypes.data))

    def apply(self, Y, out=None, stream=None):
        import torch
        n = self._data(Y)
        if out is None:
            out = torch.empty((self.Jc,) + tuple(Y.shape[1:]), dtype=torch.complex64, device=Y.device)
        if not (out.is_cuda and out.dtype == torch.complex64 and out.is_contiguous() and out.numel() == self.Jc * n):
            raise ValueError("out must be a contiguous CUDA complex64 tensor with Jc channel rows")
        self._chk(_lib.nlinv_pca_apply(self._h, ctypes.c_void_p(Y.data_ptr()), n, ctypes.c_void_p(out.data_ptr()),
                                       _stream_ptr(stream)))
        return out

    @property
    def launch_count(self) -> int:
        return int(_lib.nlinv_pca_launch_count(self._h))

    def close(self):
        if getattr(self, "_h", None):
            _lib.nlinv_pca_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
