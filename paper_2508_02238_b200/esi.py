"""Thin ctypes binding of libesi.so (include/esi.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels
of libesi.so.  There is no CPU fallback -- if the library is missing or no
CUDA device is present the calls raise.

Names follow the C ABI: ``create``, ``push_events``, ``render``,
``render_many``, ``get_state``, ``set_state``, ``reset``, ``set_stream``,
``get_error``, ``destroy`` (plus the ``Esi`` convenience class).
Buffers may be numpy arrays (host) or torch tensors (host or CUDA); device
tensors are borrowed zero-copy by ``push_events`` (see esi.h).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ESI_LIB_PATH") or os.path.join(_HERE, "libesi.so")   # override: A/B kernel variants

ESI_OK = 0
ESI_ERR_INVALID_ARG = 1
ESI_ERR_OUT_OF_BOUNDS = 2
ESI_ERR_BAD_POLARITY = 3
ESI_ERR_NEGATIVE_INTERVAL = 4
ESI_ERR_CUDA = 5
ESI_ERR_OOM = 6

# per-pixel summary of a time slice (esi_slice_map_t)
SLICE_MAP_DTYPE = np.dtype([("t_first", "<i8"), ("t_last", "<i8"), ("a", "<f4"), ("c", "<f4"), ("lo", "<f4"),
                            ("hi", "<f4"), ("n", "<i4"), ("p_first", "<i4")])
assert SLICE_MAP_DTYPE.itemsize == 40

# 16-byte packed event record (esi_event_t; SPEC S:370 layout)
EVENT_DTYPE = np.dtype([("t", "<i8"), ("x", "<u2"), ("y", "<u2"), ("p", "i1"), ("_pad", "u1", (3,))])
assert EVENT_DTYPE.itemsize == 16


class EsiParams(ctypes.Structure):
    _fields_ = [("C", ctypes.c_double), ("k", ctypes.c_double), ("b", ctypes.c_double),
                ("s_min", ctypes.c_double), ("s_max", ctypes.c_double),
                ("t_origin_us", ctypes.c_int64), ("readout_decay", ctypes.c_int32),
                ("device", ctypes.c_int32), ("validate_on_push", ctypes.c_int32),
                ("chunk_events", ctypes.c_int32), ("decay_kind", ctypes.c_int32),
                ("decay_first", ctypes.c_int32), ("state_unclamped", ctypes.c_int32),
                ("band_layout", ctypes.c_int32)]


class EsiError(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = int(code)
        msg = _lib().esi_strerror(self.code).decode() if _LIB is not None else str(code)
        super().__init__(f"{what}: {msg} (status {self.code})")


_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libesi.so not built ({LIB_PATH}); run "
                               "`python -m paper_2508_02238_b200.build` (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        L.esi_default_params.argtypes = [ctypes.POINTER(EsiParams)]
        L.esi_default_params.restype = None
        L.esi_create.argtypes = [i32, i32, ctypes.POINTER(EsiParams), ctypes.POINTER(vp)]
        L.esi_push_events.argtypes = [vp, vp, sz]
        L.esi_render.argtypes = [vp, i64, vp]
        L.esi_render_many.argtypes = [vp, vp, sz, vp]
        L.esi_get_state.argtypes = [vp, vp, vp]
        L.esi_set_state.argtypes = [vp, vp, vp]
        L.esi_reset.argtypes = [vp]
        L.esi_set_stream.argtypes = [vp, vp]
        L.esi_get_error.argtypes = [vp]
        L.esi_destroy.argtypes = [vp]
        L.esi_destroy.restype = None
        L.esi_strerror.argtypes = [ctypes.c_int]
        L.esi_strerror.restype = ctypes.c_char_p
        L.esi_enable_kernel_timing.argtypes = [vp, ctypes.c_int]
        L.esi_kernel_time.argtypes = [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64)]
        L.esi_last_render_stats.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.esi_frame_metrics.argtypes = [i32, vp, vp, i64, i32, i32, vp, vp, vp]
        L.esi_frame_metrics.restype = ctypes.c_int
        L.esi_layout.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32)]
        L.esi_debug_partition.argtypes = [vp, vp, vp, vp, sz, vp, ctypes.POINTER(i32), ctypes.POINTER(i32)]
        L.esi_router_create.argtypes = [i32, i32, vp, i32, ctypes.POINTER(vp)]
        L.esi_router_count.argtypes = [vp, vp, sz, vp, vp]
        L.esi_router_scatter.argtypes = [vp, vp, vp, vp]
        L.esi_router_destroy.argtypes = [vp]
        L.esi_router_destroy.restype = None
        L.esi_buffer_alloc.argtypes = [i32, sz, ctypes.POINTER(vp)]
        L.esi_buffer_free.argtypes = [i32, vp]
        L.esi_ipc_get_handle.argtypes = [vp, vp]
        L.esi_ipc_open.argtypes = [i32, vp, ctypes.POINTER(vp)]
        L.esi_ipc_close.argtypes = [i32, vp]
        L.esi_stream_sync.argtypes = [i32, vp]
        L.esi_slice_summarize.argtypes = [vp, vp, sz, vp]
        L.esi_slice_compose.argtypes = [vp, vp, vp, vp]
        L.esi_slice_apply.argtypes = [vp, vp]
        for f in ("esi_router_create", "esi_router_count", "esi_router_scatter", "esi_route_bands",
                  "esi_buffer_alloc", "esi_buffer_free", "esi_ipc_get_handle", "esi_ipc_open",
                  "esi_ipc_close", "esi_stream_sync"):
            getattr(L, f).restype = ctypes.c_int
        for f in ("esi_create", "esi_push_events", "esi_render", "esi_render_many", "esi_get_state",
                  "esi_set_state", "esi_reset", "esi_set_stream", "esi_get_error",
                  "esi_enable_kernel_timing", "esi_kernel_time", "esi_last_render_stats",
                  "esi_debug_partition", "esi_layout", "esi_slice_summarize", "esi_slice_compose",
                  "esi_slice_apply"):
            getattr(L, f).restype = ctypes.c_int
        _LIB = L
    return _LIB


def lib_path() -> str:
    return LIB_PATH


def _addr(buf) -> int:
    """Raw address of a numpy array or torch tensor (must be contiguous)."""
    if hasattr(buf, "data_ptr"):
        if not buf.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return int(buf.data_ptr())
    if isinstance(buf, np.ndarray):
        if not buf.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return int(buf.ctypes.data)
    if isinstance(buf, int):
        return buf
    raise TypeError(f"unsupported buffer type {type(buf)}")


def _nbytes(buf) -> int:
    if hasattr(buf, "data_ptr"):
        return buf.numel() * buf.element_size()
    return int(buf.nbytes)


def _check(rc: int, what: str):
    if rc != ESI_OK:
        raise EsiError(rc, what)


def default_params(**kw) -> EsiParams:
    p = EsiParams()
    _lib().esi_default_params(ctypes.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def create(width: int, height: int, params: Optional[EsiParams] = None) -> int:
    h = ctypes.c_void_p()
    _check(_lib().esi_create(int(width), int(height),
                             ctypes.byref(params) if params is not None else None, ctypes.byref(h)),
           "esi_create")
    return h.value


def push_events(h: int, events, n: Optional[int] = None) -> int:
    """Returns the raw status (validation errors are data, not exceptions)."""
    if n is None:
        n = _nbytes(events) // 16
    return _lib().esi_push_events(h, _addr(events) if n else None, int(n))


def render(h: int, t_frame_us: int, out) -> int:
    return _lib().esi_render(h, int(t_frame_us), _addr(out))


def render_many(h: int, t_frames_us, out) -> int:
    tf = np.ascontiguousarray(t_frames_us, dtype=np.int64)
    return _lib().esi_render_many(h, tf.ctypes.data, len(tf), _addr(out))


def get_state(h: int, S, T) -> int:
    return _lib().esi_get_state(h, _addr(S) if S is not None else None, _addr(T) if T is not None else None)


def set_state(h: int, S, T) -> int:
    return _lib().esi_set_state(h, _addr(S), _addr(T))


def reset(h: int) -> int:
    return _lib().esi_reset(h)


def set_stream(h: int, stream_handle: int) -> int:
    return _lib().esi_set_stream(h, int(stream_handle) or None)


def get_error(h: int) -> int:
    return _lib().esi_get_error(h)


def destroy(h: int) -> None:
    _lib().esi_destroy(h)


def frame_metrics(frames, truth, device: Optional[int] = None):
    """SPEC metrics on the GPU (esi_frame_metrics): frames [F, H, W]
    uint8 and truth [H, W] or [F, H, W] float32 log intensity, both CUDA tensors
    (on `device`, default: the frames' device).
    Returns (pearson[F], mse_norm[F]) as numpy float64 (NaN = missing)."""
    import torch
    if device is None:
        device = frames.device.index if frames.device.index is not None else torch.cuda.current_device()
    F = frames.shape[0]
    P = frames[0].numel()
    per = 1 if truth.dim() == 3 else 0
    pr = np.empty(F, np.float64)
    mn = np.empty(F, np.float64)
    stream = torch.cuda.current_stream(frames.device).cuda_stream
    _check(_lib().esi_frame_metrics(int(device), _addr(frames.contiguous()), _addr(truth.contiguous()), int(P), int(F),
                                    per, pr.ctypes.data, mn.ctypes.data, stream), "esi_frame_metrics")
    return pr, mn


class Esi:
    """Object wrapper of one handle (one sensor stream)."""

    def __init__(self, width: int, height: int, **params):
        self.W, self.H = int(width), int(height)
        self.P = self.W * self.H
        if "device" not in params:
            # the handle lives on the caller's current CUDA device (one process per GPU:
            # torch.cuda.set_device(local_rank)), not on device 0
            try:
                import torch
                if torch.cuda.is_available():
                    params = dict(params, device=torch.cuda.current_device())
            except ImportError:
                pass
        self.params = default_params(**params)
        self.h = create(self.W, self.H, self.params)
        self._borrowed = []          # (buffer, cumulative end): borrowed buffers kept alive until consumed
        self._pushed = 0             # events pushed since create/reset
        self._consumed = 0           # events integrated by renders since create/reset

    def close(self):
        if getattr(self, "h", None):
            destroy(self.h)
            self.h = None
            self._borrowed = []

    __del__ = close

    def push(self, events) -> int:
        rc = push_events(self.h, events)
        if rc == ESI_OK:
            self._pushed += _nbytes(events) // 16
            if hasattr(events, "is_cuda") and (events.is_cuda or events.is_pinned()):
                self._borrowed.append((events, self._pushed))   # borrowed until integrated (esi.h)
        return rc

    def push_ptr(self, ptr: int, n: int, keep=None) -> int:
        """Pushes n events at a raw device (or pinned host) address, e.g. a P2P
        receive buffer; `keep` is held until the events are integrated."""
        rc = _lib().esi_push_events(self.h, int(ptr) if n else None, int(n))
        if rc == ESI_OK:
            self._pushed += int(n)
            self._borrowed.append((keep, self._pushed))
        return rc

    def pending(self) -> int:
        """Events pushed but not yet integrated by a render."""
        return self._pushed - self._consumed

    def _release_consumed(self):
        self._consumed += self.last_render_stats()["events"]
        self._borrowed = [(b, end) for (b, end) in self._borrowed if end > self._consumed]

    def render(self, t_frame_us: int, out=None):
        if out is None:
            out = np.empty((self.H, self.W), np.uint8)
        _check(render(self.h, t_frame_us, out), "esi_render")
        self._release_consumed()
        return out

    def render_many(self, t_frames_us, out=None):
        tf = np.ascontiguousarray(t_frames_us, dtype=np.int64)
        if out is None:
            out = np.empty((len(tf), self.H, self.W), np.uint8)
        _check(render_many(self.h, tf, out), "esi_render_many")
        self._release_consumed()     # buffers with events after the last frame stay borrowed
        return out

    def render_many_rc(self, t_frames_us, out) -> int:
        rc = render_many(self.h, t_frames_us, out)
        if rc == ESI_OK:
            self._release_consumed()
        return rc

    def get_state(self):
        S = np.empty((self.H, self.W), np.float32)
        T = np.empty((self.H, self.W), np.int64)
        _check(get_state(self.h, S, T), "esi_get_state")
        return S, T

    def set_state(self, S, T):
        S = np.ascontiguousarray(S, dtype=np.float32)
        T = np.ascontiguousarray(T, dtype=np.int64)
        _check(set_state(self.h, S, T), "esi_set_state")

    def reset(self):
        _check(reset(self.h), "esi_reset")
        self._borrowed = []
        self._pushed = self._consumed = 0

    def set_stream(self, stream_handle: int):
        _check(set_stream(self.h, stream_handle), "esi_set_stream")

    def error(self) -> int:
        return get_error(self.h)

    def enable_kernel_timing(self, on: bool = True):
        _check(_lib().esi_enable_kernel_timing(self.h, int(on)), "esi_enable_kernel_timing")

    def kernel_time(self, kind: int):
        ms = ctypes.c_double()
        n = ctypes.c_int64()
        _check(_lib().esi_kernel_time(self.h, kind, ctypes.byref(ms), ctypes.byref(n)), "esi_kernel_time")
        return ms.value, n.value

    def last_render_stats(self):
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(_lib().esi_last_render_stats(self.h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)),
               "esi_last_render_stats")
        return {"kernel_launches": a.value, "events": b.value, "chunks": c.value}

    def layout(self):
        """(bands, pixels per band, warps per integrate CTA) of this handle."""
        a, b, c = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _check(_lib().esi_layout(self.h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)), "esi_layout")
        return a.value, b.value, c.value

    # ---- time-sharded streams (esi_slice_*): maps are CUDA uint8 tensors of P x 40 bytes
    def slice_maps_empty(self):
        import torch
        return torch.zeros((self.P, SLICE_MAP_DTYPE.itemsize), dtype=torch.uint8,
                           device=torch.device("cuda", self.params.device))

    def slice_summarize(self, events, out=None):
        """Per-pixel summary (esi_slice_map_t) of a time slice of events."""
        out = self.slice_maps_empty() if out is None else out
        n = _nbytes(events) // 16
        _check(_lib().esi_slice_summarize(self.h, _addr(events) if n else None, int(n), _addr(out)),
               "esi_slice_summarize")
        return out

    def slice_compose(self, first, second, out=None):
        """`first` followed by `second` (stream-ordered on the handle's stream)."""
        out = self.slice_maps_empty() if out is None else out
        _check(_lib().esi_slice_compose(self.h, _addr(first), _addr(second), _addr(out)), "esi_slice_compose")
        return out

    def slice_apply(self, maps):
        """The handle's state <- the action of `maps` (no event may be pending)."""
        _check(_lib().esi_slice_apply(self.h, _addr(maps)), "esi_slice_apply")

    def debug_partition(self, n_max: int):
        t = np.empty(n_max, np.int64)
        pid = np.empty(n_max, np.uint32)
        p = np.empty(n_max, np.int8)
        bs = np.empty(1024 + 1, np.uint32)
        nb, bp = ctypes.c_int32(), ctypes.c_int32()
        _check(_lib().esi_debug_partition(self.h, t.ctypes.data, pid.ctypes.data, p.ctypes.data, n_max,
                                          bs.ctypes.data, ctypes.byref(nb), ctypes.byref(bp)),
               "esi_debug_partition")
        nbv = nb.value
        n = int(bs[nbv])
        return t[:n], pid[:n], p[:n], bs[:nbv + 1].copy(), bp.value
