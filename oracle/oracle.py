"""ctypes binding of the C oracle (esi_oracle.c) plus a small pure-Python copy.

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

* ``Oracle`` mirrors the C oracle handle: push / render / render_many /
  flush / get_state / set_state / reset.
* ``run`` is the whole-stream convenience (push everything, render every
  frame, return frames and the final state).
* ``py_run`` is a pure-Python restatement of Algorithm 2 for small inputs; it
  is a consistency check of the C code, not a pin (pins live in
  tests/test_oracle_pins.py).
* ``stable_group_by`` is the plain definition of the per-window grouping the
  GPU path must reproduce bit-exactly: a stable sort by key.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from typing import Optional

import numpy as np

ESIO_OK = 0
ESIO_ERR_INVALID_ARG = 1
ESIO_ERR_OUT_OF_BOUNDS = 2
ESIO_ERR_BAD_POLARITY = 3
ESIO_ERR_NEGATIVE_INTERVAL = 4

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "esi_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build_oracle(force: bool = False) -> str:
    """Compile esi_oracle.c with gcc (fp64, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call([
            "gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-shared", "-fPIC",
            "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build_oracle())
        i32, i64, u64, dbl, vp = (ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t,
                                  ctypes.c_double, ctypes.c_void_p)
        L.esio_decay.argtypes = [i64, dbl, dbl]; L.esio_decay.restype = dbl
        L.esio_decay_exp.argtypes = [i64, dbl]; L.esio_decay_exp.restype = dbl
        L.esio_set_variant.argtypes = [vp, i32, i32]; L.esio_set_variant.restype = ctypes.c_int
        L.esio_set_unclamped.argtypes = [vp, i32]; L.esio_set_unclamped.restype = ctypes.c_int
        L.esio_clamp.argtypes = [dbl, dbl, dbl]; L.esio_clamp.restype = dbl
        L.esio_map.argtypes = [dbl, dbl, dbl]; L.esio_map.restype = ctypes.c_uint8
        L.esio_create.argtypes = [i32, i32, dbl, dbl, dbl, dbl, dbl, i64, i32, ctypes.POINTER(vp)]
        L.esio_create.restype = ctypes.c_int
        L.esio_destroy.argtypes = [vp]; L.esio_destroy.restype = None
        L.esio_push.argtypes = [vp, vp, vp, vp, vp, u64]; L.esio_push.restype = ctypes.c_int
        L.esio_render.argtypes = [vp, i64, vp]; L.esio_render.restype = ctypes.c_int
        L.esio_render_many.argtypes = [vp, vp, u64, vp]; L.esio_render_many.restype = ctypes.c_int
        L.esio_flush.argtypes = [vp]; L.esio_flush.restype = ctypes.c_int
        L.esio_get_state.argtypes = [vp, vp, vp]; L.esio_get_state.restype = ctypes.c_int
        L.esio_set_state.argtypes = [vp, vp, vp]; L.esio_set_state.restype = ctypes.c_int
        L.esio_reset.argtypes = [vp]; L.esio_reset.restype = ctypes.c_int
        L.esio_pending.argtypes = [vp]; L.esio_pending.restype = u64
        L.esio_run.argtypes = [i32, i32, dbl, dbl, dbl, dbl, dbl, i64, i32,
                               vp, vp, vp, vp, u64, vp, u64, vp, vp, vp]
        L.esio_run.restype = ctypes.c_int
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: oracle status {code}")
        self.code = code


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _soa(events):
    """Accept a structured array with fields t,x,y,p or a (t,x,y,p) tuple."""
    if isinstance(events, tuple):
        t, x, y, p = events
    else:
        t, x, y, p = events["t"], events["x"], events["y"], events["p"]
    return (np.ascontiguousarray(t, dtype=np.int64), np.ascontiguousarray(x, dtype=np.uint16),
            np.ascontiguousarray(y, dtype=np.uint16), np.ascontiguousarray(p, dtype=np.int8))


def decay(dt_us: int, k: float, b: float) -> float:
    """Eq. 4 as computed by the C oracle."""
    return lib().esio_decay(int(dt_us), float(k), float(b))


def clamp(v: float, s_min: float, s_max: float) -> float:
    return lib().esio_clamp(float(v), float(s_min), float(s_max))


def map_gray(v: float, s_min: float, s_max: float) -> int:
    return int(lib().esio_map(float(v), float(s_min), float(s_max)))


class Oracle:
    """Stateful oracle handle (same call structure as the C ABI)."""

    def __init__(self, width, height, C=0.15, k=10.0, b=2.0, s_min=-1.5, s_max=1.5,
                 t_origin=0, readout_decay=1, decay_kind=0, decay_first=0, state_unclamped=0):
        self.W, self.H = int(width), int(height)
        self.P = self.W * self.H
        h = ctypes.c_void_p()
        rc = lib().esio_create(self.W, self.H, C, k, b, s_min, s_max, int(t_origin),
                               int(readout_decay), ctypes.byref(h))
        if rc:
            raise OracleError(rc, "esio_create")
        self._h = h
        rc = lib().esio_set_variant(h, int(decay_kind), int(decay_first))
        if not rc:
            rc = lib().esio_set_unclamped(h, int(state_unclamped))
        if rc:
            raise OracleError(rc, "esio_set_variant")

    def close(self):
        if getattr(self, "_h", None):
            lib().esio_destroy(self._h)
            self._h = None

    __del__ = close

    def push(self, events) -> int:
        t, x, y, p = _soa(events)
        return lib().esio_push(self._h, _ptr(t), _ptr(x), _ptr(y), _ptr(p), len(t))

    def render(self, t_frame: int):
        out = np.empty(self.P, np.uint8)
        rc = lib().esio_render(self._h, int(t_frame), _ptr(out))
        if rc:
            raise OracleError(rc, "esio_render")
        return out.reshape(self.H, self.W)

    def render_many(self, t_frames):
        tf = np.ascontiguousarray(t_frames, dtype=np.int64)
        out = np.empty((len(tf), self.H, self.W), np.uint8)
        rc = lib().esio_render_many(self._h, _ptr(tf), len(tf), _ptr(out))
        if rc:
            raise OracleError(rc, "esio_render_many")
        return out

    def flush(self):
        lib().esio_flush(self._h)

    def pending(self) -> int:
        return int(lib().esio_pending(self._h))

    def get_state(self):
        S = np.empty(self.P, np.float64)
        T = np.empty(self.P, np.int64)
        lib().esio_get_state(self._h, _ptr(S), _ptr(T))
        return S.reshape(self.H, self.W), T.reshape(self.H, self.W)

    def set_state(self, S, T):
        S = np.ascontiguousarray(S, dtype=np.float64).reshape(-1)
        T = np.ascontiguousarray(T, dtype=np.int64).reshape(-1)
        return lib().esio_set_state(self._h, _ptr(S), _ptr(T))

    def reset(self):
        return lib().esio_reset(self._h)


def run(width, height, events, t_frames, C=0.15, k=10.0, b=2.0, s_min=-1.5, s_max=1.5,
        t_origin=0, readout_decay=1, decay_kind=0, decay_first=0, state_unclamped=0):
    """Whole-stream oracle: returns (frames[F,H,W] u8, S[H,W] f64, T[H,W] i64)."""
    if decay_kind or decay_first or state_unclamped:   # variants: through the handle
        o = Oracle(width, height, C=C, k=k, b=b, s_min=s_min, s_max=s_max, t_origin=t_origin,
                   readout_decay=readout_decay, decay_kind=decay_kind, decay_first=decay_first,
                   state_unclamped=state_unclamped)
        rc = o.push(events)
        if rc:
            raise OracleError(rc, "esio_push")
        frames = o.render_many(t_frames)
        S, T = o.get_state()                      # as esio_run: events after the last frame stay pending
        o.close()
        return frames, S, T
    t, x, y, p = _soa(events)
    tf = np.ascontiguousarray(t_frames, dtype=np.int64)
    P = int(width) * int(height)
    frames = np.empty((len(tf), int(height), int(width)), np.uint8)
    S = np.empty(P, np.float64)
    T = np.empty(P, np.int64)
    rc = lib().esio_run(int(width), int(height), C, k, b, s_min, s_max, int(t_origin),
                        int(readout_decay), _ptr(t), _ptr(x), _ptr(y), _ptr(p), len(t),
                        _ptr(tf), len(tf), _ptr(frames), _ptr(S), _ptr(T))
    if rc:
        raise OracleError(rc, "esio_run")
    return frames, S.reshape(int(height), int(width)), T.reshape(int(height), int(width))


def stable_group_by(keys) -> np.ndarray:
    """Plain definition of the bit-exact grouping: the permutation
    of a stable sort by key, i.e. key-major, arrival-order-minor."""
    return np.argsort(np.asarray(keys), kind="stable")


# ---------------------------------------------------------------------------
# Pure-Python restatement of Algorithm 2 for small inputs.
# ---------------------------------------------------------------------------
def _py_decay(dt_us, k, b, kind=0):
    if kind == 2:
        return 1.0                            # Eq. 2: no decay
    if kind:
        return math.exp(-k * (dt_us / 1e6))   # exponential variant
    u = 1.0 - k * (dt_us / 1e6)           # Eq. 4
    return u ** b if u > 0.0 else 0.0


def py_run(width, height, events, t_frames, C=0.15, k=10.0, b=2.0, s_min=-1.5, s_max=1.5,
           t_origin=0, readout_decay=1, decay_kind=0, decay_first=0, state_unclamped=0):
    t, x, y, p = _soa(events)
    S = [0.0] * (width * height)
    T = [int(t_origin)] * (width * height)       # P:239 (A3)
    frames = []
    i = 0
    n = len(t)
    for tf in t_frames:
        while i < n and int(t[i]) <= int(tf):     # A6: t == t_frame belongs to the frame
            q = int(y[i]) * width + int(x[i])
            dt = int(t[i]) - T[q]
            if decay_first:                                           # variant: P:247 then P:243
                S[q] = S[q] * _py_decay(dt, k, b, decay_kind)
                S[q] = S[q] + int(p[i]) * C
            else:
                S[q] = S[q] + int(p[i]) * C
                S[q] = S[q] * _py_decay(dt, k, b, decay_kind)
            T[q] = int(t[i])
            if decay_kind != 2 and not state_unclamped:               # Eq. 2 / unclamped: no clamp
                S[q] = min(max(S[q], s_min), s_max)
            i += 1
        fr = np.empty(width * height, np.uint8)
        for q in range(width * height):
            v = S[q] * _py_decay(int(tf) - T[q], k, b, decay_kind) if readout_decay else S[q]
            v = min(max(v, s_min), s_max)
            qv = 255.0 * (v - s_min) / (s_max - s_min)                # Eq. 14
            r = math.floor(qv + 0.5) if qv >= 0 else math.ceil(qv - 0.5)
            fr[q] = min(255, max(0, r))
        frames.append(fr.reshape(height, width))
    return (np.stack(frames) if frames else np.zeros((0, height, width), np.uint8),
            np.array(S).reshape(height, width), np.array(T, np.int64).reshape(height, width))
