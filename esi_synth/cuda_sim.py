"""ctypes binding of the CUDA event-camera simulator (esi_synth/csrc/esim.cu).

SURVEY 8(f) item 2 / SPEC synth: the reference-level
threshold-crossing model of PAPER.md Eq. 1 run one thread per pixel
on the GPU.  Tooling: no ESI arithmetic; the ESI library and the oracle both
consume its output.

    sim = CudaSim()                                   # builds libesim.so on first use
    t, x, y, p = sim.simulate(scene, steps, param)    # time-sorted event tensors
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csrc", "esim.cu")
_LIB = os.path.join(_HERE, "libesim.so")


def build_sim(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        nvcc = "/usr/local/cuda/bin/nvcc" if os.path.exists("/usr/local/cuda/bin/nvcc") else "nvcc"
        tmp = _LIB + ".tmp"
        subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
                               "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


class EsimScene(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("W", ctypes.c_int32), ("H", ctypes.c_int32), ("c", ctypes.c_float),
                ("tex", ctypes.c_void_p), ("R", ctypes.c_int32),
                ("ramp_min", ctypes.c_float), ("ramp_max", ctypes.c_float),
                ("radius", ctypes.c_float), ("reflect", ctypes.c_float), ("cy", ctypes.c_float)]


_L = None


def _lib():
    global _L
    if _L is None:
        L = ctypes.CDLL(build_sim())
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.esim_count.argtypes = [ctypes.POINTER(EsimScene), vp, vp, ctypes.c_int, vp, vp]
        L.esim_emit.argtypes = [ctypes.POINTER(EsimScene), vp, vp, ctypes.c_int, vp, vp, vp, vp, vp]
        L.esim_field.argtypes = [ctypes.POINTER(EsimScene), ctypes.c_float, vp, vp]
        L.esim_pack.argtypes = [vp, vp, vp, vp, i64, i32, vp, vp]
        for f in ("esim_count", "esim_emit", "esim_field", "esim_pack"):
            getattr(L, f).restype = ctypes.c_int
        _L = L
    return _L


def _chk(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed (status {rc})")


def rotation_scene(W: int, H: int, tex: torch.Tensor, c: float) -> EsimScene:
    """kind 0: an R x R float32 CUDA log texture rotated about the image centre."""
    assert tex.is_cuda and tex.dtype == torch.float32 and tex.is_contiguous() and tex.dim() == 2
    s = EsimScene()
    s.kind, s.W, s.H, s.c = 0, W, H, c
    s.tex, s.R = tex.data_ptr(), tex.shape[0]
    s._keep = tex
    return s


def circle_scene(W: int, H: int, c: float, ramp=(0.2, 1.0), radius=18.0, reflect=0.3, cy=None) -> EsimScene:
    """kind 1: the Fig. 2 scene (defaults): linear intensity
    ramp along x and a circle of 30 % reflectivity whose centre x is the scene
    parameter."""
    s = EsimScene()
    s.kind, s.W, s.H, s.c = 1, W, H, c
    s.ramp_min, s.ramp_max = ramp
    s.radius, s.reflect = radius, reflect
    s.cy = H / 2 if cy is None else cy
    return s


class CudaSim:
    def __init__(self, device: Optional[torch.device] = None):
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.L = _lib()

    def _stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def _steps(self, steps, param):
        st = torch.as_tensor(np.ascontiguousarray(steps, np.int64), device=self.device)
        pa = torch.as_tensor(np.ascontiguousarray(param, np.float32), device=self.device)
        return st, pa

    def count(self, scene: EsimScene, steps, param) -> torch.Tensor:
        """Events per pixel ([H*W] int64, device)."""
        st, pa = self._steps(steps, param)
        cnt = torch.empty(scene.W * scene.H, dtype=torch.int64, device=self.device)
        _chk(self.L.esim_count(ctypes.byref(scene), st.data_ptr(), pa.data_ptr(), len(st), cnt.data_ptr(),
                               self._stream()), "esim_count")
        return cnt

    def field(self, scene: EsimScene, param: float) -> torch.Tensor:
        out = torch.empty((scene.H, scene.W), dtype=torch.float32, device=self.device)
        _chk(self.L.esim_field(ctypes.byref(scene), float(param), out.data_ptr(), self._stream()), "esim_field")
        return out

    def simulate(self, scene: EsimScene, steps, param, pixel_major: bool = False):
        """(t, x, y, p) int64/int32/int32/int8 CUDA tensors of every threshold
        crossing, merged in time order (stable sort by t over the pixel-major
        emission order: ties by pixel id, then emission); pixel_major=True skips
        the merge."""
        st, pa = self._steps(steps, param)
        cnt = torch.empty(scene.W * scene.H, dtype=torch.int64, device=self.device)
        _chk(self.L.esim_count(ctypes.byref(scene), st.data_ptr(), pa.data_ptr(), len(st), cnt.data_ptr(),
                               self._stream()), "esim_count")
        off = torch.cumsum(cnt, 0) - cnt
        n = int(cnt.sum().item())
        t = torch.empty(n, dtype=torch.int64, device=self.device)
        pid = torch.empty(n, dtype=torch.int32, device=self.device)
        p = torch.empty(n, dtype=torch.int8, device=self.device)
        if n:
            _chk(self.L.esim_emit(ctypes.byref(scene), st.data_ptr(), pa.data_ptr(), len(st), off.data_ptr(),
                                  t.data_ptr(), pid.data_ptr(), p.data_ptr(), self._stream()), "esim_emit")
        if not pixel_major and n:
            o = torch.sort(t, stable=True).indices
            t, pid, p = t[o], pid[o], p[o]
        W = scene.W
        return t, (pid % W).to(torch.int32), (pid // W).to(torch.int32), p
