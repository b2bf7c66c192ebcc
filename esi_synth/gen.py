"""Event-camera simulator and workload recipes (see esi_synth/__init__.py)."""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional

import numpy as np
import torch

EVENT_NP_DTYPE = np.dtype([("t", "<i8"), ("x", "<u2"), ("y", "<u2"), ("p", "i1"), ("_pad", "u1", (3,))])


# ----------------------------------------------------------------------------- packing
def pack_events(t: torch.Tensor, x: torch.Tensor, y: torch.Tensor, p: torch.Tensor) -> torch.Tensor:
    """[n] tensors -> [n, 2] int64 holding n packed 16-byte esi_event_t records."""
    out = torch.empty((t.numel(), 2), dtype=torch.int64, device=t.device)
    out[:, 0] = t.to(torch.int64)
    out[:, 1] = (x.to(torch.int64) | (y.to(torch.int64) << 16) |
                 ((p.to(torch.int64) & 0xFF) << 32))
    return out


def to_numpy_struct(ev: torch.Tensor) -> np.ndarray:
    a = ev.detach().to("cpu").contiguous().numpy()
    return a.view(EVENT_NP_DTYPE).reshape(-1)


def from_numpy_struct(a: np.ndarray) -> torch.Tensor:
    a = np.ascontiguousarray(a.astype(EVENT_NP_DTYPE, copy=False))
    return torch.from_numpy(a.view(np.int64).reshape(-1, 2).copy())


def unpack(ev: torch.Tensor):
    t = ev[:, 0]
    w = ev[:, 1]
    x = (w & 0xFFFF).to(torch.int32)
    y = ((w >> 16) & 0xFFFF).to(torch.int32)
    p = ((w >> 32) & 0xFF).to(torch.int32)
    p = torch.where(p >= 128, p - 256, p)
    return t, x, y, p


def frame_times(duration_us: int, fps: int, t_origin: int = 0) -> np.ndarray:
    """Frame grid t_j = t_origin + (j+1) * period (DESIGN reading A7)."""
    period = 1_000_000 // fps
    n = duration_us // period
    return t_origin + (np.arange(1, n + 1, dtype=np.int64) * period)


def events_of_pixels(ev_np: np.ndarray, W: int, pixels: np.ndarray):
    """Sub-stream of the given pixel ids, arrival order kept (for sampled oracle checks)."""
    pid = ev_np["y"].astype(np.int64) * W + ev_np["x"].astype(np.int64)
    m = np.isin(pid, pixels)
    return ev_np[m]


# ----------------------------------------------------------------------------- scenes
def value_noise(h: int, w: int, octaves: int, base: int, gen: torch.Generator, device) -> torch.Tensor:
    """Multi-octave value noise in [-1, 1], shape [h, w]."""
    acc = torch.zeros((1, 1, h, w), device=device)
    amp, tot = 1.0, 0.0
    for o in range(octaves):
        g = base * (2 ** o)
        grid = torch.rand((1, 1, g + 1, g + 1), generator=gen, device=device) * 2 - 1
        acc += amp * torch.nn.functional.interpolate(grid, size=(h, w), mode="bicubic", align_corners=True)
        tot += amp
        amp *= 0.5
    acc = acc / tot
    acc = acc / acc.abs().max().clamp_min(1e-6)
    return acc[0, 0]


class RotatingTexture:
    """Camera rolling about the image centre over a static random log texture
    (c4/c5 'fast camera rotation over a seeded random-texture scene')."""

    def __init__(self, W, H, gen, device, log_range=1.5, octaves=5):
        self.W, self.H, self.device = W, H, device
        R = int(math.ceil(math.hypot(W, H))) + 8
        self.tex = (value_noise(R, R, octaves, 6, gen, device) * log_range)[None, None]
        self.R = R
        ys, xs = torch.meshgrid(torch.arange(H, device=device, dtype=torch.float32) + 0.5 - H / 2,
                                torch.arange(W, device=device, dtype=torch.float32) + 0.5 - W / 2,
                                indexing="ij")
        self.xs, self.ys = xs, ys

    def L(self, theta: torch.Tensor) -> torch.Tensor:
        """theta: [B] angles -> [B, H, W] log intensity."""
        c, s = torch.cos(theta)[:, None, None], torch.sin(theta)[:, None, None]
        u = c * self.xs - s * self.ys
        v = s * self.xs + c * self.ys
        grid = torch.stack((u / (self.R / 2), v / (self.R / 2)), dim=-1)
        out = torch.nn.functional.grid_sample(self.tex.expand(theta.numel(), -1, -1, -1), grid,
                                              mode="bilinear", padding_mode="reflection",
                                              align_corners=False)
        return out[:, 0]


class MovingBar:
    """c1: vertical bar, width 8 px, log contrast 2.0 over a uniform background, moving in x with wrap."""

    def __init__(self, W, H, device, width=8.0, contrast=2.0, edge=2.0):
        self.W, self.H, self.device = W, H, device
        self.xs = (torch.arange(W, device=device, dtype=torch.float32) + 0.5)[None, None, :].expand(1, H, W)
        self.width, self.contrast, self.edge = width, contrast, edge

    def L(self, pos: torch.Tensor) -> torch.Tensor:
        d = torch.remainder(self.xs - pos[:, None, None], self.W)      # distance behind the bar's left edge
        d = torch.minimum(d, self.W - d + self.width)                  # wrap
        inside = torch.clamp((d + self.edge / 2) / self.edge, 0, 1) * \
            torch.clamp((self.width - d + self.edge / 2) / self.edge, 0, 1)
        return self.contrast * inside


class AffinePatches:
    """c2: textured patches under piecewise-constant random affine motion over a flat background."""

    def __init__(self, W, H, gen, device, n=6, log_range=1.5, size=(60, 110)):
        self.W, self.H, self.device = W, H, device
        self.n = n
        self.textures = []
        self.sizes = []
        for _ in range(n):
            s = int(torch.randint(size[0], size[1], (1,), generator=gen, device="cpu"))
            self.sizes.append(s)
            self.textures.append(value_noise(s, s, 4, 3, gen, device) * log_range)
        g = torch.Generator(device="cpu").manual_seed(int(torch.randint(0, 2**31, (1,), generator=gen, device="cpu")))
        self.cx0 = torch.rand(n, generator=g) * W
        self.cy0 = torch.rand(n, generator=g) * H
        self.segments = []   # per patch: list of (t0, vx, vy, omega, sdot)
        for i in range(n):
            segs = []
            t = 0.0
            while t < 1e3:
                dur = float(0.2 + 0.6 * torch.rand(1, generator=g))
                ang = float(torch.rand(1, generator=g) * 2 * math.pi)
                spd = float(0.3 + 0.7 * torch.rand(1, generator=g))
                segs.append((t, spd * math.cos(ang), spd * math.sin(ang),
                             float(torch.randn(1, generator=g)) * 0.6, float(torch.randn(1, generator=g)) * 0.1))
                t += dur
                if len(segs) > 200:
                    break
            self.segments.append(segs)
        ys, xs = torch.meshgrid(torch.arange(H, device=device, dtype=torch.float32) + 0.5,
                                torch.arange(W, device=device, dtype=torch.float32) + 0.5, indexing="ij")
        self.xs, self.ys = xs, ys
        self.speed = 1.0

    def _pose(self, i, t):
        cx, cy, th, sc = float(self.cx0[i]), float(self.cy0[i]), 0.0, 1.0
        segs = self.segments[i]
        for k, (t0, vx, vy, om, sd) in enumerate(segs):
            t1 = segs[k + 1][0] if k + 1 < len(segs) else 1e9
            dt = max(0.0, min(t, t1) - t0)
            if dt <= 0:
                break
            cx += vx * self.speed * dt * 100
            cy += vy * self.speed * dt * 100
            th += om * self.speed * dt
            sc = min(1.6, max(0.6, sc + sd * self.speed * dt))
        return cx % self.W, cy % self.H, th, sc

    def L(self, ts: torch.Tensor) -> torch.Tensor:
        B = ts.numel()
        out = torch.zeros((B, self.H, self.W), device=self.device)
        for i in range(self.n):
            s = self.sizes[i]
            poses = [self._pose(i, float(t)) for t in ts.tolist()]
            cx = torch.tensor([q[0] for q in poses], device=self.device)[:, None, None]
            cy = torch.tensor([q[1] for q in poses], device=self.device)[:, None, None]
            th = torch.tensor([q[2] for q in poses], device=self.device)[:, None, None]
            sc = torch.tensor([q[3] for q in poses], device=self.device)[:, None, None]
            dx, dy = self.xs - cx, self.ys - cy
            u = (torch.cos(th) * dx + torch.sin(th) * dy) / (sc * s / 2)
            v = (-torch.sin(th) * dx + torch.cos(th) * dy) / (sc * s / 2)
            grid = torch.stack((u, v), -1)
            val = torch.nn.functional.grid_sample(self.textures[i][None, None].expand(B, -1, -1, -1), grid,
                                                  mode="bilinear", padding_mode="zeros", align_corners=False)[:, 0]
            alpha = torch.clamp((1.0 - torch.maximum(u.abs(), v.abs())) * 8, 0, 1)
            out = out * (1 - alpha) + (val + 0.3 * (i % 3 - 1)) * alpha
        return out


# ----------------------------------------------------------------------------- simulator
def simulate(scene_L: Callable[[torch.Tensor], torch.Tensor], param_of_t: Callable[[np.ndarray], np.ndarray],
             t_start_us: int, t_end_us: int, dt_us: int, c: float, device, batch: int = 64,
             count_only: bool = False):
    """Reference-level threshold-crossing model:
    an event fires each time |L - L_ref| reaches c; L_ref steps by +-c per event;
    crossing times are linearly interpolated inside a sample step and floored
    to 1 us.  Returns per-step lists (t, x, y, p) in emission order."""
    steps = np.arange(t_start_us, t_end_us + 1, dt_us, dtype=np.int64)
    if steps[-1] != t_end_us:
        steps = np.append(steps, t_end_us)
    params = param_of_t(steps)
    L_prev = scene_L(torch.as_tensor(params[:1], device=device, dtype=torch.float32))[0]
    H, W = L_prev.shape
    L_ref = L_prev.clone()
    out_t, out_pid, out_p = [], [], []
    total = 0
    for b0 in range(1, len(steps), batch):
        b1 = min(len(steps), b0 + batch)
        Ls = scene_L(torch.as_tensor(params[b0:b1], device=device, dtype=torch.float32))
        for k in range(b1 - b0):
            L_new = Ls[k]
            d = L_new - L_ref
            n_up = torch.floor(d / c).clamp_min(0)
            n_dn = torch.floor(-d / c).clamp_min(0)
            n = (n_up + n_dn).to(torch.int32).reshape(-1)
            if count_only:
                total += int(n.sum())
            else:
                nz = torch.nonzero(n, as_tuple=False).reshape(-1)
                if nz.numel():
                    cnt = n[nz].to(torch.int64)
                    pid = torch.repeat_interleave(nz, cnt)
                    start = torch.cumsum(cnt, 0) - cnt
                    idx = torch.arange(pid.numel(), device=device) - torch.repeat_interleave(start, cnt) + 1
                    up = (n_up.reshape(-1)[pid] > 0)
                    sgn = torch.where(up, 1.0, -1.0)
                    lv = L_ref.reshape(-1)[pid] + sgn * idx.to(torch.float32) * c
                    l0 = L_prev.reshape(-1)[pid]
                    l1 = L_new.reshape(-1)[pid]
                    den = torch.where((l1 - l0).abs() > 1e-12, l1 - l0, torch.ones_like(l1))
                    frac = ((lv - l0) / den).clamp(0.0, 1.0)
                    ts = steps[b0 + k - 1] + torch.floor(frac * float(steps[b0 + k] - steps[b0 + k - 1])).to(torch.int64)
                    out_t.append(ts)
                    out_pid.append(pid)
                    out_p.append(torch.where(up, 1, -1).to(torch.int8))
            L_ref = L_ref + c * (n_up - n_dn)
            L_prev = L_new
    if count_only:
        return total
    if out_t:
        t = torch.cat(out_t); pid = torch.cat(out_pid); p = torch.cat(out_p)
    else:
        t = torch.zeros(0, dtype=torch.int64, device=device)
        pid = torch.zeros(0, dtype=torch.int64, device=device)
        p = torch.zeros(0, dtype=torch.int8, device=device)
    return t, (pid % W).to(torch.int32), (pid // W).to(torch.int32), p


def poisson_noise(W, H, rate_hz_per_px, t0_us, t1_us, gen, device, p_on=0.5):
    """Background-activity noise: uniform pixel, uniform time, random polarity."""
    n_exp = rate_hz_per_px * W * H * (t1_us - t0_us) * 1e-6
    n = int(torch.poisson(torch.tensor([n_exp], dtype=torch.float64), generator=_cpu_gen(gen)).item()) if n_exp > 0 else 0
    t = torch.randint(t0_us, t1_us, (n,), generator=gen, device=device, dtype=torch.int64)
    x = torch.randint(0, W, (n,), generator=gen, device=device, dtype=torch.int32)
    y = torch.randint(0, H, (n,), generator=gen, device=device, dtype=torch.int32)
    p = torch.where(torch.rand(n, generator=gen, device=device) < p_on, 1, -1).to(torch.int8)
    return t, x, y, p


def _cpu_gen(gen: torch.Generator) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(torch.randint(0, 2**62, (1,), generator=gen, device=gen.device).item()) & ((1 << 62) - 1))
    return g


def merge(parts, device):
    """Concatenate parts in order and stable-sort by t (deterministic tie-break:
    signal first in emission order, then noise, then hot pixels)."""
    t = torch.cat([q[0] for q in parts]).to(device)
    x = torch.cat([q[1].to(torch.int32) for q in parts]).to(device)
    y = torch.cat([q[2].to(torch.int32) for q in parts]).to(device)
    p = torch.cat([q[3].to(torch.int8) for q in parts]).to(device)
    order = torch.sort(t, stable=True).indices
    return t[order], x[order], y[order], p[order]


# ----------------------------------------------------------------------------- workloads
@dataclass
class Workload:
    name: str
    W: int
    H: int
    events: torch.Tensor          # [n, 2] int64 packed esi_event_t
    t_frames: np.ndarray          # int64 frame times
    params: Dict[str, float]      # C, k, b, s_min, s_max
    duration_us: int
    description: str = ""
    extra: Dict[str, object] = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.events.shape[0])

    @property
    def P(self) -> int:
        return self.W * self.H


def _esi_params(C):
    # reading A10: C = simulator threshold, S_min/S_max = -+10 C, k = 10 1/s, b = 2
    return {"C": C, "k": 10.0, "b": 2.0, "s_min": -10 * C, "s_max": 10 * C}


def _c1(device, seed):
    W, H, dur = 64, 48, 100_000
    gen = torch.Generator(device=device).manual_seed(seed)
    bar = MovingBar(W, H, device)
    # 95 k signal events: each pass of the bar gives 2 * contrast / c = 20 events per pixel
    passes = 1.12 * 95_000 / (W * H * 20)   # 1.12: soft bar edges cross fewer levels
    speed = passes * W / (dur * 1e-6)                       # px / s
    sig = simulate(bar.L, lambda ts: (ts * 1e-6 * speed).astype(np.float64), 0, dur, 100, 0.2, device)
    n_noise = int(0.05 * sig[0].numel())
    noise = (torch.randint(0, dur, (n_noise,), generator=gen, device=device, dtype=torch.int64),
             torch.randint(0, W, (n_noise,), generator=gen, device=device, dtype=torch.int32),
             torch.randint(0, H, (n_noise,), generator=gen, device=device, dtype=torch.int32),
             torch.where(torch.rand(n_noise, generator=gen, device=device) < 0.5, 1, -1).to(torch.int8))
    t, x, y, p = merge([sig, noise], device)
    return Workload("c1", W, H, pack_events(t, x, y, p), frame_times(dur, 100), _esi_params(0.2), dur,
                    "64x48 moving bar, contrast 0.2, +5% uniform noise")


def _c2(device, seed, duration_us=2_000_000):
    W, H = 346, 260
    gen = torch.Generator(device=device).manual_seed(seed)
    sc = AffinePatches(W, H, gen, device)
    # calibrate speed so the signal rate is ~1 Mev/s (count over 0.2 s at unit speed)
    sc.speed = 1.0
    n_cal = simulate(sc.L, lambda ts: ts * 1e-6, 0, 200_000, 1000, 0.2, device, count_only=True)
    sc.speed = max(0.05, 1.0e6 * 0.2 / max(n_cal, 1))
    sig = simulate(sc.L, lambda ts: ts * 1e-6, 0, duration_us, 500, 0.2, device)
    noise = poisson_noise(W, H, 0.1, 0, duration_us, gen, device)
    t, x, y, p = merge([sig, noise], device)
    return Workload("c2", W, H, pack_events(t, x, y, p), frame_times(duration_us, 100), _esi_params(0.2),
                    duration_us, "346x260 textured patches, random affine motion, BA 0.1 Hz/px")


def _c3(device, seed, duration_us=5_000_000):
    W, H = 640, 480
    gen = torch.Generator(device=device).manual_seed(seed)
    ba = poisson_noise(W, H, 2.0, 0, duration_us, gen, device, p_on=0.6)
    # 10 % of pixels are hot-burst pixels: bursts of ~20 ms at ~1 kHz, random off-times,
    # together supplying the remaining ~11.9 M events (reading of config 3 in DESIGN.md)
    n_hot = (W * H) // 10
    hot_pid = torch.randperm(W * H, generator=gen, device=device)[:n_hot]
    target = 11_900_000 * duration_us / 5_000_000
    per_px = target / n_hot                            # events per hot pixel
    bursts = max(1, int(round(per_px / 20)))           # ~20 events per burst
    starts = torch.rand((n_hot, bursts), generator=gen, device=device) * (duration_us - 20_000)
    k_ev = 20
    offs = torch.sort(torch.rand((n_hot, bursts, k_ev), generator=gen, device=device) * 20_000, dim=-1).values
    t = (starts[:, :, None] + offs).reshape(-1).to(torch.int64)
    pid = hot_pid[:, None, None].expand(n_hot, bursts, k_ev).reshape(-1)
    p = torch.where(torch.rand(t.numel(), generator=gen, device=device) < 0.6, 1, -1).to(torch.int8)
    hot = (t, (pid % W).to(torch.int32), (pid // W).to(torch.int32), p)
    t, x, y, p = merge([ba, hot], device)
    # +-50 us jitter, kept non-decreasing by a stable re-sort
    t = (t + torch.randint(-50, 51, t.shape, generator=gen, device=device)).clamp(0, duration_us - 1)
    o = torch.sort(t, stable=True).indices
    t, x, y, p = t[o], x[o], y[o], p[o]
    return Workload("c3", W, H, pack_events(t, x, y, p), frame_times(duration_us, 100), _esi_params(0.15),
                    duration_us, "640x480 noise-dominated: BA 2 Hz/px + 10% hot-burst pixels, P(ON)=0.6")


def _rotation(W, H, device, seed, duration_us, rate_fn, c=0.15, dt_us=500, name="c4", desc="", sim=None):
    """Camera roll over a seeded random log texture with a calibrated event rate.
    On CUDA the threshold-crossing walk runs in the CUDA simulator
    (esi_synth/csrc/esim.cu); on CPU in torch (``simulate``)."""
    gen = torch.Generator(device=device).manual_seed(seed)
    sc = RotatingTexture(W, H, gen, device)
    use_cuda = device.type == "cuda" and (sim or os.environ.get("ESI_SYNTH_SIM", "cuda")) == "cuda"
    if use_cuda:
        from .cuda_sim import CudaSim, rotation_scene
        cs = CudaSim(device)
        scene = rotation_scene(W, H, sc.tex[0, 0].contiguous(), c)

        def count(rad):
            st = np.arange(0, int(rad * 1e6) + 1, 1000, dtype=np.int64)
            return int(cs.count(scene, st, (st.astype(np.float64) * 1e-6).astype(np.float32)).sum().item())
    else:
        def count(rad):
            return simulate(sc.L, lambda ts: ts.astype(np.float64) * 1e-6, 0, int(rad * 1e6), 1000, c, device,
                            count_only=True)
    # events per radian: calibrated with a short count-only run (steady state only:
    # the first 0.1 rad charges the reference levels up), then omega is scaled
    ev_per_rad = max(1.0, (count(0.4) - count(0.1)) / 0.3)
    # theta(t) = integral of omega, omega(t) = rate(t) / ev_per_rad
    tt = np.arange(0, duration_us + dt_us, dt_us, dtype=np.int64)
    rates = rate_fn(tt)
    theta = np.concatenate([[0.0], np.cumsum(0.5 * (rates[1:] + rates[:-1]) * dt_us * 1e-6)]) / ev_per_rad

    def param_of_t(ts):
        return np.interp(ts.astype(np.float64), tt.astype(np.float64), theta)

    if use_cuda:
        steps = np.arange(0, duration_us + 1, dt_us, dtype=np.int64)
        if steps[-1] != duration_us:
            steps = np.append(steps, duration_us)
        t, x, y, p = cs.simulate(scene, steps, param_of_t(steps).astype(np.float32))
        return (t, x, y, p), sc
    sig = simulate(sc.L, param_of_t, 0, duration_us, dt_us, c, device, batch=32)
    t, x, y, p = sig
    o = torch.sort(t, stable=True).indices
    return (t[o], x[o], y[o], p[o]), sc


def _c4_rate(tt):
    r = np.full(tt.shape, 15.79e6)
    ts = tt * 1e-6
    for i in range(10):
        r[(ts >= 0.5 + i) & (ts < 0.55 + i)] = 100e6
    return r


def _c4(device, seed, duration_us=10_000_000, fps=100):
    W, H = 1280, 720
    (t, x, y, p), _ = _rotation(W, H, device, seed, duration_us,
                                lambda tt: _c4_rate(tt) if duration_us == 10_000_000 else np.full(tt.shape, 20e6))
    return Workload("c4", W, H, pack_events(t, x, y, p), frame_times(duration_us, fps), _esi_params(0.15),
                    duration_us, f"1280x720 rotating texture, 20 Mev/s avg with 100 Mev/s bursts, {fps} FPS")


def _c5a(device, seed, duration_us=10_000_000):
    W, H = 1280, 720
    (t, x, y, p), _ = _rotation(W, H, device, seed, duration_us, lambda tt: np.full(tt.shape, 10e6))
    return Workload("c5a", W, H, pack_events(t, x, y, p), frame_times(duration_us, 100), _esi_params(0.15),
                    duration_us, "1280x720 rotating texture at 10 Mev/s (one of 64 streams)")


def _c5b(device, seed, duration_us=10_000_000):
    W, H = 2560, 1440
    (t, x, y, p), _ = _rotation(W, H, device, seed, duration_us, lambda tt: np.full(tt.shape, 80e6))
    return Workload("c5b", W, H, pack_events(t, x, y, p), frame_times(duration_us, 100), _esi_params(0.15),
                    duration_us, "2560x1440 rotating texture at 80 Mev/s")


CONFIGS = {
    "c1": (_c1, 1),
    "c2": (_c2, 2),
    "c3": (_c3, 3),
    "c4": (_c4, 4),
    "c5a": (_c5a, 5000),
    "c5b": (_c5b, 5),
}


def make_workload(name: str, device="cpu", seed: Optional[int] = None, **kw) -> Workload:
    fn, default_seed = CONFIGS[name]
    with torch.no_grad():
        return fn(torch.device(device), default_seed if seed is None else seed, **kw)
