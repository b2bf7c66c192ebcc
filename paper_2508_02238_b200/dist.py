"""Multi-GPU sharding of the ESI hot path.

ESI has no spatial coupling: an event changes only its own pixel (Alg. 2,
PAPER.md P:242-253) and a frame is a per-pixel map of the state (Eq. 14,
P:227), so the path shards two ways, one process per GPU (torch.distributed,
NCCL over NVLink on the GPU box, gloo in the CPU tests):

* ``StreamSharded`` -- independent event streams (BASELINE config 5a) are
  assigned round-robin to ranks; every rank integrates its streams with
  ordinary handles.  No data-path collective.
* ``RowBandSharded`` -- one large sensor (config 5b) is split into G row bands
  (``row_bands``).  Each rank holds a time-contiguous shard of the raw stream
  (rank order = time order); it stably partitions the shard by band on its GPU
  (``esi_route_bands``), exchanges the band buckets with one all-to-all, and
  integrates its band's events -- received in source-rank order, i.e. time
  order -- with an ordinary handle of height = band rows (y rebased by the
  router).  Frames are assembled with all_gather_into_tensor: bands are
  row-contiguous, so rank order is row-major order and every frame lands in
  place.  The collectives only move bytes; all arithmetic runs in libesi's
  kernels.

The band handle and the router are injectable (``band_factory``, ``router``)
so that the host logic -- routing plan, exchange, assembly -- is testable with
world_size 2 on CPU (gloo) against a full-sensor reference; the product path
uses libesi handles and the device router and has no CPU fallback.
"""
from __future__ import annotations

import ctypes
from typing import Callable, List, Optional, Sequence

import numpy as np
import torch
import torch.distributed as dist


def row_bands(height: int, n_bands: int) -> List[int]:
    """Row starts of n_bands contiguous bands (len n_bands + 1): ceil(H/G) rows
    each, the last band taking the remainder."""
    if n_bands < 1 or height < n_bands:
        raise ValueError(f"cannot split {height} rows into {n_bands} bands")
    bh = -(-height // n_bands)
    starts = [min(height, b * bh) for b in range(n_bands)] + [height]
    if any(starts[b + 1] <= starts[b] for b in range(n_bands)):
        raise ValueError(f"{height} rows do not split into {n_bands} non-empty bands of {bh}")
    return starts


def time_shard_bounds(n: int, world: int) -> List[int]:
    """Split n time-ordered events into `world` contiguous shards (rank order = time order)."""
    return [n * r // world for r in range(world + 1)]


def device_router(device: int, height: int) -> Callable:
    """Router of the product path: esi_route_bands on the events' GPU."""
    from .esi import _lib

    def route(events: torch.Tensor, starts: Sequence[int]):
        n = events.shape[0]
        G = len(starts) - 1
        out = torch.empty_like(events)
        counts = np.zeros(G, np.int64)
        rs = (ctypes.c_int32 * (G + 1))(*starts)
        stream = torch.cuda.current_stream(events.device).cuda_stream
        rc = _lib().esi_route_bands(int(device), ctypes.c_void_p(events.data_ptr() if n else 0),
                                    ctypes.c_size_t(n), int(height), rs, int(G),
                                    ctypes.c_void_p(out.data_ptr() if n else 0),
                                    counts.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(stream))
        if rc != 0:
            from .esi import EsiError
            raise EsiError(rc, "esi_route_bands")
        return out, counts

    return route


class RowBandSharded:
    """One sensor split into row bands, one band per rank (see module docstring)."""

    def __init__(self, width: int, height: int, group=None, band_factory: Optional[Callable] = None,
                 router: Optional[Callable] = None, device: Optional[torch.device] = None, **params):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.W, self.H = int(width), int(height)
        self.starts = row_bands(self.H, self.world)
        self.bh = self.starts[1] - self.starts[0]           # padded band height (all but the last band)
        self.rows = self.starts[self.rank + 1] - self.starts[self.rank]
        self.device = device if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu"))
        if band_factory is None:
            from .esi import Esi
            band_factory = lambda w, h, **p: Esi(w, h, **p)   # noqa: E731
        self.band = band_factory(self.W, self.rows, **params)
        self.router = router if router is not None else device_router(self.device.index or 0, self.H)
        self._keep = []
        self.stats = {"routed": 0, "sent": 0, "received": 0}

    def close(self):
        if getattr(self, "band", None) is not None and hasattr(self.band, "close"):
            self.band.close()
        self.band = None
        self._keep = []

    # -- routing + exchange -------------------------------------------------
    def exchange(self, shard: torch.Tensor) -> torch.Tensor:
        """Route this rank's time shard ([n, 2] int64 packed events) by band and
        exchange: returns this rank's band events (y rebased), time-ordered."""
        routed, counts = self.router(shard, self.starts)
        send = torch.as_tensor(np.asarray(counts, np.int64), device=shard.device)
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send, group=self.group)
        in_splits = [int(c) for c in np.asarray(counts)]
        out_splits = [int(c) for c in recv.tolist()]
        out = torch.empty((sum(out_splits), 2), dtype=torch.int64, device=shard.device)
        # rows of 16 bytes: split sizes count events (dim 0)
        dist.all_to_all_single(out, routed, out_splits, in_splits, group=self.group)
        self.stats["routed"] += int(shard.shape[0])
        self.stats["sent"] += int(sum(in_splits) - in_splits[self.rank])
        self.stats["received"] += int(out.shape[0])
        return out

    def push_shard(self, shard: torch.Tensor) -> int:
        """Collective: every rank calls it once per round with its shard of the
        round's time slice; the concatenation of the shards in rank order must be
        time-ordered, and each round must follow the previous one in time."""
        band_events = self.exchange(shard)
        self._keep.append(band_events)                      # device pushes are borrowed zero-copy
        return self.band.push(band_events)

    # -- rendering + assembly -----------------------------------------------
    def render_many(self, t_frames, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Renders this rank's band for every frame time and assembles the full
        [F, H, W] frames on every rank (all_gather over the group)."""
        tf = np.ascontiguousarray(t_frames, dtype=np.int64)
        F = len(tf)
        band = torch.zeros((F, self.bh, self.W), dtype=torch.uint8, device=self.device)
        if self.rows == self.bh:
            self.band.render_many(tf, band)
        else:                                                # short last band: render, then pad
            part = torch.empty((F, self.rows, self.W), dtype=torch.uint8, device=self.device)
            self.band.render_many(tf, part)
            band[:, :self.rows].copy_(part)
        full_h = self.bh * self.world
        direct = out is not None and full_h == self.H and out.is_contiguous()
        buf = out if direct else torch.empty((F, full_h, self.W), dtype=torch.uint8, device=self.device)
        for j in range(F):                                   # frame j: rank-major = row-major
            dist.all_gather_into_tensor(buf[j].view(-1), band[j].view(-1), group=self.group)
        self._keep = []
        if direct:
            return out
        res = buf[:, :self.H]
        if out is not None:
            out.copy_(res)
            return out
        return res.contiguous()

    def get_state(self):
        return self.band.get_state()


class StreamSharded:
    """Independent streams assigned round-robin to ranks (config 5a); no collective
    on the data path.  ``streams`` are (width, height, params) triples; this rank
    owns streams s with s % world == rank."""

    def __init__(self, streams: Sequence, group=None, handle_factory: Optional[Callable] = None):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        if handle_factory is None:
            from .esi import Esi
            handle_factory = lambda w, h, **p: Esi(w, h, **p)   # noqa: E731
        self.owned = [s for s in range(len(streams)) if s % self.world == self.rank]
        self.handles = {s: handle_factory(streams[s][0], streams[s][1], **streams[s][2]) for s in self.owned}

    def push(self, s: int, events) -> int:
        return self.handles[s].push(events)

    def render_many(self, s: int, t_frames, out=None):
        return self.handles[s].render_many(t_frames, out)

    def close(self):
        for h in self.handles.values():
            if hasattr(h, "close"):
                h.close()
        self.handles = {}
