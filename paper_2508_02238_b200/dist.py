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
  and the band buckets are exchanged so that every rank integrates its band's
  events -- received in source-rank order, i.e. time order -- with an ordinary
  handle of height = band rows (y rebased by the router).  Two exchanges:
    - ``transport=PeerTransport(...)`` (the product path on NVLink): the
      router's scatter kernel stores every event straight into the receive
      arena of the rank that owns its band (CUDA IPC mapping, P2P stores), so
      the all-to-all IS the partition kernel; only the per-band counts go
      through a collective (a G x G all_gather) to place each source's run;
    - otherwise ``esi_route_bands`` into a local buffer + NCCL
      ``all_to_all_single`` (the baseline).
  Frames are assembled with all_gather_into_tensor: bands are row-contiguous,
  so rank order is row-major order and every frame lands in place.  All
  arithmetic runs in libesi's kernels.

The band handle, the router and the transport are injectable (``band_factory``,
``router``, ``transport``) so that the host logic -- routing plan, receive
offsets, arena growth, exchange, assembly -- is testable with world_size 2 on
CPU (gloo) against a full-sensor reference; the product path uses libesi
handles and kernels and has no CPU fallback.
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


class PeerTransport:
    """P2P exchange of the row-band split on the GPUs (product path).

    count(): esi_router_count of this rank's shard (per-band counts, host).
    scatter(): esi_router_scatter -- band g's run is stored by the kernel
    directly into dst[g] (rank g's receive arena, mapped into this process with
    CUDA IPC; this rank's own arena by its pointer) at the given record offset.
    Arenas are plain cudaMalloc buffers (esi_buffer_alloc) so that their IPC
    handles cover them exactly."""

    def __init__(self, device: int, height: int, starts: Sequence[int], stream: Optional[int] = None):
        from .esi import _lib
        self.L = _lib()
        self.device = int(device)
        self.G = len(starts) - 1
        rs = (ctypes.c_int32 * (self.G + 1))(*starts)
        r = ctypes.c_void_p()
        self._check(self.L.esi_router_create(self.device, int(height), rs, self.G, ctypes.byref(r)), "router_create")
        self.r = r
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        self._shard = None

    @staticmethod
    def _check(rc, what):
        if rc != 0:
            from .esi import EsiError
            raise EsiError(rc, f"esi_{what}")

    def count(self, shard: torch.Tensor) -> np.ndarray:
        counts = np.zeros(self.G, np.int64)
        n = int(shard.shape[0])
        self._shard = shard                       # must stay valid until scatter
        self._check(self.L.esi_router_count(self.r, shard.data_ptr() if n else None, n,
                                            counts.ctypes.data, self.stream), "router_count")
        return counts

    def scatter(self, dst: Sequence[int], offsets: np.ndarray):
        ptrs = (ctypes.c_void_p * self.G)(*[int(d) for d in dst])
        off = np.ascontiguousarray(offsets, np.int64)
        self._check(self.L.esi_router_scatter(self.r, ptrs, off.ctypes.data, self.stream), "router_scatter")

    def sync(self):
        self._check(self.L.esi_stream_sync(self.device, self.stream), "stream_sync")
        self._shard = None

    def alloc(self, nrec: int) -> int:
        p = ctypes.c_void_p()
        self._check(self.L.esi_buffer_alloc(self.device, int(nrec) * 16, ctypes.byref(p)), "buffer_alloc")
        return int(p.value)

    def free(self, addr: int):
        self._check(self.L.esi_buffer_free(self.device, addr), "buffer_free")

    def export(self, addr: int) -> bytes:
        h = ctypes.create_string_buffer(64)
        self._check(self.L.esi_ipc_get_handle(addr, h), "ipc_get_handle")
        return h.raw

    def open(self, handle: bytes) -> int:
        p = ctypes.c_void_p()
        self._check(self.L.esi_ipc_open(self.device, handle, ctypes.byref(p)), "ipc_open")
        return int(p.value)

    def unmap(self, addr: int):
        self._check(self.L.esi_ipc_close(self.device, addr), "ipc_close")

    def push(self, band, addr: int, off: int, n: int) -> int:
        return band.push_ptr(addr + 16 * int(off), int(n)) if n else 0

    def quiesce(self):
        """Every stream of the device idle (the band handle's renders included)."""
        torch.cuda.synchronize(self.device)

    def close(self):
        if getattr(self, "r", None) is not None:
            self.L.esi_router_destroy(self.r)
            self.r = None


class RowBandSharded:
    """One sensor split into row bands, one band per rank (see module docstring)."""

    MIN_ARENA = 1 << 20                                     # records (16 MB) per receive arena

    def __init__(self, width: int, height: int, group=None, band_factory: Optional[Callable] = None,
                 router: Optional[Callable] = None, device: Optional[torch.device] = None,
                 transport=None, **params):
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
        # The band handle works on torch's current stream: the NCCL exchange output it
        # borrows zero-copy and the frame buffer zero-fill are ordered on that stream,
        # so the handle's kernels must be too (a private stream would race with both).
        if self.device.type == "cuda" and hasattr(self.band, "set_stream"):
            self.band.set_stream(torch.cuda.current_stream(self.device).cuda_stream)
        self.p2p = transport
        if transport is None:
            self.router = router if router is not None else device_router(self.device.index or 0, self.H)
        self._keep = []
        self.stats = {"routed": 0, "sent": 0, "received": 0}
        # P2P receive arenas: every rank tracks every arena's capacity and fill,
        # which evolve deterministically from the all-gathered counts.
        self._cap = [0] * self.world
        self._fill = [0] * self.world
        self._arena = None                                   # this rank's arena (transport id)
        self._dst = [None] * self.world                      # where this rank writes band g
        self._old = []                                       # replaced arenas, freed once consumed

    def close(self):
        if getattr(self, "band", None) is not None and hasattr(self.band, "close"):
            self.band.close()
        self.band = None
        self._keep = []
        if self.p2p is not None:                             # collective: every rank closes
            for g, d in enumerate(self._dst):
                if d is not None and g != self.rank:
                    self.p2p.unmap(d)
            dist.barrier(group=self.group)                   # no peer maps an arena once it is freed
            for a in self._old + ([self._arena] if self._arena is not None else []):
                self.p2p.free(a)
            self._old, self._arena, self._dst = [], None, [None] * self.world
            self.p2p.close()

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
        if self.p2p is not None:
            return self._push_shard_p2p(shard)
        band_events = self.exchange(shard)
        self._keep.append(band_events)                      # device pushes are borrowed zero-copy
        return self.band.push(band_events)

    def _push_shard_p2p(self, shard: torch.Tensor) -> int:
        T, G, r = self.p2p, self.world, self.rank
        counts = torch.as_tensor(np.asarray(T.count(shard), np.int64), device=self.device)
        M = torch.empty((G, G), dtype=torch.int64, device=self.device)
        dist.all_gather_into_tensor(M.view(-1), counts, group=self.group)
        M = M.cpu().numpy()                                  # M[s, g]: events of source s for band g
        R = M.sum(axis=0)                                    # this round's events per band
        grow = [self._fill[g] + int(R[g]) > self._cap[g] for g in range(G)]
        if any(grow):                                        # deterministic on every rank
            for g in range(G):
                if grow[g]:
                    self._cap[g] = max(2 * self._cap[g], int(R[g]), self.MIN_ARENA)
                    self._fill[g] = 0
            if grow[r]:
                if self._arena is not None:
                    self._old.append(self._arena)            # may hold pending events: freed after render
                self._arena = T.alloc(self._cap[r])
            handles = [None] * G
            dist.all_gather_object(handles, T.export(self._arena) if grow[r] else None, group=self.group)
            for g in range(G):
                if not grow[g]:
                    continue
                if g == r:
                    self._dst[g] = self._arena
                else:
                    if self._dst[g] is not None:
                        T.unmap(self._dst[g])
                    self._dst[g] = T.open(handles[g])
        off = np.array([self._fill[g] + int(M[:r, g].sum()) for g in range(G)], np.int64)
        T.scatter(self._dst, off)                            # the exchange: P2P stores by the router kernel
        T.sync()
        dist.barrier(group=self.group)                       # every source's stores have landed
        n_mine = int(R[r])
        rc = T.push(self.band, self._arena, self._fill[r], n_mine)
        for g in range(G):
            self._fill[g] += int(R[g])
        self.stats["routed"] += int(shard.shape[0])
        self.stats["sent"] += int(M[r].sum() - M[r, r])
        self.stats["received"] += n_mine
        return rc

    # -- rendering + assembly -----------------------------------------------
    ASSEMBLY_BATCH = 64                                     # frames per coalesced (grouped) all-gather

    def _assemble(self, band: torch.Tensor, buf: torch.Tensor):
        """Frame assembly: all_gather_into_tensor of every frame's band slice into
        frame j of buf (rank-major = row-major, so each frame lands in place).
        On NCCL, batches of frames are issued as one coalesced group
        (ncclGroupStart/End of the per-frame all-gathers: one launch per batch)."""
        F = band.shape[0]
        coalesce = dist.get_backend(self.group) == "nccl"
        for j0 in range(0, F, self.ASSEMBLY_BATCH):
            j1 = min(F, j0 + self.ASSEMBLY_BATCH)
            if coalesce:
                from torch.distributed.distributed_c10d import _coalescing_manager
                with _coalescing_manager(group=self.group, device=self.device, async_ops=True) as cm:
                    for j in range(j0, j1):
                        dist.all_gather_into_tensor(buf[j].view(-1), band[j].view(-1), group=self.group)
                cm.wait()
            else:
                for j in range(j0, j1):
                    dist.all_gather_into_tensor(buf[j].view(-1), band[j].view(-1), group=self.group)

    def render_many(self, t_frames, out: Optional[torch.Tensor] = None, stage_ms: Optional[dict] = None) -> torch.Tensor:
        """Renders this rank's band for every frame time and assembles the full
        [F, H, W] frames on every rank (all_gather over the group).  stage_ms:
        if given, the band render and the assembly are timed separately (CUDA
        events on the current stream) and accumulated into it."""
        tf = np.ascontiguousarray(t_frames, dtype=np.int64)
        F = len(tf)
        timing = stage_ms is not None and self.device.type == "cuda"
        if timing:
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
        band = torch.empty((F, self.bh, self.W), dtype=torch.uint8, device=self.device)
        if self.rows == self.bh:
            self.band.render_many(tf, band)
        else:                                                # short last band: render, then pad
            band[:, self.rows:].zero_()
            part = torch.empty((F, self.rows, self.W), dtype=torch.uint8, device=self.device)
            self.band.render_many(tf, part)
            band[:, :self.rows].copy_(part)
        if timing:
            e1.record()
        full_h = self.bh * self.world
        direct = out is not None and full_h == self.H and out.is_contiguous()
        if self.world == 1 and direct:                       # one band = the whole frame: no assembly
            out.copy_(band)
            buf = out
        else:
            buf = out if direct else torch.empty((F, full_h, self.W), dtype=torch.uint8, device=self.device)
            self._assemble(band, buf)
        if timing:
            e2.record()
            e2.synchronize()
            stage_ms["band_render"] = stage_ms.get("band_render", 0.0) + e0.elapsed_time(e1)
            stage_ms["assembly"] = stage_ms.get("assembly", 0.0) + e1.elapsed_time(e2)
        self._keep = []
        if self.p2p is not None:
            self._recycle_arenas()
        if direct:
            return out
        res = buf[:, :self.H]
        if out is not None:
            out.copy_(res)
            return out
        return res.contiguous()

    def _recycle_arenas(self):
        """After a render: arenas whose events are all integrated are reused from
        the start (every rank must agree, so the decision is all-gathered)."""
        (self.p2p.quiesce if hasattr(self.p2p, "quiesce") else self.p2p.sync)()
        pending = int(self.band.pending()) if hasattr(self.band, "pending") else 1
        flags = torch.tensor([1 if pending == 0 else 0], dtype=torch.int64, device=self.device)
        allf = torch.empty(self.world, dtype=torch.int64, device=self.device)
        dist.all_gather_into_tensor(allf, flags, group=self.group)
        for g, f in enumerate(allf.cpu().tolist()):
            if f:
                self._fill[g] = 0
        if pending == 0:
            for a in self._old:
                self.p2p.free(a)
            self._old = []

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


def time_slices(t_events: np.ndarray, t_frames: np.ndarray, world: int):
    """Split one stream in time for `world` ranks: rank r
    renders frames [F r / G, F (r+1) / G) and integrates the events with
    t in (b_r, b_{r+1}], b_r = the last frame time of rank r-1 (events at a frame
    time belong to that frame, reading A6).  Returns (event bounds, frame bounds)."""
    F = len(t_frames)
    fb = [F * r // world for r in range(world + 1)]
    eb = [0]
    for r in range(1, world):
        b = int(t_frames[fb[r] - 1]) if fb[r] > 0 else np.iinfo(np.int64).min
        eb.append(int(np.searchsorted(t_events, b, side="right")))
    eb.append(len(t_events))
    return eb, fb


class TimeSharded:
    """one stream sharded in time (rank order = time order).

    A time slice acts on each pixel's state through the first event's decay
    (which sees the incoming T) followed by one clamped affine map (the Eq. 5
    product of decays composes; esi.h ``esi_slice_map_t``), so:
      1. every rank summarises its slice (``esi_slice_summarize``, P x 40 B);
      2. the summaries are all-gathered (one collective; NCCL over NVLink);
      3. rank r composes the summaries of ranks < r (the exclusive scan,
         ``esi_slice_compose``) and applies it to the initial state
         (``esi_slice_apply``): its slice's incoming state;
      4. rank r integrates its slice and renders its frames.
    The handle is injectable (``handle_factory``) so the orchestration runs in
    the gloo CPU tests with an oracle-backed stand-in; the product path uses
    libesi handles (all arithmetic in its kernels)."""

    def __init__(self, width: int, height: int, group=None, handle_factory: Optional[Callable] = None, **params):
        if handle_factory is None:
            from .esi import Esi as handle_factory
        self.group = group
        init = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if init else 0
        self.world = dist.get_world_size(group) if init else 1
        self.h = handle_factory(width, height, **params)
        if torch.cuda.is_available() and hasattr(self.h, "set_stream"):
            # on torch's current stream: ordered after NCCL's all_gather of the maps
            # and visible to CUDA events recorded on that stream
            self.h.set_stream(torch.cuda.current_stream().cuda_stream)

    def close(self):
        if self.h is not None:
            self.h.close()
            self.h = None

    def incoming_state_maps(self, events_slice):
        """Steps 1-3: the exclusive prefix of the slices' maps (None on rank 0)."""
        if self.world == 1:
            return None
        maps = self.h.slice_summarize(events_slice)
        gathered = [torch.empty_like(maps) for _ in range(self.world)]
        dist.all_gather(gathered, maps, group=self.group)
        if self.rank == 0:
            return None
        pre = gathered[0]
        for s in range(1, self.rank):
            pre = self.h.slice_compose(pre, gathered[s])
        return pre

    def run(self, events_slice, t_frames_slice, out=None):
        pre = self.incoming_state_maps(events_slice)
        self.h.reset()
        if pre is not None:
            self.h.slice_apply(pre)
        rc = self.h.push(events_slice)
        if rc != 0:
            raise RuntimeError(f"push of the time slice failed (status {rc})")
        return self.h.render_many(t_frames_slice, out)

    def get_state(self):
        return self.h.get_state()
