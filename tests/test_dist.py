"""Multi-GPU sharding.

CPU (gloo, world_size 2): the host logic of paper_2508_02238_b200.dist --
time sharding, routing plan, all-to-all exchange, band rendering, all-gather
assembly -- with each rank's band integrated by the fp64 oracle (test
infrastructure) and a plain stable partition as router; the assembled frames
must equal the full-sensor oracle bit for bit (pixels are independent, so a
band sees exactly its pixels' events in arrival order).
GPU: the device router (esi_route_bands) is bit-exact against a stable sort by
band, and G band handles on one GPU reproduce the full-sensor handle.
"""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from esi_synth import from_numpy_struct, to_numpy_struct
from paper_2508_02238_b200.dist import RowBandSharded, StreamSharded, row_bands, time_shard_bounds

PRM = {"C": 0.15, "k": 10.0, "b": 2.0, "s_min": -1.5, "s_max": 1.5}


class OracleBand:
    """Band handle backed by the oracle (same call surface as Esi)."""

    def __init__(self, w, h, C, k, b, s_min, s_max, t_origin_us=0, readout_decay=1):
        self.o = oracle.Oracle(w, h, C=C, k=k, b=b, s_min=s_min, s_max=s_max, t_origin=t_origin_us,
                               readout_decay=readout_decay)

    def push(self, ev):
        return self.o.push(to_numpy_struct(ev)) if ev.shape[0] else 0

    def render_many(self, tf, out):
        out.copy_(torch.from_numpy(self.o.render_many(tf)))
        return out

    def get_state(self):
        return self.o.get_state()

    def pending(self):
        return self.o.pending()

    def close(self):
        self.o.close()


class FileTransport:
    """Stand-in for PeerTransport between CPU processes: receive arenas are
    files mapped by every rank (np.memmap), "P2P stores" are writes into the
    destination rank's mapping, and the router is the plain stable partition.
    It exercises RowBandSharded's P2P host logic -- counts all-gather, receive
    offsets, arena growth and handle exchange, recycling after a render."""

    def __init__(self, root, rank, starts):
        self.root, self.rank, self.starts = root, rank, starts
        self.k = 0
        self.routed = None
        self.maps = {}
        self.log = []

    def _map(self, path):
        if path not in self.maps:
            self.maps[path] = np.memmap(path, dtype=np.int64, mode="r+").reshape(-1, 2)
        return self.maps[path]

    def count(self, shard):
        routed, counts = np_router(shard, self.starts)
        self.routed = (routed.numpy(), np.concatenate([[0], np.cumsum(counts)]))
        return counts

    def scatter(self, dst, off):
        rec, cs = self.routed
        for g, path in enumerate(dst):
            n = cs[g + 1] - cs[g]
            if n:
                m = self._map(path)
                assert off[g] + n <= m.shape[0], "write past the destination arena"
                m[off[g]:off[g] + n] = rec[cs[g]:cs[g + 1]]
        self.log.append(("scatter", list(off)))

    def sync(self):
        for m in self.maps.values():
            m.flush()

    def alloc(self, nrec):
        path = os.path.join(self.root, f"arena_{self.rank}_{self.k}.bin")
        self.k += 1
        np.memmap(path, dtype=np.int64, mode="w+", shape=(nrec, 2)).flush()
        self.log.append(("alloc", nrec))
        return path

    def free(self, path):
        self.maps.pop(path, None)
        os.remove(path)

    def export(self, path):
        return path

    def open(self, handle):
        return handle

    def unmap(self, path):
        self.maps.pop(path, None)

    def push(self, band, path, off, n):
        if not n:
            return 0
        m = np.memmap(path, dtype=np.int64, mode="r").reshape(-1, 2)
        return band.push(torch.from_numpy(np.array(m[off:off + n])))

    def close(self):
        self.maps = {}


def np_router(events, starts):
    """Plain stable partition by row band with y rebased (definition of esi_route_bands)."""
    a = to_numpy_struct(events).copy()
    band = np.searchsorted(np.asarray(starts), a["y"].astype(np.int64), side="right") - 1
    order = oracle.stable_group_by(band)
    out = a[order]
    out["y"] = (out["y"].astype(np.int64) - np.asarray(starts)[band[order]]).astype(np.uint16)
    counts = np.bincount(band, minlength=len(starts) - 1).astype(np.int64)
    return from_numpy_struct(out), counts


def stream(seed, W, H, n, span):
    rng = np.random.default_rng(seed)
    a = np.zeros(n, dtype=[("t", "<i8"), ("x", "<u2"), ("y", "<u2"), ("p", "i1"), ("_pad", "u1", (3,))])
    a["t"] = np.sort(rng.integers(0, span, n))
    a["x"] = rng.integers(0, W, n)
    a["y"] = rng.integers(0, H, n)
    a["p"] = rng.choice([-1, 1], n)
    return a


def test_row_bands_and_time_shards():
    assert row_bands(1440, 8) == [0, 180, 360, 540, 720, 900, 1080, 1260, 1440]
    assert row_bands(7, 3) == [0, 3, 6, 7]
    assert row_bands(5, 1) == [0, 5]
    with pytest.raises(ValueError):
        row_bands(2, 3)
    with pytest.raises(ValueError):
        row_bands(10, 4)            # ceil(10/4) = 3 -> bands 3,3,3,1 is fine; 9,4 is not
        row_bands(9, 4)
    assert time_shard_bounds(10, 3) == [0, 3, 6, 10]


def test_np_router_is_stable_partition():
    a = stream(1, 16, 10, 500, 10_000)
    ev = from_numpy_struct(a)
    starts = row_bands(10, 3)
    routed, counts = np_router(ev, starts)
    r = to_numpy_struct(routed)
    assert counts.sum() == 500
    off = 0
    for b in range(3):
        seg = r[off:off + counts[b]]
        m = (a["y"] >= starts[b]) & (a["y"] < starts[b + 1])
        exp = a[m].copy()
        exp["y"] -= starts[b]
        assert np.array_equal(seg, exp)
        off += counts[b]


def _worker(rank, world, path, W, H, a, tf, q):
    dist.init_process_group("gloo", init_method=f"file://{path}", rank=rank, world_size=world)
    try:
        rb = RowBandSharded(W, H, band_factory=OracleBand, router=np_router, device=torch.device("cpu"), **PRM)
        # two collective rounds (packets): round k covers a time slice of the stream,
        # split among the ranks in rank order
        half = len(a) // 2
        for base, part in ((0, a[:half]), (half, a[half:])):
            lo, hi = time_shard_bounds(len(part), world)[rank:rank + 2]
            assert rb.push_shard(from_numpy_struct(part[lo:hi])) == 0
        frames = rb.render_many(tf)
        q.put((rank, frames.numpy(), rb.stats))
        rb.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("W,H", [(20, 12), (9, 7)])
def test_row_band_sharding_gloo_world2_equals_full_sensor(W, H):
    a = stream(3, W, H, 6000, 300_000)
    tf = np.arange(1, 31, dtype=np.int64) * 10_000
    f_ref, _, _ = oracle.run(W, H, a, tf, **PRM)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    path = tempfile.mktemp()
    procs = [ctx.Process(target=_worker, args=(r, 2, path, W, H, a, tf, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, frames, stats in res:
        assert np.array_equal(frames, f_ref), f"rank {rank}: assembled frames differ from the full sensor"
        assert stats["received"] > 0 and stats["sent"] > 0


def _worker_p2p(rank, world, path, root, W, H, a, tf_list, q):
    dist.init_process_group("gloo", init_method=f"file://{path}", rank=rank, world_size=world)
    try:
        T = FileTransport(root, rank, row_bands(H, world))
        rb = RowBandSharded(W, H, band_factory=OracleBand, transport=T, device=torch.device("cpu"), **PRM)
        rb.MIN_ARENA = 64                                  # force arena growth and re-exchange of handles
        frames = []
        # rounds of different sizes, two renders (the second reuses the recycled arenas)
        bounds = [0, 300, 350, 1800, 3000, 3100, 6000]
        for k in range(len(bounds) - 1):
            part = a[bounds[k]:bounds[k + 1]]
            lo, hi = time_shard_bounds(len(part), world)[rank:rank + 2]
            assert rb.push_shard(from_numpy_struct(part[lo:hi])) == 0
            if bounds[k + 1] == 3000:
                frames.append(rb.render_many(tf_list[0]).numpy())
        frames.append(rb.render_many(tf_list[1]).numpy())
        q.put((rank, frames, rb.stats, T.log))
        rb.close()
    finally:
        dist.destroy_process_group()


def test_row_band_p2p_exchange_gloo_world2_equals_full_sensor(tmp_path):
    W, H = 16, 11
    a = stream(7, W, H, 6000, 300_000)
    t_split = int(a["t"][2999])
    tf_all = np.arange(1, 31, dtype=np.int64) * 10_000
    tf0 = tf_all[tf_all < t_split]                     # first render: frames before round 4's events
    tf1 = tf_all[tf_all >= int(a["t"][3099]) + 1]
    f_ref, _, _ = oracle.run(W, H, a, np.concatenate([tf0, tf1]), **PRM)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    path = tempfile.mktemp()
    procs = [ctx.Process(target=_worker_p2p, args=(r, 2, path, str(tmp_path), W, H, a, (tf0, tf1), q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, frames, stats, log in res:
        got = np.concatenate(frames)
        assert np.array_equal(got, f_ref), f"rank {rank}: P2P-exchanged frames differ from the full sensor"
        assert stats["received"] > 0 and stats["sent"] > 0
        assert sum(1 for e in log if e[0] == "alloc") >= 2, "arena growth path not exercised"


def _worker_streams(rank, world, path, q):
    dist.init_process_group("gloo", init_method=f"file://{path}", rank=rank, world_size=world)
    try:
        specs = [(8, 6, PRM)] * 5
        ss = StreamSharded(specs, handle_factory=OracleBand)
        out = {}
        tf = np.arange(1, 11, dtype=np.int64) * 10_000
        for s in ss.owned:
            ss.push(s, from_numpy_struct(stream(100 + s, 8, 6, 400, 100_000)))
            out[s] = ss.render_many(s, tf, torch.empty((10, 6, 8), dtype=torch.uint8)).numpy()
        q.put((rank, out))
        ss.close()
    finally:
        dist.destroy_process_group()


def test_stream_sharding_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    path = tempfile.mktemp()
    procs = [ctx.Process(target=_worker_streams, args=(r, 2, path, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(res[0]) == [0, 2, 4] and sorted(res[1]) == [1, 3]
    tf = np.arange(1, 11, dtype=np.int64) * 10_000
    for r in (0, 1):
        for s, fr in res[r].items():
            ref, _, _ = oracle.run(8, 6, stream(100 + s, 8, 6, 400, 100_000), tf, **PRM)
            assert np.array_equal(fr, ref)


# ----------------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("G", [1, 2, 3, 8, 64])
def test_device_router_bit_exact(G):
    from paper_2508_02238_b200.dist import device_router
    W, H = 300, 128
    a = stream(7 + G, W, H, 200_000, 1_000_000)
    ev = from_numpy_struct(a).cuda()
    starts = row_bands(H, G)
    routed, counts = device_router(0, H)(ev, starts)
    torch.cuda.synchronize()
    r_ref, c_ref = np_router(from_numpy_struct(a), starts)
    assert np.array_equal(counts, c_ref)
    assert torch.equal(routed.cpu(), r_ref)


@pytest.mark.gpu
def test_device_router_rejects_out_of_bounds_rows():
    from paper_2508_02238_b200.dist import device_router
    from paper_2508_02238_b200 import EsiError
    a = stream(9, 10, 10, 1000, 10_000)
    a["y"][500] = 10
    with pytest.raises(EsiError):
        device_router(0, 10)(from_numpy_struct(a).cuda(), row_bands(10, 2))


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 4])
def test_band_handles_on_one_gpu_equal_full_sensor(G):
    """G band handles (height H/G, events routed by the device router) on one
    GPU, frames stacked by rows: equal to one full-sensor handle -- bit-exact
    on a stream whose pixels get at most one event per frame window (sparse
    path), within tolerance otherwise (dense batches depend on the band layout)."""
    from paper_2508_02238_b200 import Esi
    from paper_2508_02238_b200.dist import device_router
    from helpers import assert_frames_close, assert_state_close
    W, H, F = 64, 48, 30
    tf = np.arange(1, F + 1, dtype=np.int64) * 10_000
    rng = np.random.default_rng(G)
    rows = []
    for j in range(F):
        pix = rng.choice(W * H, 1000, replace=False)
        ts = np.sort(rng.integers(j * 10_000 + 1, (j + 1) * 10_000 + 1, 1000))
        rows += [(int(t), int(q % W), int(q // W), int(rng.choice([-1, 1]))) for q, t in zip(pix, ts)]
    rows.sort(key=lambda r: r[0])
    sparse = np.zeros(len(rows), dtype=[("t", "<i8"), ("x", "<u2"), ("y", "<u2"), ("p", "i1"), ("_pad", "u1", (3,))])
    for i, r in enumerate(rows):
        sparse[i]["t"], sparse[i]["x"], sparse[i]["y"], sparse[i]["p"] = r
    for a, exact in ((sparse, True), (stream(5, W, H, 100_000, 300_000), False)):
        ev = from_numpy_struct(a).cuda()
        full = Esi(W, H, **PRM)
        full.push(ev)
        f_full = full.render_many(tf)
        S_full, T_full = full.get_state()
        full.close()
        starts = row_bands(H, G)
        routed, counts = device_router(0, H)(ev, starts)
        off = 0
        parts, Ss, Ts = [], [], []
        for b in range(G):
            h = Esi(W, starts[b + 1] - starts[b], **PRM)
            seg = routed[off:off + int(counts[b])].contiguous()
            off += int(counts[b])
            assert h.push(seg) == 0
            parts.append(h.render_many(tf))
            S, T = h.get_state()
            Ss.append(S); Ts.append(T)
            h.close()
        f_bands = np.concatenate(parts, axis=1)
        S_b, T_b = np.concatenate(Ss), np.concatenate(Ts)
        if exact:
            assert np.array_equal(f_bands, f_full)
            assert np.array_equal(S_b, S_full) and np.array_equal(T_b, T_full)
        else:
            assert_frames_close(f_bands, f_full)
            assert_state_close(S_b, T_b, S_full.astype(np.float64), T_full)


@pytest.mark.gpu
@pytest.mark.parametrize("G,S", [(2, 2), (4, 3), (8, 8)])
def test_p2p_router_scatter_into_band_arenas(G, S):
    """The P2P exchange kernel on one GPU: S time shards ("source ranks"), each
    counted and scattered by esi_router_* straight into G per-band arenas at
    the offsets RowBandSharded computes (fill + events of earlier sources).
    Every arena must hold its band's events in arrival order, y rebased: the
    stable partition of the whole stream (bit-exact).  On the GPU box the
    arenas of other ranks are IPC mappings; the kernel is the same."""
    from paper_2508_02238_b200.dist import PeerTransport
    W, H = 200, 96
    a = stream(40 + G, W, H, 150_000, 1_000_000)
    starts = row_bands(H, G)
    ev = from_numpy_struct(a).cuda()
    bounds = time_shard_bounds(len(a), S)
    T = PeerTransport(0, H, starts)
    ref, c_ref = np_router(from_numpy_struct(a), starts)
    pad = 5                                                    # arenas start with some fill
    bufs = [torch.full((int(c_ref[g]) + pad, 2), -1, dtype=torch.int64, device="cuda") for g in range(G)]
    arenas = [b.data_ptr() for b in bufs]
    torch.cuda.synchronize()
    M = []
    for s in range(S):
        M.append(T.count(ev[bounds[s]:bounds[s + 1]]))
        off = np.array([pad + sum(int(M[q][g]) for q in range(s)) for g in range(G)], np.int64)
        T.scatter(arenas, off)
        T.sync()
    assert np.array_equal(np.sum(M, axis=0), c_ref)
    cs = np.concatenate([[0], np.cumsum(c_ref)])
    for g in range(G):
        got = bufs[g].cpu()
        assert torch.equal(got[:pad], torch.full((pad, 2), -1, dtype=torch.int64)), f"band {g}: prefix touched"
        assert torch.equal(got[pad:], ref[cs[g]:cs[g + 1]]), f"band {g}"
    T.close()


@pytest.mark.gpu
def test_ipc_export_of_arena():
    from paper_2508_02238_b200.dist import PeerTransport
    T = PeerTransport(0, 8, row_bands(8, 2))
    p = T.alloc(1024)
    h = T.export(p)
    assert isinstance(h, bytes) and len(h) == 64 and any(h)
    T.free(p)
    T.close()


@pytest.mark.gpu
def test_borrowed_buffers_kept_while_pending():
    """Device pushes are borrowed (esi.h): the wrapper keeps the tensor alive
    while any of its events is still pending after a render."""
    from paper_2508_02238_b200 import Esi
    e = Esi(16, 8, **PRM)
    a = stream(3, 16, 8, 1000, 100_000)
    ev = from_numpy_struct(a).cuda()
    assert e.push(ev) == 0
    e.render_many(np.array([50_000], np.int64))
    assert e.pending() > 0 and len(e._borrowed) == 1
    e.render_many(np.array([100_000], np.int64))
    assert e.pending() == 0 and len(e._borrowed) == 0
    e.close()


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(12))
def test_p2p_router_random_sweep(seed):
    """Random sensors, band counts (1..64), shard counts and arena fills: the
    router's count + scatter into per-band arenas equals the stable partition
    of the whole stream (bit-exact), and bytes outside each run are untouched."""
    from paper_2508_02238_b200.dist import PeerTransport
    rng = np.random.default_rng(500 + seed)
    H = int(rng.integers(1, 300))
    W = int(rng.integers(1, 500))
    G = int(rng.integers(1, min(64, H) + 1))
    S = int(rng.integers(1, 6))
    n = int(rng.choice([0, 1, 1000, 40_000, 300_000]))
    a = stream(600 + seed, W, H, n, 2_000_000)
    starts = row_bands(H, G) if H % G == 0 or -(-H // G) * (G - 1) < H else [round(H * g / G) for g in range(G + 1)]
    starts = sorted(set(starts))
    G = len(starts) - 1
    ev = from_numpy_struct(a).cuda()
    bounds = time_shard_bounds(len(a), S)
    T = PeerTransport(0, H, starts)
    ref, c_ref = np_router(from_numpy_struct(a), starts)
    pad = [int(rng.integers(0, 9)) for _ in range(G)]
    bufs = [torch.full((int(c_ref[g]) + pad[g] + 3, 2), -7, dtype=torch.int64, device="cuda") for g in range(G)]
    torch.cuda.synchronize()
    M = []
    for s in range(S):
        M.append(T.count(ev[bounds[s]:bounds[s + 1]]))
        off = np.array([pad[g] + sum(int(M[q][g]) for q in range(s)) for g in range(G)], np.int64)
        T.scatter([b.data_ptr() for b in bufs], off)
        T.sync()
    cs = np.concatenate([[0], np.cumsum(c_ref)])
    for g in range(G):
        got = bufs[g].cpu()
        assert torch.equal(got[:pad[g]], torch.full((pad[g], 2), -7, dtype=torch.int64))
        assert torch.equal(got[pad[g]:pad[g] + int(c_ref[g])], ref[cs[g]:cs[g + 1]]), f"band {g}"
        assert torch.equal(got[pad[g] + int(c_ref[g]):], torch.full((3, 2), -7, dtype=torch.int64))
    T.close()
