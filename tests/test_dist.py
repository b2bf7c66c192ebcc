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

    def close(self):
        self.o.close()


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
