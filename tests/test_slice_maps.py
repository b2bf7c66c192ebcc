"""time-sharded single streams through per-pixel slice maps.

CPU (-m "not gpu"): the oracle's slice maps (oracle/slice_map.py) are pinned to
the sequential oracle (Alg. 2, itself pinned in test_oracle_pins):
applying the map of a slice -- or the composition of the maps of its parts,
at every split point -- to a state gives exactly the state the event-by-event
run gives; composition is associative; the orchestration (dist.TimeSharded:
summaries, all_gather, exclusive scan, apply, integrate) runs on gloo world 2
against the full-stream oracle.
GPU (-m gpu): esi_slice_summarize / compose / apply against the oracle maps,
and a time-sharded render on one GPU (G slices in sequence) against the
full-stream oracle at the north-star tolerances.
"""
import math
import os

import numpy as np
import pytest
import torch

import oracle
from oracle import slice_map as sm

VARIANTS = [dict(), dict(decay_kind=1), dict(decay_first=1), dict(decay_kind=2), dict(state_unclamped=1),
            dict(b=0.5, k=100.0), dict(s_min=-0.4, s_max=0.3)]


def _stream(seed, W, H, n, span, hot=True):
    rng = np.random.default_rng(seed)
    t = np.sort(rng.integers(0, span, n)).astype(np.int64)
    if hot:   # equal timestamps and bursts on a few pixels, gaps around 1/k
        t[n // 3: n // 3 + 8] = t[n // 3]
    x = rng.integers(0, W, n).astype(np.uint16)
    y = rng.integers(0, H, n).astype(np.uint16)
    if hot:
        x[::5] = 1
        y[::5] = 0
    p = rng.choice(np.array([-1, 1], np.int8), n)
    a = np.zeros(n, dtype=[("t", "<i8"), ("x", "<u2"), ("y", "<u2"), ("p", "i1"), ("_pad", "u1", (3,))])
    a["t"], a["x"], a["y"], a["p"] = t, x, y, p
    return a


def _params(v):
    p = dict(C=0.15, k=10.0, b=2.0, s_min=-1.5, s_max=1.5)
    p.update(v)
    return p


def _sequential(W, H, ev, S0, T0, **params):
    o = oracle.Oracle(W, H, **params)
    assert o.set_state(S0, T0) == 0
    assert o.push(ev) == 0
    o.flush()
    S, T = o.get_state()
    o.close()
    return S.ravel(), T.ravel()


def _maps(W, ev, **params):
    return sm.slice_maps(W, None, ev["t"], ev["x"], ev["y"], ev["p"], **params)


@pytest.mark.parametrize("v", VARIANTS, ids=lambda v: ",".join(f"{k}={x}" for k, x in v.items()) or "esi")
def test_slice_map_action_equals_sequential_run_at_every_split(v):
    """apply(map(A) . map(B), S0) == Alg. 2 run over A then B, for every split point,
    from a random incoming state (T0 within and beyond the decay horizon)."""
    W, H = 4, 3
    params = _params(v)
    ev = _stream(3, W, H, 60, 400_000)
    rng = np.random.default_rng(7)
    lim = 1.0 if not (v.get("decay_kind") == 2 or v.get("state_unclamped")) else 3.0
    S0 = rng.uniform(max(params["s_min"], -lim), min(params["s_max"], lim), W * H)
    T0 = -rng.integers(0, 300_000, W * H).astype(np.int64)
    S_ref, T_ref = _sequential(W, H, ev, S0, T0, **params)
    S_m, T_m = sm.apply(_maps(W, ev, **params), S0, T0, **params)
    assert np.array_equal(T_m, T_ref)
    assert np.allclose(S_m, S_ref, rtol=1e-12, atol=1e-12)
    for cut in range(0, len(ev) + 1, 3):
        A, B = _maps(W, ev[:cut], **params), _maps(W, ev[cut:], **params)
        S_c, T_c = sm.apply(sm.compose(A, B, **params), S0, T0, **params)
        assert np.array_equal(T_c, T_ref), cut
        assert np.allclose(S_c, S_ref, rtol=1e-12, atol=1e-12), cut


def test_slice_map_composition_is_associative_and_empty_is_identity():
    W, H = 5, 2
    params = _params({})
    ev = _stream(11, W, H, 90, 600_000)
    parts = [ev[:25], ev[25:25], ev[25:70], ev[70:]]
    M = [_maps(W, p, **params) for p in parts]
    left = sm.compose(sm.compose(sm.compose(M[0], M[1], **params), M[2], **params), M[3], **params)
    right = sm.compose(M[0], sm.compose(M[1], sm.compose(M[2], M[3], **params), **params), **params)
    S0 = np.linspace(-1.2, 1.2, W * H)
    T0 = np.zeros(W * H, np.int64)
    a = sm.apply(left, S0, T0, **params)
    b = sm.apply(right, S0, T0, **params)
    assert np.array_equal(a[1], b[1]) and np.allclose(a[0], b[0], rtol=1e-12, atol=1e-13)
    assert M[1] == {}                                           # an empty slice is the identity
    Sx, Tx = sm.apply({}, S0, T0, **params)
    assert np.array_equal(Sx, S0) and np.array_equal(Tx, T0)


def test_slice_map_closed_forms():
    """Same-polarity events every dt after a fully decayed state: the geometric
    closed form S_n = C d (1 - d^n)/(1 - d) (test_oracle_pins' pin), here through
    the map (a = d^(n-1), c = sum) of the slice; a gap >= 1/k zeroes the slice's
    history (Eq. 4: d = 0, reading A14)."""
    params = _params({})
    dt = 10_000
    n = 12
    t = np.arange(1, n + 1, dtype=np.int64) * dt
    M = sm.slice_maps(1, 1, t, np.zeros(n), np.zeros(n), np.ones(n, np.int8), **params)
    d = (1 - 10.0 * dt * 1e-6) ** 2
    nn, tf, pf, G, tl = M[0]
    assert (nn, tf, pf, tl) == (n, dt, 1, n * dt)
    assert math.isclose(G[0], d ** (n - 1), rel_tol=1e-13)
    S, _ = sm.apply(M, [0.0], [0], **params)
    assert math.isclose(S[0], 0.15 * d * (1 - d ** n) / (1 - d), rel_tol=1e-12)
    gap = np.array([0, 100_000], np.int64)                      # dt = 1/k exactly
    M = sm.slice_maps(1, 1, gap, np.zeros(2), np.zeros(2), np.array([1, -1], np.int8), **params)
    S, T = sm.apply(M, [1.0], [0], **params)
    assert S[0] == 0.0 and T[0] == 100_000


class _OracleTimeHandle:
    """Oracle stand-in for a libesi handle in the gloo orchestration test (maps as float64 tensors)."""

    def __init__(self, W, H, **params):
        self.W, self.H, self.P = W, H, W * H
        self.params = params
        self.o = oracle.Oracle(W, H, **params)

    def _pack(self, M):
        n, tf, tl, pf, G = sm.to_arrays(M, self.P)
        return torch.tensor(np.column_stack([n, tf, tl, pf, G]), dtype=torch.float64)

    def _unpack(self, X):
        X = X.numpy()
        return {q: (int(X[q, 0]), int(X[q, 1]), int(X[q, 3]), tuple(X[q, 4:8]), int(X[q, 2]))
                for q in range(self.P) if X[q, 0] > 0}

    def slice_summarize(self, ev):
        return self._pack(_maps(self.W, ev, **self.params))

    def slice_compose(self, A, B):
        return self._pack(sm.compose(self._unpack(A), self._unpack(B), **self.params))

    def slice_apply(self, X):
        S, T = self.o.get_state()
        S, T = sm.apply(self._unpack(X), S, T, **self.params)
        self.o.set_state(S, T)

    def reset(self):
        self.o.reset()

    def push(self, ev):
        return self.o.push(ev)

    def render_many(self, tf, out=None):
        return self.o.render_many(tf)

    def get_state(self):
        return self.o.get_state()

    def close(self):
        self.o.close()


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2508_02238_b200.dist import TimeSharded, time_slices
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W, H = 6, 5
        ev = _stream(21, W, H, 400, 300_000)
        tf = np.arange(1, 31, dtype=np.int64) * 10_000
        eb, fb = time_slices(ev["t"], tf, world)
        ts = TimeSharded(W, H, handle_factory=_OracleTimeHandle)
        fr = ts.run(ev[eb[rank]:eb[rank + 1]], tf[fb[rank]:fb[rank + 1]])
        S, T = ts.get_state()
        ts.close()
        q.put((rank, fr, S, T))
    finally:
        dist.destroy_process_group()


def test_time_sharded_gloo_world2_equals_full_stream():
    import torch.multiprocessing as mp
    from paper_2508_02238_b200.dist import time_slices
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (f, S, T)) for r, f, S, T in (q.get(timeout=120) for _ in range(2)))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    W, H = 6, 5
    ev = _stream(21, W, H, 400, 300_000)
    tf = np.arange(1, 31, dtype=np.int64) * 10_000
    f_ref, S_ref, T_ref = oracle.run(W, H, ev, tf)
    eb, fb = time_slices(ev["t"], tf, 2)
    assert np.array_equal(np.concatenate([res[0][0], res[1][0]]), f_ref)
    assert np.array_equal(res[1][2], T_ref)
    assert np.allclose(res[1][1], S_ref, rtol=1e-12, atol=1e-12)
    assert 0 < eb[1] < len(ev) and fb[1] == 15


# ---------------------------------------------------------------------- GPU
def _gpu_maps_to_np(X):
    from paper_2508_02238_b200.esi import SLICE_MAP_DTYPE
    return X.cpu().numpy().view(SLICE_MAP_DTYPE).reshape(-1)


@pytest.mark.gpu
@pytest.mark.parametrize("v", VARIANTS[:4], ids=["esi", "exp", "decay_first", "naive"])
def test_gpu_slice_summary_matches_oracle_maps(v):
    from esi_synth import make_workload, to_numpy_struct
    from paper_2508_02238_b200 import Esi
    w = make_workload("c2", "cpu", duration_us=300_000)
    ev = to_numpy_struct(w.events)
    params = dict(w.params)
    params.update(v)
    h = Esi(w.W, w.H, **params)
    try:
        X = _gpu_maps_to_np(h.slice_summarize(w.events.cuda()))
    finally:
        h.close()
    keep = ("C", "k", "b", "s_min", "s_max", "decay_kind", "decay_first", "state_unclamped")
    n, tf, tl, pf, G = sm.to_arrays(_maps(w.W, ev, **{k: x for k, x in params.items() if k in keep}), w.P)
    assert np.array_equal(X["n"], n)
    m = n > 0
    assert np.array_equal(X["t_first"][m], tf[m]) and np.array_equal(X["t_last"][m], tl[m])
    assert np.array_equal(X["p_first"][m], pf[m])
    m2 = n > 1
    for j, f in enumerate(("a", "c")):
        ref = G[m2, j]
        assert np.all(np.abs(X[f][m2] - ref) <= 1e-6 + 1e-5 * np.abs(ref)), f


@pytest.mark.gpu
@pytest.mark.parametrize("G_,layout", [(2, 0), (3, 0), (5, 0), (3, 1)])
def test_gpu_time_sharded_render_equals_full_stream(G_, layout):
    """G time shards processed in sequence on one GPU, each from the composed maps
    of the earlier shards (esi_slice_summarize / compose / apply), against the
    full-stream oracle: frames within +-1 on <= 0.01 % of pixel-frames, state
    within the fp32 tolerance, T exact."""
    from esi_synth import make_workload, to_numpy_struct
    from paper_2508_02238_b200 import Esi
    from paper_2508_02238_b200.dist import time_slices
    w = make_workload("c2", "cpu", duration_us=600_000)
    ev = to_numpy_struct(w.events)
    tf = np.asarray(w.t_frames)
    f_ref, S_ref, T_ref = oracle.run(w.W, w.H, ev, tf, **w.params)
    eb, fb = time_slices(ev["t"], tf, G_)
    dev = w.events.cuda()
    h = Esi(w.W, w.H, band_layout=layout, **w.params)      # layout 1: interleaved bands (K5's map addressing)
    try:
        maps = [h.slice_summarize(dev[eb[r]:eb[r + 1]]) for r in range(G_)]
        frames = []
        for r in range(G_):
            h.reset()
            if r > 0:
                pre = maps[0].clone()
                for s in range(1, r):
                    pre = h.slice_compose(pre, maps[s])
                h.slice_apply(pre)
            assert h.push(dev[eb[r]:eb[r + 1]]) == 0
            out = torch.empty((fb[r + 1] - fb[r], w.H, w.W), dtype=torch.uint8, device="cuda")
            h.render_many(tf[fb[r]:fb[r + 1]], out)
            frames.append(out.cpu().numpy())
        S, T = h.get_state()
    finally:
        h.close()
    fr = np.concatenate(frames)
    d = np.abs(fr.astype(int) - f_ref.astype(int))
    assert d.max() <= 1 and (d != 0).mean() <= 1e-4, (d.max(), (d != 0).mean())
    assert np.array_equal(T, T_ref)
    assert np.all(np.abs(S - S_ref) <= np.maximum(1e-6, 1e-5 * np.abs(S_ref)))


@pytest.mark.gpu
def test_gpu_slice_rejects_invalid_events_and_pending_apply():
    from paper_2508_02238_b200 import Esi, esi
    ev = np.zeros(3, dtype=esi.EVENT_DTYPE)
    ev["t"] = [5, 4, 6]                                        # t goes back
    ev["p"] = 1
    h = Esi(8, 8)
    try:
        with pytest.raises(esi.EsiError) as e:
            h.slice_summarize(torch.from_numpy(ev.view(np.uint8)).cuda())
        assert e.value.code == esi.ESI_ERR_NEGATIVE_INTERVAL
        ok = ev.copy()
        ok["t"] = [1, 2, 3]
        m = h.slice_summarize(torch.from_numpy(ok.view(np.uint8)).cuda())
        assert h.push(torch.from_numpy(ok.view(np.uint8)).cuda()) == 0
        with pytest.raises(esi.EsiError) as e:
            h.slice_apply(m)                                   # events pending
        assert e.value.code == esi.ESI_ERR_INVALID_ARG
    finally:
        h.close()
