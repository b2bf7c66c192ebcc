"""Shared test helpers: run the CUDA path and the oracle on the same inputs."""
import numpy as np

import oracle
from esi_synth import to_numpy_struct

# tolerances of BASELINE.json north_star
S_ABS, S_REL = 1e-6, 1e-5
FRAME_FLIP_FRAC = 1e-4


def oracle_run(W, H, ev_np, t_frames, params, readout_decay=1, t_origin=0):
    return oracle.run(W, H, ev_np, t_frames, C=params["C"], k=params["k"], b=params["b"],
                      s_min=params["s_min"], s_max=params["s_max"], t_origin=t_origin,
                      readout_decay=readout_decay, decay_kind=params.get("decay_kind", 0),
                      decay_first=params.get("decay_first", 0), state_unclamped=params.get("state_unclamped", 0))


def gpu_run(W, H, events, t_frames, params, readout_decay=1, t_origin=0, chunk_events=0,
            device_events=True, device_out=True):
    import torch
    from paper_2508_02238_b200 import Esi
    e = Esi(W, H, C=params["C"], k=params["k"], b=params["b"], s_min=params["s_min"],
            s_max=params["s_max"], t_origin_us=t_origin, readout_decay=readout_decay,
            chunk_events=chunk_events, decay_kind=params.get("decay_kind", 0),
            decay_first=params.get("decay_first", 0), state_unclamped=params.get("state_unclamped", 0),
            band_layout=params.get("band_layout", 0))
    try:
        ev = events.to("cuda") if device_events else events.cpu().contiguous()
        if not device_events:
            ev = ev.numpy()
        rc = e.push(ev)
        assert rc == 0, rc
        F = len(t_frames)
        if device_out:
            out = torch.empty((F, H, W), dtype=torch.uint8, device="cuda")
            e.render_many(t_frames, out)
            frames = out.cpu().numpy()
        else:
            frames = e.render_many(t_frames)
        S, T = e.get_state()
        stats = e.last_render_stats()
        return frames, S, T, stats
    finally:
        e.close()


def assert_state_close(S_gpu, T_gpu, S_ref, T_ref):
    np.testing.assert_array_equal(T_gpu, T_ref)
    diff = np.abs(S_gpu.astype(np.float64) - S_ref)
    ok = (diff <= S_ABS) | (diff <= S_REL * np.abs(S_ref))
    assert ok.all(), f"{(~ok).sum()} pixels off, max |dS| = {diff.max():.3g}"


def assert_frames_close(f_gpu, f_ref):
    assert f_gpu.shape == f_ref.shape
    d = np.abs(f_gpu.astype(np.int16) - f_ref.astype(np.int16))
    assert d.max() <= 1, f"max frame diff {d.max()}"
    frac = (d != 0).mean() if d.size else 0.0
    assert frac <= FRAME_FLIP_FRAC, f"{frac:.3g} of pixel-frames differ by 1 LSB"
    return frac


def ev_np_of(w):
    return to_numpy_struct(w.events)
