"""Throughput of the hot path on every single-GPU BASELINE config (device-resident
inputs, frames into HBM, CUDA-event timing, median of 5 runs after 2 warm-ups).
Prints one JSON line per config.

    python tools/bench_configs.py [c1 c2 c3 c4 c4@1000]
    python tools/bench_configs.py c4:decay_kind=1 c4:decay_first=1 c4:decay_kind=2 c4:state_unclamped=1

`name:key=value,...` runs the config with ESI parameters overridden (the decay
variants of reading A20: exp decay and decay-then-add run on the fast fp32
kernel, the naive Eq. 2 integrator and the unclamped state on the fp64 one).
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from esi_synth import make_workload, frame_times  # noqa: E402
from paper_2508_02238_b200 import Esi  # noqa: E402


def run(name, fps=100, over=None):
    t0 = time.time()
    w = make_workload(name, "cuda", fps=fps) if name == "c4" else make_workload(name, "cpu")
    w.events = w.events.cuda()
    gen_s = time.time() - t0
    tf = w.t_frames if name == "c4" else frame_times(w.duration_us, fps)
    F = len(tf)
    params = dict(w.params)
    params.update(over or {})
    e = Esi(w.W, w.H, **params)
    out = torch.empty((F, w.H, w.W), dtype=torch.uint8, device="cuda")
    st = torch.cuda.Stream()
    e.set_stream(st.cuda_stream)

    def step():
        e.reset()
        assert e.push(w.events) == 0
        e.render_many(tf, out)

    for _ in range(2):
        step()
    times = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        step()
        b.record(st)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    ms = float(np.median(times))
    stats = e.last_render_stats()
    e.close()
    alg = 16.0 * w.n + w.P * F + 24.0 * w.P * max(1, stats["chunks"])
    return {"config": name, "fps": fps, "params": over or {}, "sensor": f"{w.W}x{w.H}", "events": w.n, "frames": F,
            "ms": ms, "events_per_s": w.n / (ms / 1e3), "frames_per_s": F / (ms / 1e3),
            "step_hbm_frac": alg / (ms / 1e3) / 6546.6e9, "chunks": stats["chunks"], "generation_s": gen_s}


def main():
    names = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c4@1000"]
    for n in names:
        n, _, ov = n.partition(":")
        name, _, fps = n.partition("@")
        over = {k: (float(v) if "." in v else int(v)) for k, v in (kv.split("=") for kv in ov.split(",") if kv)}
        print(json.dumps(run(name, int(fps) if fps else 100, over)), flush=True)


if __name__ == "__main__":
    main()
