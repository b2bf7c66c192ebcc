"""Throughput of the time-slice kernels (csrc/esi_slice.cu) on
one GPU: the c4 stream (1280x720, 10 s, ~194 M events) cut into G time slices
(dist.time_slices); per slice esi_slice_summarize (K1 band partition + K5), then
the exclusive scan of G-1 compositions (K6) and one apply (K7).  CUDA events on
the handle's stream, median of 3.  Prints one JSON line.

Algorithmic bytes: summarize 16 B per event (the packed record) + 40 B per pixel
per slice (the map written); compose 3 x 40 B per pixel; apply 40 + 24 B per pixel.
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from esi_synth import make_workload  # noqa: E402
from paper_2508_02238_b200 import Esi  # noqa: E402
from paper_2508_02238_b200.dist import time_slices  # noqa: E402


def main():
    G = int(os.environ.get("SLICES", 8))
    w = make_workload("c4", "cuda")
    tf = np.asarray(w.t_frames)
    eb, _ = time_slices(w.events[:, 0].cpu().numpy(), tf, G)
    h = Esi(w.W, w.H, **w.params)
    st = torch.cuda.Stream()
    h.set_stream(st.cuda_stream)
    maps = [h.slice_maps_empty() for _ in range(G)]
    pre = h.slice_maps_empty()

    def ev_ms(fn):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        return a.elapsed_time(b)

    def summarize():
        for r in range(G):
            h.slice_summarize(w.events[eb[r]:eb[r + 1]], maps[r])

    def scan():
        h.slice_compose(maps[0], maps[1], pre)
        for r in range(2, G):
            h.slice_compose(pre, maps[r], pre)

    def apply():
        h.reset()
        h.slice_apply(pre)

    for f in (summarize, scan, apply):
        f()
    torch.cuda.synchronize()
    t_sum = statistics.median(ev_ms(summarize) for _ in range(3))
    t_scan = statistics.median(ev_ms(scan) for _ in range(3))
    t_app = statistics.median(ev_ms(apply) for _ in range(3))
    h.close()
    peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    P = w.P
    b_sum = 16.0 * w.n + 40.0 * P * G
    b_scan = 120.0 * P * (G - 1)
    print(json.dumps({
        "workload": f"c4 stream ({w.n} events, {w.W}x{w.H}) in {G} time slices", "slices": G,
        "summarize_ms": t_sum, "summarize_events_per_s": w.n / (t_sum / 1e3),
        "summarize_gbs": b_sum / (t_sum / 1e3) / 1e9, "summarize_frac": b_sum / (t_sum / 1e3) / 1e9 / peak,
        "scan_ms": t_scan, "scan_gbs": b_scan / (t_scan / 1e3) / 1e9, "apply_ms": t_app,
        "note": "summarize includes the per-call validation pass and per-chunk host checks (esi_slice_summarize)",
        "peak_gbs": peak}))


if __name__ == "__main__":
    main()
