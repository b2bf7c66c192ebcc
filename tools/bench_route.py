"""Throughput of the multi-GPU row-band router (csrc/esi_route.cu) on one GPU:
a 2560x1440 stream (config 5b shape: 80 Mev/s -> one 1 s shard of 80 M events)
routed into G = 8 row bands through the product path's router object
(esi_router_create / count / scatter; scratch allocated once and kept).

Timed with CUDA events on the router's stream, median of `REPS` calls:
* scatter: the stream-ordered scatter kernel alone (no host sync inside);
* count: the histogram + scan kernels plus the API's 8-count read-back and
  stream sync (the host needs the counts to place the runs);
* both: count + scatter back to back.
Algorithmic bytes per event: 16 B read by the histogram pass, 16 B read + 16 B
written by the scatter pass (48 B in total; 32 B for the scatter alone).
Prints one JSON line.
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2508_02238_b200.dist import PeerTransport, row_bands  # noqa: E402


def main():
    W, H, G = 2560, 1440, 8
    n = int(os.environ.get("ROUTE_EVENTS", 80_000_000))
    reps = int(os.environ.get("ROUTE_REPS", 7))
    g = torch.Generator(device="cuda").manual_seed(5)
    t = torch.sort(torch.randint(0, 1_000_000, (n,), generator=g, device="cuda", dtype=torch.int64)).values
    x = torch.randint(0, W, (n,), generator=g, device="cuda", dtype=torch.int64)
    y = torch.randint(0, H, (n,), generator=g, device="cuda", dtype=torch.int64)
    p = torch.where(torch.rand(n, generator=g, device="cuda") < 0.5, 1, 255).to(torch.int64)
    ev = torch.stack([t, x | (y << 16) | (p << 32)], 1).contiguous()
    del t, x, y, p
    out = torch.empty_like(ev)
    stream = torch.cuda.Stream()
    tr = PeerTransport(0, H, row_bands(H, G), stream=stream.cuda_stream)

    def ev_pair():
        return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    counts = tr.count(ev)
    offs = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
    dst = [out.data_ptr()] * G
    for _ in range(2):
        tr.count(ev)
        tr.scatter(dst, offs)
    tr.sync()
    t_cnt, t_sc, t_both = [], [], []
    for _ in range(reps):
        a, b = ev_pair()
        a.record(stream)
        tr.count(ev)                      # synchronises the stream (counts read back)
        b.record(stream)
        b.synchronize()
        t_cnt.append(a.elapsed_time(b))
        a, b = ev_pair()
        a.record(stream)
        tr.scatter(dst, offs)
        b.record(stream)
        b.synchronize()
        t_sc.append(a.elapsed_time(b))
        a, b = ev_pair()
        a.record(stream)
        tr.count(ev)
        tr.scatter(dst, offs)
        b.record(stream)
        b.synchronize()
        t_both.append(a.elapsed_time(b))
    tr.close()
    ms_c, ms_s, ms_b = (statistics.median(v) for v in (t_cnt, t_sc, t_both))
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    gbs = lambda b, ms: b * n / (ms / 1e3) / 1e9
    print(json.dumps({
        "kernel": "esi_router (count: hist + scan; scatter: stable ballot multi-split)", "events": n, "bands": G,
        "sensor": f"{W}x{H}", "reps": reps, "timing": "CUDA events on the router stream, median",
        "count_ms": ms_c, "scatter_ms": ms_s, "count_plus_scatter_ms": ms_b,
        "events_per_s": n / (ms_b / 1e3), "algorithmic_bytes_per_event": 48,
        "achieved_gbs": gbs(48, ms_b), "scatter_gbs": gbs(32, ms_s), "count_gbs": gbs(16, ms_c),
        "peak_gbs": peak, "frac": gbs(48, ms_b) / peak, "scatter_frac": gbs(32, ms_s) / peak,
        "counts": [int(c) for c in counts],
        "samples_ms": {"count": t_cnt, "scatter": t_sc, "both": t_both}}))


if __name__ == "__main__":
    main()
