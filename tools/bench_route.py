"""Throughput of the multi-GPU row-band router (esi_route_bands, csrc/esi_route.cu)
on one GPU: a 2560x1440 stream (config 5b shape: 80 Mev/s -> one 1 s shard of
80 M events) routed into G = 8 row bands.  Prints one JSON line.

Algorithmic bytes per event: 16 B read (histogram pass) + 16 B read + 16 B
written (scatter pass) = 48 B.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2508_02238_b200.dist import device_router, row_bands  # noqa: E402


def main():
    W, H, G = 2560, 1440, 8
    n = int(os.environ.get("ROUTE_EVENTS", 80_000_000))
    g = torch.Generator(device="cuda").manual_seed(5)
    t = torch.sort(torch.randint(0, 1_000_000, (n,), generator=g, device="cuda", dtype=torch.int64)).values
    x = torch.randint(0, W, (n,), generator=g, device="cuda", dtype=torch.int64)
    y = torch.randint(0, H, (n,), generator=g, device="cuda", dtype=torch.int64)
    p = torch.where(torch.rand(n, generator=g, device="cuda") < 0.5, 1, 255).to(torch.int64)
    ev = torch.stack([t, x | (y << 16) | (p << 32)], 1).contiguous()
    del t, x, y, p
    route = device_router(0, H)
    starts = row_bands(H, G)
    for _ in range(3):
        route(ev, starts)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        out, counts = route(ev, starts)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    gbs = 48.0 * n / (ms / 1e3) / 1e9
    print(json.dumps({"kernel": "esi_route_bands (hist + scan + stable scatter)", "events": n, "bands": G,
                      "sensor": f"{W}x{H}", "ms_per_call": ms, "events_per_s": n / (ms / 1e3),
                      "algorithmic_bytes_per_event": 48, "achieved_gbs": gbs, "peak_gbs": peak,
                      "frac": gbs / peak, "counts": [int(c) for c in counts],
                      "note": "includes the host-synchronous counts read-back of each call"}))


if __name__ == "__main__":
    main()
