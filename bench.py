#!/usr/bin/env python
"""ESI hot-path benchmark (BASELINE.json metric: events/s integrated and frames/s
at 1280x720 @100 FPS, % of the HBM roofline).

One step = one pass of the whole hot path over one batch of synthetic input:
reset the handle, push the c4 stream (200 M events, already in HBM, borrowed
zero-copy), render its 1000 frames @100 FPS into HBM.  The stream (3.2 GB) and
the frames (0.92 GB) are far larger than L2, so no flush is needed between
steps.  N > 1 GPUs (torchrun): every rank integrates its own independent c4
stream (stream sharding, config 5a style), no data-path collective; value =
all ranks' events / max-over-ranks time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {esi,reference}]
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "events/s integrated and frames/s at 1280x720@100FPS, 1/2/4/8 B200, % HBM roofline"
UNIT = "events/s"


def load_json(path, default=None):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return default


def dist_setup(n_gpus):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        t0, t1 = getattr(self, "window", (0, 1e30))
        for ts, ln in self.lines:
            if not (t0 <= ts <= t1 + 0.15):
                continue
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); mx.append(float(f[2]))
            except ValueError:
                continue
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


def workload_for(rank, args):
    from esi_synth import make_workload
    seed = 4 + 1000 * rank       # rank 0 = the c4 stream; other ranks: independent streams
    t0 = time.time()
    w = make_workload("c4", "cuda", seed=seed, fps=args.fps)
    torch.cuda.synchronize()
    return w, time.time() - t0


def cpu_baseline(w, sample_s):
    """The oracle (as it stands, single thread) on the first sample_s seconds of the stream."""
    import oracle
    from esi_synth import to_numpy_struct
    tmax = int(sample_s * 1e6)
    t_all = w.events[:, 0]
    n = int(torch.searchsorted(t_all, torch.tensor([tmax], device=t_all.device), right=True).item())
    ev = to_numpy_struct(w.events[:n])
    tf = w.t_frames[w.t_frames <= tmax]
    t0 = time.perf_counter()
    oracle.run(w.W, w.H, ev, tf, **w.params)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"first {sample_s:g} s of the c4 stream: {n} events, {len(tf)} frames of 1280x720",
            "frames_per_s": len(tf) / dt, "seconds": dt}


def run_reference(args, rank, world):
    """--impl reference: the fp64 oracle timed on host cores (rank 0 only)."""
    if rank != 0:
        return
    from esi_synth import make_workload
    w = make_workload("c4", "cuda", seed=4, fps=args.fps)
    import oracle
    from esi_synth import to_numpy_struct
    tmax = int(args.ref_sample_s * 1e6)
    n = int(torch.searchsorted(w.events[:, 0], torch.tensor([tmax], device="cuda"), right=True).item())
    ev = to_numpy_struct(w.events[:n])
    tf = w.t_frames[w.t_frames <= tmax]
    for _ in range(args.warmup):
        oracle.run(w.W, w.H, ev[: max(1, n // 20)], tf[: max(1, len(tf) // 20)], **w.params)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.run(w.W, w.H, ev, tf, **w.params)
        times.append(time.perf_counter() - t0)
    dt = float(np.mean(times))
    v = n / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(w, world) | {"sample": f"first {args.ref_sample_s:g} s: {n} events, {len(tf)} frames"},
            "frames_per_s": len(tf) / dt,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"first {args.ref_sample_s:g} s of the c4 stream ({n} events, {len(tf)} frames)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(w, world):
    return {"workload": f"c4: {w.W}x{w.H} sensor, {w.duration_us / 1e6:g} s stream, {w.n} events "
                        f"(20 Mev/s avg, 100 Mev/s bursts), {len(w.t_frames)} frames @{int(round(len(w.t_frames) / (w.duration_us / 1e6)))} FPS",
            "sensor": f"{w.W}x{w.H}", "events_per_step_per_gpu": w.n, "frames_per_step_per_gpu": len(w.t_frames),
            "esi_params": w.params, "parallelism": f"stream-sharded x{world} (independent streams, no collective)",
            "l2": "inputs (16 B x events) and frames far larger than the 126 MB L2; no flush needed"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="esi", choices=["esi", "reference"])
    ap.add_argument("--fps", type=int, default=100)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-sample-s", type=float, default=1.5)
    ap.add_argument("--ref-sample-s", type=float, default=0.5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-kernel-timing", action="store_true",
                    help="skip the per-launch CUDA events (roofline 'achieved' then unavailable)")
    args = ap.parse_args()
    rank, world, local = dist_setup(args.gpus)

    if args.impl == "reference":
        run_reference(args, rank, world)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    from paper_2508_02238_b200 import Esi
    peaks = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json"), {}) or {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "B200_PROFILING.md fallback 6.65 TB/s"

    w, gen_s = workload_for(rank, args)
    F = len(w.t_frames)
    P = w.P
    stream = torch.cuda.Stream()
    e = Esi(w.W, w.H, **w.params)
    e.set_stream(stream.cuda_stream)
    out = torch.empty((F, w.H, w.W), dtype=torch.uint8, device="cuda")

    def step():
        e.reset()
        rc = e.push(w.events)
        assert rc == 0, rc
        e.render_many(w.t_frames, out)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        step()                      # keeps the GPU busy while nvidia-smi starts
        time.sleep(0.5)
        step()
        torch.cuda.synchronize()
        barrier(world)              # timed region bracketed by barrier + synchronize on both sides
        torch.cuda.synchronize()
        t_wall0 = time.time()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        clk.mark(t_wall0, time.time())
        barrier(world)
        # Per-kernel launch durations: a second timed pass of the same steps with a
        # CUDA event pair around every launch, each on the stream the kernel is
        # launched on.  Kept out of the main timed region because the per-launch
        # events serialise the overlap of K1 (aux stream) and K2 (~15 % slower).
        kt_steps = 0 if args.no_kernel_timing else max(1, min(args.steps, 5))
        e.enable_kernel_timing(kt_steps > 0)
        kt0, kt1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kt0.record(stream)
        for _ in range(kt_steps):
            step()
        kt1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    ms_local = ev0.elapsed_time(ev1)
    ms_total = max_over_ranks(ms_local, world)
    ms_step = ms_total / args.steps
    stats = e.last_render_stats()
    kt = {k: e.kernel_time(k) for k in range(4)}
    kt_pass_ms_step = kt0.elapsed_time(kt1) / kt_steps if kt_steps else None
    e.enable_kernel_timing(False)

    events_total = w.n * world * args.steps
    value = events_total / (ms_total / 1e3)
    frames_per_s = F * world * args.steps / (ms_total / 1e3)

    # roofline of the dominant kernel (algorithmic bytes per launch / mean launch time)
    n_chunks = max(1, stats["chunks"])
    kt_ms = {k: kt[k][0] for k in kt}
    kt_n = {k: kt[k][1] for k in kt}
    dom = max((0, 1), key=lambda k: kt_ms[k])
    names = {0: "esi_partition_kernel", 1: "esi_integrate_kernel"}
    if dom == 0:
        alg_bytes_per_launch = 16.0 * w.n / n_chunks
        unit_note = "16 B per event read (SURVEY 8(d)) x events per chunk"
    else:
        alg_bytes_per_launch = (P * F + 24.0 * P * n_chunks) / n_chunks
        unit_note = "1 B per pixel-frame written + 24 B per pixel state round trip (SURVEY 8(d)), per chunk"
    mean_ms = kt_ms[dom] / max(1, kt_n[dom])
    achieved = alg_bytes_per_launch / (mean_ms / 1e3) / 1e9 if mean_ms > 0 else None
    traffic = None
    prof = load_json(os.path.join(ROOT, "profiles", "traffic.json"), {}) or {}
    if names[dom] in prof:
        traffic = prof[names[dom]].get("dram_bytes_per_launch")
    step_alg = 16.0 * w.n + P * F + 24.0 * P * n_chunks
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak if achieved else None, "traffic": traffic, "kernel": names[dom],
                "algorithmic_bytes_per_launch": alg_bytes_per_launch, "per_unit": unit_note,
                "peak_source": peak_src + " (burst copy; kernel timed inside a long step)",
                "mean_launch_ms": mean_ms, "launches_timed": kt_n[dom]}
    step_roof = {"kernel_timing_pass": {"steps": kt_steps, "ms_per_step": kt_pass_ms_step,
                                        "note": "per-launch CUDA events, separate pass after the timed region"},
                 "algorithmic_bytes": step_alg, "achieved_gbs": step_alg / (ms_step / 1e3) / 1e9,
                 "frac": step_alg / (ms_step / 1e3) / 1e9 / hbm_peak,
                 "kernel_ms_per_step": {names[0]: kt_ms[0] / max(1, kt_steps), names[1]: kt_ms[1] / max(1, kt_steps),
                                        "readout_only": kt_ms[2] / max(1, kt_steps)}}
    launches_per_step = stats["kernel_launches"] + 2   # + reset's two fill kernels
    gpu_launches = launches_per_step * args.steps

    # end to end through the C ABI with host buffers (H2D of the events, D2H of the frames)
    e2e = None
    if args.e2e_steps > 0:
        ev_host = w.events.cpu().pin_memory()
        out_host = torch.empty((F, w.H, w.W), dtype=torch.uint8).pin_memory()
        eh = Esi(w.W, w.H, **w.params)
        eh.set_stream(stream.cuda_stream)

        def step_host():
            eh.reset()
            assert eh.push(ev_host) == 0
            eh.render_many(w.t_frames, out_host)
        step_host()
        barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            step_host()
        torch.cuda.synchronize()
        dt = max_over_ranks(time.perf_counter() - t0, world)
        e2e = {"value": w.n * world * args.e2e_steps / dt, "unit": UNIT,
               "h2d_bytes_per_step": int(w.events.numel() * 8), "d2h_bytes_per_step": int(F * P),
               "ms_per_step": dt * 1e3 / args.e2e_steps}
        eh.close()
        del ev_host, out_host

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w, args.cpu_sample_s)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": config_dict(w, world), "frames_per_s": frames_per_s,
                "roofline": roofline, "step_roofline": step_roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": gpu_launches, "clocks": clk.summary(),
                "notes": {"generation_s": gen_s, "chunks_per_step": stats["chunks"],
                          "paper_context": "ESI 21.3e6 ev/s on an i7-1185G7E CPU (PAPER.md Table 1, P:284)"}}
        print(json.dumps(line), flush=True)
    e.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
