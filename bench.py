#!/usr/bin/env python
"""ESI hot-path benchmark (BASELINE.json metric: events/s integrated and frames/s
at 1280x720 @100 FPS, 1/2/4/8 B200, % of the HBM roofline).

One step = one pass of the whole hot path over one batch of synthetic input.

  --config c4 (default): reset the handle, push the c4 stream (1280x720, 10 s,
      194 M events, already in HBM, borrowed zero-copy; validated on push, the
      library's default atomic-push contract) and render its 1000 frames @100 FPS
      into HBM.  N > 1 GPUs: every rank integrates its own independent c4-like
      stream (stream sharding, weak scaling, no data-path collective).
  --config c5a: BASELINE config 5(a): 64 independent 1280x720 streams of 10 s at
      10 Mev/s, 64/N per rank (stream sharding, strong scaling).
  --config c5b: BASELINE config 5(b): one 2560x1440 sensor at 80 Mev/s split in
      N row bands; each rank holds a time shard, routes it by band over peer
      memory (router kernel P2P stores into IPC-mapped arenas) and the frames
      are assembled by grouped NCCL all-gathers.  The three stages (routing +
      exchange, band integration + readout, assembly) are timed separately.

The stream (3.1 GB) and the frames (0.92 GB) exceed the 126 MB L2, so no flush
is needed between steps.  `--gpus N` without torchrun re-launches itself under
torch.distributed.run with N ranks (127.0.0.1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {esi,reference}]
                    [--config {c4,c5a,c5b}] [--fps F]
"""
import argparse
import json
import os
import socket
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


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_spawn(args, argv):
    """--gpus N outside torchrun: re-run this script under torch.distributed.run with
    N ranks on this node and exit with its status."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *argv]
        sys.exit(subprocess.call(cmd))


def dist_setup(args, backend="nccl"):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if backend == "nccl":
        torch.cuda.set_device(local)
    if world > 1 or args.config == "c5b":
        import torch.distributed as dist
        if backend == "nccl":
            if world == 1:
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
                os.environ.setdefault("MASTER_PORT", str(_free_port()))
                os.environ.setdefault("RANK", "0")
                os.environ.setdefault("WORLD_SIZE", "1")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def barrier(world):
    import torch.distributed as dist
    if dist.is_initialized() and world > 1:
        dist.barrier()


def max_over_ranks(x, world, device="cuda"):
    import torch.distributed as dist
    if world == 1 or not dist.is_initialized():
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, world, device="cuda"):
    import torch.distributed as dist
    if world == 1 or not dist.is_initialized():
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index, enabled=True):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.enabled = enabled

    def __enter__(self):
        if not self.enabled:
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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

    def in_window(self):
        t0, t1 = getattr(self, "window", (0, 1e30))
        return sum(1 for ts, _ in self.lines if t0 <= ts <= t1 + 0.15)

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


def host_cpu():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        model = next((l.split(":", 1)[1].strip() for l in out.splitlines() if l.startswith("Model name")), None)
    except Exception:
        model = None
    return {"cpu_model": model, "nproc": os.cpu_count()}


# --------------------------------------------------------------------------- timing harness
class Ctx:
    """What the step functions need from the environment (injectable for the
    gloo CPU test of the multi-rank orchestration)."""

    def __init__(self, rank, world, local, device="cuda"):
        self.rank, self.world, self.local, self.device = rank, world, local, device

    def sync(self):
        if self.device == "cuda":
            torch.cuda.synchronize()

    def timed(self, step, steps, stream=None):
        """Times exactly `steps` calls of step(): barrier + synchronize on both
        sides, CUDA events on the launching stream; returns the max over ranks (ms)."""
        self.sync()
        barrier(self.world)
        self.sync()
        if self.device == "cuda":
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            for _ in range(steps):
                step()
            ev1.record(stream)
            torch.cuda.synchronize()
            ms = ev0.elapsed_time(ev1)
        else:
            t0 = time.perf_counter()
            for _ in range(steps):
                step()
            ms = (time.perf_counter() - t0) * 1e3
        barrier(self.world)
        return max_over_ranks(ms, self.world, self.device)


def roofline_of(e, w, F, n_chunks, kt_steps, hbm_peak, peak_src):
    """Roofline of the dominant kernel: algorithmic bytes per launch / mean launch time."""
    kt = {k: e.kernel_time(k) for k in range(4)}
    kt_ms = {k: kt[k][0] for k in kt}
    kt_n = {k: kt[k][1] for k in kt}
    P = w.P
    dom = max((0, 1), key=lambda k: kt_ms[k])
    names = {0: "esi_partition_kernel", 1: "esi_integrate_kernel"}
    if dom == 0:
        alg = 16.0 * w.n / n_chunks
        unit_note = "16 B per event read (SURVEY 8(d)) x events per chunk"
    else:
        alg = (P * F + 24.0 * P * n_chunks) / n_chunks
        unit_note = "1 B per pixel-frame written + 24 B per pixel state round trip (SURVEY 8(d)), per chunk"
    mean_ms = kt_ms[dom] / max(1, kt_n[dom])
    achieved = alg / (mean_ms / 1e3) / 1e9 if mean_ms > 0 else None
    prof = load_json(os.path.join(ROOT, "profiles", "traffic.json"), {}) or {}
    traffic = prof.get(names[dom], {}).get("dram_bytes_per_launch")
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
            "frac": achieved / hbm_peak if achieved else None, "traffic": traffic, "kernel": names[dom],
            "algorithmic_bytes_per_launch": alg, "per_unit": unit_note,
            "peak_source": peak_src + " (burst copy; kernel timed inside a long step)",
            "mean_launch_ms": mean_ms, "launches_timed": kt_n[dom]}
    per_step = {names[0]: kt_ms[0] / max(1, kt_steps), names[1]: kt_ms[1] / max(1, kt_steps),
                "readout_only": kt_ms[2] / max(1, kt_steps), "validate": kt_ms[3] / max(1, kt_steps)}
    return roof, per_step


# --------------------------------------------------------------------------- c4 / c5a: stream sharding
def make_stream(name, rank, idx, args):
    from esi_synth import make_workload
    if name == "c4":
        seed = 4 + 1000 * rank + idx          # rank 0 = the c4 stream; other ranks: independent streams
        w = make_workload("c4", "cuda", seed=seed, fps=args.fps)
        if getattr(args, "roi", None):        # local activity: keep only the events inside a rectangle
            x0, y0, x1, y1 = (float(v) for v in args.roi.split(","))
            xy = w.events[:, 1]
            x, y = xy & 0xffff, (xy >> 16) & 0xffff
            keep = (x >= int(x0 * w.W)) & (x < int(x1 * w.W)) & (y >= int(y0 * w.H)) & (y < int(y1 * w.H))
            w.events = w.events[keep].contiguous()
        return w
    seed = 5000 + 64 * rank + idx
    return make_workload("c5a", "cuda", seed=seed)


def run_streams(args, ctx, peaks, handle_factory=None, stream_factory=None):
    """c4 / c5a: stream sharding.  handle_factory / stream_factory are injectable
    (the gloo CPU test of the multi-rank orchestration uses stand-ins)."""
    if handle_factory is None:
        from paper_2508_02238_b200 import Esi as handle_factory
    stream_factory = stream_factory or make_stream
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "B200_PROFILING.md fallback 6.65 TB/s"
    rank, world = ctx.rank, ctx.world
    cuda = ctx.device == "cuda"
    if args.config == "c4":
        n_streams, n_distinct = 1, 1
    else:
        if 64 % world:
            raise SystemExit("c5a needs N dividing 64")
        n_streams = 64 // world
        n_distinct = min(n_streams, args.c5a_distinct)
    t0 = time.time()
    ws = [stream_factory(args.config, rank, i, args) for i in range(n_distinct)]
    ctx.sync()
    gen_s = time.time() - t0
    w = ws[0]
    F = len(w.t_frames)
    stream = torch.cuda.Stream() if cuda else None
    validate = 1 if args.validation == "push" else 0
    e = handle_factory(w.W, w.H, validate_on_push=validate, **w.params)
    if cuda:
        e.set_stream(stream.cuda_stream)
    outs = [torch.empty((F, w.H, w.W), dtype=torch.uint8, device=ctx.device) for _ in range(min(2, n_streams))]
    events_step = sum(ws[s % n_distinct].n for s in range(n_streams))
    frames_step = F * n_streams

    def step():
        for s in range(n_streams):
            ws_ = ws[s % n_distinct]
            e.reset()
            rc = e.push(ws_.events)
            assert rc == 0, rc
            e.render_many(ws_.t_frames, outs[s % len(outs)])

    for _ in range(args.warmup):
        step()
    with ClockSampler(ctx.local, enabled=cuda) as clk:
        step()                      # keeps the GPU busy while nvidia-smi starts
        if cuda:
            time.sleep(0.5)
        step()
        t_wall0 = time.time()
        ms_total = ctx.timed(step, args.steps, stream)
        clk.mark(t_wall0, time.time())
        stats = e.last_render_stats()
        # a short timed region (20 x 4 ms) may fall between two nvidia-smi samples (20 ms
        # apart, delivered late): keep the GPU on the same step until two samples are in
        t_busy = time.time()
        while cuda and clk.proc is not None and clk.in_window() < 2 and time.time() - t_busy < 1.0:
            step()
            torch.cuda.synchronize()
        # Per-kernel launch durations: a separate pass with a CUDA event pair around
        # every launch (they serialise the K1/K2 overlap, so not in the timed region).
        kt_steps = 0 if args.no_kernel_timing else max(1, min(args.steps, 3))
        e.enable_kernel_timing(kt_steps > 0)
        kt_ms = ctx.timed(step, kt_steps, stream) if kt_steps else None
    ms_step = ms_total / args.steps
    events_total = sum_over_ranks(events_step, world, ctx.device) * args.steps
    value = events_total / (ms_total / 1e3)
    frames_per_s = sum_over_ranks(frames_step, world, ctx.device) * args.steps / (ms_total / 1e3)
    n_chunks = max(1, stats["chunks"])
    roof, k_ms = roofline_of(e, w, F, n_chunks, kt_steps * n_streams, hbm_peak, peak_src)
    e.enable_kernel_timing(False)
    P = w.P
    step_alg = 16.0 * events_step + P * frames_step + 24.0 * P * n_chunks * n_streams
    step_roof = {"kernel_timing_pass": {"steps": kt_steps, "ms_per_step": kt_ms / kt_steps if kt_steps else None,
                                        "note": "per-launch CUDA events, separate pass after the timed region"},
                 "algorithmic_bytes": step_alg, "achieved_gbs": step_alg / (ms_step / 1e3) / 1e9,
                 "frac": step_alg / (ms_step / 1e3) / 1e9 / hbm_peak, "kernel_ms_per_step": k_ms,
                 "bytes_note": "16 B x events + 1 B x pixel-frames + 24 B x pixels x chunks (SURVEY 8(d))"}
    launches_per_step = (stats["kernel_launches"] + 2 + (1 if validate else 0)) * n_streams   # + reset fills, validate
    extra = {}
    # the other validation mode, a short pass (same workload)
    if args.config == "c4" and not args.no_alt_validation:
        e.close()
        e = handle_factory(w.W, w.H, validate_on_push=1 - validate, **w.params)
        if cuda:
            e.set_stream(stream.cuda_stream)
        step()
        n_alt = max(1, min(args.steps, 5))
        ms_alt = ctx.timed(step, n_alt, stream) / n_alt
        extra["other_validation_mode"] = {
            "validation": "fused" if validate else "push",
            "value": sum_over_ranks(events_step, world, ctx.device) / (ms_alt / 1e3), "ms_per_step": ms_alt,
            "note": ("validate_on_push=0: the checks run inside the ingest kernel K1 (no extra read of the "
                     "events); a failing render restores S/T, its frames are unspecified (DESIGN reading A21)")
            if validate else "validate_on_push=1: atomic push, one extra read of the events"}
    e2e = None
    if args.e2e_steps > 0 and args.config == "c4" and cuda:
        e2e = run_e2e(args, ctx, w, stream)
    e.close()
    cfg = stream_config(w, world, args, n_streams, n_distinct)
    return {"value": value, "ms_per_step": ms_step, "frames_per_s": frames_per_s, "roofline": roof,
            "step_roofline": step_roof, "gpu_launches": launches_per_step * args.steps, "clocks": clk.summary(),
            "config": cfg, "e2e": e2e, "scaling": "weak" if args.config == "c4" else "strong",
            "notes": {"generation_s": gen_s, "chunks_per_step": stats["chunks"] * n_streams,
                      "paper_context": "ESI 21.3e6 ev/s on an i7-1185G7E CPU (PAPER.md Table 1, P:284)"},
            **extra}, w


def run_e2e(args, ctx, w, stream):
    """The same metric through the C ABI with host buffers: pinned H2D of the events
    (validated on push) and D2H of all frames inside the timed region."""
    from paper_2508_02238_b200 import Esi
    F = len(w.t_frames)
    ev_host = w.events.cpu().pin_memory()
    out_host = torch.empty((F, w.H, w.W), dtype=torch.uint8).pin_memory()
    eh = Esi(w.W, w.H, **w.params)
    eh.set_stream(stream.cuda_stream)

    def step_host():
        eh.reset()
        assert eh.push(ev_host) == 0
        eh.render_many(w.t_frames, out_host)
    step_host()
    ctx.sync()
    barrier(ctx.world)
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        step_host()
    ctx.sync()
    dt = max_over_ranks(time.perf_counter() - t0, ctx.world)
    eh.close()
    return {"value": sum_over_ranks(w.n, ctx.world) * args.e2e_steps / dt, "unit": UNIT,
            "h2d_bytes_per_step": int(w.events.numel() * 8), "d2h_bytes_per_step": int(F * w.P),
            "ms_per_step": dt * 1e3 / args.e2e_steps}


def stream_config(w, world, args, n_streams, n_distinct):
    if args.config == "c4":
        wl = (f"c4: {w.W}x{w.H} sensor, {w.duration_us / 1e6:g} s stream, {w.n} events "
              f"(20 Mev/s avg, 100 Mev/s bursts), {len(w.t_frames)} frames @{args.fps} FPS")
        par = f"stream-sharded x{world} (one independent c4-like stream per rank, no collective)"
    else:
        wl = (f"c5a: 64 independent {w.W}x{w.H} streams of {w.duration_us / 1e6:g} s at 10 Mev/s "
              f"({w.n} events, {len(w.t_frames)} frames each), {n_streams} per rank")
        par = (f"stream-sharded x{world} ({n_streams} streams per rank, no collective; "
               f"{n_distinct} distinct generated streams per rank are cycled as inputs)")
    return {"workload": wl, "sensor": f"{w.W}x{w.H}", "events_per_step_per_gpu": w.n * n_streams,
            "frames_per_step_per_gpu": len(w.t_frames) * n_streams, "esi_params": w.params,
            "validation": args.validation, "parallelism": par,
            "band_layout": {"1": "interleaved", "2": "auto"}.get(os.environ.get("ESI_BAND_LAYOUT", ""), "contiguous (default)"),
            "l2": "inputs (16 B x events) and frames far larger than the 126 MB L2; no flush needed"}


# --------------------------------------------------------------------------- c5b: row bands
def run_c5b(args, ctx, peaks):
    import torch.distributed as dist
    from esi_synth import make_workload
    from paper_2508_02238_b200.dist import PeerTransport, RowBandSharded, row_bands, time_shard_bounds
    rank, world = ctx.rank, ctx.world
    dur = int(args.c5b_seconds * 1e6)
    t0 = time.time()
    w = make_workload("c5b", "cuda", duration_us=dur)
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    b = time_shard_bounds(w.n, world)
    n_total = w.n
    shard = w.events[b[rank]:b[rank + 1]].contiguous()
    w.events = w.events[:0]
    torch.cuda.empty_cache()
    F = len(w.t_frames)
    starts = row_bands(w.H, world)
    stage = {}

    def build():
        tr = PeerTransport(ctx.local, w.H, starts)
        return RowBandSharded(w.W, w.H, transport=tr, validate_on_push=1 if args.validation == "push" else 0,
                              **w.params)

    rb = build()
    out = torch.empty((F, w.H, w.W), dtype=torch.uint8, device="cuda")

    def step(record=None):
        rb.band.reset()
        if record is not None:
            ev_a, ev_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev_a.record()
        rc = rb.push_shard(shard)
        assert rc == 0, rc
        if record is not None:
            ev_b.record()
            ev_b.synchronize()
            record["route_exchange"] = record.get("route_exchange", 0.0) + ev_a.elapsed_time(ev_b)
        rb.render_many(w.t_frames, out, stage_ms=record)

    for _ in range(args.warmup):
        step()
    with ClockSampler(ctx.local) as clk:
        t_wall0 = time.time()
        ms_total = ctx.timed(step, args.steps)
        clk.mark(t_wall0, time.time())
    n_stage = max(1, min(args.steps, 3))
    for _ in range(n_stage):
        step(stage)
    stage_ms = {k: max_over_ranks(v / n_stage, world) for k, v in stage.items()}
    ms_step = ms_total / args.steps
    value = n_total * args.steps / (ms_total / 1e3)
    rows = starts[rank + 1] - starts[rank]
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    band_bytes = 16.0 * (n_total / world) + rows * w.W * F + 24.0 * rows * w.W
    asm_bytes = (world - 1) / world * w.P * F
    stages = {
        "route_exchange": {"ms": stage_ms.get("route_exchange"),
                           "bytes_per_rank": 16.0 * (b[rank + 1] - b[rank]) * 2,
                           "note": "router count + scatter (P2P stores into the band owners' arenas)"},
        "band_integration_readout": {"ms": stage_ms.get("band_render"), "bytes_per_rank": band_bytes,
                                     "hbm_frac": (band_bytes / (stage_ms["band_render"] / 1e3) / 1e9 / hbm_peak)
                                     if stage_ms.get("band_render") else None},
        "assembly": {"ms": stage_ms.get("assembly"), "bytes_received_per_rank": asm_bytes,
                     "gbs": asm_bytes / (stage_ms["assembly"] / 1e3) / 1e9 if stage_ms.get("assembly") else None,
                     "note": "grouped NCCL all_gather_into_tensor of the band slices (64 frames per group)"},
    }
    rb.close()
    cfg = {"workload": f"c5b: {w.W}x{w.H} sensor, first {dur / 1e6:g} s of the 80 Mev/s stream "
                       f"({n_total} events, {F} frames @100 FPS)",
           "sensor": f"{w.W}x{w.H}", "events_per_step_per_gpu": n_total / world, "frames_per_step": F,
           "esi_params": w.params, "validation": args.validation,
           "parallelism": f"row bands x{world} (router P2P exchange + NCCL frame assembly)"}
    return {"value": value, "ms_per_step": ms_step, "frames_per_s": F * args.steps / (ms_total / 1e3),
            "stages": stages, "clocks": clk.summary(), "config": cfg, "e2e": None, "scaling": "strong",
            "gpu_launches": None, "notes": {"generation_s": gen_s}}, w


# --------------------------------------------------------------------------- c4t: time shards
def run_c4t(args, ctx, peaks):
    """the c4 stream sharded in time over the ranks
    (dist.TimeSharded): every rank summarises its slice into per-pixel maps,
    the maps are all-gathered (NCCL), rank r composes the maps of the earlier
    slices, applies them to its initial state and integrates + renders its own
    slice.  value = events of the whole stream / max-over-ranks step time."""
    from esi_synth import make_workload
    from paper_2508_02238_b200.dist import TimeSharded, time_slices
    rank, world = ctx.rank, ctx.world
    t0 = time.time()
    w = make_workload("c4", "cuda", fps=args.fps)
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    tf = np.asarray(w.t_frames)
    t_ev = w.events[:, 0].cpu().numpy()
    eb, fb = time_slices(t_ev, tf, world)
    ev = w.events[eb[rank]:eb[rank + 1]]
    tfr = tf[fb[rank]:fb[rank + 1]]
    out = torch.empty((len(tfr), w.H, w.W), dtype=torch.uint8, device="cuda")
    ts = TimeSharded(w.W, w.H, validate_on_push=1 if args.validation == "push" else 0, **w.params)

    def step():
        ts.run(ev, tfr, out)

    for _ in range(args.warmup):
        step()
    with ClockSampler(ctx.local) as clk:
        t_wall0 = time.time()
        ms_total = ctx.timed(step, args.steps)
        clk.mark(t_wall0, time.time())
    # the scan's share: summarise + gather + compose + apply alone
    n_sc = max(1, min(args.steps, 3))
    ms_scan = ctx.timed(lambda: ts.incoming_state_maps(ev), n_sc) / n_sc
    ts.close()
    ms_step = ms_total / args.steps
    cfg = {"workload": f"c4 time-sharded: {w.W}x{w.H}, {w.duration_us / 1e6:g} s stream, {w.n} events, "
                       f"{len(tf)} frames @{args.fps} FPS, split in {world} time slices",
           "sensor": f"{w.W}x{w.H}", "events_per_step": w.n, "events_per_step_per_gpu": eb[rank + 1] - eb[rank],
           "frames_per_step": len(tf), "esi_params": w.params, "validation": args.validation,
           "parallelism": f"time slices x{world} (per-pixel slice maps all-gathered + exclusive scan)"}
    return {"value": w.n * args.steps / (ms_total / 1e3), "ms_per_step": ms_step,
            "frames_per_s": len(tf) * args.steps / (ms_total / 1e3),
            "stages": {"slice_map_scan_ms": ms_scan,
                       "note": "esi_slice_summarize + all_gather + compose + apply (skipped at N=1)"},
            "clocks": clk.summary(), "config": cfg, "e2e": None, "scaling": "strong", "gpu_launches": None,
            "notes": {"generation_s": gen_s}}, w


# --------------------------------------------------------------------------- streaming latency
def run_latency(args, frames_max=300):
    """Analogue of the paper's per-frame reconstruction time (Fig. rec_time,
    PAPER.md P:299-311): events arrive in 10 ms packets (the
    100 Hz driver cadence), each packet is pushed from pinned host memory
    (validated on push) and esi_render is called once per frame into a pinned
    host frame.  Per-frame time = (packet push + its frames' renders) / frames."""
    from esi_synth import make_workload
    from paper_2508_02238_b200 import Esi
    res = {}
    for cfg in ("c2", "c4"):
        w = make_workload(cfg, "cuda", duration_us=2_000_000) if cfg == "c4" else make_workload(cfg, "cpu")
        ev = w.events.cpu()
        t_all = ev[:, 0].numpy()
        for fps in (100, 1000):
            period = 1_000_000 // fps
            e = Esi(w.W, w.H, **w.params)
            out = torch.empty((w.H, w.W), dtype=torch.uint8).pin_memory()
            n_packets = min(int(w.duration_us // 10_000), max(1, frames_max * period // 10_000))
            bounds = np.searchsorted(t_all, np.arange(0, n_packets + 1) * 10_000, side="right")
            packets = [ev[bounds[k]:bounds[k + 1]].pin_memory() for k in range(n_packets)]
            per_frame, render_ms = [], []
            for k in range(n_packets):
                t0 = time.perf_counter()
                assert e.push(packets[k]) == 0
                t1 = time.perf_counter()
                nf = 10_000 // period
                rs = []
                for f in range(nf):
                    a = time.perf_counter()
                    e.render(k * 10_000 + (f + 1) * period, out)
                    rs.append(time.perf_counter() - a)
                push_ms = (t1 - t0) * 1e3
                for r in rs:
                    render_ms.append(r * 1e3)
                    per_frame.append(r * 1e3 + push_ms / nf)
            e.close()
            skip = max(1, len(per_frame) // 10)              # warm-up packets
            pf = np.array(per_frame[skip:])
            rm = np.array(render_ms[skip:])
            res[f"{cfg}@{fps}"] = {"sensor": f"{w.W}x{w.H}", "frames": int(len(pf)),
                                   "mean_ms_per_frame": float(pf.mean()), "p99_ms_per_frame": float(np.percentile(pf, 99)),
                                   "render_mean_ms": float(rm.mean()), "render_p99_ms": float(np.percentile(rm, 99)),
                                   "pct_of_frame_period_mean": float(100 * pf.mean() / (period / 1e3)),
                                   "pct_of_frame_period_p99": float(100 * np.percentile(pf, 99) / (period / 1e3))}
    return res


# --------------------------------------------------------------------------- oracle arms
def cpu_baseline(w, sample_s):
    """The oracle (as it stands, single thread) on the first sample_s seconds of the stream."""
    import oracle
    from esi_synth import to_numpy_struct
    tmax = int(sample_s * 1e6)
    t_all = w.events[:, 0].contiguous()
    n = int(torch.searchsorted(t_all, torch.tensor([tmax], device=t_all.device), right=True).item())
    ev = to_numpy_struct(w.events[:n])
    tf = w.t_frames[w.t_frames <= tmax]
    t0 = time.perf_counter()
    oracle.run(w.W, w.H, ev, tf, **w.params)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"first {sample_s:g} s of the {w.name} stream: {n} events, {len(tf)} frames of {w.W}x{w.H}",
            "frames_per_s": len(tf) / dt, "seconds": dt, **host_cpu()}


def run_reference(args, rank, world):
    """--impl reference: the fp64 oracle timed on host cores (rank 0 only)."""
    if rank != 0:
        return
    from esi_synth import make_workload
    w = make_workload("c4", "cuda", seed=4, fps=args.fps)
    import oracle
    from esi_synth import to_numpy_struct
    tmax = int(args.ref_sample_s * 1e6)
    n = int(torch.searchsorted(w.events[:, 0].contiguous(), torch.tensor([tmax], device="cuda"), right=True).item())
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
    cfg = {"workload": f"c4: {w.W}x{w.H} sensor, {w.duration_us / 1e6:g} s stream, {w.n} events "
                       f"(20 Mev/s avg, 100 Mev/s bursts), {len(w.t_frames)} frames @{args.fps} FPS",
           "sensor": f"{w.W}x{w.H}", "esi_params": w.params,
           "sample": f"first {args.ref_sample_s:g} s: {n} events, {len(tf)} frames"}
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
            "frames_per_s": len(tf) / dt,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"first {args.ref_sample_s:g} s of the c4 stream ({n} events, {len(tf)} frames)",
                             **host_cpu()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def bench_line(args, res, world, cpu=None, lat=None):
    res = dict(res)
    return {"metric": METRIC, "value": res.pop("value"), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res.pop("ms_per_step"),
            "higher_is_better": True, "scaling": res.pop("scaling"), "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": res.pop("config"), "frames_per_s": res.pop("frames_per_s"),
            "cpu_baseline": cpu, "latency": lat, **res}


def parse_args(argv):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="esi", choices=["esi", "reference"])
    ap.add_argument("--config", default="c4", choices=["c4", "c5a", "c5b", "c4t"])
    ap.add_argument("--fps", type=int, default=100)
    ap.add_argument("--roi", default=None,
                    help="c4 only: x0,y0,x1,y1 as fractions of the sensor; events outside are dropped "
                         "(a locally active scene; not the BASELINE workload)")
    ap.add_argument("--validation", default="push", choices=["push", "fused"],
                    help="push: validate_on_push=1 (the library default, atomic push); fused: checks in K1")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-sample-s", type=float, default=1.5)
    ap.add_argument("--ref-sample-s", type=float, default=0.5)
    ap.add_argument("--c5a-distinct", type=int, default=2)
    ap.add_argument("--c5b-seconds", type=float, default=2.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--no-alt-validation", action="store_true")
    ap.add_argument("--no-kernel-timing", action="store_true",
                    help="skip the per-launch CUDA events (roofline 'achieved' then unavailable)")
    return ap.parse_args(argv)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse_args(argv)
    maybe_spawn(args, argv)
    rank, world, local = dist_setup(args)
    ctx = Ctx(rank, world, local)

    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        peaks = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json"), {}) or {}
        if args.config == "c5b":
            res, w = run_c5b(args, ctx, peaks)
        elif args.config == "c4t":
            res, w = run_c4t(args, ctx, peaks)
        else:
            res, w = run_streams(args, ctx, peaks)
        cpu = None
        if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config == "c4":
            cpu = cpu_baseline(w, args.cpu_sample_s)
        lat = None
        if rank == 0 and world == 1 and not args.no_latency and args.config == "c4":
            lat = run_latency(args)
        if rank == 0:
            print(json.dumps(bench_line(args, res, world, cpu, lat)), flush=True)
    import torch.distributed as dist
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
