"""bench.py's multi-rank code path on CPU (gloo, world_size 2).

The orchestration -- per-rank streams, barrier + max-over-ranks timing, the
whole-job aggregate value, the JSON line -- runs with a stand-in handle that
does no arithmetic (the CUDA handle needs a GPU; its numerics are covered by
the GPU parity tests).  `--gpus N` without torchrun re-launches under
torch.distributed.run with N ranks on 127.0.0.1.
"""
import os
import sys
import tempfile
import time

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


class _W:
    def __init__(self, rank, idx, n=1000, W=16, H=8, F=5):
        self.name, self.W, self.H = "fake", W, H
        self.events = torch.zeros((n + 100 * rank + idx, 2), dtype=torch.int64)
        self.t_frames = np.arange(1, F + 1, dtype=np.int64) * 10_000
        self.params = {"C": 0.15, "k": 10.0, "b": 2.0, "s_min": -1.5, "s_max": 1.5}
        self.duration_us = 50_000

    @property
    def n(self):
        return int(self.events.shape[0])

    @property
    def P(self):
        return self.W * self.H


class FakeHandle:
    calls = []

    def __init__(self, W, H, **p):
        self.n, self.delay = 0, 0.002 * (1 + dist.get_rank())

    def reset(self):
        pass

    def push(self, ev):
        self.n = int(ev.shape[0])
        return 0

    def render_many(self, tf, out):
        time.sleep(self.delay)
        return out

    def last_render_stats(self):
        return {"kernel_launches": 4, "events": self.n, "chunks": 1}

    def enable_kernel_timing(self, on):
        pass

    def kernel_time(self, k):
        return (0.0, 0)

    def close(self):
        pass


def _worker(rank, world, path, config, q):
    dist.init_process_group("gloo", init_method=f"file://{path}", rank=rank, world_size=world)
    try:
        args = bench.parse_args(["--gpus", str(world), "--steps", "3", "--warmup", "1", "--config", config,
                                 "--e2e-steps", "0", "--no-alt-validation", "--c5a-distinct", "2"])
        ctx = bench.Ctx(rank, world, rank, device="cpu")
        res, w = bench.run_streams(args, ctx, {}, handle_factory=FakeHandle,
                                   stream_factory=lambda cfg, r, i, a: _W(r, i))
        line = bench.bench_line(args, res, world)
        q.put((rank, line))
    finally:
        dist.destroy_process_group()


def _run(config):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    path = tempfile.mktemp()
    procs = [ctx.Process(target=_worker, args=(r, 2, path, config, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_bench_c4_two_ranks_weak_scaling():
    res = _run("c4")
    line = res[0]
    assert line["n_gpus"] == 2 and line["steps"] == 3 and line["scaling"] == "weak"
    # whole-job aggregate: both ranks' events over the slowest rank's time
    ev = (1000 + 0) + (1000 + 100)
    t_max = line["ms_per_step"] * 3 / 1e3
    assert abs(line["value"] - ev * 3 / t_max) / line["value"] < 1e-9
    # the slowest rank (rank 1 sleeps 4 ms per render) sets the time
    assert line["ms_per_step"] >= 4.0
    assert res[1]["ms_per_step"] == line["ms_per_step"]          # max over ranks on every rank
    assert line["config"]["events_per_step_per_gpu"] == 1000
    assert line["gpu_launches"] == (4 + 2 + 1) * 3


def test_bench_c5a_two_ranks_stream_sharding():
    res = _run("c5a")
    line = res[0]
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert "32 per rank" in line["config"]["workload"]
    # 32 streams per rank cycling 2 distinct inputs: rank r streams have 1000 + 100 r + (s % 2) events
    ev = sum(16 * (2000 + 1 + 200 * r) for r in range(2))
    t_max = line["ms_per_step"] * 3 / 1e3
    assert abs(line["value"] - ev * 3 / t_max) / line["value"] < 1e-9


def test_gpus_flag_relaunches_under_torchrun(monkeypatch):
    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    args = bench.parse_args(["--gpus", "4", "--steps", "2"])
    try:
        bench.maybe_spawn(args, ["--gpus", "4", "--steps", "2"])
    except SystemExit as e:
        assert e.code == 0
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]


def test_world_size_mismatch_fails_loudly(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "2")
    args = bench.parse_args(["--gpus", "4"])
    try:
        bench.dist_setup(args, backend="gloo")
        raise AssertionError("expected SystemExit")
    except SystemExit as e:
        assert "WORLD_SIZE=2" in str(e)
