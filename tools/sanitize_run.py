"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck):
c1 plus a hot-pixel random stream with multiple chunks, through the C ABI, checked
against the oracle (test infrastructure)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from esi_synth import make_workload, to_numpy_struct, from_numpy_struct  # noqa: E402
from helpers import assert_frames_close, assert_state_close, gpu_run  # noqa: E402


def main():
    w = make_workload("c1", "cpu")
    f, S, T, st = gpu_run(w.W, w.H, w.events, w.t_frames, w.params, chunk_events=16384)
    fr, Sr, Tr = oracle.run(w.W, w.H, to_numpy_struct(w.events), w.t_frames, **w.params)
    assert_frames_close(f, fr)
    assert_state_close(S, T, Sr, Tr)
    rng = np.random.default_rng(0)
    n, W, H = 60_000, 96, 40
    a = np.zeros(n, dtype=[("t", "<i8"), ("x", "<u2"), ("y", "<u2"), ("p", "i1"), ("_pad", "u1", (3,))])
    a["t"] = np.sort(rng.integers(0, 300_000, n)) // 5 * 5
    a["x"] = rng.integers(0, W, n)
    a["y"] = rng.integers(0, H, n)
    hot = rng.random(n) < 0.3
    a["x"][hot] = 7
    a["y"][hot] = 3
    a["p"] = rng.choice([-1, 1], n)
    tf = np.arange(1, 31, dtype=np.int64) * 10_000
    prm = {"C": 0.15, "k": 10.0, "b": 2.0, "s_min": -1.5, "s_max": 1.5}
    f, S, T, st = gpu_run(W, H, from_numpy_struct(a), tf, prm, chunk_events=16384)
    fr, Sr, Tr = oracle.run(W, H, a, tf, **prm)
    assert_frames_close(f, fr)
    assert_state_close(S, T, Sr, Tr)
    print("sanitize run ok", st)


if __name__ == "__main__":
    main()
