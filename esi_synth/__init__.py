"""Seeded synthetic event streams shaped like the BASELINE.json workloads.

This module holds NO ESI arithmetic: it simulates an event camera (the
threshold-crossing model of PAPER.md Eq. 1 / Sec. III-A; SPEC synth
S:290-348) over procedural scenes, adds noise / hot pixels (Fig. 3),
and merges everything into one time-sorted stream.  Both the CUDA path and
the oracle consume its output; neither side's code is imported here.

Events are returned as a contiguous int64 tensor of shape [n, 2] whose bytes
are exactly n esi_event_t records (16 B each):  col 0 = t_us,
col 1 = x | y << 16 | (p & 0xff) << 32.  ``to_numpy_struct`` views it as a
structured array with fields t, x, y, p.

Configs (BASELINE.json ``configs``; recipe in DESIGN.md section 5):
  c1  64x48,    0.1 s, ~100 k ev, moving bar (contrast 0.2) + 5 % uniform noise, 10 frames @100 FPS
  c2  346x260,  2 s,   ~1 Mev/s, 6 textured patches, random affine motion, BA 0.1 Hz/px, 200 frames
  c3  640x480,  5 s,   ~3 Mev/s, BA 2 Hz/px + 10 % hot-burst pixels, P(ON)=0.6, +-50 us jitter, 500 frames
  c4  1280x720, 10 s,  20 Mev/s avg (15.79 base + ten 50 ms bursts at 100 Mev/s), rotating texture, c=0.15
  c5a 1280x720 stream at 10 Mev/s (one of the 64 independent streams; seed 5000+s)
  c5b 2560x1440, 10 s, 80 Mev/s rotating texture
"""
from .gen import (  # noqa: F401
    CONFIGS, Workload, make_workload, pack_events, to_numpy_struct, from_numpy_struct,
    frame_times, events_of_pixels,
)
