"""Step time of c4 @100 FPS for several chunk sizes (esi_params_t.chunk_events):
    python tools/chunk_sweep.py
"""
import sys, os, time, json
sys.path.insert(0, os.getcwd())
import torch
from esi_synth import make_workload
from paper_2508_02238_b200 import Esi
w = make_workload("c4", "cuda", fps=100)
out = torch.empty((len(w.t_frames), w.H, w.W), dtype=torch.uint8, device="cuda")
for ce in (4 << 20, 6 << 20, 7 << 20, 8 << 20):
    e = Esi(w.W, w.H, chunk_events=ce, **w.params)
    st = torch.cuda.Stream(); e.set_stream(st.cuda_stream)
    def step():
        e.reset(); assert e.push(w.events) == 0; e.render_many(w.t_frames, out)
    for _ in range(3): step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(10): step()
        b.record(st); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) / 10)
    ts.sort()
    print(json.dumps({"chunk_events": ce, "ms": ts[2]}), flush=True)
    e.close()
