"""Events per K2 band per 8 Mi-event chunk of the c4 stream: contiguous bands (pid // band_px)
vs interleaved 64-pixel groups ((pid // 64) % nb).  K2's launch time follows the busiest band."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from esi_synth import make_workload
from paper_2508_02238_b200 import Esi

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
w = make_workload(cfg, "cuda")
e = Esi(w.W, w.H, **w.params)
nb, band_px, _ = e.layout()
e.close()
ev = w.events
# packed 16-B records: int64 t, u16 x, u16 y, i8 p
w1 = ev[:, 1]                                  # [n, 2] int64: t | x, y (u16 each), p
pid = ((w1 >> 16) & 0xffff) * w.W + (w1 & 0xffff)
n = pid.numel()
chunk = 8 << 20
out = {"config": cfg, "n": n, "nb": nb, "band_px": band_px, "chunks": []}
G = 64
for c0 in range(0, n, chunk):
    p = pid[c0:c0 + chunk]
    a = torch.bincount(p // band_px, minlength=nb).double()
    b = torch.bincount((p // G) % nb, minlength=nb).double()
    out["chunks"].append({"contig_max_over_mean": float(a.max() / a.mean()), "contig_p95_over_mean": float(a.quantile(0.95) / a.mean()),
                          "inter_max_over_mean": float(b.max() / b.mean())})
# per-SM sums with the default block -> SM assignment guess (b % 148)
print(json.dumps(out))
cm = [c["contig_max_over_mean"] for c in out["chunks"]]
im = [c["inter_max_over_mean"] for c in out["chunks"]]
print("contiguous max/mean: mean %.3f max %.3f; interleaved: mean %.3f max %.3f" % (sum(cm) / len(cm), max(cm), sum(im) / len(im), max(im)), file=sys.stderr)
