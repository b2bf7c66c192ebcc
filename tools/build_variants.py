"""Build compile-time variants of libesi.so for A/B runs (ESI_LIB_PATH=...)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_02238_b200 import build as b
VARIANTS = {
    "k2c2": ["-DESI_K2_CTAS=2"],
    "k2c2_t2048": ["-DESI_K2_CTAS=2", "-DESI_TILE=2048", "-DESI_PART_THREADS=256", "-DESI_PART_CTAS=2"],
    "t2048c3": ["-DESI_TILE=2048", "-DESI_PART_THREADS=256", "-DESI_PART_CTAS=3"],
}
names = sys.argv[1:] or list(VARIANTS)
os.makedirs(os.path.join(b.HERE, "variants"), exist_ok=True)
for n in names:
    out = os.path.join(b.HERE, "variants", f"libesi_{n}.so")
    b.build(out=out, objdir=os.path.join(b.HERE, "build_" + n), extra=tuple(VARIANTS[n]))
    print(out)
