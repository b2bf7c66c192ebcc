"""Build compile-time variants of libesi.so for A/B runs (ESI_LIB_PATH=...)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_02238_b200 import build as b
VARIANTS = {
    # interleaved bands: pixel groups of 128 / 256 / 512 ids (default 64)
    "g7": ["-DESI_GROUP_SHIFT=7"],
    "g8": ["-DESI_GROUP_SHIFT=8"],
    "g9": ["-DESI_GROUP_SHIFT=9"],
    "k2c4": ["-DESI_K2_CTAS=4"],
    "k2c2w12": ["-DESI_K2_CTAS=2", "-DESI_K2_WARPS=12"],
    "k2c2w16": ["-DESI_K2_CTAS=2", "-DESI_K2_WARPS=16"],
    "k2c2w12sb3072": ["-DESI_K2_CTAS=2", "-DESI_K2_WARPS=12", "-DESI_K2_SB=3072"],
    "k2c2w8sb3072": ["-DESI_K2_CTAS=2", "-DESI_K2_WARPS=8", "-DESI_K2_SB=3072"],
    "k2c2w16sb3072": ["-DESI_K2_CTAS=2", "-DESI_K2_WARPS=16", "-DESI_K2_SB=3072"],
    "k2c2": ["-DESI_K2_CTAS=2"],
    "k2c2_t2048": ["-DESI_K2_CTAS=2", "-DESI_TILE=2048", "-DESI_PART_THREADS=256", "-DESI_PART_CTAS=2"],
    "t2048c3": ["-DESI_TILE=2048", "-DESI_PART_THREADS=256", "-DESI_PART_CTAS=3"],
    # K1 with 8 warps per 4096-event tile: fewer registers per CTA, so that a K1 CTA
    # fits beside two K2 CTAs on an SM (register file: 2 x 18.4 K + 20 K < 64 K)
    "p256": ["-DESI_PART_THREADS=256", "-DESI_PART_CTAS=2"],
    "p256c3": ["-DESI_PART_THREADS=256", "-DESI_PART_CTAS=3"],
    # K2 at 2 CTAs per SM with a 3-CTA register budget + a light K1 (8 warps, 3072-event
    # tiles, 6 Mi-event chunks) that fits beside them: K1 of chunk c+1 co-resident with K2 of c
    "overlap": ["-DESI_K2_CTAS=2", "-DESI_K2_MINB=3", "-DESI_TILE=3072", "-DESI_PART_THREADS=256",
                "-DESI_PART_CTAS=3"],
    "overlap4k": ["-DESI_K2_CTAS=2", "-DESI_K2_MINB=3", "-DESI_PART_THREADS=256", "-DESI_PART_CTAS=3"],
}
names = sys.argv[1:] or list(VARIANTS)
os.makedirs(os.path.join(b.HERE, "variants"), exist_ok=True)
for n in names:
    out = os.path.join(b.HERE, "variants", f"libesi_{n}.so")
    b.build(out=out, objdir=os.path.join(b.HERE, "build_" + n), extra=tuple(VARIANTS[n]))
    print(out)
