"""CPU-side checks of the C ABI library: it builds, loads, and exports every
symbol include/esi.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "esi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(esi_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("esi_create", "esi_push_events", "esi_render", "esi_destroy", "esi_render_many"):
        assert s in syms


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2508_02238_b200 import build
    lib = build.build()
    L = ctypes.CDLL(lib)
    for s in declared_symbols():
        assert hasattr(L, s), s


def test_library_is_sm100a():
    import subprocess
    from paper_2508_02238_b200 import build
    lib = build.build()
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2508_02238_b200 import Esi, EsiError
    with pytest.raises(EsiError) as ei:
        Esi(64, 48)
    assert ei.value.code == 5   # ESI_ERR_CUDA: no silent CPU fallback


def test_invalid_arguments_rejected_on_host():
    from paper_2508_02238_b200 import esi
    L = esi._lib()
    p = esi.default_params()
    h = ctypes.c_void_p()
    assert L.esi_create(0, 10, ctypes.byref(p), ctypes.byref(h)) == 1
    assert L.esi_create(10, 70000, ctypes.byref(p), ctypes.byref(h)) == 1
    bad = esi.default_params(s_min=1.0, s_max=1.0)
    assert L.esi_create(10, 10, ctypes.byref(bad), ctypes.byref(h)) == 1
    bad = esi.default_params(k=0.0)
    assert L.esi_create(10, 10, ctypes.byref(bad), ctypes.byref(h)) == 1
    for kw in (dict(decay_kind=3), dict(decay_first=3), dict(decay_kind=-1), dict(state_unclamped=2)):
        bad = esi.default_params(**kw)
        assert L.esi_create(10, 10, ctypes.byref(bad), ctypes.byref(h)) == 1
    assert L.esi_strerror(4) == b"negative time interval (events or frames out of order)"


def test_router_and_ipc_reject_bad_arguments_on_host():
    """Row-band router / IPC entry points validate their arguments before any
    CUDA call (so this runs without a GPU)."""
    from paper_2508_02238_b200 import esi
    L = esi._lib()
    r = ctypes.c_void_p()
    i32 = ctypes.c_int32
    bad_rows = [((i32 * 3)(0, 5, 9), 10, 2),      # last start != height
                ((i32 * 3)(1, 5, 10), 10, 2),     # first start != 0
                ((i32 * 3)(0, 5, 5), 5, 2),       # empty band
                ((i32 * 2)(0, 10), 10, 0),        # no bands
                ((i32 * 2)(0, 10), 0, 1)]         # height 0
    for rows, h, g in bad_rows:
        assert L.esi_router_create(0, h, rows, g, ctypes.byref(r)) == 1
    assert L.esi_router_create(0, 10, None, 1, ctypes.byref(r)) == 1
    assert L.esi_router_count(None, None, 0, None, None) == 1
    assert L.esi_router_scatter(None, None, None, None) == 1
    assert L.esi_ipc_get_handle(None, None) == 1
    assert L.esi_ipc_open(0, None, ctypes.byref(r)) == 1
    assert L.esi_buffer_alloc(0, 0, ctypes.byref(r)) == 1
    counts = (ctypes.c_int64 * 2)()
    assert L.esi_route_bands(0, None, 0, 10, (i32 * 3)(0, 4, 9), 2, None, counts, None) == 1
