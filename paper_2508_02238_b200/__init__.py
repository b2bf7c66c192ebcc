"""B200-native ESI (Event-based Single Integration, arXiv 2508.02238).

The hot path lives in libesi.so (CUDA, sm_100a) behind the C ABI declared in
include/esi.h; ``paper_2508_02238_b200.esi`` is the ctypes binding.
"""
from . import esi  # noqa: F401
from .esi import (  # noqa: F401
    Esi, EsiError, EVENT_DTYPE, create, push_events, render, render_many, get_state, set_state,
    reset, set_stream, get_error, destroy, default_params,
)

__all__ = ["esi", "Esi", "EsiError", "EVENT_DTYPE", "create", "push_events", "render",
           "render_many", "get_state", "set_state", "reset", "set_stream", "get_error",
           "destroy", "default_params"]
