"""ESI oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of Event-based Single
Integration (arXiv 2508.02238, Algorithm 2 at PAPER.md lines 233-262, readout
Eq. 14 at line 227), in fp64.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may import
this package.  It shares no code with the CUDA library in
``paper_2508_02238_b200/``; neither imports the other.
"""
from .oracle import (  # noqa: F401
    ESIO_OK, ESIO_ERR_INVALID_ARG, ESIO_ERR_OUT_OF_BOUNDS, ESIO_ERR_BAD_POLARITY,
    ESIO_ERR_NEGATIVE_INTERVAL, Oracle, OracleError, decay, clamp, map_gray,
    run, stable_group_by, py_run, build_oracle, lib,
)
