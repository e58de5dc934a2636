"""Seeded synthetic workloads shared by the CUDA path's tests/bench and the oracle.

This package holds NO arithmetic of the BatMap method (no hashing, no layout, no
intersection): it only draws vertical tidlists (CSR ``offsets``/``tids``) shaped like
the paper's workloads (§4) and the BASELINE.json configs.
Both ``oracle/`` and ``paper_1102_1003_b200/`` consume its output; neither is
imported here.
"""
from .gen import (  # noqa: F401
    CONFIGS,
    fimi_text,
    Workload,
    make_config,
    quest,
    to_horizontal,
    uniform,
    zipf,
)
