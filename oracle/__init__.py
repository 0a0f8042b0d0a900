"""TEST INFRASTRUCTURE ONLY — the CPU oracle (see oracle.cpp header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.
"""
from .oracle import Oracle, build, hop_delay_exact, ring_sim, pipeline, pipeline_ilv, op_order, hamilton, needs_reshard, maxmin  # noqa: F401
