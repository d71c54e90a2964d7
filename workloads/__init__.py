"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the method: it only produces inputs —
dependency DAGs (edge lists), workload shapes, bf16 random bytes and a paged
memory layout (which physical pages hold which token range).  Level/segment
computation, segment binding, attention and append live separately in
`oracle/` (CPU reference) and `paper_2510_24390_b200/` (CUDA path); neither
imports the other.  Recipe: DESIGN.md §"Input recipe".
"""
from .dags import (EDGE_NULL, EDGE_CONTEXTUAL, EDGE_DEPENDENT, DAGS, diamond, fig4,
                   mixed8, mixed16, wide, chain, edgeless, random_dag)
from .configs import CONFIGS, Config, get_config
from .tensors import bf16_randn_u16, make_layout, Layout, make_qkv

__all__ = [
    "EDGE_NULL", "EDGE_CONTEXTUAL", "EDGE_DEPENDENT", "DAGS", "diamond", "fig4", "mixed8",
    "mixed16", "wide", "chain", "edgeless", "random_dag", "CONFIGS", "Config", "get_config",
    "bf16_randn_u16", "make_layout", "Layout", "make_qkv",
]
