"""Seeded synthetic inputs shared by the tests, smoke() and bench.py.

This package holds no PCPM arithmetic: it only draws graphs and vectors from a
counter-based generator (``rng``) and canonicalises them into CSR
(``graphs``).  Both the oracle (``oracle/``) and the CUDA path
(``paper_1709_07122_b200``) consume its output; neither is imported here.
"""
from .rng import counter_hash_np, counter_hash_torch  # noqa: F401
from .graphs import (  # noqa: F401
    CONFIGS, GraphCSR, make_config, rmat_edges, er_edges, edges_to_csr, random_permutation,
)
