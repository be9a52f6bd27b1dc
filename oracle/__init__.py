"""DIGEST CPU oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, fp64 CPU implementation of the partitioned stale-halo GCN that
DIGEST (arXiv 2206.00057) trains.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / `--impl reference` leg may import, call or execute
anything in this package.  The product path (`paper_2206_00057_b200`) never does,
and the two share no code: the only common inputs come from `synth/`.

Citations: `P:n` = PAPER.md line n (section / equation noted), `S:n` = SPEC.md
line n.  Every function names the passage it follows; DESIGN.md lists the readings
taken where the paper is silent, garbled or inconsistent (A1..A26 of SURVEY §8.c.2).

Parity status: every function here is pinned by `tests/test_oracle_*.py`
(worked examples, closed forms, brute force, finite differences, special cases),
except the ones whose docstring says "parity unpinned".
"""
from .propagation import prop_values, degrees
from .partition import oracle_partition, OraclePartition
from .gcn import (layer_forward, layer_backward, cross_entropy, sgd_step, adam_step,
                  normalize_rows)
from .train import oracle_train, OracleRun, full_graph_forward, full_graph_backward
from .bound import theorem1_bound, staleness_bound_check

__all__ = ["prop_values", "degrees", "oracle_partition", "OraclePartition",
           "layer_forward", "layer_backward", "cross_entropy", "sgd_step", "adam_step",
           "normalize_rows", "oracle_train", "OracleRun", "full_graph_forward",
           "full_graph_backward", "theorem1_bound", "staleness_bound_check"]
