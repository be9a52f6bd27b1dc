"""Small test-input builders (no DIGEST arithmetic)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def csr_from_edges(n, edges):
    """Symmetric CSR with sorted, deduplicated rows and no self loops."""
    s = set()
    for a, b in edges:
        if a != b:
            s.add((a, b))
            s.add((b, a))
    rows = [[] for _ in range(n)]
    for a, b in sorted(s):
        rows[a].append(b)
    indptr = np.zeros(n + 1, dtype=np.int64)
    indptr[1:] = np.cumsum([len(r) for r in rows])
    indices = np.array([b for r in rows for b in r], dtype=np.int32)
    return indptr, indices


def random_graph(n, p, rng):
    edges = [(a, b) for a in range(n) for b in range(a + 1, n) if rng.random() < p]
    return csr_from_edges(n, edges)


def random_parts(n, M, rng):
    p = rng.integers(0, M, n)
    p[rng.permutation(n)[:M]] = np.arange(M)
    return p.astype(np.int32)
