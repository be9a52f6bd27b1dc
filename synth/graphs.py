"""Planted-partition Chung-Lu graphs and the other seeded inputs.

Construction (generation only; no DIGEST arithmetic lives here):
  1. K contiguous blocks, block(v) = floor(v*K/N).
  2. Mean-1 log-normal weights w_v = exp(sigma*z - sigma^2/2), capped.
  3. Undirected pairs: u ~ w globally; with prob 1-mu, v ~ w inside block(u),
     otherwise inside a uniformly chosen other block.
  4. Drop self pairs, deduplicate, drop a seeded random excess so exactly nnz/2
     unique pairs remain, symmetrise to a CSR with sorted, duplicate-free rows.
  5. Partition part_of(v) = floor(block(v)*M/K): contiguous id ranges, so the
     1/2/4/8-part runs share one graph.
"""
from dataclasses import dataclass
import numpy as np
import torch

from .configs import GraphConfig


def _searchsorted(sorted_arr: np.ndarray, q: np.ndarray) -> np.ndarray:
    """Right-sided searchsorted (multithreaded through torch's CPU kernel)."""
    return torch.searchsorted(torch.from_numpy(sorted_arr), torch.from_numpy(q),
                              right=True).numpy()


def _block_of(n: int, k: int) -> np.ndarray:
    return (np.arange(n, dtype=np.int64) * k) // n


def make_graph(cfg: GraphConfig):
    """Return (indptr int64[N+1], indices int32[nnz]) of a symmetric graph.

    Rows are sorted ascending, have no duplicates and no self loops."""
    n, need = cfg.num_nodes, cfg.nnz // 2
    if need > n * (n - 1) // 2:
        raise ValueError("more edges requested than a simple graph can hold")
    k = max(1, min(cfg.blocks, n))
    rng = np.random.default_rng(cfg.seed)
    block = _block_of(n, k)
    bstart = np.searchsorted(block, np.arange(k), side="left")
    bend = np.searchsorted(block, np.arange(k), side="right")
    z = rng.standard_normal(n)
    w = np.exp(cfg.sigma * z - 0.5 * cfg.sigma ** 2)
    avg_deg = max(cfg.nnz / n, 1e-9)
    w = np.minimum(w, max(1.0, 0.2 * (n / k) / avg_deg))
    cw = np.cumsum(w)
    lo_w = np.where(bstart > 0, cw[np.maximum(bstart - 1, 0)], 0.0)
    hi_w = cw[bend - 1]

    keys = np.empty(0, dtype=np.int64)
    for _ in range(10000):
        have = keys.size
        if have >= need:
            break
        batch = int((need - have) * 1.08) + 1024
        u = _searchsorted(cw, rng.random(batch) * cw[-1])
        np.minimum(u, n - 1, out=u)
        bu = block[u]
        if k > 1:
            cross = rng.random(batch) < cfg.mu
            other = (bu + 1 + rng.integers(0, k - 1, batch)) % k
            tb = np.where(cross, other, bu)
        else:
            tb = bu
        v = _searchsorted(cw, lo_w[tb] + rng.random(batch) * (hi_w[tb] - lo_w[tb]))
        v = np.clip(v, bstart[tb], bend[tb] - 1)
        keep = u != v
        a = np.minimum(u[keep], v[keep])
        b = np.maximum(u[keep], v[keep])
        keys = np.concatenate([keys, a * n + b])
        keys.sort()
        keys = keys[np.concatenate([[True], keys[1:] != keys[:-1]])]
    else:  # pragma: no cover
        raise RuntimeError("edge sampling did not converge")
    if keys.size > need:  # drop a seeded random excess so exactly nnz/2 pairs remain
        drop = rng.choice(keys.size, keys.size - need, replace=False)
        keys = np.delete(keys, drop)

    a, b = keys // n, keys % n
    sym = np.concatenate([a * n + b, b * n + a])
    sym.sort()
    rows = sym // n
    indices = (sym - rows * n).astype(np.int32)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=indptr[1:])
    return indptr, indices


def make_features(cfg: GraphConfig) -> np.ndarray:
    """X ~ U(-1, 1), fp32 [N, d0_pad], padding columns zero."""
    rng = np.random.default_rng(cfg.seed + 1)
    x = np.zeros((cfg.num_nodes, cfg.d0_pad), dtype=np.float32)
    x[:, :cfg.d0] = rng.random((cfg.num_nodes, cfg.d0), dtype=np.float32) * 2.0 - 1.0
    return x


def make_labels(cfg: GraphConfig) -> np.ndarray:
    """y_v = block(v) mod C with probability 0.8, else uniform in [0, C)."""
    rng = np.random.default_rng(cfg.seed + 2)
    n, c = cfg.num_nodes, cfg.num_classes
    y = _block_of(n, max(1, min(cfg.blocks, n))) % c
    flip = rng.random(n) >= 0.8
    y = np.where(flip, rng.integers(0, c, n), y)
    return y.astype(np.int32)


def make_train_mask(cfg: GraphConfig) -> np.ndarray:
    """First round(frac*N) nodes of a seeded permutation are training nodes."""
    rng = np.random.default_rng(cfg.seed + 3)
    n = cfg.num_nodes
    m = np.zeros(n, dtype=np.uint8)
    m[rng.permutation(n)[: int(round(cfg.train_frac * n))]] = 1
    return m


def make_weights(cfg: GraphConfig) -> list:
    """Glorot-uniform W^(l) of shape [dims[l-1], dims[l]] (fp32).

    Only the unpadded block [raw d_{l-1}, raw d_l] is random; padded rows (feature
    padding) and padded columns (class padding) are zero."""
    dims, raw = cfg.dims, cfg.raw_dims
    out = []
    for l in range(1, len(dims)):
        rng = np.random.default_rng(cfg.seed + 10 + l)
        a = np.sqrt(6.0 / (raw[l - 1] + raw[l]))
        w = np.zeros((dims[l - 1], dims[l]), dtype=np.float32)
        w[: raw[l - 1], : raw[l]] = (rng.random((raw[l - 1], raw[l])) * 2 * a - a).astype(np.float32)
        out.append(w)
    return out


def make_block_parts(cfg: GraphConfig, num_parts: int) -> np.ndarray:
    """part_of(v) = floor(block(v) * M / K) (contiguous id ranges)."""
    n = cfg.num_nodes
    k = max(1, min(cfg.blocks, n))
    if num_parts > k:
        # more parts than planted blocks: split contiguous id ranges evenly instead
        return ((np.arange(n, dtype=np.int64) * num_parts) // n).astype(np.int32)
    return ((_block_of(n, k) * num_parts) // k).astype(np.int32)


def make_random_parts(num_nodes: int, num_parts: int, seed: int) -> np.ndarray:
    """A seeded random assignment with every part non-empty (non-contiguous parts)."""
    if num_parts > num_nodes:
        raise ValueError("more parts than nodes")
    rng = np.random.default_rng(seed)
    p = rng.integers(0, num_parts, num_nodes)
    p[rng.permutation(num_nodes)[:num_parts]] = np.arange(num_parts)
    return p.astype(np.int32)


@dataclass
class SyntheticInputs:
    cfg: GraphConfig
    indptr: np.ndarray
    indices: np.ndarray
    x: np.ndarray
    y: np.ndarray
    train_mask: np.ndarray
    weights: list


def make_inputs(cfg: GraphConfig) -> SyntheticInputs:
    indptr, indices = make_graph(cfg)
    return SyntheticInputs(cfg, indptr, indices, make_features(cfg), make_labels(cfg),
                           make_train_mask(cfg), make_weights(cfg))
