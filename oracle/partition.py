"""O2-O6: the per-partition split of P (TEST INFRASTRUCTURE ONLY, see oracle/__init__).

Follows the matrix form of the stale-representation layer, Eq. 5:
"P_in^(m) and P_out^(m) denotes the propagation matrix for in-subgraph nodes and
out-of-subgraph nodes of G_m ... P_m = P_in^(m) + P_out^(m)", and the halo set of
§3.2: H~_out^(l,m) = { h~_u : u in N(v) \\ V_m, for all v in V_m }.

Orderings (reading A4, paper silent):
  * V_m: ascending global id; loc(v) = rank in V_m.
  * H_m: ordered by (part_of[u], u); ext(u) = n_m + rank in H_m.
  * row loc(v) of P_m holds {(ext(u), P_vu) : u in N(v)} U {(loc(v), P_vv)},
    sorted by extended column; columns < n_m form P_in, the rest P_out.
  * S_{m->k} = {u in V_m : N(u) ∩ V_k != ∅} ascending, concatenated over k != m
    in ascending k (the boundary rows part m pushes to part k, "push").
  * reverse-halo CSR (P_out transposed): halo row j lists (i, P) for local i with
    H_m[j] in N(V_m[i]), ascending i.
"""
from dataclasses import dataclass
import numpy as np

from .propagation import degrees, prop_values


@dataclass
class OraclePartition:
    num_parts: int
    rank: int
    local_ids: np.ndarray   # int32 [n_m]      V_m
    halo_ids: np.ndarray    # int32 [h_m]      H_m
    row_ptr: np.ndarray     # int64 [n_m+1]
    col: np.ndarray         # int32 [E_m]      extended column index
    val: np.ndarray         # fp32  [E_m]
    send_idx: np.ndarray    # int32 [sum_k |S_m->k|] local indices
    send_count: np.ndarray  # int64 [M]
    send_off: np.ndarray    # int64 [M]
    recv_count: np.ndarray  # int64 [M]
    recv_off: np.ndarray    # int64 [M]
    rh_ptr: np.ndarray      # int64 [h_m+1]   reverse-halo CSR
    rh_col: np.ndarray      # int32
    rh_val: np.ndarray      # fp32

    @property
    def n_local(self) -> int:
        return int(self.local_ids.size)

    @property
    def n_halo(self) -> int:
        return int(self.halo_ids.size)

    @property
    def nnz(self) -> int:
        return int(self.col.size)

    @property
    def nnz_in(self) -> int:
        return int(np.count_nonzero(self.col < self.n_local))


def _unique_sorted(a: np.ndarray) -> np.ndarray:
    """Sorted distinct values (a library sort, then a neighbour comparison)."""
    a = np.sort(a)
    if a.size == 0:
        return a
    return a[np.concatenate([[True], a[1:] != a[:-1]])]


def _row_gather(indptr, indices, rows):
    """For each row r in `rows` (in order): (position of r in rows, neighbour u)."""
    cnt = indptr[rows + 1] - indptr[rows]
    total = int(cnt.sum())
    owner = np.repeat(np.arange(rows.size, dtype=np.int64), cnt)
    first = np.repeat(indptr[rows] - (np.cumsum(cnt) - cnt), cnt)
    nbr = indices[first + np.arange(total, dtype=np.int64)]
    return owner, nbr.astype(np.int64)


def oracle_partition(indptr, indices, part_of, num_parts: int, rank: int) -> OraclePartition:
    indptr = np.asarray(indptr, dtype=np.int64)
    indices = np.asarray(indices, dtype=np.int64)
    part_of = np.asarray(part_of, dtype=np.int64)
    n_nodes = indptr.size - 1
    if num_parts < 1 or num_parts > n_nodes or part_of.min() < 0 or part_of.max() >= num_parts:
        raise ValueError("invalid partition")
    if np.bincount(part_of, minlength=num_parts).min() == 0:
        raise ValueError("empty part")  # A26 / S:110 every part non-empty
    m = rank
    deg = degrees(indptr)

    # O2: V_m ascending, loc(v)
    V = np.flatnonzero(part_of == m)
    n = V.size

    # O3: halo = neighbours of V_m outside V_m, ordered by (owner, id)
    src, nbr = _row_gather(indptr, indices, V)
    H = _unique_sorted(nbr[part_of[nbr] != m])
    H = H[np.argsort(part_of[H], kind="stable")]
    h = H.size
    ext = np.full(n_nodes, -1, dtype=np.int64)
    ext[V] = np.arange(n)
    ext[H] = n + np.arange(h)

    # O4: local CSR over extended columns, plus the self loop, sorted by column
    rows = np.concatenate([src, np.arange(n)])
    cols = np.concatenate([ext[nbr], np.arange(n)])
    vals = np.concatenate([prop_values(deg[V][src], deg[nbr]), prop_values(deg[V], deg[V])])
    order = np.lexsort((cols, rows))
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    col = cols[order].astype(np.int32)
    val = vals[order]

    # O5: send lists and receive counts
    nbr_part = part_of[nbr]
    send_lists, send_count = [], np.zeros(num_parts, dtype=np.int64)
    for k in range(num_parts):
        if k == m:
            continue
        s = _unique_sorted(src[nbr_part == k])     # local indices i with a neighbour in V_k
        send_lists.append(s)
        send_count[k] = s.size
    send_idx = (np.concatenate(send_lists) if send_lists else np.zeros(0, np.int64)).astype(np.int32)
    send_off = np.concatenate([[0], np.cumsum(send_count)[:-1]]).astype(np.int64)
    recv_count = np.bincount(part_of[H], minlength=num_parts).astype(np.int64)
    recv_off = np.concatenate([[0], np.cumsum(recv_count)[:-1]]).astype(np.int64)

    # O6: reverse-halo CSR = transpose of the P_out block
    is_h = ext[nbr] >= n
    hrow = ext[nbr[is_h]] - n
    hcol = src[is_h]
    hval = prop_values(deg[V][hcol], deg[nbr[is_h]])
    order = np.lexsort((hcol, hrow))
    rh_ptr = np.zeros(h + 1, dtype=np.int64)
    np.cumsum(np.bincount(hrow, minlength=h), out=rh_ptr[1:])

    return OraclePartition(num_parts, m, V.astype(np.int32), H.astype(np.int32), row_ptr,
                           col, val, send_idx, send_count, send_off, recv_count, recv_off,
                           rh_ptr, hcol[order].astype(np.int32), hval[order])
