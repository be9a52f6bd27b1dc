"""Dense brute force from the definitions, for tiny graphs (n <= 64).

Independent of oracle/: it builds the dense P = D~^{-1/2}(A+I)D~^{-1/2} with
matrix operations, splits it with Python loops and index sets, and applies Eq. 5,
Eq. 6 and P:783-794 with dense matrix products.  Used only to pin the oracle.
"""
import numpy as np


def dense_adjacency(indptr, indices):
    n = len(indptr) - 1
    A = np.zeros((n, n))
    for v in range(n):
        for e in range(indptr[v], indptr[v + 1]):
            A[v, indices[e]] = 1.0
    return A


def dense_P(indptr, indices, round_fp32=True):
    A = dense_adjacency(indptr, indices)
    At = A + np.eye(A.shape[0])
    Dm = np.diag(1.0 / np.sqrt(At.sum(axis=1)))
    P = Dm @ At @ Dm
    if round_fp32:
        P = P.astype(np.float32).astype(np.float64)
    return P


def brute_partition(indptr, indices, part_of, num_parts, m):
    """Pure-Python loops over the definitions of V_m, H_m, the CSR rows and send lists."""
    n = len(indptr) - 1
    nbrs = [list(indices[indptr[v]:indptr[v + 1]]) for v in range(n)]
    P = dense_P(indptr, indices)
    V = [v for v in range(n) if part_of[v] == m]
    loc = {v: i for i, v in enumerate(V)}
    hs = set()
    for v in V:
        for u in nbrs[v]:
            if part_of[u] != m:
                hs.add(int(u))
    H = sorted(hs, key=lambda u: (int(part_of[u]), u))
    ext = dict(loc)
    for j, u in enumerate(H):
        ext[u] = len(V) + j
    row_ptr, col, val = [0], [], []
    for v in V:
        ent = [(ext[int(u)], P[v, u]) for u in nbrs[v]] + [(ext[v], P[v, v])]
        ent.sort()
        col += [c for c, _ in ent]
        val += [x for _, x in ent]
        row_ptr.append(len(col))
    send, scount = [], [0] * num_parts
    for k in range(num_parts):
        if k == m:
            continue
        s = [loc[v] for v in V if any(part_of[u] == k for u in nbrs[v])]
        send += s
        scount[k] = len(s)
    rcount = [sum(1 for u in H if part_of[u] == k) for k in range(num_parts)]
    rh_ptr, rh_col, rh_val = [0], [], []
    for u in H:
        ent = sorted((loc[int(v)], P[v, u]) for v in nbrs[u] if part_of[v] == m)
        rh_col += [c for c, _ in ent]
        rh_val += [x for _, x in ent]
        rh_ptr.append(len(rh_col))
    return dict(V=V, H=H, row_ptr=row_ptr, col=col, val=val, send=send, send_count=scount,
                recv_count=rcount, rh_ptr=rh_ptr, rh_col=rh_col, rh_val=rh_val)


def brute_block(P, V, H):
    """P_m = P[V_m, V_m ++ H_m] (dense)."""
    return P[np.ix_(list(V), list(V) + list(H))]


def brute_layer_forward(Pm, x_ext, w, relu):
    A = Pm @ x_ext
    Z = A @ w
    return A, Z, (np.maximum(Z, 0) if relu else Z)


def brute_layer_backward(Pm, n_local, x_ext, w, Z, g_out, relu):
    D = g_out * (Z > 0) if relu else g_out
    G_W = (Pm @ x_ext).T @ D
    G_in = Pm[:, :n_local].T @ D @ w.T
    return G_W, G_in
