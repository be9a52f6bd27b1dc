"""O7-O12: the stale store, Alg. 1's schedule and the epoch loop; full-graph GCN.

TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Schedule, Alg. 1, 1-based epochs r, levels l in [1, L-1] only
("l != L"; reading A6 -- layer 1's halo inputs are the exact features):
  * PULL  if r % N == 0:        halo^(l,m) <- committed^(l)[H_m]
  * PUSH  if (r-1) % N == 0:    pending^(l)[V_m] <- H^(l)[V_m]
  * pushes are committed at the end of epoch r, so a pull only ever sees versions
    < r (reading A7; "After the end of a epoch ... pushed").  All of epoch
    r's pulls happen at epoch start (Alg. 1 pulls level l before computing it).
  * cold start (A8): committed = halo = 0 ('zero'), or the exact full-graph
    representations at W^(1) ('prime').
  * one forward, one backward and one optimizer step per epoch (A10); AGG
     = sum of the parts' gradients then one identical step (A11).
  * loss weighting (A12): 'count' = sum over all training nodes / #train (the
    full-graph objective); 'per_part' = (1/M) sum_m mean over V_m ∩ train
    (Eq. 3 P:100 with the (1/M) sum of P:702).
  * mode 'fresh' (reading A15, a test hook): after every part computed
    level l, halo^(l,m) is set to the CURRENT epoch's values (zero staleness).
  * store_dtype 'bf16': the store keeps the pushed rows rounded to
    bfloat16 (fp32 first, then round-to-nearest-even to 8 significant bits), so the
    pulled halo rows carry that rounding.
"""
from dataclasses import dataclass, field
import numpy as np
import scipy.sparse as sp

from .partition import oracle_partition
from .gcn import (layer_forward, layer_backward, cross_entropy, sgd_step, adam_step,
                  normalize_rows, prop_matrix)


def bf16_round(x):
    """fp64 -> fp32 (RNE) -> bfloat16 (RNE on the top 16 bits of the fp32 pattern), as fp64.
    Finite inputs only (the store never holds NaN/Inf)."""
    f = np.ascontiguousarray(np.asarray(x, np.float32)).view(np.uint32).astype(np.uint64)
    lsb = (f >> 16) & 1
    r = ((f + 0x7FFF + lsb) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32).astype(np.float64)


# ---------------------------------------------------------------- full graph (O12 i)
def full_prop_matrix(indptr, indices) -> sp.csr_matrix:
    """P = D~^{-1/2}(A+I)D~^{-1/2} (Kipf), entries rounded to fp32 (A2)."""
    n = len(indptr) - 1
    A = sp.csr_matrix((np.ones(len(indices)), np.asarray(indices, np.int64),
                       np.asarray(indptr, np.int64)), shape=(n, n))
    At = A + sp.identity(n, format="csr")
    dinv = 1.0 / np.sqrt(np.asarray(At.sum(axis=1)).ravel())
    P = (sp.diags(dinv) @ At @ sp.diags(dinv)).tocsr()
    P.data = P.data.astype(np.float32).astype(np.float64)
    return P


def full_graph_forward(P, x, weights):
    """Single-machine GCN: Z = P H W, H = relu(Z) (identity last)."""
    L = len(weights)
    H = [np.asarray(x, np.float64)]
    Z = []
    for l in range(L):
        z = (P @ H[-1]) @ np.asarray(weights[l], np.float64)
        Z.append(z)
        H.append(np.maximum(z, 0) if l < L - 1 else z)
    return H, Z


def full_graph_backward(P, H, Z, weights, g_logits):
    """G_H = P^T D W^T, G_W = (P H)^T D, D = G o sigma'(Z)."""
    L = len(weights)
    grads = [None] * L
    G = np.asarray(g_logits, np.float64)
    for l in range(L - 1, -1, -1):
        D = G if l == L - 1 else G * (Z[l] > 0)
        grads[l] = (P @ H[l]).T @ D
        if l > 0:
            G = P.T @ (D @ np.asarray(weights[l], np.float64).T)
    return grads


# ---------------------------------------------------------------- partitioned training
@dataclass
class EpochRecord:
    epoch: int
    loss: float
    grads: list                   # aggregated G_W per layer (fp64)
    weights_used: list            # W at the start of the epoch
    pulled: bool
    pushed: bool
    halo_versions: dict = field(default_factory=dict)   # (l, m) -> int array
    halo_used: dict = field(default_factory=dict)       # (l, m) -> halo values used
    reps: dict = field(default_factory=dict)            # l -> global [N, d_l] DIGEST H^(l)
    part_out: dict = field(default_factory=dict)        # (l, m) -> dict(A,Z,H)
    eps: dict = field(default_factory=dict)             # l -> max_u ||h~_u - h_u||
    part_d: dict = field(default_factory=dict)          # (l, m) -> D^(l) of the part
    halo_grad_sent: dict = field(default_factory=dict)  # (l, m) -> G_halo rows returned


@dataclass
class OracleRun:
    parts: list
    records: list
    weights: list
    pull_count: int = 0
    push_count: int = 0


def oracle_train(indptr, indices, x, y, train_mask, weights, num_classes, part_of,
                 num_parts, sync_interval, epochs, lr=0.01, optimizer="sgd",
                 cold_start="zero", mode="stale", normalize_pushed=False,
                 loss_weighting="count", record_outputs=False, parts=None,
                 halo_grad="none", store_dtype="fp32") -> OracleRun:
    """halo_grad (the gradient a part sends back for its halo rows):
      'none'        halo inputs are constants of the iteration (Eq. 6) -- default;
      'prev_epoch'  the appendix's DIGEST backward, literally:
                    G~_H^(t) = P_in^T D~^(t) (W~^(t))^T + P_out^T D~^(t-1) (W~^(t))^T, i.e.
                    each part keeps S^(t) = P_out^T D~^(t) of its halo rows and, in
                    iteration t+1, returns S^(t) (W^(t+1))^T to the owners (zero at t=1);
      'same_epoch'  the exact (zero-staleness) variant: P_out^T D~^(t) (W^(t))^T returned in
                    the same iteration t -- with fresh halos every G_W equals full-graph GCN
                    (reading A16).  Not the paper's term; the exact reference for it."""
    if halo_grad not in ("none", "same_epoch", "prev_epoch"):
        raise ValueError(halo_grad)
    if store_dtype not in ("fp32", "bf16"):
        raise ValueError(store_dtype)
    store = bf16_round if store_dtype == "bf16" else (lambda v: v)
    if sync_interval < 1 or epochs < 1:
        raise ValueError("sync interval and epochs must be >= 1")
    M, Ns = num_parts, sync_interval
    W = [np.asarray(w, np.float64).copy() for w in weights]
    L = len(W)
    dims = [W[0].shape[0]] + [w.shape[1] for w in W]
    n_nodes = len(indptr) - 1
    x = np.asarray(x, np.float64)
    train = np.asarray(train_mask).astype(bool)
    if parts is None:
        parts = [oracle_partition(indptr, indices, part_of, M, m) for m in range(M)]
    n_train = int(train.sum())
    if loss_weighting == "count":
        wl = [1.0 / n_train if n_train else 0.0] * M
    else:
        wl = []
        for p in parts:
            t = int(train[p.local_ids].sum())
            wl.append(1.0 / (M * t) if t else 0.0)

    committed = {l: np.zeros((n_nodes, dims[l])) for l in range(1, L)}
    version = {l: np.zeros(n_nodes, np.int64) for l in range(1, L)}
    if cold_start == "prime":
        Pf = full_prop_matrix(indptr, indices)
        Hs, _ = full_graph_forward(Pf, x, W)
        for l in range(1, L):
            committed[l] = Hs[l].copy()
    elif cold_start != "zero":
        raise ValueError(cold_start)
    halo = {(l, m): committed[l][p.halo_ids].copy() for l in range(1, L) for m, p in enumerate(parts)}
    halo_ver = {(l, m): version[l][p.halo_ids].copy() for l in range(1, L) for m, p in enumerate(parts)}
    opt_state = [(np.zeros_like(w), np.zeros_like(w)) for w in W]
    # prev_epoch: S^(t-1) = P_out^T D~^(t-1) per (layer l >= 2, part m), zero before t = 1
    s_prev = {(l, m): np.zeros((p.n_halo, dims[l])) for l in range(2, L + 1)
              for m, p in enumerate(parts)}

    run = OracleRun(parts, [], W)
    for r in range(1, epochs + 1):
        pull = mode == "stale" and r % Ns == 0
        push = (r - 1) % Ns == 0
        rec = EpochRecord(r, 0.0, [], [w.copy() for w in W], pull, push)
        if pull:
            for l in range(1, L):
                for m, p in enumerate(parts):
                    halo[(l, m)] = committed[l][p.halo_ids].copy()
                    halo_ver[(l, m)] = version[l][p.halo_ids].copy()
                    run.pull_count += 1
        pending = {}
        outs = {}
        loc_in = {m: x[p.local_ids] for m, p in enumerate(parts)}
        halo_in = {m: x[p.halo_ids] for m, p in enumerate(parts)}
        inputs = {}
        for l in range(1, L + 1):
            glob = np.zeros((n_nodes, dims[l])) if l < L else None
            for m, p in enumerate(parts):
                inputs[(l, m)] = (loc_in[m], halo_in[m])
                o = layer_forward(p, loc_in[m], halo_in[m], W[l - 1], relu=l < L)
                outs[(l, m)] = o
                if glob is not None:
                    glob[p.local_ids] = o["H"]
            if l == L:
                break
            if mode == "fresh":
                for m, p in enumerate(parts):
                    halo[(l, m)] = store(glob[p.halo_ids])
                    halo_ver[(l, m)] = np.full(p.n_halo, r, np.int64)
            rec.eps[l] = max([float(np.sqrt(((halo[(l, m)] - glob[p.halo_ids]) ** 2).sum(1)).max())
                              if p.n_halo else 0.0 for m, p in enumerate(parts)])
            for m, p in enumerate(parts):
                rec.halo_versions[(l, m)] = halo_ver[(l, m)].copy()
                if record_outputs:
                    rec.halo_used[(l, m)] = halo[(l, m)].copy()
                loc_in[m] = outs[(l, m)]["H"]
                halo_in[m] = halo[(l, m)]
            if push:
                pending[l] = store(normalize_rows(glob) if normalize_pushed else glob)
                run.push_count += M
            rec.reps[l] = glob
        # loss, backward (layer-major over the parts), AGG, update
        total = [np.zeros_like(w) for w in W]
        g = {}
        for m, p in enumerate(parts):
            loss, g[m] = cross_entropy(outs[(L, m)]["H"], y[p.local_ids], train[p.local_ids],
                                       num_classes, wl[m])
            rec.loss += loss
        for l in range(L, 0, -1):
            gin, ghalo = {}, {}
            for m, p in enumerate(parts):
                xl, xh = inputs[(l, m)]
                mask = None if l == L else outs[(l, m)]["Z"] > 0
                b = layer_backward(p, xl, xh, W[l - 1], g[m], mask, need_g_in=l >= 2,
                                   need_g_halo=(halo_grad == "same_epoch" and l >= 2))
                total[l - 1] += b["G_W"]
                gin[m], ghalo[m] = b["G_in"], b["G_halo"]
                if record_outputs:
                    rec.part_d[(l, m)] = b["D"]
                if halo_grad == "prev_epoch" and l >= 2:
                    # P_out^T D~^(t-1) (W~^(t))^T -- last iteration's D, this one's W
                    P_out = prop_matrix(p)[:, p.n_local:]
                    ghalo[m] = s_prev[(l, m)] @ W[l - 1].T
                    s_prev[(l, m)] = P_out.T @ b["D"]
            if l >= 2 and halo_grad != "none":
                # the returned term: rows of G_halo of part m go to the owners of its halo
                # nodes and add into their G^(l-1) before sigma'
                for m, p in enumerate(parts):
                    if record_outputs:
                        rec.halo_grad_sent[(l, m)] = ghalo[m].copy()
                    owner = np.asarray(part_of)[p.halo_ids]
                    for k, pk in enumerate(parts):
                        sel = np.flatnonzero(owner == k)
                        if sel.size:
                            loc_k = np.searchsorted(pk.local_ids, p.halo_ids[sel])
                            np.add.at(gin[k], loc_k, ghalo[m][sel])
            g = gin
        rec.grads = total
        if record_outputs:
            rec.part_out = outs
        for l in range(L):
            if optimizer == "sgd":
                W[l] = sgd_step(W[l], total[l], lr)
            else:
                mm, vv = opt_state[l]
                W[l], mm, vv = adam_step(W[l], total[l], mm, vv, r, lr)
                opt_state[l] = (mm, vv)
        for l, val in pending.items():   # commit at epoch end: visible to later epochs only
            for p in parts:
                committed[l][p.local_ids] = val[p.local_ids]
                version[l][p.local_ids] = r
        run.records.append(rec)
    run.weights = W
    return run
