"""DIGEST-A, the asynchronous mode (SPEC train_async S:380-388).

TEST INFRASTRUCTURE ONLY (see oracle/__init__).

The paper: "To support the asynchronous mode (DIGEST-A), we can simply remove the loop
of training epoch and move the parameter aggregation (Line 13) into the subgraph loop"
(P:243); each subgraph "directly pulls/pushes stale representations of other subgraphs
from the shared KVS and downloads/uploads parameters from the PS without blindly
waiting for the slowest subgraph".  Readings (DIGEST-A):

  * R1: a worker's local epoch = download W_global, one local epoch of
    Alg. 1 (pull if r_m % N == 0 and push if (r_m - 1) % N == 0, keyed on its OWN local
    epoch counter r_m, levels 1..L-1), one local optimizer step, upload; the PS mixes
    W_global <- (1 - alpha) W_global + alpha W_m (alpha = 1/M by default), atomically
    per upload.
  * R2: the local objective is the part's own mean loss over its training nodes (Eq. 3,
    P:100, L_m with w_loss = 1/|V_m ∩ train|); the step is SGD or Adam with a
    per-worker optimizer state whose step count is r_m.
  * R3: asynchrony is an input: `events` lists which worker completes its next local
    epoch, in completion order (synth.async_sched).  Events are applied one after the
    other; a push is visible to every later event (the KVS is shared), a pull
    copies the latest committed rows of every owner.
  * Cold start: zero halos (A8), as in the synchronous oracle.
"""
from dataclasses import dataclass, field

import numpy as np

from .partition import oracle_partition
from .gcn import layer_forward, layer_backward, cross_entropy, sgd_step, adam_step


@dataclass
class AsyncRecord:
    worker: int
    local_epoch: int
    loss: float
    pulled: bool
    pushed: bool
    uploaded: list = field(default_factory=list)       # W_m uploaded (record_weights)
    halo_versions: dict = field(default_factory=dict)  # l -> event index of each halo row
    halos: dict = field(default_factory=dict)          # l -> halo rows used (record_halos)


@dataclass
class AsyncRun:
    parts: list
    records: list
    weights: list            # W_global after the last upload
    ps_updates: int = 0
    pull_count: int = 0
    push_count: int = 0


def oracle_train_async(indptr, indices, x, y, train_mask, weights, num_classes, part_of,
                       num_parts, sync_interval, events, lr=0.01, optimizer="sgd", alpha=None,
                       parts=None, record_weights=False, record_halos=False) -> AsyncRun:
    if sync_interval < 1:
        raise ValueError("sync interval must be >= 1")
    M, Ns = num_parts, sync_interval
    a = 1.0 / M if alpha is None else float(alpha)
    Wg = [np.asarray(w, np.float64).copy() for w in weights]
    L = len(Wg)
    dims = [Wg[0].shape[0]] + [w.shape[1] for w in Wg]
    n_nodes = len(indptr) - 1
    x = np.asarray(x, np.float64)
    train = np.asarray(train_mask).astype(bool)
    if parts is None:
        parts = [oracle_partition(indptr, indices, part_of, M, m) for m in range(M)]
    wl = []
    for p in parts:
        t = int(train[p.local_ids].sum())
        wl.append(1.0 / t if t else 0.0)
    committed = {l: np.zeros((n_nodes, dims[l])) for l in range(1, L)}
    cver = {l: np.full(n_nodes, -1, np.int64) for l in range(1, L)}    # event of the push
    halo = {(l, m): np.zeros((p.n_halo, dims[l])) for l in range(1, L) for m, p in enumerate(parts)}
    hver = {(l, m): np.full(p.n_halo, -1, np.int64) for l in range(1, L) for m, p in enumerate(parts)}
    opt = [[(np.zeros_like(w), np.zeros_like(w)) for w in Wg] for _ in range(M)]
    r = [0] * M
    run = AsyncRun(parts, [], Wg)
    for ev, m in enumerate(events):
        p = parts[m]
        r[m] += 1
        rm = r[m]
        Wm = [w.copy() for w in Wg]                       # download
        pull, push = rm % Ns == 0, (rm - 1) % Ns == 0      # Alg. 1 guards on r_m
        rec = AsyncRecord(m, rm, 0.0, pull, push)
        if pull:
            for l in range(1, L):
                halo[(l, m)] = committed[l][p.halo_ids].copy()
                hver[(l, m)] = cver[l][p.halo_ids].copy()
                run.pull_count += 1
        xl, xh = x[p.local_ids], x[p.halo_ids]
        inputs, outs = {}, {}
        for l in range(1, L + 1):                          # Eq. 5 per layer
            inputs[l] = (xl, xh)
            o = layer_forward(p, xl, xh, Wm[l - 1], relu=l < L)
            outs[l] = o
            if l < L:
                rec.halo_versions[l] = hver[(l, m)].copy()
                if record_halos:
                    rec.halos[l] = halo[(l, m)].copy()
                if push:                                   # visible to later events
                    committed[l][p.local_ids] = o["H"]
                    cver[l][p.local_ids] = ev
                    run.push_count += 1
                xl, xh = o["H"], halo[(l, m)]
        loss, g = cross_entropy(outs[L]["H"], y[p.local_ids], train[p.local_ids], num_classes,
                                wl[m])
        rec.loss = loss
        G = [None] * L
        for l in range(L, 0, -1):                          # Eq. 6, halo constant
            a_l, h_l = inputs[l]
            mask = None if l == L else outs[l]["Z"] > 0
            b = layer_backward(p, a_l, h_l, Wm[l - 1], g, mask, need_g_in=l >= 2)
            G[l - 1] = b["G_W"]
            g = b["G_in"]
        for l in range(L):                                 # local update
            if optimizer == "sgd":
                Wm[l] = sgd_step(Wm[l], G[l], lr)
            else:
                mm, vv = opt[m][l]
                Wm[l], mm, vv = adam_step(Wm[l], G[l], mm, vv, rm, lr)
                opt[m][l] = (mm, vv)
        for l in range(L):                                 # upload: PS mixing
            Wg[l] = (1.0 - a) * Wg[l] + a * Wm[l]
        run.ps_updates += 1
        if record_weights:
            rec.uploaded = [w.copy() for w in Wm]
        run.records.append(rec)
    run.weights = Wg
    return run
