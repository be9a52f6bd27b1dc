"""O8-O11: one GCN layer forward/backward, loss and updates in fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Forward, Eq. 5:
    H_in^(l+1) = sigma( P_in H_in^(l) W + P_out H~_out^(l) W )
written with the extended input X_ext = [H_in ; H~_out] and P_m = [P_in | P_out]:
    A = P_m X_ext,  Z = A W,  H = sigma(Z)            (reading A5: no bias)
sigma = ReLU on hidden layers, identity on the output layer (A5).

Backward, Eq. 6 and the appendix GCN backward, with the
stale halo block a constant of the current iteration (reading A14):
    D   = G_out o sigma'(Z)           (ReLU'(0) := 0)
    G_W = (P_in H_in + P_out H~_out)^T D = A^T D
    G_in = P_in^T D W^T               (local rows only; no gradient to the halo)
"""
import numpy as np
import scipy.sparse as sp


def prop_matrix(part) -> sp.csr_matrix:
    """P_m = [P_in | P_out] as an fp64 CSR over extended columns."""
    return sp.csr_matrix((part.val.astype(np.float64), part.col.astype(np.int64), part.row_ptr),
                         shape=(part.n_local, part.n_local + part.n_halo))


def _x_ext(x_local, x_halo, n_halo):
    xl = np.asarray(x_local, dtype=np.float64)
    if n_halo == 0:
        return xl
    return np.vstack([xl, np.asarray(x_halo, dtype=np.float64)])


def layer_forward(part, x_local, x_halo, w, relu: bool):
    """Eq. 5 for partition `part`; returns dict(A, Z, H) in fp64."""
    P = prop_matrix(part)
    A = P @ _x_ext(x_local, x_halo, part.n_halo)
    Z = A @ np.asarray(w, dtype=np.float64)
    H = np.maximum(Z, 0.0) if relu else Z
    return {"A": A, "Z": Z, "H": H}


def layer_backward(part, x_local, x_halo, w, g_out, act_mask, need_g_in: bool,
                   need_g_halo: bool = False):
    """Eq. 6 and P:785-792 with constant halo.

    act_mask: boolean sigma'(Z) (None for the identity output layer).  It is passed
    in so that a caller comparing against another implementation can share that
    implementation's ReLU decisions (integer decisions taken once, in one precision).

    need_g_halo: also return G_halo = P_out^T D W^T (n_halo rows), the gradient this
    partition's rows send back to the owners of its halo nodes in the SAME iteration --
    the exact (zero-staleness) variant of the appendix's term; the paper's own term uses
    the previous iteration's D~^(t-1) (oracle_train halo_grad='prev_epoch').  It
    is not part of Eq. 6's constant-halo reading.
    """
    P = prop_matrix(part)
    D = np.asarray(g_out, dtype=np.float64)
    if act_mask is not None:
        D = D * np.asarray(act_mask, dtype=np.float64)
    A = P @ _x_ext(x_local, x_halo, part.n_halo)
    G_W = A.T @ D
    G_in = G_halo = None
    if need_g_in:
        P_in = P[:, : part.n_local]
        G_in = P_in.T @ (D @ np.asarray(w, dtype=np.float64).T)
    if need_g_halo:
        P_out = P[:, part.n_local:]
        G_halo = P_out.T @ (D @ np.asarray(w, dtype=np.float64).T)
    return {"D": D, "G_W": G_W, "G_in": G_in, "G_halo": G_halo}


def cross_entropy(logits, labels, train_mask, num_classes: int, w_loss: float):
    """Eq. 3 with the loss restricted to training nodes (reading A13).

    For v in train: l_v = logsumexp(z_v[0:C]) - z_v[y_v].
    Returns (loss = w_loss * sum_v l_v, G_logits) with
    G_logits[v, 0:C] = w_loss * (softmax(z_v[0:C]) - e_{y_v}) on train rows, 0 elsewhere
    (padded columns >= C stay 0, reading A25).
    """
    z = np.asarray(logits, dtype=np.float64)
    n, c_pad = z.shape
    zc = z[:, :num_classes]
    zmax = zc.max(axis=1, keepdims=True) if n else np.zeros((0, 1))
    e = np.exp(zc - zmax)
    s = e.sum(axis=1, keepdims=True)
    lse = (zmax + np.log(s))[:, 0]
    y = np.asarray(labels, dtype=np.int64)
    t = np.asarray(train_mask).astype(bool)
    lv = lse - zc[np.arange(n), y]
    loss = w_loss * float(lv[t].sum())
    g = np.zeros((n, c_pad))
    soft = e / s
    soft[np.arange(n), y] -= 1.0
    g[t, :num_classes] = w_loss * soft[t]
    return loss, g


def sgd_step(w, g, lr):
    """Alg. 1 'update local parameters': W <- W - eta * grad."""
    return np.asarray(w, dtype=np.float64) - lr * np.asarray(g, dtype=np.float64)


def adam_step(w, g, m, v, step, lr, b1=0.9, b2=0.999, eps=1e-8):
    """Adam (the paper's optimizer), bias-corrected, S:191 constants."""
    g = np.asarray(g, dtype=np.float64)
    m = b1 * m + (1 - b1) * g
    v = b2 * v + (1 - b2) * g * g
    mh = m / (1 - b1 ** step)
    vh = v / (1 - b2 ** step)
    return np.asarray(w, dtype=np.float64) - lr * mh / (np.sqrt(vh) + eps), m, v


def normalize_rows(h):
    """Alg. 1 representation normalisation h <- h/||h||_2; zero rows stay 0."""
    h = np.asarray(h, dtype=np.float64)
    nrm = np.sqrt((h * h).sum(axis=1, keepdims=True))
    return np.where(nrm > 0, h / np.where(nrm > 0, nrm, 1.0), 0.0)
