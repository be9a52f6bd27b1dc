"""Theorem 1 and its representation-level precursor (TEST INFRASTRUCTURE ONLY).

theorem1_bound: the right-hand side of Theorem 1 (formal P:698)
    (tau/M) * sum_{l=1}^{L-1} eps^(l) r1^(L-l) r2^(L-l) sum_m Delta(G_m)^(L-l).
The gradient-level inequality itself needs tau, which the paper gives no way to
compute: "parity unpinned" for the gradient form (reported only, reading A17/A18).

staleness_bound_check: the per-representation bound the proof starts from
(from GNNAutoscale Thm. 2), made rigorous for a ReLU/identity GCN:
    delta^(1) = 0,  delta^(l+1) <= c_{l+1} (delta^(l) + eps^(l)),
    c_k = ||W^(k)||_2 * max_v sum_u P_vu          (Lip(ReLU) = 1)
and the paper's looser form with r1 = max P_vu, r2 = max_k ||W^(k)||_2,
Delta = max_v deg(v)+1:  delta^(L) <= sum_l eps^(l) (r1 r2 Delta)^(L-l).
"""
import numpy as np


def theorem1_bound(tau, num_parts, eps, r1, r2, deltas):
    """eps: [eps^(1) .. eps^(L-1)]; deltas: [Delta(G_1) .. Delta(G_M)]."""
    L = len(eps) + 1
    deltas = np.asarray(deltas, dtype=np.float64)
    s = 0.0
    for l in range(1, L):
        k = L - l
        s += eps[l - 1] * (r1 ** k) * (r2 ** k) * float((deltas ** k).sum())
    return tau / num_parts * s


def staleness_bound_check(P_full, deg, weights, digest_reps, exact_reps, eps):
    """Return (delta_L, tight_bound, paper_bound).

    digest_reps / exact_reps: lists [H^(1), ..., H^(L)] over all nodes (fp64), the
    DIGEST representations and the exact full-graph ones at the same weights.
    eps: {l: max over halo u of ||h~_u - h_u||} for l in 1..L-1.
    """
    L = len(weights)
    rowsum = float(np.asarray(P_full.sum(axis=1)).max())
    c = [np.linalg.norm(np.asarray(w, np.float64), 2) * rowsum for w in weights]
    delta = [0.0]  # delta^(1) = 0: layer 1 uses exact features everywhere
    for l in range(1, L):
        delta.append(c[l] * (delta[-1] + eps[l]))
    tight = delta[-1]
    r1 = float(P_full.data.max())
    r2 = max(np.linalg.norm(np.asarray(w, np.float64), 2) for w in weights)
    Delta = float(deg.max() + 1)
    paper = sum(eps[l] * (r1 * r2 * Delta) ** (L - l) for l in range(1, L))
    dL = float(np.sqrt(((digest_reps[L - 1] - exact_reps[L - 1]) ** 2).sum(1)).max())
    return dL, tight, paper
