"""Round-2 pins of the oracle against values fixed outside it (VERDICT r1 "oracle gaps"):

* Adam beyond step 1 (the paper's optimizer; S:191 constants): a closed form for
  a constant gradient and a hand-derived three-step case (tests/golden/adam_hand.json).
* The representation staleness bound: a hand-derived formula case that separates
  the spectral norm from the Frobenius / infinity / max norms, and a hand-derived run of
  the oracle's own training loop on a two-node graph (tests/golden/bound_hand.json).
* halo_grad='prev_epoch', the appendix's literal DIGEST backward:
  G~_H^(t) = P_in^T D~^(t) W~^(t)T + P_out^T D~^(t-1) W~^(t)T, pinned by (i) epoch 1 equals
  the constant-halo run, (ii) with eta = 0 the returned term is the 'same_epoch' term of
  the previous epoch, (iii) a dense, global brute force of the formula over the whole
  graph (no send lists, no owners, no per-part CSR).
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import adam_step, oracle_train, staleness_bound_check
from synth import make_inputs, make_random_parts, small_config
from tests.brute import dense_P

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- Adam
@pytest.mark.parametrize("g", [3.0, -0.2, 1e-3, -7.5])
def test_adam_constant_gradient_closed_form(g):
    """Constant g: m_t = (1-b1^t) g and v_t = (1-b2^t) g^2, so after bias correction
    mhat_t = g and vhat_t = g^2 at EVERY t: each step moves W by -lr g/(|g| + eps).
    A dropped bias correction or a wrong moment carry-over breaks it at t >= 2."""
    lr, eps = 0.01, 1e-8
    w = np.full((2, 3), 0.5)
    m = np.zeros_like(w)
    v = np.zeros_like(w)
    for t in range(1, 9):
        w_new, m, v = adam_step(w, np.full_like(w, g), m, v, t, lr)
        np.testing.assert_allclose(w_new - w, -lr * g / (abs(g) + eps), rtol=1e-12)
        np.testing.assert_allclose(m, (1 - 0.9 ** t) * g, rtol=1e-13)
        np.testing.assert_allclose(v, (1 - 0.999 ** t) * g * g, rtol=1e-12)
        w = w_new


def test_adam_hand_three_steps():
    """Three steps with changing gradients against the hand derivation (exact rationals)."""
    ex = _gold("adam_hand.json")
    w = np.array([[ex["w0"]]])
    m = v = 0.0
    for t, g in enumerate(ex["g"], 1):
        w, m, v = adam_step(w, np.array([[g]]), m, v, t, ex["lr"])
        assert abs(m[0, 0] - float(Fraction(ex["m"][t - 1]))) <= 1e-15
        assert abs(v[0, 0] - float(Fraction(ex["v"][t - 1]))) <= 1e-17
        assert abs(w[0, 0] - float(ex["w"][t - 1])) <= 1e-14, (t, w[0, 0], ex["w"][t - 1])


def test_adam_zero_gradient_after_a_step_decays_moments():
    """g = (2, 0): the second step still moves W (m carries over), by lr*mhat/sqrt(vhat)
    with mhat = 0.9*0.2/0.19, vhat = 0.999*0.004/0.001999 (hand)."""
    w, m, v = adam_step(np.array([[1.0]]), np.array([[2.0]]), 0.0, 0.0, 1, 0.1)
    w2, m, v = adam_step(w, np.array([[0.0]]), m, v, 2, 0.1)
    mh, vh = 0.18 / 0.19, 0.003996 / 0.001999
    assert abs((w2 - w)[0, 0] + 0.1 * mh / (np.sqrt(vh) + 1e-8)) <= 1e-14


# ---------------------------------------------------------------- staleness bound
def test_bound_formula_case_hand_derived():
    ex = _gold("bound_hand.json")["formula_case"]
    r6 = 1 / np.sqrt(6.0)
    P = sp.csr_matrix(np.array([[0.5, r6, 0.0], [r6, 1 / 3, r6], [0.0, r6, 0.5]]))
    deg = np.array([1, 2, 1])
    W = [np.array(w, np.float64) for w in ex["weights"]]
    eps = {int(k): v for k, v in ex["eps"].items()}
    dig = [None, None, np.array(ex["digest_last"])]
    exa = [None, None, np.array(ex["exact_last"])]
    dL, tight, paper = staleness_bound_check(P, deg, W, dig, exa, eps)
    assert abs(dL - float(ex["delta_L"])) <= 1e-15
    assert abs(tight - float(ex["tight"])) <= 1e-14 * float(ex["tight"])
    assert abs(paper - float(ex["paper"])) <= 1e-14 * float(ex["paper"])


def test_bound_through_the_training_loop_hand_derived():
    """Two nodes, one per part, zero cold start: every quantity of the bound is a small
    integer derived by hand (tests/golden/bound_hand.json train_case)."""
    ex = _gold("bound_hand.json")["train_case"]
    indptr = np.array([0, 1, 2])
    indices = np.array([1, 0], np.int32)
    part = np.array([0, 1], np.int32)
    x = np.array(ex["x"])
    W = [np.array(w) for w in ex["weights"]]
    run = oracle_train(indptr, indices, x, np.zeros(2, np.int64), np.ones(2, bool), W, 1, part,
                       2, sync_interval=1, epochs=1, lr=0.0, record_outputs=True)
    rec = run.records[0]
    assert rec.eps[1] == ex["eps1"]
    P = sp.csr_matrix(np.full((2, 2), 0.5))
    out_L = np.zeros((2, 1))
    for m, p in enumerate(run.parts):
        out_L[p.local_ids] = rec.part_out[(2, m)]["H"]
    exact_h1 = np.full((2, 1), 4.0)
    exact_h2 = np.full((2, 1), 12.0)
    dL, tight, paper = staleness_bound_check(P, np.array([1, 1]), W, [rec.reps[1], out_L],
                                             [exact_h1, exact_h2], rec.eps)
    assert (dL, tight, paper) == (ex["delta_L"], ex["tight"], ex["paper"])


# ---------------------------------------------------------------- prev_epoch
def _inp(seed, n=44, nnz=200, hidden=(6, 5)):
    cfg = small_config(num_nodes=n, nnz=nnz, d0=5, hidden=hidden, num_classes=3, c_pad=4,
                       seed=seed, train_frac=0.6)
    return cfg, make_inputs(cfg)


def _run(inp, cfg, part, M, **kw):
    return oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                        cfg.num_classes, part, M, record_outputs=True, **kw)


def test_prev_epoch_first_epoch_is_the_constant_halo_run():
    """At t = 1 there is no D~^(0): the returned term is zero."""
    cfg, inp = _inp(110)
    part = make_random_parts(cfg.num_nodes, 3, 1)
    a = _run(inp, cfg, part, 3, sync_interval=1, epochs=1, lr=0.2)
    b = _run(inp, cfg, part, 3, sync_interval=1, epochs=1, lr=0.2, halo_grad="prev_epoch")
    for x, y in zip(a.records[0].grads, b.records[0].grads):
        np.testing.assert_array_equal(x, y)
    for k, v in b.records[0].halo_grad_sent.items():
        assert not v.any(), k


@pytest.mark.parametrize("L_hidden", [(6,), (6, 5)])
def test_prev_epoch_with_frozen_weights_is_same_epoch_shifted(L_hidden):
    """eta = 0 freezes W, so the forward and every D of the top layer are the same in both
    runs; the top layer's returned rows at epoch t (prev_epoch) are then the rows
    'same_epoch' returned at epoch t-1."""
    cfg, inp = _inp(120, hidden=L_hidden)
    part = make_random_parts(cfg.num_nodes, 3, 2)
    kw = dict(sync_interval=1, epochs=4, lr=0.0)
    a = _run(inp, cfg, part, 3, halo_grad="same_epoch", **kw)
    b = _run(inp, cfg, part, 3, halo_grad="prev_epoch", **kw)
    L = len(L_hidden) + 1
    for t in range(1, 4):
        for m in range(3):
            x = a.records[t - 1].halo_grad_sent[(L, m)]
            y = b.records[t].halo_grad_sent[(L, m)]
            np.testing.assert_allclose(y, x, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("M,N,seed", [(2, 1, 0), (3, 2, 1), (4, 1, 2)])
def test_prev_epoch_matches_the_global_dense_formula(M, N, seed):
    """P:816 written over the whole graph with dense matrices: for node v of part k,
        G_v^(t) = sum_{u in V_k} P_uv (D^(t) W^(t)T)_u + sum_{u not in V_k} P_uv (D^(t-1) W^(t)T)_u
    (S = same-part indicator: G = (P o S)^T D^(t) W^T + (P o (1-S))^T D^(t-1) W^T),
    then D^(l-1) = G o 1[Z^(l-1) > 0].  Weights change between epochs (eta > 0), so the
    W^(t) (not W^(t-1)) of the formula is pinned too."""
    cfg, inp = _inp(130 + seed)
    part = make_random_parts(cfg.num_nodes, M, seed)
    run = _run(inp, cfg, part, M, sync_interval=N, epochs=3, lr=0.3, halo_grad="prev_epoch")
    P = dense_P(inp.indptr, inp.indices)
    po = np.asarray(part)
    S = (po[:, None] == po[None, :]).astype(np.float64)
    L = len(inp.weights)
    n = cfg.num_nodes
    prevD = {l: np.zeros((n, inp.weights[l - 1].shape[1])) for l in range(2, L + 1)}
    for rec in run.records:
        for l in range(L, 1, -1):
            Dt = np.zeros((n, inp.weights[l - 1].shape[1]))
            Zm = np.zeros((n, inp.weights[l - 2].shape[1]))
            for m, p in enumerate(run.parts):
                Dt[p.local_ids] = rec.part_d[(l, m)]
                Zm[p.local_ids] = rec.part_out[(l - 1, m)]["Z"]
            Wt = rec.weights_used[l - 1]
            G = (P * S).T @ Dt @ Wt.T + (P * (1 - S)).T @ prevD[l] @ Wt.T
            want = G * (Zm > 0)
            for m, p in enumerate(run.parts):
                np.testing.assert_allclose(rec.part_d[(l - 1, m)], want[p.local_ids],
                                           rtol=1e-11, atol=1e-14)
            prevD[l] = Dt
