"""Pins for oracle O8-O11: layer forward/backward, loss, optimizers, normalisation."""
import numpy as np
import pytest

from oracle import (oracle_partition, layer_forward, layer_backward, cross_entropy,
                    sgd_step, adam_step, normalize_rows)
from tests.brute import (brute_block, brute_layer_backward, brute_layer_forward, dense_P)
from tests.helpers import csr_from_edges, golden, random_graph, random_parts

G = golden("spec_examples.json")


def _two_node_part():
    ip, ix = csr_from_edges(2, [(0, 1)])
    return oracle_partition(ip, ix, np.array([0, 1], np.int32), 2, 0)


def test_forward_worked_example():
    p = _two_node_part()  # P_in=[[.5]], P_out=[[.5]]
    o = layer_forward(p, [[2.0]], [[4.0]], [[1.0]], relu=False)
    assert o["H"][0, 0] == G["layer_forward_1node"]["out"]


def test_backward_worked_example():
    p = _two_node_part()
    b = layer_backward(p, [[2.0]], [[4.0]], [[1.0]], [[1.0]], None, need_g_in=True)
    assert b["G_W"][0, 0] == G["layer_backward_1node"]["G_W"]
    assert b["G_in"][0, 0] == G["layer_backward_1node"]["G_in"]


def test_relu_clamp_and_dead_relu():
    p = _two_node_part()
    o = layer_forward(p, [[2.0]], [[4.0]], [[-1.0]], relu=True)
    assert o["H"][0, 0] == 0.0
    b = layer_backward(p, [[2.0]], [[4.0]], [[-1.0]], [[1.0]], o["Z"] > 0, True)
    assert b["G_W"][0, 0] == 0.0 and b["G_in"][0, 0] == 0.0


def test_empty_halo_is_local_layer():
    rng = np.random.default_rng(3)
    ip, ix = random_graph(20, 0.2, rng)
    p = oracle_partition(ip, ix, np.zeros(20, np.int32), 1, 0)
    x = rng.standard_normal((20, 4))
    w = rng.standard_normal((4, 3))
    o = layer_forward(p, x, np.zeros((0, 4)), w, relu=True)
    np.testing.assert_allclose(o["H"], np.maximum(dense_P(ip, ix) @ x @ w, 0), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("seed", range(40))
def test_layer_vs_dense_brute_force(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(4, 64))
    ip, ix = random_graph(n, float(rng.uniform(0.05, 0.3)), rng)
    M = int(rng.integers(1, 5))
    part = random_parts(n, M, rng)
    Pd = dense_P(ip, ix)
    din, dout = int(rng.integers(1, 7)), int(rng.integers(1, 7))
    X = rng.standard_normal((n, din))
    w = rng.standard_normal((din, dout))
    for m in range(M):
        p = oracle_partition(ip, ix, part, M, m)
        xl, xh = X[p.local_ids], rng.standard_normal((p.n_halo, din))  # arbitrary stale values
        Pm = brute_block(Pd, p.local_ids, p.halo_ids)
        xe = np.vstack([xl, xh])
        for relu in (False, True):
            o = layer_forward(p, xl, xh, w, relu)
            A, Z, H = brute_layer_forward(Pm, xe, w, relu)
            np.testing.assert_allclose(o["A"], A, rtol=1e-12, atol=1e-12)
            np.testing.assert_allclose(o["H"], H, rtol=1e-12, atol=1e-12)
            g = rng.standard_normal((p.n_local, dout))
            b = layer_backward(p, xl, xh, w, g, (o["Z"] > 0) if relu else None, True)
            GW, Gin = brute_layer_backward(Pm, p.n_local, xe, w, Z, g, relu)
            np.testing.assert_allclose(b["G_W"], GW, rtol=1e-12, atol=1e-12)
            np.testing.assert_allclose(b["G_in"], Gin, rtol=1e-12, atol=1e-12)


def test_linearity_identity_activation():
    """with identity activation the layer is linear in the local and halo inputs."""
    rng = np.random.default_rng(9)
    ip, ix = random_graph(30, 0.2, rng)
    part = random_parts(30, 3, rng)
    p = oracle_partition(ip, ix, part, 3, 1)
    w = rng.standard_normal((3, 2))
    a, b = 0.7, -1.3
    x1, x2 = rng.standard_normal((p.n_local, 3)), rng.standard_normal((p.n_local, 3))
    h1, h2 = rng.standard_normal((p.n_halo, 3)), rng.standard_normal((p.n_halo, 3))
    lhs = layer_forward(p, a * x1 + b * x2, a * h1 + b * h2, w, False)["H"]
    rhs = a * layer_forward(p, x1, h1, w, False)["H"] + b * layer_forward(p, x2, h2, w, False)["H"]
    np.testing.assert_allclose(lhs, rhs, rtol=1e-12, atol=1e-12)


def _local_loss(p, xl, xh, ws, y, t, C):
    h_l, h_h = xl, xh
    for l, w in enumerate(ws):
        o = layer_forward(p, h_l, h_h, w, relu=l < len(ws) - 1)
        h_l, h_h = o["H"], np.zeros((p.n_halo, w.shape[1]))  # halo inputs of layer>=2 held fixed (zero)
    return cross_entropy(h_l, y, t, C, 1.0)[0]


@pytest.mark.parametrize("seed", range(4))
def test_finite_differences_local_loss(seed):
    """central differences of the LOCAL loss, halo inputs held fixed."""
    rng = np.random.default_rng(50 + seed)
    n = 14
    ip, ix = random_graph(n, 0.3, rng)
    part = random_parts(n, 2, rng)
    p = oracle_partition(ip, ix, part, 2, 0)
    C = 3
    ws = [rng.standard_normal((4, 5)), rng.standard_normal((5, C))]
    xl, xh = rng.standard_normal((p.n_local, 4)), rng.standard_normal((p.n_halo, 4))
    y = rng.integers(0, C, p.n_local)
    t = np.ones(p.n_local, bool)
    # analytic gradient
    o1 = layer_forward(p, xl, xh, ws[0], True)
    o2 = layer_forward(p, o1["H"], np.zeros((p.n_halo, 5)), ws[1], False)
    assert np.abs(o1["Z"]).min() > 1e-3  # away from ReLU kinks
    _, g = cross_entropy(o2["H"], y, t, C, 1.0)
    b2 = layer_backward(p, o1["H"], np.zeros((p.n_halo, 5)), ws[1], g, None, True)
    b1 = layer_backward(p, xl, xh, ws[0], b2["G_in"], o1["Z"] > 0, False)
    grads = [b1["G_W"], b2["G_W"]]
    h = 1e-5
    for li in range(2):
        for idx in np.ndindex(ws[li].shape):
            wp = [w.copy() for w in ws]
            wm = [w.copy() for w in ws]
            wp[li][idx] += h
            wm[li][idx] -= h
            fd = (_local_loss(p, xl, xh, wp, y, t, C) - _local_loss(p, xl, xh, wm, y, t, C)) / (2 * h)
            assert abs(fd - grads[li][idx]) <= 1e-6 * max(1.0, abs(fd)), (li, idx, fd, grads[li][idx])


def test_cross_entropy_examples():
    ex = G["xent_uniform"]
    loss, _ = cross_entropy(np.zeros((1, 8)), [2], [1], ex["C"], 1.0)
    assert abs(loss - ex["loss"]) < 1e-12
    ex = G["xent_gap"]
    loss, g = cross_entropy(np.array([ex["logits"]]), [ex["label"]], [1], 2, 1.0)
    assert abs(loss - ex["loss"]) < 1e-6 * ex["loss"]


def test_cross_entropy_mask_padding_and_fd():
    rng = np.random.default_rng(4)
    z = rng.standard_normal((6, 8))
    y = rng.integers(0, 5, 6)
    t = np.array([1, 0, 1, 1, 0, 1])
    loss, g = cross_entropy(z, y, t, 5, 0.25)
    assert np.all(g[t == 0] == 0) and np.all(g[:, 5:] == 0)
    h = 1e-6
    for idx in np.ndindex(6, 5):
        zp, zm = z.copy(), z.copy()
        zp[idx] += h
        zm[idx] -= h
        fd = (cross_entropy(zp, y, t, 5, 0.25)[0] - cross_entropy(zm, y, t, 5, 0.25)[0]) / (2 * h)
        assert abs(fd - g[idx]) < 1e-7


def test_optimizers():
    ex = G["sgd"]
    assert abs(sgd_step([[ex["W"]]], [[ex["G"]]], ex["lr"])[0, 0] - ex["out"]) < 1e-15
    assert sgd_step([[1.5]], [[0.0]], 0.3)[0, 0] == 1.5
    for gval in (3.0, -0.2, 1e-3):
        w, m, v = adam_step(np.array([[1.0]]), np.array([[gval]]), 0.0, 0.0, 1, 0.01)
        assert abs((w[0, 0] - 1.0) + 0.01 * np.sign(gval)) < 1e-6  # S:243 step-1 sign step


def test_normalize_rows():
    ex = G["normalize"]
    np.testing.assert_allclose(normalize_rows(ex["in"]), ex["out"], rtol=1e-15)
    assert np.all(normalize_rows([[0.0, 0.0]]) == 0)
    h = np.random.default_rng(0).standard_normal((5, 4))
    np.testing.assert_allclose(normalize_rows(normalize_rows(h)), normalize_rows(h), atol=1e-12)
