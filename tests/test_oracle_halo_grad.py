"""Pins for the oracle's same-iteration halo-gradient return (halo_grad='same_epoch', the
exact variant of the appendix term; the literal stale term P:816 is pinned in
tests/test_oracle_pins.py)."""
import numpy as np
import pytest

import oracle
from oracle.gcn import layer_backward, cross_entropy
from oracle.train import full_prop_matrix, full_graph_forward, full_graph_backward
from synth import make_inputs, make_random_parts, small_config
from tests.brute import brute_block, dense_P


def _inp(seed, n=48, nnz=220, hidden=(6, 5)):
    cfg = small_config(num_nodes=n, nnz=nnz, d0=5, hidden=hidden, num_classes=3, c_pad=4,
                       seed=seed, train_frac=0.6)
    return cfg, make_inputs(cfg)


@pytest.mark.parametrize("M,seed", [(2, 0), (3, 1), (4, 2)])
def test_fresh_with_returned_halo_gradient_equals_full_graph(M, seed):
    """Zero staleness + the returned P_out^T D W^T term: every layer's G_W equals full-graph
    GCN (A16's gap closes), for arbitrary (random) partitions."""
    cfg, inp = _inp(60 + seed)
    part = make_random_parts(cfg.num_nodes, M, seed)
    run = oracle.oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                              cfg.num_classes, part, M, sync_interval=1, epochs=1, mode="fresh",
                              halo_grad="same_epoch")
    P = full_prop_matrix(inp.indptr, inp.indices)
    W = [w.astype(np.float64) for w in inp.weights]
    H, Z = full_graph_forward(P, inp.x, W)
    _, g = cross_entropy(H[-1], inp.y, inp.train_mask, cfg.num_classes, 1.0 / inp.train_mask.sum())
    ref = full_graph_backward(P, H, Z, W, g)
    for a, b in zip(run.records[0].grads, ref):
        np.testing.assert_allclose(a, b, rtol=1e-11, atol=1e-13)


def test_single_part_has_nothing_to_return():
    cfg, inp = _inp(70)
    part = np.zeros(cfg.num_nodes, np.int32)
    a = oracle.oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                            cfg.num_classes, part, 1, sync_interval=1, epochs=2, lr=0.3)
    b = oracle.oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                            cfg.num_classes, part, 1, sync_interval=1, epochs=2, lr=0.3,
                            halo_grad="same_epoch")
    for x, y in zip(a.weights, b.weights):
        assert x.tobytes() == y.tobytes()


@pytest.mark.parametrize("seed", range(10))
def test_g_halo_vs_dense_brute_force(seed):
    rng = np.random.default_rng(300 + seed)
    cfg, inp = _inp(80 + seed, n=40, nnz=180)
    M = int(rng.integers(2, 5))
    part = make_random_parts(cfg.num_nodes, M, seed)
    Pd = dense_P(inp.indptr, inp.indices)
    for m in range(M):
        p = oracle.oracle_partition(inp.indptr, inp.indices, part, M, m)
        din, dout = 4, 3
        xl, xh = rng.standard_normal((p.n_local, din)), rng.standard_normal((p.n_halo, din))
        w, g = rng.standard_normal((din, dout)), rng.standard_normal((p.n_local, dout))
        b = layer_backward(p, xl, xh, w, g, None, True, need_g_halo=True)
        Pm = brute_block(Pd, p.local_ids, p.halo_ids)
        np.testing.assert_allclose(b["G_halo"], Pm[:, p.n_local:].T @ g @ w.T, rtol=1e-12,
                                   atol=1e-13)


def test_returned_gradient_changes_the_stale_trajectory():
    """With staleness the returned term is a real change of the update (not a no-op)."""
    cfg, inp = _inp(90)
    part = make_random_parts(cfg.num_nodes, 3, 5)
    kw = dict(sync_interval=2, epochs=3, lr=0.3)
    a = oracle.oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                            cfg.num_classes, part, 3, **kw)
    b = oracle.oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                            cfg.num_classes, part, 3, halo_grad="same_epoch", **kw)
    assert np.abs(a.weights[0] - b.weights[0]).max() > 1e-6
    np.testing.assert_array_equal(a.records[0].grads[-1], b.records[0].grads[-1])  # last layer
