"""Pins for oracle O7-O12: schedule, store semantics, special cases, staleness bound."""
import numpy as np
import pytest

from oracle import oracle_train, oracle_partition, theorem1_bound, staleness_bound_check, degrees
from oracle.train import full_prop_matrix, full_graph_forward, full_graph_backward
from oracle.gcn import cross_entropy
from synth import small_config, make_inputs, make_random_parts, make_block_parts
from tests.brute import brute_block, brute_layer_backward, brute_layer_forward, dense_P
from tests.helpers import golden

G = golden("spec_examples.json")


def _inputs(seed=7, n=40, nnz=160, hidden=(6,), C=3, c_pad=4, d0=5):
    cfg = small_config(num_nodes=n, nnz=nnz, d0=d0, hidden=hidden, num_classes=C, c_pad=c_pad,
                       seed=seed, train_frac=0.6)
    return cfg, make_inputs(cfg)


def _train(inp, cfg, part, M, **kw):
    return oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                        cfg.num_classes, part, M, **kw)


def _full_reference(inp, cfg, epochs, lr):
    """Full-graph GCN training with the same count-weighted loss."""
    P = full_prop_matrix(inp.indptr, inp.indices)
    W = [w.astype(np.float64) for w in inp.weights]
    out = []
    n_train = int(inp.train_mask.sum())
    for _ in range(epochs):
        H, Z = full_graph_forward(P, inp.x, W)
        loss, g = cross_entropy(H[-1], inp.y, inp.train_mask, cfg.num_classes, 1.0 / n_train)
        grads = full_graph_backward(P, H, Z, W, g)
        out.append((loss, grads, H))
        W = [w - lr * gw for w, gw in zip(W, grads)]
    return out, W


def test_m1_equals_full_graph_training():
    cfg, inp = _inputs(hidden=(6, 5))
    run = _train(inp, cfg, np.zeros(cfg.num_nodes, np.int32), 1, sync_interval=1, epochs=5, lr=0.5)
    ref, Wref = _full_reference(inp, cfg, 5, 0.5)
    for rec, (loss, grads, _) in zip(run.records, ref):
        assert abs(rec.loss - loss) <= 1e-12 * abs(loss)
        for a, b in zip(rec.grads, grads):
            np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-14)
    for a, b in zip(run.weights, Wref):
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("M", [2, 3, 4])
def test_fresh_mode_forward_equals_full_graph(M):
    """A15/A16: zero staleness => every layer output, the loss and G_W^(L) equal the full graph;
    G_W^(l<L) equals the brute force of the PARTITIONED formula (halo constant)."""
    cfg, inp = _inputs(seed=11 + M, n=48, nnz=220, hidden=(6, 5))
    part = make_random_parts(cfg.num_nodes, M, 3 + M)
    run = _train(inp, cfg, part, M, sync_interval=1, epochs=1, mode="fresh", record_outputs=True)
    rec = run.records[0]
    ref, _ = _full_reference(inp, cfg, 1, 0.0)
    loss, grads, H = ref[0]
    L = len(inp.weights)
    for l in range(1, L):
        np.testing.assert_allclose(rec.reps[l], H[l], rtol=1e-12, atol=1e-13)
    for m, p in enumerate(run.parts):
        np.testing.assert_allclose(rec.part_out[(L, m)]["H"], H[L][p.local_ids], rtol=1e-12, atol=1e-13)
    assert abs(rec.loss - loss) <= 1e-12 * abs(loss)
    np.testing.assert_allclose(rec.grads[L - 1], grads[L - 1], rtol=1e-11, atol=1e-13)
    # earlier layers: the partitioned definition, by dense brute force
    Pd = dense_P(inp.indptr, inp.indices)
    n_train = int(inp.train_mask.sum())
    tot = [np.zeros_like(w, dtype=np.float64) for w in inp.weights]
    for m, p in enumerate(run.parts):
        Pm = brute_block(Pd, p.local_ids, p.halo_ids)
        xe = [np.vstack([inp.x[p.local_ids], inp.x[p.halo_ids]])]
        Zs = []
        for l in range(L):
            A, Z, Hh = brute_layer_forward(Pm, xe[-1], inp.weights[l].astype(np.float64), l < L - 1)
            Zs.append(Z)
            if l < L - 1:
                xe.append(np.vstack([Hh, H[l + 1][p.halo_ids]]))
        _, g = cross_entropy(Hh, inp.y[p.local_ids], inp.train_mask[p.local_ids], cfg.num_classes,
                             1.0 / n_train)
        for l in range(L - 1, -1, -1):
            GW, Gin = brute_layer_backward(Pm, p.n_local, xe[l], inp.weights[l].astype(np.float64),
                                           Zs[l], g, l < L - 1)
            tot[l] += GW
            g = Gin
    for a, b in zip(rec.grads, tot):
        np.testing.assert_allclose(a, b, rtol=1e-11, atol=1e-13)
    # and the first-layer gradient is NOT the full-graph one (finding 3 / A16)
    rel = np.abs(rec.grads[0] - grads[0]).max() / np.abs(grads[0]).max()
    assert rel > 1e-3


@pytest.mark.parametrize("N", G["schedule_counts"]["N"])
def test_schedule_counts_and_ages(N):
    sc = G["schedule_counts"]
    R, L, M = sc["R"], sc["L"], sc["M"]
    cfg, inp = _inputs(seed=21, n=32, nnz=120, hidden=(3, 3))
    part = make_block_parts(cfg, M)
    run = _train(inp, cfg, part, M, sync_interval=N, epochs=R, lr=0.0)
    assert run.pull_count == (R // N) * (L - 1) * M
    assert run.push_count == ((R - 1) // N + 1) * (L - 1) * M
    for rec in run.records:
        r = rec.epoch
        assert rec.pulled == (r % N == 0) and rec.pushed == ((r - 1) % N == 0)
        for (l, m), ver in rec.halo_versions.items():
            if ver.size == 0:
                continue
            assert np.all(ver == ver[0]) and np.all(ver < r)      # pulls see only older epochs
            if N == 1:
                assert ver[0] == r - 1                             # age 1 (epoch 1: cold, v=0)
            elif r < N:
                assert ver[0] == 0                                 # cold start until epoch N
            else:
                assert N - 1 <= r - ver[0] <= 2 * N - 2            # age cycles N-1 .. 2N-2


def test_n1_frozen_weights_pull_previous_epoch_exactly():
    """S:409 example: N=1, eta=0: the halo pulled at epoch r equals epoch r-1's values,
    bit-exactly, and eps^(l) = 0 once the levels below have stabilised (r >= l+1)."""
    cfg, inp = _inputs(seed=5, n=40, nnz=180, hidden=(4, 4))
    part = make_random_parts(cfg.num_nodes, 3, 1)
    run = _train(inp, cfg, part, 3, sync_interval=1, epochs=5, lr=0.0, record_outputs=True)
    for prev, rec in zip(run.records[:-1], run.records[1:]):
        for (l, m), used in rec.halo_used.items():
            np.testing.assert_array_equal(used, prev.reps[l][run.parts[m].halo_ids])
        for l, e in rec.eps.items():
            if rec.epoch >= l + 1:
                assert e == 0.0


def test_prime_cold_start_first_epoch_is_full_graph():
    cfg, inp = _inputs(seed=8, n=40, nnz=180, hidden=(4,))
    part = make_random_parts(cfg.num_nodes, 2, 2)
    run = _train(inp, cfg, part, 2, sync_interval=5, epochs=1, cold_start="prime")
    ref, _ = _full_reference(inp, cfg, 1, 0.0)
    assert abs(run.records[0].loss - ref[0][0]) <= 1e-12 * abs(ref[0][0])


def test_zero_cold_start_drops_halo_term():
    """A8: with zero halos the first epoch's hidden layers see only P_in (global normalisation)."""
    cfg, inp = _inputs(seed=9, n=30, nnz=120, hidden=(4,))
    part = make_random_parts(cfg.num_nodes, 2, 4)
    run = _train(inp, cfg, part, 2, sync_interval=3, epochs=1, record_outputs=True)
    for (l, m), used in run.records[0].halo_used.items():
        assert np.all(used == 0)


def test_per_part_weighting_equals_count_on_equal_split():
    cfg, inp = _inputs(seed=12, n=40, nnz=150, hidden=(4,))
    part = make_block_parts(cfg, 2)
    tr = inp.train_mask.copy()
    tr[:] = 0
    tr[:10] = 1
    tr[20:30] = 1  # 10 training nodes in each half
    inp.train_mask = tr
    a = _train(inp, cfg, part, 2, sync_interval=1, epochs=2, lr=0.3)
    b = _train(inp, cfg, part, 2, sync_interval=1, epochs=2, lr=0.3, loss_weighting="per_part")
    for ra, rb in zip(a.records, b.records):
        assert abs(ra.loss - rb.loss) < 1e-13
        for x, y in zip(ra.grads, rb.grads):
            np.testing.assert_allclose(x, y, rtol=1e-12, atol=1e-15)


def test_determinism():
    cfg, inp = _inputs(seed=13)
    part = make_random_parts(cfg.num_nodes, 2, 0)
    a = _train(inp, cfg, part, 2, sync_interval=2, epochs=4, lr=0.1, optimizer="adam")
    b = _train(inp, cfg, part, 2, sync_interval=2, epochs=4, lr=0.1, optimizer="adam")
    for x, y in zip(a.weights, b.weights):
        assert x.tobytes() == y.tobytes()


def test_theorem1_arithmetic():
    for key in ("theorem1_a", "theorem1_b"):
        ex = G[key]
        got = theorem1_bound(ex["tau"], ex["M"], ex["eps"], ex["r1"], ex["r2"], ex["deltas"])
        assert abs(got - ex["bound"]) < 1e-12
    assert theorem1_bound(3.0, 2, [0.0, 0.0], 1.0, 2.0, [5, 6]) == 0.0


@pytest.mark.parametrize("N,lr,seed", [(2, 0.1, 0), (5, 0.1, 1), (10, 0.01, 2), (5, 0.5, 3)])
def test_staleness_bound_holds(N, lr, seed):
    """P:714 representation bound, in the tight and the paper's form, at every epoch."""
    cfg, inp = _inputs(seed=30 + seed, n=48, nnz=200, hidden=(5, 5))
    part = make_random_parts(cfg.num_nodes, 3, seed)
    run = _train(inp, cfg, part, 3, sync_interval=N, epochs=2 * N + 2, lr=lr, record_outputs=True)
    P = full_prop_matrix(inp.indptr, inp.indices)
    deg = degrees(inp.indptr)
    L = len(inp.weights)
    checked = 0
    for rec in run.records:
        Hs, _ = full_graph_forward(P, inp.x, rec.weights_used)
        out_L = np.zeros((cfg.num_nodes, inp.weights[-1].shape[1]))
        for m, p in enumerate(run.parts):
            out_L[p.local_ids] = rec.part_out[(L, m)]["H"]
        digest = [rec.reps[l] for l in range(1, L)] + [out_L]
        dL, tight, paper = staleness_bound_check(P, deg, rec.weights_used, digest, Hs[1:], rec.eps)
        assert dL <= tight * (1 + 1e-9) + 1e-12 and tight <= paper * (1 + 1e-9) + 1e-12
        checked += dL > 0
    assert checked > 0
