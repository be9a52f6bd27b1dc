"""Pins for the DIGEST-A oracle (oracle/async_train.py) and the
seeded asynchronous schedules (synth/async_sched.py)."""
import numpy as np
import pytest

from oracle import oracle_train
from oracle.async_train import oracle_train_async
from oracle.train import full_prop_matrix, full_graph_forward, full_graph_backward
from oracle.gcn import cross_entropy
from synth import small_config, make_inputs, make_random_parts
from synth.async_sched import async_events, straggler_delays
from tests.helpers import csr_from_edges


def _inputs(seed=7, n=40, nnz=160, hidden=(6,), C=3, c_pad=4, d0=5):
    cfg = small_config(num_nodes=n, nnz=nnz, d0=d0, hidden=hidden, num_classes=C, c_pad=c_pad,
                       seed=seed, train_frac=0.6)
    return cfg, make_inputs(cfg)


def _async(inp, cfg, part, M, events, **kw):
    return oracle_train_async(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                              cfg.num_classes, part, M, events=events, **kw)


@pytest.mark.parametrize("opt,N", [("sgd", 1), ("sgd", 3), ("adam", 2)])
def test_one_worker_async_is_sync(opt, N):
    """M=1 async == M=1 sync (alpha = 1): identical weight trajectory."""
    cfg, inp = _inputs(hidden=(6, 5))
    part = np.zeros(cfg.num_nodes, np.int32)
    R, lr = 6, (0.3 if opt == "sgd" else 0.05)
    a = _async(inp, cfg, part, 1, [0] * R, sync_interval=N, lr=lr, optimizer=opt)
    s = oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                     cfg.num_classes, part, 1, sync_interval=N, epochs=R, lr=lr, optimizer=opt)
    for ra, rs in zip(a.records, s.records):
        assert abs(ra.loss - rs.loss) <= 1e-12 * abs(rs.loss)
    for wa, ws in zip(a.weights, s.weights):
        np.testing.assert_allclose(wa, ws, rtol=1e-12, atol=1e-15)
    assert a.ps_updates == R


def test_zero_learning_rate_keeps_the_global_weights():
    """Mixing identical weights is the identity (convex combination)."""
    cfg, inp = _inputs(seed=3)
    M = 3
    part = make_random_parts(cfg.num_nodes, M, 2)
    ev = async_events(4, [1.0, 1.3, 2.1])
    run = _async(inp, cfg, part, M, ev, sync_interval=2, lr=0.0)
    for w, w0 in zip(run.weights, inp.weights):
        np.testing.assert_allclose(w, w0, rtol=1e-15, atol=1e-16)


def test_mixing_closed_form():
    """After n uploads U_1..U_n: W = (1-a)^n W0 + sum_j a (1-a)^(n-j) U_j."""
    cfg, inp = _inputs(seed=5, hidden=(6, 5))
    M = 3
    part = make_random_parts(cfg.num_nodes, M, 4)
    ev = async_events(3, [1.0, 0.7, 1.9])
    run = _async(inp, cfg, part, M, ev, sync_interval=1, lr=0.2, record_weights=True)
    a, n = 1.0 / M, len(ev)
    for l, w0 in enumerate(inp.weights):
        ref = (1 - a) ** n * np.asarray(w0, np.float64)
        for j, rec in enumerate(run.records, start=1):
            ref = ref + a * (1 - a) ** (n - j) * rec.uploaded[l]
        np.testing.assert_allclose(run.weights[l], ref, rtol=1e-12, atol=1e-14)


def _two_components(seed):
    """Two disjoint random graphs (ids [0, n1) and [n1, n1+n2)): parts without halos."""
    rng = np.random.default_rng(seed)
    n1, n2 = 14, 11
    edges = [(a, b) for a in range(n1) for b in range(a + 1, n1) if rng.random() < 0.35]
    edges += [(n1 + a, n1 + b) for a in range(n2) for b in range(a + 1, n2) if rng.random() < 0.4]
    ip, ix = csr_from_edges(n1 + n2, edges)
    return ip, ix, n1, n2


def test_disconnected_parts_match_dense_replay():
    """With one connected component per part there is no halo, so every local epoch is
    plain full-graph GCN on its component at the downloaded W (dense P of the component,
    P:778), followed by the mixing rule -- replayed here independently of the partition
    and layer code."""
    ip, ix, n1, n2 = _two_components(8)
    n = n1 + n2
    rng = np.random.default_rng(1)
    d0, h, C = 5, 6, 3
    x = rng.uniform(-1, 1, (n, d0))
    y = rng.integers(0, C, n).astype(np.int32)
    tm = (rng.random(n) < 0.7).astype(np.uint8)
    tm[0] = tm[n1] = 1
    W0 = [rng.uniform(-0.5, 0.5, (d0, h)), rng.uniform(-0.5, 0.5, (h, C))]
    part = np.array([0] * n1 + [1] * n2, np.int32)
    ev = [0, 1, 1, 0, 1, 0, 0]
    lr = 0.4
    run = oracle_train_async(ip, ix, x, y, tm, W0, C, part, 2, sync_interval=1, events=ev, lr=lr)
    Pf = full_prop_matrix(ip, ix).toarray()
    comps = [np.arange(n1), np.arange(n1, n)]
    Wg = [w.copy() for w in W0]
    losses = []
    for m in ev:
        ids = comps[m]
        P = Pf[np.ix_(ids, ids)]
        H, Z = full_graph_forward(P, x[ids], Wg)
        loss, g = cross_entropy(H[-1], y[ids], tm[ids], C, 1.0 / tm[ids].sum())
        grads = full_graph_backward(P, H, Z, Wg, g)
        Wm = [w - lr * gw for w, gw in zip(Wg, grads)]
        Wg = [0.5 * a + 0.5 * b for a, b in zip(Wg, Wm)]
        losses.append(loss)
    np.testing.assert_allclose([r.loss for r in run.records], losses, rtol=1e-12)
    for a, b in zip(run.weights, Wg):
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("N", [1, 2, 3])
def test_schedule_counts_and_halo_sources(N):
    """Alg. 1 guards on each worker's own counter; every pulled halo row comes from its
    owner's latest push event before the pull (shared KVS)."""
    cfg, inp = _inputs(seed=9, n=44, nnz=200, hidden=(6, 5))
    M = 3
    part = make_random_parts(cfg.num_nodes, M, 6)
    R = 7
    ev = async_events(R, [1.0, 1.6, 0.9], straggler_delays(M, R, 1, 0.5, 1.5, seed=2))
    run = _async(inp, cfg, part, M, ev, sync_interval=N, lr=0.1)
    L = 3
    assert run.ps_updates == M * R == len(ev)
    assert run.pull_count == M * (R // N) * (L - 1)
    assert run.push_count == M * ((R - 1) // N + 1) * (L - 1)
    # replay the owners' push events from the event list alone
    last_push = {}            # owner -> event index of its latest push so far
    last_pull_src = {}        # worker -> snapshot of last_push at its latest pull
    cnt = [0] * M
    for j, (m, rec) in enumerate(zip(ev, run.records)):
        cnt[m] += 1
        assert rec.worker == m and rec.local_epoch == cnt[m]
        if cnt[m] % N == 0:
            last_pull_src[m] = dict(last_push)
        p = run.parts[m]
        owner = part[p.halo_ids]
        want = np.array([last_pull_src.get(m, {}).get(int(k), -1) for k in owner], np.int64)
        for l in (1, 2):
            np.testing.assert_array_equal(rec.halo_versions[l], want)
        if (cnt[m] - 1) % N == 0:
            last_push[m] = j


def test_async_events_and_delays():
    """Discrete-event clock and inject_delay."""
    ev = async_events(3, [1.0, 1.0])
    assert ev == [0, 1, 0, 1, 0, 1]                       # ties -> worker id
    ev = async_events(4, [1.0, 2.5])
    assert ev == [0, 0, 1, 0, 0, 1, 1, 1]                  # ends 1,2,2.5,3,4,5,7.5,10
    d = straggler_delays(4, 10000, 2, 8000.0, 10000.0, seed=0)
    assert (d[[0, 1, 3]] == 0).all()
    assert abs(d[2].mean() - 9000.0) <= 3 * (2000 / np.sqrt(12)) / np.sqrt(10000)
    assert d[2].min() >= 8000 and d[2].max() <= 10000
    np.testing.assert_array_equal(straggler_delays(2, 3, 0, 8000.0, 8000.0, 1)[0], 8000.0)
    with pytest.raises(ValueError):
        straggler_delays(2, 3, 0, 2.0, 1.0, 1)
    ev = async_events(20, [1.0] * 4, straggler_delays(4, 20, 3, 8.0, 10.0, seed=1))
    assert len(ev) == 80 and all(ev.count(m) == 20 for m in range(4))
    # the straggler completes far later: its first epoch ends after everyone's 8th
    assert ev.index(3) > 4 * 8 - 5
