"""DIGEST-A on the GPU vs the oracle on the same seeded
event schedule (synth.async_sched: discrete-event clock with a straggler).
Bar: every event's local loss and the final W_global within 1e-4 (north_star)."""
import numpy as np
import pytest
import torch

from oracle import oracle_train
from oracle.async_train import oracle_train_async
from synth import make_block_parts, make_inputs, make_random_parts, small_config
from synth.async_sched import async_events, straggler_delays

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def read_rows(addr, n, ld, width):
    from tests.test_gpu_parity import read_rows as rr
    return rr(addr, n, ld, width)


def rel(got, ref):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    return np.abs(got - ref).max() / np.abs(ref).max()


@pytest.mark.parametrize("M,N,opt,straggler", [(1, 1, "sgd", None), (2, 1, "sgd", None),
                                               (3, 2, "sgd", 1), (4, 3, "adam", 2)])
def test_async_loopback_vs_oracle(M, N, opt, straggler):
    from paper_2206_00057_b200 import capi as D
    from paper_2206_00057_b200.engine import TrainConfig, build_workers, AsyncLoopbackGroup
    cfg = small_config(num_nodes=1000, nnz=11000, d0=20, hidden=(32, 16), num_classes=6, c_pad=8,
                       seed=70 + M, train_frac=0.5)
    inp = make_inputs(cfg)
    part = make_block_parts(cfg, M) if M != 3 else make_random_parts(cfg.num_nodes, M, 5)
    R, lr = 5, (0.05 if opt == "sgd" else 0.01)
    delays = straggler_delays(M, R, straggler, 2.0, 3.0, seed=M)
    ev = async_events(R, [1.0 + 0.1 * m for m in range(M)], delays)
    tc = TrainConfig(dims=cfg.dims, num_classes=cfg.num_classes, sync_interval=N, lr=lr,
                     optimizer=opt, pull_mode=D.PULL_COPY)
    ws = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights, part,
                       M, tc, loss_weighting="local")
    grp = AsyncLoopbackGroup(ws)
    run = oracle_train_async(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                             cfg.num_classes, part, M, sync_interval=N, events=ev, lr=lr,
                             optimizer=opt, record_halos=True)
    for j, m in enumerate(ev):
        grp.event(m)
        torch.cuda.synchronize()
        rec = run.records[j]
        got, ref = ws[m].loss.item(), rec.loss
        assert abs(got - ref) <= TOL * abs(ref), (j, m, got, ref)
        # the halo rows the event used, row by row: never-pushed rows (version -1) are
        # exactly zero, the others are the owner's latest push before the pull
        for l, hv in rec.halo_versions.items():
            if ws[m].part.n_halo == 0:
                continue
            p, ld, _ = D.digest_store_front(ws[m].store, l)
            front = read_rows(p, ws[m].part.n_halo, ld, cfg.dims[l]).cpu().numpy()
            cold = hv < 0
            assert not front[cold].any(), (j, m, l, "rows never pushed must be zero")
            if (~cold).any():
                h = rec.halos[l][~cold]
                err = np.abs(front[~cold] - h).max() / max(np.abs(h).max(), 1e-30)
                assert err <= TOL, (j, m, l, err)
    wref = np.concatenate([w.ravel() for w in run.weights])
    assert rel(grp.W_global.cpu().numpy(), wref) <= TOL
    assert grp.ps_updates == M * R
    assert sum(w.pulls for w in ws) == run.pull_count
    assert sum(w.pushes for w in ws) == run.push_count
    if M == 1:   # one worker, alpha = 1: DIGEST-A is the synchronous run
        s = oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                         cfg.num_classes, part, 1, sync_interval=N, epochs=R, lr=lr,
                         optimizer=opt)
        assert rel(grp.W_global.cpu().numpy(), np.concatenate([w.ravel() for w in s.weights])) <= TOL
    grp.close()
