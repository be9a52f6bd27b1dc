"""bf16 stale store (DIGEST_STORE_BF16) on the GPU.

* Exchange: after a push and a pull, every part's fp32 front buffer is BIT-exactly the
  bf16 round-to-nearest-even of its owners' fp32 rows (oracle.train.bf16_round applied to
  the GPU's own H), for the loopback, the normalised push and every pull mode.
* Trajectories vs the oracle with store_dtype='bf16'.  Tolerance 5e-4 instead of 1e-4:
  both sides round the same pushed values to 8 significant bits, but the GPU rounds its
  fp32 H and the oracle its fp64 H; an element within ~1e-7 (relative) of a rounding
  boundary lands one bf16 ulp (2^-8 relative) apart, and a handful of such halo inputs
  per epoch move a layer output by up to ~2^-8 / sqrt(degree * width) ~ 1e-4 relative."""
import numpy as np
import pytest
import torch

import oracle
from oracle.train import bf16_round
from synth import make_block_parts, make_inputs, make_random_parts, small_config
from tests.test_gpu_parity import D, read_rows, rel

pytestmark = pytest.mark.gpu
TOL_BF16 = 5e-4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("pull_mode,norm", [(0, False), (1, False), (0, True)])
def test_bf16_exchange_is_exact_rounding(pull_mode, norm):
    Dm = D()
    from paper_2206_00057_b200.engine import TrainConfig, build_workers, LoopbackGroup
    cfg = small_config(num_nodes=700, nnz=7000, d0=8, hidden=(12, 8), num_classes=3, c_pad=4,
                       seed=19)
    inp = make_inputs(cfg)
    M = 3
    part = make_random_parts(cfg.num_nodes, M, 7)
    tc = TrainConfig(dims=cfg.dims, num_classes=3, store_bf16=True, pull_mode=pull_mode,
                     normalize_pushed=norm)
    ws = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights, part,
                       M, tc)
    grp = LoopbackGroup(ws)
    for w in ws:
        w.forward(1, push=True)
    torch.cuda.synchronize()
    glob = {l: np.zeros((cfg.num_nodes, cfg.dims[l]), np.float32) for l in (1, 2)}
    exps = [w.part.export() for w in ws]
    for w, ex in zip(ws, exps):
        ids = ex["local_ids"].cpu().numpy()
        for l in (1, 2):
            glob[l][ids] = w.H[l].cpu().numpy()
    for w in ws:
        w.pull(2)
    torch.cuda.synchronize()
    for w, ex in zip(ws, exps):
        hids = ex["halo_ids"].cpu().numpy()
        for l in (1, 2):
            p, ld, ver = Dm.digest_store_front(w.store, l)
            assert ver == 1
            front = read_rows(p, w.part.n_halo, ld, cfg.dims[l]).cpu().numpy()
            src = glob[l][hids].astype(np.float64)
            if norm:   # the GPU scales in fp32 by 1/sqrt(sum of squares): compare within 1 ulp
                n = np.sqrt((src ** 2).sum(1, keepdims=True))
                want = bf16_round(np.where(n > 0, src / np.where(n > 0, n, 1), 0))
                assert np.abs(front - want).max() <= 2.0 ** -7 * np.abs(want).max()
            else:
                assert front.astype(np.float32).tobytes() == bf16_round(src).astype(np.float32).tobytes()
    grp.close()


@pytest.mark.parametrize("M,N,opt,fresh", [(2, 1, "sgd", False), (3, 2, "adam", False),
                                           (2, 1, "sgd", True), (4, 3, "sgd", False)])
def test_bf16_store_trajectory_vs_oracle(M, N, opt, fresh):
    from paper_2206_00057_b200.engine import TrainConfig, build_workers, LoopbackGroup
    cfg = small_config(num_nodes=1200, nnz=14000, d0=20, hidden=(32, 16), num_classes=6, c_pad=8,
                       seed=41 + M, train_frac=0.4)
    inp = make_inputs(cfg)
    part = make_block_parts(cfg, M) if M != 3 else make_random_parts(cfg.num_nodes, M, 1)
    R, lr = 6, (0.05 if opt == "sgd" else 0.01)
    tc = TrainConfig(dims=cfg.dims, num_classes=cfg.num_classes, sync_interval=N, lr=lr,
                     optimizer=opt, store_bf16=True, fresh=fresh)
    ws = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights, part,
                       M, tc)
    grp = LoopbackGroup(ws)
    run = oracle.oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                              cfg.num_classes, part, M, sync_interval=N, epochs=R, lr=lr,
                              optimizer=opt, store_dtype="bf16",
                              mode="fresh" if fresh else "stale")
    for r in range(1, R + 1):
        grp.epoch(r)
        torch.cuda.synchronize()
        loss = sum(w.loss.item() for w in ws)
        ref = run.records[r - 1].loss
        assert abs(loss - ref) <= TOL_BF16 * abs(ref), (r, loss, ref)
    for l, wref in enumerate(run.weights):
        assert rel(ws[0].W[l].cpu().numpy(), wref) <= TOL_BF16
    grp.close()
