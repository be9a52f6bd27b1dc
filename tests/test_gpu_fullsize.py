"""Full-size and long-row parity of the GPU path against the oracle,
plus the P:714 staleness bound asserted on the GPU's own outputs.

* products-shaped, full size, M = 8, N_sync = 1: after two full epochs every part's
  halo buffers hold the owners' previous-epoch rows (non-cold, pulled); epoch 3 is run
  up to (not including) AGG and compared in lockstep on two parts: the pulled halo rows
  bit for bit with what their owners computed in epoch 2, sampled output rows of every
  layer from the GPU's own inputs, and every layer's FULL weight gradient.
* Reddit-shaped (average degree ~490, hub rows of thousands), 0.25 scale, M = 2: one
  transform-first layer (602 -> 256) forward and backward per call.
* Bound: at probe epochs of a stale M = 3 run, the oracle takes the GPU's weights, halo
  buffers and representations, computes the exact full-graph H*, eps and delta, and the
  rigorous form of P:714 must hold (slack 1e-4 max|H*| for fp32).
"""
import numpy as np
import pytest
import scipy.sparse as sp
import torch

import oracle
from oracle.gcn import layer_backward, layer_forward, prop_matrix
from oracle.train import full_graph_forward, full_prop_matrix
from synth import (get_config, make_graph, make_inputs, make_block_parts, make_random_parts,
                   small_config)
from synth.configs import scaled
from tests.test_gpu_parity import D, TOL, gpu_partition, read_rows, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _rows_product(P, rows, X):
    """(P X)[rows] in fp64 touching only the source rows those rows need."""
    Pr = P[rows]
    cols = np.unique(Pr.indices)
    Pc = sp.csr_matrix((Pr.data, np.searchsorted(cols, Pr.indices), Pr.indptr),
                       shape=(len(rows), len(cols)))
    return Pc @ np.asarray(X[cols], np.float64)


def _front(w, level, width):
    p, ld, _ = D().digest_store_front(w.store, level)
    return read_rows(p, w.part.n_halo, ld, width).cpu().numpy()


@pytest.mark.slow
def test_full_size_products_stale_halos_lockstep():
    from paper_2206_00057_b200.engine import TrainConfig, build_workers, LoopbackGroup
    cfg = get_config("products")
    inp = make_inputs(cfg)
    M = 8
    part = make_block_parts(cfg, M)
    tc = TrainConfig(dims=cfg.dims, num_classes=cfg.num_classes, sync_interval=1, lr=0.01,
                     optimizer="adam")
    ws = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights, part, M,
                       tc)
    grp = LoopbackGroup(ws)
    L = len(cfg.dims) - 1
    grp.epoch(1)
    grp.epoch(2)
    torch.cuda.synchronize()
    # what every owner pushed in epoch 2 (the rows epoch 3 pulls), by global id
    pushed = {l: np.zeros((cfg.num_nodes, cfg.dims[l]), np.float32) for l in range(1, L)}
    lids = {}
    for m, w in enumerate(ws):
        ids = torch.empty(w.part.n_local, dtype=torch.int32, device="cuda")
        D().digest_part_export(w.part.handle, local_ids=ids)
        lids[m] = ids.cpu().numpy()
        for l in range(1, L):
            pushed[l][lids[m]] = w.H[l].cpu().numpy()
    # epoch 3 up to AGG (pull, forward with the push, loss, backward)
    for w in ws:
        w.pull(3)
    for w in ws:
        w.forward(3, push=True)
    for w in ws:
        w.loss_and_backward()
    torch.cuda.synchronize()
    rng = np.random.default_rng(3)
    for m in (0, 5):
        w = ws[m]
        op = oracle.oracle_partition(inp.indptr, inp.indices, part, M, m)
        P = prop_matrix(op)
        Wt = [x.double().cpu().numpy() for x in w.W]          # the weights epoch 3 used
        fronts = {l: _front(w, l, cfg.dims[l]) for l in range(1, L)}
        for l in range(1, L):                                # pulled halo = owners' rows, bitwise
            assert fronts[l].tobytes() == pushed[l][op.halo_ids].tobytes(), (m, l)
            assert np.abs(fronts[l]).max() > 0                # non-cold
        H = {l: w.H[l].cpu().numpy() for l in range(1, L + 1)}
        x_ext = np.vstack([inp.x[op.local_ids], inp.x[op.halo_ids]])
        deg = np.diff(op.row_ptr)
        rows = np.unique(np.concatenate([rng.choice(op.n_local, 1500, replace=False),
                                         np.argsort(deg)[-50:], [0, op.n_local - 1]]))
        srcs = {1: x_ext}
        for l in range(2, L + 1):
            srcs[l] = np.vstack([H[l - 1], fronts[l - 1]])
        for l in range(1, L + 1):                            # sampled rows, lockstep
            Z = _rows_product(P, rows, srcs[l]) @ Wt[l - 1]
            ref = np.maximum(Z, 0) if l < L else Z
            e = rel(H[l][rows], ref)
            print(f"part {m} layer {l} sampled-row rel err {e:.3g}")
            assert e <= TOL, (m, l, e)
        for l in range(1, L + 1):                            # full G_W of every layer
            A = P @ np.asarray(srcs[l], np.float64)
            Dl = w.G[l].cpu().numpy().astype(np.float64)    # D^(l) (G_IS_D chain; logits grad at L)
            e = rel(w.GW[l - 1].cpu().numpy(), A.T @ Dl)
            print(f"part {m} full G_W{l} rel err {e:.3g}")
            assert e <= TOL, (m, l, e)
    grp.close()


@pytest.mark.slow
@pytest.mark.parametrize("m", [0, 1])
def test_reddit_shaped_layer_parity(m):
    """Long rows (Reddit-shaped: avg degree ~490, hubs of thousands), 0.25 scale, M = 2:
    the transform-first layer 602(604) -> 256 forward and backward per call."""
    Dm = D()
    cfg = scaled(get_config("reddit"), 0.25)
    ip, ix = make_graph(cfg)
    M = 2
    part = make_block_parts(cfg, M)
    p, _ = gpu_partition(ip, ix, part, M, m)
    op = oracle.oracle_partition(ip, ix, part, M, m)
    assert np.diff(op.row_ptr).mean() > 200
    d_in, d_out, order = cfg.dims[0], 256, 0          # AUTO: 604 > 256 -> transform-first
    g = torch.Generator().manual_seed(11 + m)
    xl = torch.rand(p.n_local, d_in, generator=g) * 2 - 1
    xh = torch.rand(p.n_halo, d_in, generator=g) * 2 - 1
    w = (torch.rand(d_in, d_out, generator=g) * 2 - 1) / np.sqrt(d_in)
    gout = torch.randn(p.n_local, d_out, generator=g)
    sv, sc = Dm.digest_layer_workspace(p.handle, d_in, d_out, order)
    saved = torch.empty(max(sv, 256), dtype=torch.uint8, device="cuda")
    scratch = torch.empty(max(sc, 256), dtype=torch.uint8, device="cuda")
    H = torch.empty(p.n_local, d_out, device="cuda")
    Dm.digest_layer_fwd(p.handle, xl.cuda(), xh.cuda(), d_in, w.cuda(), d_in, d_out, 1, order, H,
                        saved, scratch)
    GW = torch.empty(d_in, d_out, device="cuda")
    Gin = torch.empty(p.n_local, d_in, device="cuda")
    Dm.digest_layer_bwd(p.handle, xl.cuda(), xh.cuda(), d_in, w.cuda(), d_in, d_out, 1, order,
                        saved, H, gout.cuda(), GW, Gin, scratch)
    torch.cuda.synchronize()
    ref = layer_forward(op, xl.numpy(), xh.numpy(), w.numpy(), relu=True)
    e = rel(H.cpu().numpy(), ref["H"])
    print(f"reddit part {m} H rel err {e:.3g}")
    assert e <= TOL
    b = layer_backward(op, xl.numpy(), xh.numpy(), w.numpy(), gout.numpy(),
                       H.cpu().numpy() > 0, True)
    assert rel(GW.cpu().numpy(), b["G_W"]) <= TOL
    assert rel(Gin.cpu().numpy(), b["G_in"]) <= TOL
    p.close()


@pytest.mark.parametrize("N,seed", [(3, 0), (5, 1)])
def test_staleness_bound_on_gpu_outputs(N, seed):
    """P:714 (rigorous ReLU-GCN form, reading A18) with the GPU's W, halo buffers and
    representations: delta^(L) <= sum_l eps^(l) prod_{k>l} c_k (+ fp32 slack)."""
    from paper_2206_00057_b200.engine import TrainConfig, build_workers, LoopbackGroup
    cfg = small_config(num_nodes=900, nnz=9000, d0=16, hidden=(24, 16), num_classes=5, c_pad=8,
                       seed=90 + seed, train_frac=0.5)
    inp = make_inputs(cfg)
    M = 3
    part = make_random_parts(cfg.num_nodes, M, seed)
    tc = TrainConfig(dims=cfg.dims, num_classes=cfg.num_classes, sync_interval=N, lr=0.1)
    ws = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights, part,
                       M, tc)
    grp = LoopbackGroup(ws)
    P = full_prop_matrix(inp.indptr, inp.indices)
    deg = oracle.degrees(inp.indptr)
    L = len(cfg.dims) - 1
    ops = [oracle.oracle_partition(inp.indptr, inp.indices, part, M, m) for m in range(M)]
    checked = 0
    for r in range(1, 2 * N + 3):
        W = [x.double().cpu().numpy() for x in ws[0].W]    # weights this epoch uses
        grp.epoch(r)
        torch.cuda.synchronize()
        # GPU representations of every level (global), and the halo rows each part used
        reps = {l: np.zeros((cfg.num_nodes, cfg.dims[l])) for l in range(1, L + 1)}
        for m, w in enumerate(ws):
            for l in range(1, L + 1):
                reps[l][ops[m].local_ids] = w.H[l].double().cpu().numpy()
        eps = {}
        for l in range(1, L):
            e = 0.0
            for m, w in enumerate(ws):
                if ops[m].n_halo:
                    fr = _front(w, l, cfg.dims[l]).astype(np.float64)
                    d = np.sqrt(((fr - reps[l][ops[m].halo_ids]) ** 2).sum(1)).max()
                    e = max(e, d)
            eps[l] = e
        Hs, _ = full_graph_forward(P, inp.x, W)
        dL, tight, paper = oracle.staleness_bound_check(P, deg, W, [reps[l] for l in range(1, L + 1)],
                                                        Hs[1:], eps)
        slack = 1e-4 * np.abs(Hs[L]).max()
        assert dL <= tight + slack and tight <= paper * (1 + 1e-9) + 1e-12, (r, dL, tight, paper)
        checked += dL > slack
    assert checked > 0   # the bound was exercised with real staleness
    grp.close()
