"""GPU path vs oracle for the halo-gradient return: the paper's stale term
P_out^T D~^(t-1) W~^(t)T (halo_grad='prev_epoch') and its exact same-iteration
variant (halo_grad='same_epoch')."""
import numpy as np
import pytest
import torch

import oracle
from oracle.gcn import layer_backward, cross_entropy
from oracle.train import full_prop_matrix, full_graph_forward, full_graph_backward
from synth import make_graph, make_inputs, make_random_parts, small_config
from tests.test_gpu_parity import D, TOL, gpu_partition, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("d_in,d_out,order", [(24, 40, 1), (40, 24, 2), (256, 48, 0),
                                              (100, 256, 0)])
def test_g_halo_per_call(d_in, d_out, order):
    Dm = D()
    cfg = small_config(num_nodes=900, nnz=9000, d0=d_in, hidden=(d_out,), seed=5 + d_in)
    ip, ix = make_graph(cfg)
    part = make_random_parts(cfg.num_nodes, 3, 1)
    p, _ = gpu_partition(ip, ix, part, 3, 2)
    op = oracle.oracle_partition(ip, ix, part, 3, 2)
    g = torch.Generator().manual_seed(d_in + d_out)
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
    Gh = torch.full((p.n_halo, d_in), 9.0, device="cuda")
    Dm.digest_layer_bwd(p.handle, xl.cuda(), xh.cuda(), d_in, w.cuda(), d_in, d_out, 1, order,
                        saved, H, gout.cuda(), GW, Gin, scratch, G_halo=Gh)
    torch.cuda.synchronize()
    b = layer_backward(op, xl.numpy(), xh.numpy(), w.numpy(), gout.numpy(),
                       H.cpu().numpy() > 0, True, need_g_halo=True)
    assert rel(Gh.cpu().numpy(), b["G_halo"]) <= TOL
    assert rel(GW.cpu().numpy(), b["G_W"]) <= TOL
    p.close()


@pytest.mark.parametrize("M,fresh,N", [(2, True, 1), (3, True, 1), (3, False, 2)])
def test_trajectory_with_halo_grad(M, fresh, N):
    from paper_2206_00057_b200.engine import TrainConfig, build_workers, LoopbackGroup
    cfg = small_config(num_nodes=1000, nnz=11000, d0=20, hidden=(32, 16), num_classes=6, c_pad=8,
                       seed=60 + M, train_frac=0.5)
    inp = make_inputs(cfg)
    part = make_random_parts(cfg.num_nodes, M, 9)
    tc = TrainConfig(dims=cfg.dims, num_classes=cfg.num_classes, sync_interval=N, lr=0.05,
                     fresh=fresh, halo_grad=True)
    ws = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights, part, M, tc)
    grp = LoopbackGroup(ws)
    R = 3
    run = oracle.oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                              cfg.num_classes, part, M, sync_interval=N, epochs=R, lr=0.05,
                              mode="fresh" if fresh else "stale", halo_grad="same_epoch")
    for r in range(1, R + 1):
        grp.epoch(r)
        torch.cuda.synchronize()
        loss = sum(w.loss.item() for w in ws)
        assert abs(loss - run.records[r - 1].loss) <= TOL * abs(run.records[r - 1].loss)
        if r == 1 and fresh:
            # exact: every layer's aggregated gradient equals full-graph GCN's (A16 closed)
            P = full_prop_matrix(inp.indptr, inp.indices)
            W = [x.astype(np.float64) for x in inp.weights]
            H, Z = full_graph_forward(P, inp.x, W)
            _, g = cross_entropy(H[-1], inp.y, inp.train_mask, cfg.num_classes,
                                 1.0 / inp.train_mask.sum())
            ref = full_graph_backward(P, H, Z, W, g)
            for l, gref in enumerate(ref):
                assert rel(ws[0].GW[l].cpu().numpy(), gref) <= TOL, l
    for l, wref in enumerate(run.weights):
        assert rel(ws[0].W[l].cpu().numpy(), wref) <= TOL
    grp.close()


@pytest.mark.parametrize("d_in,d_out,order", [(24, 40, 1), (40, 24, 2), (256, 48, 0),
                                              (100, 256, 0)])
def test_saved_s_per_call(d_in, d_out, order):
    """DIGEST_BWD_HALO_SAVE_S: G_halo receives S = P_out^T D (width d_out) and G_W is
    unchanged; S W^T through digest_gemm(bt) is the oracle's G_halo."""
    Dm = D()
    cfg = small_config(num_nodes=900, nnz=9000, d0=d_in, hidden=(d_out,), seed=15 + d_in)
    ip, ix = make_graph(cfg)
    part = make_random_parts(cfg.num_nodes, 3, 2)
    p, _ = gpu_partition(ip, ix, part, 3, 1)
    op = oracle.oracle_partition(ip, ix, part, 3, 1)
    g = torch.Generator().manual_seed(3 * d_in + d_out)
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
    S = torch.full((p.n_halo, d_out), 9.0, device="cuda")
    Dm.digest_layer_bwd(p.handle, xl.cuda(), xh.cuda(), d_in, w.cuda(), d_in, d_out, 1, order,
                        saved, H, gout.cuda(), GW, Gin, scratch, G_halo=S,
                        flags=Dm.BWD_HALO_SAVE_S)
    Gh = torch.empty(p.n_halo, d_in, device="cuda")
    Dm.digest_gemm(S, w.cuda(), Gh, bt=True)
    torch.cuda.synchronize()
    b = layer_backward(op, xl.numpy(), xh.numpy(), w.numpy(), gout.numpy(),
                       H.cpu().numpy() > 0, True, need_g_halo=True)
    P_out = oracle.gcn.prop_matrix(op)[:, op.n_local:]
    assert rel(S.cpu().numpy(), P_out.T @ b["D"]) <= TOL
    assert rel(Gh.cpu().numpy(), b["G_halo"]) <= TOL
    assert rel(GW.cpu().numpy(), b["G_W"]) <= TOL
    assert rel(Gin.cpu().numpy(), b["G_in"]) <= TOL
    p.close()


@pytest.mark.parametrize("M,N,opt", [(2, 1, "sgd"), (3, 1, "sgd"), (3, 2, "adam")])
def test_trajectory_with_stale_halo_grad(M, N, opt):
    """halo_grad='prev_epoch' (P:816 literal) vs the oracle, per epoch; the stale term
    changes the trajectory (it is not the constant-halo run)."""
    from paper_2206_00057_b200.engine import TrainConfig, build_workers, LoopbackGroup
    cfg = small_config(num_nodes=1000, nnz=11000, d0=20, hidden=(32, 16), num_classes=6, c_pad=8,
                       seed=80 + M, train_frac=0.5)
    inp = make_inputs(cfg)
    part = make_random_parts(cfg.num_nodes, M, 4)
    lr = 0.05 if opt == "sgd" else 0.01
    tc = TrainConfig(dims=cfg.dims, num_classes=cfg.num_classes, sync_interval=N, lr=lr,
                     optimizer=opt, halo_grad="prev_epoch")
    ws = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights, part, M, tc)
    grp = LoopbackGroup(ws)
    R = 4
    kw = dict(sync_interval=N, epochs=R, lr=lr, optimizer=opt)
    run = oracle.oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                              cfg.num_classes, part, M, halo_grad="prev_epoch", **kw)
    base = oracle.oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                               cfg.num_classes, part, M, **kw)
    for r in range(1, R + 1):
        grp.epoch(r)
        torch.cuda.synchronize()
        loss = sum(w.loss.item() for w in ws)
        assert abs(loss - run.records[r - 1].loss) <= TOL * abs(run.records[r - 1].loss), r
        for l, gref in enumerate(run.records[r - 1].grads):
            assert rel(ws[0].GW[l].cpu().numpy(), gref) <= TOL, (r, l)
    for l, wref in enumerate(run.weights):
        assert rel(ws[0].W[l].cpu().numpy(), wref) <= TOL
    # the returned term is real: the first layer's weights leave the constant-halo run
    assert rel(run.weights[0], base.weights[0]) > 10 * TOL
    grp.close()


@pytest.mark.parametrize("d_in,d_out,order,save_s", [(24, 40, 1, False), (40, 24, 2, False),
                                                     (256, 48, 0, False), (256, 48, 0, True),
                                                     (40, 8, 2, True)])
def test_loss_rows_products_equal_full_products(d_in, d_out, order, save_s):
    """digest_part_set_loss_mask + DIGEST_BWD_LOSS_ROWS (the last layer's P_in / P_out^T
    products over the training-row columns only) = the full products when G_out is
    zero outside the mask; and both = the oracle."""
    Dm = D()
    cfg = small_config(num_nodes=900, nnz=9000, d0=d_in, hidden=(d_out,), seed=11 + d_in)
    ip, ix = make_graph(cfg)
    part = make_random_parts(cfg.num_nodes, 3, 2)
    p, _ = gpu_partition(ip, ix, part, 3, 1)
    op = oracle.oracle_partition(ip, ix, part, 3, 1)
    g = torch.Generator().manual_seed(d_in * 7 + d_out)
    xl = torch.rand(p.n_local, d_in, generator=g) * 2 - 1
    xh = torch.rand(p.n_halo, d_in, generator=g) * 2 - 1
    w = (torch.rand(d_in, d_out, generator=g) * 2 - 1) / np.sqrt(d_in)
    tmask = (torch.rand(p.n_local, generator=g) < 0.1).to(torch.uint8)
    gout = torch.randn(p.n_local, d_out, generator=g) * tmask[:, None].float()
    sv, sc = Dm.digest_layer_workspace(p.handle, d_in, d_out, order)
    saved = torch.empty(max(sv, 256), dtype=torch.uint8, device="cuda")
    scratch = torch.empty(max(sc, 256), dtype=torch.uint8, device="cuda")
    H = torch.empty(p.n_local, d_out, device="cuda")
    Dm.digest_layer_fwd(p.handle, xl.cuda(), xh.cuda(), d_in, w.cuda(), d_in, d_out, 0, order, H,
                        saved, scratch)
    outs = []
    for lrows in (False, True):
        if lrows:
            Dm.digest_part_set_loss_mask(p.handle, tmask.cuda())
        GW = torch.empty(d_in, d_out, device="cuda")
        Gin = torch.empty(p.n_local, d_in, device="cuda")
        Gh = torch.full((p.n_halo, d_out if save_s else d_in), 9.0, device="cuda")
        fl = (Dm.BWD_LOSS_ROWS if lrows else 0) | (Dm.BWD_HALO_SAVE_S if save_s else 0)
        Dm.digest_layer_bwd(p.handle, xl.cuda(), xh.cuda(), d_in, w.cuda(), d_in, d_out, 0, order,
                            saved, H, gout.cuda(), GW, Gin, scratch, G_halo=Gh, flags=fl)
        torch.cuda.synchronize()
        outs.append([GW.cpu().numpy(), Gin.cpu().numpy(), Gh.cpu().numpy()])
    for a, b in zip(*outs):
        assert rel(b, a) <= 1e-6
    ref = layer_backward(op, xl.numpy(), xh.numpy(), w.numpy(), gout.numpy(), None, True,
                         need_g_halo=not save_s)
    assert rel(outs[1][0], ref["G_W"]) <= TOL
    assert rel(outs[1][1], ref["G_in"]) <= TOL
    if not save_s:
        assert rel(outs[1][2], ref["G_halo"]) <= TOL
    Dm.digest_part_set_loss_mask(p.handle, None)
    p.close()


def test_loss_rows_flag_without_mask_is_refused():
    Dm = D()
    cfg = small_config(num_nodes=300, nnz=2400, d0=8, hidden=(8,), seed=3)
    ip, ix = make_graph(cfg)
    part = make_random_parts(cfg.num_nodes, 2, 1)
    p, _ = gpu_partition(ip, ix, part, 2, 0)
    sv, sc = Dm.digest_layer_workspace(p.handle, 8, 8, 2)
    saved = torch.empty(max(sv, 256), dtype=torch.uint8, device="cuda")
    scratch = torch.empty(max(sc, 256), dtype=torch.uint8, device="cuda")
    x = torch.rand(p.n_local, 8, device="cuda")
    xh = torch.rand(max(p.n_halo, 1), 8, device="cuda")
    w = torch.rand(8, 8, device="cuda")
    H = torch.empty(p.n_local, 8, device="cuda")
    Dm.digest_layer_fwd(p.handle, x, xh, 8, w, 8, 8, 0, 2, H, saved, scratch)
    GW = torch.empty(8, 8, device="cuda")
    with pytest.raises(Dm.DigestError):
        Dm.digest_layer_bwd(p.handle, x, xh, 8, w, 8, 8, 0, 2, saved, H, H, GW, None, scratch,
                            flags=Dm.BWD_LOSS_ROWS)
    p.close()
