"""GPU path (libdigest.so through the C ABI) vs the CPU oracle.

Bit-exact: partition arrays, send lists, counts/offsets, reverse-halo CSR, halo
exchange copies.  Float: rel = max|gpu - ref| / max|ref| <= 1e-4 (north_star's
fp32 tolerance), with the oracle computed in fp64 from the GPU's own inputs for
per-call parity, and from the shared seeded inputs for trajectories.
"""
import hashlib

import numpy as np
import pytest
import torch

import oracle
from oracle.gcn import layer_forward, layer_backward, cross_entropy
from synth import (get_config, make_graph, make_inputs, make_block_parts, make_random_parts,
                   small_config)
from synth.configs import scaled

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def D():
    from paper_2206_00057_b200 import capi
    return capi


def rel(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.abs(ref).max() if ref.size else 0.0
    num = np.abs(got - ref).max() if ref.size else 0.0
    return num / den if den > 0 else num


def read_rows(addr, n, ld, width):
    """Copy an n x width block at a raw device address (row stride ld) into a tensor."""
    Dm = D()
    out = torch.empty(n, width, device="cuda")
    idx = torch.arange(n, dtype=torch.int32, device="cuda")
    st = Dm.lib.digest_gather_rows(addr, ld, idx.data_ptr(), n, out.data_ptr(), width, width,
                                   Dm.stream_ptr())
    assert st == 0, Dm.digest_last_error()
    torch.cuda.synchronize()
    return out


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gpu_partition(indptr, indices, part_of, M, m):
    from paper_2206_00057_b200.engine import Partition
    d = lambda a, dt: torch.as_tensor(a, dtype=dt).cuda()
    p = Partition(d(indptr, torch.int64), d(indices, torch.int32), d(part_of, torch.int32), M, m)
    ex = {k: (v.cpu().numpy() if torch.is_tensor(v) else v) for k, v in p.export().items()}
    return p, ex


def assert_partition_equal(ex, o):
    assert ex["local_ids"].dtype == np.int32 and ex["col"].dtype == np.int32
    for k in ("local_ids", "halo_ids", "row_ptr", "col", "val", "send_idx", "rh_ptr", "rh_col",
              "rh_val"):
        a, b = ex[k], getattr(o, k)
        assert a.dtype == b.dtype, (k, a.dtype, b.dtype)
        assert a.shape == b.shape and sha(a) == sha(b), k
    for k in ("send_count", "send_off", "recv_count", "recv_off"):
        np.testing.assert_array_equal(ex[k], getattr(o, k), err_msg=k)


# ------------------------------------------------------------------ partition (a1)
@pytest.mark.parametrize("seed", range(6))
def test_partition_bitexact_random(seed):
    rng = np.random.default_rng(seed)
    cfg = small_config(num_nodes=int(rng.integers(50, 400)), nnz=0, seed=seed)
    n = cfg.num_nodes
    from dataclasses import replace
    cfg = replace(cfg, nnz=int(n * rng.uniform(2, 12)) // 2 * 2)
    ip, ix = make_graph(cfg)
    M = int(rng.integers(1, 9))
    part = make_random_parts(n, M, seed) if seed % 2 else make_block_parts(cfg, M)
    for m in range(M):
        p, ex = gpu_partition(ip, ix, part, M, m)
        assert_partition_equal(ex, oracle.oracle_partition(ip, ix, part, M, m))
        p.close()


@pytest.mark.parametrize("name,M,ranks", [("cora", 2, [0, 1]), ("flickr", 4, [0, 3]),
                                          ("arxiv", 8, [2, 7])])
def test_partition_bitexact_configs(name, M, ranks):
    cfg = get_config(name)
    ip, ix = make_graph(cfg)
    part = make_block_parts(cfg, M)
    for m in ranks:
        p, ex = gpu_partition(ip, ix, part, M, m)
        assert_partition_equal(ex, oracle.oracle_partition(ip, ix, part, M, m))
        p.close()


@pytest.mark.slow
@pytest.mark.parametrize("name,M,ranks", [("products", 8, [0, 5]), ("reddit", 4, [1])])
def test_partition_bitexact_full_size(name, M, ranks):
    cfg = get_config(name)
    ip, ix = make_graph(cfg)
    part = make_block_parts(cfg, M)
    for m in ranks:
        p, ex = gpu_partition(ip, ix, part, M, m)
        assert_partition_equal(ex, oracle.oracle_partition(ip, ix, part, M, m))
        p.close()


def test_partition_rejects_bad_inputs():
    Dm = D()
    ip = torch.tensor([0, 1, 2], dtype=torch.int64).cuda()
    ix = torch.tensor([1, 0], dtype=torch.int32).cuda()
    for po, M in (([0, 0], 2), ([0, 3], 2)):
        with pytest.raises(Dm.DigestError) as e:
            Dm.digest_partition(2, 2, ip, ix, torch.tensor(po, dtype=torch.int32).cuda(), M, 0)
        assert e.value.status == 1
    bad = torch.tensor([0, 0], dtype=torch.int32).cuda()  # self loop
    with pytest.raises(Dm.DigestError):
        Dm.digest_partition(2, 2, ip, bad, torch.tensor([0, 1], dtype=torch.int32).cuda(), 2, 0)


# ------------------------------------------------------------------ one layer (a3-a5, a8)
def _layer_case(seed, n=900, nnz=9000, M=3, m=1, d_in=24, d_out=40):
    cfg = small_config(num_nodes=n, nnz=nnz, d0=d_in, hidden=(d_out,), seed=seed)
    ip, ix = make_graph(cfg)
    part = make_random_parts(n, M, seed)
    p, _ = gpu_partition(ip, ix, part, M, m)
    op = oracle.oracle_partition(ip, ix, part, M, m)
    return p, op


@pytest.mark.parametrize("d_in,d_out", [(24, 40), (40, 24), (100, 256), (256, 48), (16, 8),
                                        (128, 128), (604, 256)])
@pytest.mark.parametrize("order", [0, 1, 2])
def test_layer_forward_backward_per_call(d_in, d_out, order):
    Dm = D()
    p, op = _layer_case(7 + d_in + d_out, d_in=d_in, d_out=d_out)
    g = torch.Generator().manual_seed(d_in * 1000 + d_out)
    xl = torch.rand(p.n_local, d_in, generator=g) * 2 - 1
    xh = torch.rand(p.n_halo, d_in, generator=g) * 2 - 1
    w = (torch.rand(d_in, d_out, generator=g) * 2 - 1) / np.sqrt(d_in)
    gout = torch.randn(p.n_local, d_out, generator=g)
    xl_d, xh_d, w_d, go_d = xl.cuda(), xh.cuda(), w.cuda(), gout.cuda()
    sv, sc = Dm.digest_layer_workspace(p.handle, d_in, d_out, order)
    saved = torch.empty(max(sv, 256), dtype=torch.uint8, device="cuda")
    scratch = torch.empty(max(sc, 256), dtype=torch.uint8, device="cuda")
    for act in (0, 1):
        H = torch.empty(p.n_local, d_out, device="cuda")
        Dm.digest_layer_fwd(p.handle, xl_d, xh_d, d_in, w_d, d_in, d_out, act, order, H, saved,
                            scratch)
        GW = torch.empty(d_in, d_out, device="cuda")
        Gin = torch.empty(p.n_local, d_in, device="cuda")
        Dm.digest_layer_bwd(p.handle, xl_d, xh_d, d_in, w_d, d_in, d_out, act, order, saved,
                            H if act else None, go_d, GW, Gin, scratch)
        torch.cuda.synchronize()
        ref = layer_forward(op, xl.numpy(), xh.numpy(), w.numpy(), relu=bool(act))
        assert rel(H.cpu().numpy(), ref["H"]) <= TOL
        mask = (H.cpu().numpy() > 0) if act else None   # share the kernel's ReLU decisions
        b = layer_backward(op, xl.numpy(), xh.numpy(), w.numpy(), gout.numpy(), mask, True)
        assert rel(GW.cpu().numpy(), b["G_W"]) <= TOL, (act, rel(GW.cpu().numpy(), b["G_W"]))
        assert rel(Gin.cpu().numpy(), b["G_in"]) <= TOL
        # fused variants: G_out already masked (G_IS_D) and G_in emitted masked by gin_mask
        gm = torch.randn(p.n_local, d_in, generator=g)
        Dpre = torch.as_tensor(b["D"], dtype=torch.float32).cuda()
        GW2 = torch.empty_like(GW)
        Gin2 = torch.empty_like(Gin)
        Dm.digest_layer_bwd(p.handle, xl_d, xh_d, d_in, w_d, d_in, d_out, act, order, saved,
                            None, Dpre, GW2, Gin2, scratch, flags=Dm.BWD_G_IS_D,
                            gin_mask=gm.cuda())
        torch.cuda.synchronize()
        assert rel(GW2.cpu().numpy(), b["G_W"]) <= TOL
        assert rel(Gin2.cpu().numpy(), b["G_in"] * (gm.numpy() > 0)) <= TOL
        # the same with the previous layer's ReLU' as a 1-bit mask
        gmb = torch.from_numpy(pack_bits(gm.numpy() > 0, ld_words(d_in))).cuda()
        Gin3 = torch.empty_like(Gin)
        Dm.digest_layer_bwd(p.handle, xl_d, xh_d, d_in, w_d, d_in, d_out, act, order, saved,
                            None, Dpre, GW2, Gin3, scratch, flags=Dm.BWD_G_IS_D,
                            gin_mask=(gmb.data_ptr(), gmb.shape[1]))
        torch.cuda.synchronize()
        assert torch.equal(Gin3, Gin2)
        if act:   # the forward's 1-bit mask is exactly 1[H > 0] of its own output
            bits = saved_bits(Dm, p, d_in, d_out, order, saved)
            nw = (d_out + 31) // 32   # words past nw are row padding (never read)
            np.testing.assert_array_equal(bits[:, :nw],
                                          pack_bits(H.cpu().numpy() > 0, bits.shape[1])[:, :nw])
    p.close()


def ld_words(d):
    return -(-((d + 31) // 32) // 4) * 4


def pack_bits(b, ldw):
    """bool [n, d] -> int32 [n, ldw]: bit j % 32 of word j // 32 = b[:, j]."""
    n, d = b.shape
    full = np.zeros((n, ldw * 32), dtype=np.uint64)
    full[:, :d] = b
    words = (full.reshape(n, ldw, 32) << np.arange(32, dtype=np.uint64)).sum(axis=2)
    return words.astype(np.uint32).view(np.int32)


def saved_bits(Dm, p, d_in, d_out, order, saved):
    addr, ldw = Dm.digest_layer_mask(p.handle, d_in, d_out, order, saved)
    off = addr - saved.data_ptr()
    assert 0 <= off and off + 4 * p.n_local * ldw <= saved.numel()
    return saved[off:off + 4 * p.n_local * ldw].view(torch.int32).reshape(
        p.n_local, ldw).cpu().numpy()


def test_layer_empty_halo_and_argument_errors():
    Dm = D()
    cfg = small_config(num_nodes=200, nnz=1000, seed=3)
    ip, ix = make_graph(cfg)
    p, _ = gpu_partition(ip, ix, np.zeros(200, np.int32), 1, 0)
    op = oracle.oracle_partition(ip, ix, np.zeros(200, np.int32), 1, 0)
    assert p.n_halo == 0
    x = torch.rand(200, 8)
    w = torch.rand(8, 12)
    sv, sc = Dm.digest_layer_workspace(p.handle, 8, 12, 0)
    saved = torch.empty(max(sv, 256), dtype=torch.uint8, device="cuda")
    scratch = torch.empty(max(sc, 256), dtype=torch.uint8, device="cuda")
    H = torch.empty(200, 12, device="cuda")
    Dm.digest_layer_fwd(p.handle, x.cuda(), None, 0, w.cuda(), 8, 12, 1, 0, H, saved, scratch)
    torch.cuda.synchronize()
    assert rel(H.cpu().numpy(), layer_forward(op, x.numpy(), None, w.numpy(), True)["H"]) <= TOL
    with pytest.raises(Dm.DigestError) as e:   # d_in not a multiple of 4
        Dm.digest_layer_fwd(p.handle, x.cuda(), None, 0, w.cuda(), 6, 12, 1, 0, H, saved, scratch)
    assert e.value.status == 2
    p.close()


# ------------------------------------------------------------------ loss, update, gemm
@pytest.mark.parametrize("C,Cp", [(41, 48), (7, 8), (64, 64), (70, 72)])
def test_xent_parity(C, Cp):
    """Both kernels: the register path (ld_g <= 64) and the generic loop (ld_g > 64)."""
    Dm = D()
    n = 5000
    g = torch.Generator().manual_seed(1)
    z = torch.randn(n, Cp, generator=g) * 3
    y = torch.randint(0, C, (n,), generator=g, dtype=torch.int32)
    t = (torch.rand(n, generator=g) < 0.6).to(torch.uint8)
    G = torch.full((n, Cp), 7.0, device="cuda")
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    scr = torch.empty(Dm.digest_xent_workspace(n), dtype=torch.uint8, device="cuda")
    Dm.digest_xent(z.cuda(), C, y.cuda(), t.cuda(), 1.0 / 3000, G, loss, scr)
    ref_loss, ref_g = cross_entropy(z.numpy(), y.numpy(), t.numpy(), C, 1.0 / 3000)
    assert abs(loss.item() - ref_loss) <= TOL * abs(ref_loss)
    assert rel(G.cpu().numpy(), ref_g) <= TOL
    assert torch.all(G[:, C:] == 0) and torch.all(G[t.cuda() == 0] == 0)


def test_optimizers_parity():
    Dm = D()
    g = torch.Generator().manual_seed(2)
    W = torch.randn(10000, generator=g)
    G = torch.randn(10000, generator=g)
    Wd = W.cuda()
    Dm.digest_sgd_step(Wd, G.cuda(), 0.1)
    assert rel(Wd.cpu().numpy(), oracle.sgd_step(W.numpy(), G.numpy(), 0.1)) <= 1e-6
    Wd = W.cuda()
    m, v = torch.zeros_like(Wd), torch.zeros_like(Wd)
    wr, mr, vr = W.numpy().astype(np.float64), 0.0, 0.0
    for step in (1, 2, 3):
        Dm.digest_adam_step(Wd, G.cuda() * step, m, v, 0.01, 0.9, 0.999, 1e-8, step)
        wr, mr, vr = oracle.adam_step(wr, G.numpy() * step, mr, vr, step, 0.01)
    assert rel(Wd.cpu().numpy(), wr) <= 1e-5
    # device-resident step count (CUDA-graph epochs): the same three updates
    Wd2 = W.cuda()
    m, v = torch.zeros_like(Wd2), torch.zeros_like(Wd2)
    step_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
    for step in (1, 2, 3):
        Dm.digest_adam_step_dev(Wd2, G.cuda() * step, m, v, 0.01, 0.9, 0.999, 1e-8, step_dev)
    assert int(step_dev.item()) == 3
    assert rel(Wd2.cpu().numpy(), wr) <= 1e-5


def test_cuda_graph_epoch_replay_matches_eager():
    """An M=1 epoch captured in a CUDA graph (Adam step on the device) and replayed gives the
    eager run's weights and losses, bit for bit (same kernels, same arguments)."""
    from paper_2206_00057_b200.engine import TrainConfig, build_workers
    cfg = small_config(num_nodes=1500, nnz=16000, d0=20, hidden=(32, 16), num_classes=6, c_pad=8,
                       seed=91, train_frac=0.5)
    inp = make_inputs(cfg)
    part = np.zeros(cfg.num_nodes, np.int32)
    runs = []
    for use_graph in (False, True):
        tc = TrainConfig(dims=cfg.dims, num_classes=cfg.num_classes, sync_interval=1, lr=0.01,
                         optimizer="adam", device_step=True)
        (w,) = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                             part, 1, tc)
        w.epoch(1)                          # warm-up (lazy workspaces, attributes)
        losses = []
        if use_graph:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                w.epoch(2)
            for _ in range(4):
                g.replay()
                torch.cuda.synchronize()
                losses.append(w.loss.item())
        else:
            for r in range(2, 6):
                w.epoch(r)
                torch.cuda.synchronize()
                losses.append(w.loss.item())
        runs.append((losses, w.W_flat.cpu().numpy(), int(w.step_dev.item())))
        w.close()
    assert runs[0][0] == runs[1][0]
    assert runs[0][1].tobytes() == runs[1][1].tobytes()
    assert runs[0][2] == runs[1][2] == 5


@pytest.mark.parametrize("M,N,K", [(1000, 256, 100), (777, 48, 256), (4096, 16, 1436),
                                   (129, 8, 16), (3000, 256, 256), (5000, 8, 16), (300, 128, 604),
                                   (2049, 64, 500), (70000, 256, 256), (9000, 256, 36),
                                   (3000, 256, 68), (4100, 48, 4)])
def test_gemm_parity(M, N, K):
    Dm = D()
    g = torch.Generator().manual_seed(M + N + K)
    A = torch.rand(M, K, generator=g) * 2 - 1
    B = torch.rand(K, N, generator=g) * 2 - 1
    Cm = torch.empty(M, N, device="cuda")
    Dm.digest_gemm(A.cuda(), B.cuda(), Cm, relu=True)
    ref = np.maximum(A.double().numpy() @ B.double().numpy(), 0)
    assert rel(Cm.cpu().numpy(), ref) <= TOL
    # the 3xTF32 tensor-core path is near-fp32 accurate (plain TF32 would be ~1e-3)
    assert rel(Cm.cpu().numpy(), ref) <= 3e-5, rel(Cm.cpu().numpy(), ref)


@pytest.mark.parametrize("M,N,K", [(1000, 256, 48), (3000, 100, 256), (777, 36, 52)])
def test_gemm_transposed_b_parity(M, N, K):
    """DIGEST_GEMM_BT (C = A B^T, B given N x K): the stale halo-gradient term S W^T."""
    Dm = D()
    g = torch.Generator().manual_seed(3 * M + N + K)
    A = torch.rand(M, K, generator=g) * 2 - 1
    B = torch.rand(N, K, generator=g) * 2 - 1
    Cm = torch.empty(M, N, device="cuda")
    Dm.digest_gemm(A.cuda(), B.cuda(), Cm, bt=True)
    ref = A.double().numpy() @ B.double().numpy().T
    assert rel(Cm.cpu().numpy(), ref) <= 3e-5


# ------------------------------------------------------------------ store (a2, a6)
def test_push_pull_is_an_exact_copy_and_follows_versions():
    Dm = D()
    from paper_2206_00057_b200.engine import TrainConfig, build_workers
    cfg = small_config(num_nodes=600, nnz=6000, d0=8, hidden=(12, 8), num_classes=3, c_pad=4, seed=9)
    inp = make_inputs(cfg)
    M = 3
    part = make_random_parts(cfg.num_nodes, M, 4)
    tc = TrainConfig(dims=cfg.dims, num_classes=3)
    ws = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights, part, M, tc)
    from paper_2206_00057_b200.engine import LoopbackGroup
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
    # before the pull, fronts are still the cold (zero) buffers
    for w in ws:
        p, ld, ver = Dm.digest_store_front(w.store, 1)
        assert ver == 0
    with pytest.raises(Dm.DigestError) as e:     # a pull in the pushing epoch is refused
        Dm.digest_pull(ws[0].store, 1, 1)
    assert e.value.status == 3
    for w in ws:
        w.pull(2)
    torch.cuda.synchronize()
    for w, ex in zip(ws, exps):
        hids = ex["halo_ids"].cpu().numpy()
        for l in (1, 2):
            p, ld, ver = Dm.digest_store_front(w.store, l)
            assert ver == 1
            front = read_rows(p, w.part.n_halo, ld, cfg.dims[l]).cpu().numpy()
            assert front.tobytes() == glob[l][hids].tobytes()
    # a second pull without a new push is a no-op
    for w in ws:
        w.pull(3)
        assert Dm.digest_store_front(w.store, 1)[2] == 1
    grp.close()


# ------------------------------------------------------------------ trajectories (whole epoch)
@pytest.mark.parametrize("M,N,opt", [(1, 1, "sgd"), (2, 1, "sgd"), (3, 2, "sgd"), (4, 3, "adam"),
                                     (2, 1, "adam")])
def test_epoch_trajectory_vs_oracle(M, N, opt):
    from paper_2206_00057_b200.engine import TrainConfig, build_workers, LoopbackGroup
    cfg = small_config(num_nodes=1200, nnz=14000, d0=20, hidden=(32, 16), num_classes=6, c_pad=8,
                       seed=11 + M, train_frac=0.4)
    inp = make_inputs(cfg)
    part = make_block_parts(cfg, M) if M != 3 else make_random_parts(cfg.num_nodes, M, 1)
    R, lr = 6, (0.05 if opt == "sgd" else 0.01)
    tc = TrainConfig(dims=cfg.dims, num_classes=cfg.num_classes, sync_interval=N, lr=lr,
                     optimizer=opt)
    ws = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights, part, M, tc)
    grp = LoopbackGroup(ws)
    run = oracle.oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                              cfg.num_classes, part, M, sync_interval=N, epochs=R, lr=lr,
                              optimizer=opt)
    for r in range(1, R + 1):
        grp.epoch(r)
        torch.cuda.synchronize()
        loss = sum(w.loss.item() for w in ws)
        ref = run.records[r - 1].loss
        assert abs(loss - ref) <= TOL * abs(ref), (r, loss, ref)
    for w in ws[1:]:    # weights bitwise identical on every partition (A11 invariant)
        assert torch.equal(w.W_flat, ws[0].W_flat)
    for l, wref in enumerate(run.weights):
        assert rel(ws[0].W[l].cpu().numpy(), wref) <= TOL
    assert sum(w.pulls for w in ws) == (R // N) * 2 * M
    assert sum(w.pushes for w in ws) == ((R - 1) // N + 1) * 2 * M
    grp.close()


def test_normalized_push_matches_oracle():
    from paper_2206_00057_b200.engine import TrainConfig, build_workers, LoopbackGroup
    cfg = small_config(num_nodes=500, nnz=5000, d0=12, hidden=(16,), num_classes=4, c_pad=4, seed=5)
    inp = make_inputs(cfg)
    part = make_block_parts(cfg, 2)
    tc = TrainConfig(dims=cfg.dims, num_classes=4, sync_interval=1, lr=0.1, normalize_pushed=True)
    ws = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights, part, 2, tc)
    grp = LoopbackGroup(ws)
    run = oracle.oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                              4, part, 2, sync_interval=1, epochs=3, lr=0.1, normalize_pushed=True)
    for r in (1, 2, 3):
        grp.epoch(r)
    torch.cuda.synchronize()
    loss = sum(w.loss.item() for w in ws)
    assert abs(loss - run.records[-1].loss) <= TOL * abs(run.records[-1].loss)
    grp.close()


@pytest.mark.parametrize("d_in,d_out,order", [(100, 256, 1), (256, 48, 2)])
def test_layer_parity_large_k(d_in, d_out, order):
    """Products-shaped partition with ~0.5M rows: the weight gradient reduces over K = rows,
    exercising the split-K tensor-core path and its chunked TMEM flushes."""
    Dm = D()
    cfg = scaled(get_config("products"), 0.2)
    ip, ix = make_graph(cfg)
    M = 2
    part = make_block_parts(cfg, M)
    p, _ = gpu_partition(ip, ix, part, M, 0)
    op = oracle.oracle_partition(ip, ix, part, M, 0)
    g = torch.Generator().manual_seed(5)
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
    assert rel(H.cpu().numpy(), ref["H"]) <= TOL
    b = layer_backward(op, xl.numpy(), xh.numpy(), w.numpy(), gout.numpy(),
                       H.cpu().numpy() > 0, True)
    e = rel(GW.cpu().numpy(), b["G_W"])
    print("large-K G_W rel err", e)
    assert e <= TOL
    assert rel(Gin.cpu().numpy(), b["G_in"]) <= TOL
    p.close()


def _sample_rows(n, rng, deg):
    top = np.argsort(deg)[-50:]                       # hubs (longest rows)
    return np.unique(np.concatenate([rng.choice(n, 1500, replace=False), top, [0, n - 1]]))


def _rows_product(P, rows, X):
    """(P X)[rows] in fp64 touching only the needed source rows (oracle's P, any X)."""
    Pr = P[rows]
    cols = np.unique(Pr.indices)
    sub = np.asarray(X[cols], dtype=np.float64)
    import scipy.sparse as sp
    Pc = sp.csr_matrix((Pr.data, np.searchsorted(cols, Pr.indices), Pr.indptr),
                       shape=(len(rows), len(cols)))
    return Pc @ sub


@pytest.mark.slow
@pytest.mark.parametrize("M", [1, 8])
def test_full_size_products_epoch_sampled_rows(M):
    """bench.py's workload (products-shaped, dims 100-256-256-48, Adam) at full size:
    sampled output rows of every layer (lockstep: each layer from the GPU's own input),
    and the full layer-1 weight gradient, vs the oracle on rank 0 of M parts."""
    from paper_2206_00057_b200.engine import TrainConfig, build_workers, LoopbackGroup
    from oracle.gcn import prop_matrix
    cfg = get_config("products")
    inp = make_inputs(cfg)
    part = make_block_parts(cfg, M)
    tc = TrainConfig(dims=cfg.dims, num_classes=cfg.num_classes, sync_interval=cfg.sync_interval,
                     lr=0.01, optimizer="adam", async_push=False)
    ws = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights, part, M,
                       tc)
    grp = LoopbackGroup(ws)
    # epoch 1 up to (not including) AGG, so rank 0's own G_W can be compared
    for w in ws:
        w.forward(1, push=True)
    for w in ws:
        w.loss_and_backward()
    torch.cuda.synchronize()
    w0 = ws[0]
    op = oracle.oracle_partition(inp.indptr, inp.indices, part, M, 0)
    P = prop_matrix(op)
    rng = np.random.default_rng(0)
    rows = _sample_rows(op.n_local, rng, np.diff(op.row_ptr))
    x_ext = np.vstack([inp.x[op.local_ids], inp.x[op.halo_ids]]) if op.n_halo else inp.x[op.local_ids]
    W = [w.astype(np.float64) for w in inp.weights]
    L = len(W)
    H_gpu = {l: w0.H[l].cpu().numpy() for l in range(1, L + 1)}
    for l in range(1, L + 1):
        if l == 1:
            src = x_ext
        else:   # lockstep: GPU layer l-1 output; epoch 1 halo of level l-1 is the cold (zero) store
            src = np.vstack([H_gpu[l - 1], np.zeros((op.n_halo, H_gpu[l - 1].shape[1]), np.float32)])
        Z = _rows_product(P, rows, src) @ W[l - 1]
        ref = np.maximum(Z, 0) if l < L else Z
        e = rel(H_gpu[l][rows], ref)
        print(f"M={M} layer {l} sampled-row rel err {e:.3g}")
        assert e <= TOL
    # full layer-1 weight gradient: G_W1 = (P X_ext)^T D1, D1 = the GPU's masked gradient
    A1 = P @ np.asarray(x_ext, np.float64)
    D1 = w0.G[1].cpu().numpy().astype(np.float64)
    GW1 = A1.T @ D1
    e = rel(w0.GW[0].cpu().numpy(), GW1)
    print(f"M={M} full G_W1 rel err {e:.3g}")
    assert e <= TOL
    grp.close()


@pytest.mark.parametrize("M,pull_mode", [(2, 0), (3, 1)])
def test_fresh_mode_vs_oracle_and_full_graph(M, pull_mode):
    """zero-staleness exchange per level.  The GPU trajectory follows the
    oracle's fresh mode, and the first epoch's loss equals full-graph GCN's."""
    from paper_2206_00057_b200.engine import TrainConfig, build_workers, LoopbackGroup
    from oracle.train import full_prop_matrix, full_graph_forward
    cfg = small_config(num_nodes=900, nnz=9000, d0=16, hidden=(24, 16), num_classes=5, c_pad=8,
                       seed=41 + M, train_frac=0.5)
    inp = make_inputs(cfg)
    part = make_random_parts(cfg.num_nodes, M, 2)
    tc = TrainConfig(dims=cfg.dims, num_classes=cfg.num_classes, lr=0.05, fresh=True,
                     pull_mode=pull_mode)
    ws = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights, part, M, tc)
    grp = LoopbackGroup(ws)
    run = oracle.oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                              cfg.num_classes, part, M, sync_interval=1, epochs=3, lr=0.05,
                              mode="fresh")
    Pf = full_prop_matrix(inp.indptr, inp.indices)
    H, _ = full_graph_forward(Pf, inp.x, [w.astype(np.float64) for w in inp.weights])
    n_train = int(inp.train_mask.sum())
    full_loss, _ = cross_entropy(H[-1], inp.y, inp.train_mask, cfg.num_classes, 1.0 / n_train)
    for r in (1, 2, 3):
        grp.epoch(r)
        torch.cuda.synchronize()
        loss = sum(w.loss.item() for w in ws)
        assert abs(loss - run.records[r - 1].loss) <= TOL * abs(run.records[r - 1].loss)
        if r == 1:
            assert abs(loss - full_loss) <= TOL * abs(full_loss)
    for l, wref in enumerate(run.weights):
        assert rel(ws[0].W[l].cpu().numpy(), wref) <= TOL
    grp.close()


def test_layer1_aggregation_cache_is_exact():
    """A1 = P_m X_ext^(0) aggregated once and reused; the trajectory equals
    the oracle's (which recomputes it every epoch)."""
    from paper_2206_00057_b200.engine import TrainConfig, build_workers, LoopbackGroup
    cfg = small_config(num_nodes=1000, nnz=12000, d0=36, hidden=(24,), num_classes=5, c_pad=8,
                       seed=77, train_frac=0.5)
    inp = make_inputs(cfg)
    part = make_block_parts(cfg, 2)
    tc = TrainConfig(dims=cfg.dims, num_classes=cfg.num_classes, sync_interval=2, lr=0.05,
                     cache_l1=True)     # d0=36 > 24: layer 1 would be transform-first without it
    ws = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights, part, 2, tc)
    grp = LoopbackGroup(ws)
    run = oracle.oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                              cfg.num_classes, part, 2, sync_interval=2, epochs=4, lr=0.05)
    for r in range(1, 5):
        grp.epoch(r)
        torch.cuda.synchronize()
        loss = sum(w.loss.item() for w in ws)
        assert abs(loss - run.records[r - 1].loss) <= TOL * abs(run.records[r - 1].loss)
    for l, wref in enumerate(run.weights):
        assert rel(ws[0].W[l].cpu().numpy(), wref) <= TOL
    grp.close()
