"""world_size-2 (and 3) gloo tests of the multi-process host logic on CPU.

Each rank builds its partition with the oracle (the GPU build is bit-exact with it), then:
  * the exchange plan check agrees across ranks and catches a corrupted plan;
  * a boundary exchange performed with the library's protocol (send rows H[send_idx]
    per peer, receive into halo[recv_off[k] : +recv_count[k]]) over gloo point-to-point
    delivers exactly H_global[halo_ids] -- the no-unpack property the NCCL path relies on;
  * the NCCL unique-id broadcast helper delivers rank 0's ids;
  * the gradient sum over ranks (AGG) equals the oracle's aggregated gradient.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2206_00057_b200.dist import (Schedule, all_gather_bytes, broadcast_ids,
                                        check_exchange_plan, grad_count)
from synth import make_inputs, make_block_parts, make_random_parts, small_config


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, random_parts, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = small_config(num_nodes=200, nnz=1600, d0=8, hidden=(12,), num_classes=3, c_pad=4,
                           seed=17)
        inp = make_inputs(cfg)
        part = (make_random_parts(cfg.num_nodes, world, 3) if random_parts
                else make_block_parts(cfg, world))
        p = oracle.oracle_partition(inp.indptr, inp.indices, part, world, rank)
        # 1) plan check
        S = check_exchange_plan(p.send_count, p.recv_count, world)
        bad_caught = False
        if world > 1:
            corrupt = p.send_count.copy()
            corrupt[(rank + 1) % world] += 1
            try:
                check_exchange_plan(corrupt, p.recv_count, world)
            except RuntimeError:
                bad_caught = True
        # 2) exchange with the library's protocol over gloo send/recv
        rng = np.random.default_rng(123)
        H_global = rng.standard_normal((cfg.num_nodes, 12)).astype(np.float32)
        H_local = H_global[p.local_ids]
        halo = np.zeros((p.n_halo, 12), np.float32)
        reqs = []
        for k in range(world):
            if k == rank:
                continue
            if p.send_count[k]:
                rows = p.send_idx[p.send_off[k]:p.send_off[k] + p.send_count[k]]
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(H_local[rows])), k))
        bufs = {}
        for k in range(world):
            if k != rank and p.recv_count[k]:
                bufs[k] = torch.zeros(int(p.recv_count[k]), 12)
                reqs.append(dist.irecv(bufs[k], k))
        for r in reqs:
            r.wait()
        for k, b in bufs.items():
            halo[p.recv_off[k]:p.recv_off[k] + p.recv_count[k]] = b.numpy()
        exact = halo.tobytes() == H_global[p.halo_ids].tobytes()
        # 3) id broadcast; the peer-transport handle exchange (rank-order blobs of any size,
        #    including an empty blob from a rank whose window failed)
        ids = broadcast_ids(lambda: bytes(range(128)), 2, rank)
        blobs = all_gather_bytes(bytes([rank]) * (64 + rank), world)
        empty = all_gather_bytes(b"" if rank == world - 1 else b"x", world)
        gather_ok = (blobs == [bytes([k]) * (64 + k) for k in range(world)] and
                     empty[-1] == b"" and all(e == b"x" for e in empty[:-1]))
        # 4) AGG: sum of per-part gradients over ranks == oracle aggregated gradient
        run = oracle.oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask,
                                  inp.weights, cfg.num_classes, part, world, sync_interval=1,
                                  epochs=1, record_outputs=True)
        # recompute this rank's own gradient contribution
        from oracle.gcn import cross_entropy, layer_backward
        L = len(inp.weights)
        rec = run.records[0]
        outs = rec.part_out
        n_train = int(inp.train_mask.sum())
        _, g = cross_entropy(outs[(L, rank)]["H"], inp.y[p.local_ids], inp.train_mask[p.local_ids],
                             cfg.num_classes, 1.0 / n_train)
        mine = []
        x_in = {1: (inp.x[p.local_ids], inp.x[p.halo_ids])}
        x_in[2] = (outs[(1, rank)]["H"], np.zeros((p.n_halo, 12)))  # epoch 1: cold halo
        for l in range(L, 0, -1):
            mask = None if l == L else outs[(l, rank)]["Z"] > 0
            b = layer_backward(p, x_in[l][0], x_in[l][1], inp.weights[l - 1], g, mask, l >= 2)
            mine.append(torch.from_numpy(b["G_W"].ravel()))
            g = b["G_in"]
        flat = torch.cat(mine[::-1])
        dist.all_reduce(flat)
        agg = np.concatenate([gw.ravel() for gw in rec.grads])
        agg_ok = np.allclose(flat.numpy(), agg, rtol=1e-12, atol=1e-14)
        q.put((rank, S.tolist(), bad_caught, exact, ids[0] == bytes(range(128)) and gather_ok,
               agg_ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,random_parts", [(2, False), (2, True), (3, True)])
def test_multi_process_host_logic(world, random_parts):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, random_parts, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, S, bad_caught, exact, ids_ok, agg_ok in res:
        assert np.all(np.diag(S) == 0)
        assert bad_caught
        assert exact, f"rank {rank}: exchanged halo rows differ from the owners' rows"
        assert ids_ok and agg_ok


def test_schedule_guards():
    s = Schedule(10)
    assert [r for r in range(1, 41) if s.pull(r)] == [10, 20, 30, 40]
    assert [r for r in range(1, 41) if s.push(r)] == [1, 11, 21, 31]
    assert s.counts(40, 2) == ((40 // 10) * 2, ((40 - 1) // 10 + 1) * 2)
    with pytest.raises(ValueError):
        Schedule(0)


def test_grad_count_matches_the_flat_weight_layout():
    """The peer window's AGG slot size: sum of d_l * d_{l+1} (the flat W / G buffers)."""
    assert grad_count((100, 256, 256, 48)) == 100 * 256 + 256 * 256 + 256 * 48 == 103424
    assert grad_count((604, 256, 48)) == 166912
    assert grad_count((8, 4)) == 32
