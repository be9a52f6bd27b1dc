"""Worker body of the multi-process peer-transport tests (tests/test_gpu_peer.py).

Each spawned process is one DIGEST rank (Alg. 1) with its own CUDA context;
all ranks share cuda:0 here (the pool gives one GPU per call), which exercises the same
CUDA-IPC mappings, flag protocol and kernels as one process per GPU.  The host process
group is gloo on 127.0.0.1 (handle exchange only).  Rank 0 writes every rank's
per-epoch loss and final weights to `out_path` (npz)."""
import os

import numpy as np
import torch
import torch.distributed as dist


def run_rank(rank, world, port, spec, out_path):
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    torch.cuda.set_device(0)
    from paper_2206_00057_b200 import capi as D
    from paper_2206_00057_b200.dist import connect_peer_comm, grad_count
    from paper_2206_00057_b200.engine import TrainConfig, build_workers
    from synth import small_config, make_inputs, make_block_parts, make_random_parts

    from synth import get_config
    cfg = get_config(spec["config"]) if "config" in spec else small_config(**spec["graph"])
    inp = make_inputs(cfg)
    part = (make_block_parts(cfg, world) if spec.get("parts_seed") is None
            else make_random_parts(cfg.num_nodes, world, spec["parts_seed"]))
    comm = connect_peer_comm(world, rank, grad_count(cfg.dims))
    tc = TrainConfig(dims=cfg.dims, num_classes=cfg.num_classes, transport="peer",
                     **spec["train"])
    (w,) = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                         part, world, tc, ranks=[rank], comm_grad=comm, comm_halo=comm)
    n0 = D.digest_launch_count()
    losses = []
    for r in range(1, spec["epochs"] + 1):
        w.epoch(r)
        torch.cuda.synchronize()
        losses.append(float(w.loss.item()))
    launches = D.digest_launch_count() - n0
    res = {"loss": np.array(losses), "W": w.W_flat.cpu().numpy(), "pulls": w.pulls,
           "pushes": w.pushes, "launches": launches}
    allres = [None] * world
    dist.all_gather_object(allres, res)
    dist.barrier()          # nobody unmaps a window a peer may still read
    w.close()
    D.digest_comm_destroy(comm)
    if rank == 0:
        np.savez(out_path, loss=np.stack([r["loss"] for r in allres]),
                 W=np.stack([r["W"] for r in allres]),
                 pulls=np.array([r["pulls"] for r in allres]),
                 pushes=np.array([r["pushes"] for r in allres]),
                 launches=np.array([r["launches"] for r in allres]))
    dist.destroy_process_group()


def run_rank_async(rank, world, port, spec, out_path):
    """DIGEST-A rank: local epochs at its own pace against the PS in rank
    0's window; the straggler (spec['straggler']) sleeps spec['delay_ms'] per epoch."""
    import time
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    torch.cuda.set_device(0)
    from paper_2206_00057_b200 import capi as D
    from paper_2206_00057_b200.dist import connect_peer_comm, grad_count
    from paper_2206_00057_b200.engine import TrainConfig, build_workers, run_digest_a_peer
    from synth import small_config, make_inputs, make_block_parts

    cfg = small_config(**spec["graph"])
    inp = make_inputs(cfg)
    part = make_block_parts(cfg, world)
    comm = connect_peer_comm(world, rank, grad_count(cfg.dims))
    tc = TrainConfig(dims=cfg.dims, num_classes=cfg.num_classes, transport="peer",
                     async_store=True, pull_mode=D.PULL_SNAPSHOT, **spec["train"])
    (w,) = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                         part, world, tc, ranks=[rank], comm_grad=comm, comm_halo=comm,
                         loss_weighting="local")
    if rank == 0:
        D.digest_ps_init_peer(comm, w.W_flat)
    torch.cuda.synchronize()
    dist.barrier()
    R = spec["epochs"]
    delays = None
    if spec.get("straggler") == rank:
        delays = [int(spec["delay_ms"] * 1e6)] * R
    t0 = time.perf_counter()
    losses = torch.zeros(R, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    for r in range(1, R + 1):   # run_digest_a_peer one epoch at a time, keeping the losses
        D.digest_ps_download_peer(comm, w.W_flat, stream)
        if delays:
            D.digest_delay(delays[r - 1], stream)
        w.local_epoch(r, stream)
        losses[r - 1].copy_(w.loss[0])
        D.digest_ps_upload_peer(comm, w.W_flat, 1.0 / world, stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    dist.barrier()                      # every upload has landed
    res = {"loss": losses.cpu().numpy(), "wall": wall}
    if rank == 0:
        Wg = torch.empty_like(w.W_flat)
        D.digest_ps_download_peer(comm, Wg)
        torch.cuda.synchronize()
        res["W_global"] = Wg.cpu().numpy()
        res["updates"] = D.digest_ps_updates_peer(comm)
    allres = [None] * world
    dist.all_gather_object(allres, res)
    dist.barrier()
    w.close()
    D.digest_comm_destroy(comm)
    if rank == 0:
        np.savez(out_path, loss=np.stack([r["loss"] for r in allres]),
                 wall=np.array([r["wall"] for r in allres]), W_global=allres[0]["W_global"],
                 updates=allres[0]["updates"])
    dist.destroy_process_group()
