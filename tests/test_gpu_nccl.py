"""The NCCL transport's calls on one GPU (the NCCL path had never run).

NCCL refuses two ranks on one device, and the pool gives one GPU per call, so these
tests run the library's NCCL code through a 1-rank communicator: ncclAllReduce
(AGG, the same call a multi-rank AGG makes) and the grouped ncclSend/ncclRecv of
the boundary exchange as a self transfer, bit-exact; then a full M=1 training
run whose AGG goes through that communicator every epoch, against the oracle."""
import numpy as np
import pytest
import torch

import oracle
from synth import make_inputs, make_block_parts, small_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def test_nccl_one_rank_allreduce_and_grouped_send_recv():
    from paper_2206_00057_b200 import capi as D
    comm = D.digest_comm_init(D.digest_comm_unique_id(), 1, 0)
    try:
        g = torch.randn(100003, device="cuda")
        want = g * 0.5
        D.digest_grad_allreduce(comm, g, 0.5)
        torch.cuda.synchronize()
        assert torch.equal(g, want)
        for n in (1, 4097, 3_000_000):
            send = torch.randn(n, device="cuda")
            recv = torch.full((n,), 7.0, device="cuda")
            D.digest_comm_alltoallv(comm, [send], [recv])
            torch.cuda.synchronize()
            assert torch.equal(recv, send), n
        with pytest.raises(D.DigestError):   # a peer-memory communicator has no NCCL
            pc = D.digest_comm_init_peer(1, 0, 16)
            try:
                D.digest_comm_alltoallv(pc, [send], [recv])
            finally:
                D.digest_comm_destroy(pc)
    finally:
        D.digest_comm_destroy(comm)


def test_training_with_nccl_agg_one_rank():
    from paper_2206_00057_b200 import capi as D
    from paper_2206_00057_b200.engine import TrainConfig, build_workers
    cfg = small_config(num_nodes=800, nnz=8000, d0=16, hidden=(24,), num_classes=5, c_pad=8,
                       seed=55, train_frac=0.5)
    inp = make_inputs(cfg)
    part = make_block_parts(cfg, 1)
    comm = D.digest_comm_init(D.digest_comm_unique_id(), 1, 0)
    tc = TrainConfig(dims=cfg.dims, num_classes=cfg.num_classes, lr=0.05, optimizer="adam",
                     transport="nccl")
    (w,) = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights, part,
                         1, tc, ranks=[0], comm_grad=comm, comm_halo=comm)
    run = oracle.oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                              cfg.num_classes, part, 1, sync_interval=1, epochs=4, lr=0.05,
                              optimizer="adam")
    for r in range(1, 5):
        w.epoch(r)
        torch.cuda.synchronize()
        ref = run.records[r - 1].loss
        assert abs(w.loss.item() - ref) <= 1e-4 * abs(ref)
    for l, wref in enumerate(run.weights):
        got = w.W[l].double().cpu().numpy()
        assert np.abs(got - wref).max() / np.abs(wref).max() <= 1e-4
    w.close()
    D.digest_comm_destroy(comm)
