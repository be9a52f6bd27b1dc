"""Multi-process plumbing around libdigest.so (host logic only).

* `Schedule`        -- Alg. 1's pull/push guards, 1-based epochs.
* `broadcast_ids`   -- carry rank 0's NCCL unique ids to every rank over the caller's
                       torch.distributed group (any backend; gloo in the CPU tests).
* `check_exchange_plan` -- before the first boundary exchange, verify on every rank that
                       what rank m sends to k equals what k expects from m (otherwise
                       the grouped ncclSend/ncclRecv would hang).
* `all_gather_bytes`, `connect_peer_comm`, `connect_peer_store` -- bootstrap of the
                       peer-memory transport: every rank's CUDA IPC handles travel over
                       the caller's process group, the library maps them.
"""
from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Schedule:
    """Alg. 1 guards: PULL if r % N == 0, PUSH if (r-1) % N == 0, levels 1..L-1."""
    sync_interval: int

    def __post_init__(self):
        if self.sync_interval < 1:
            raise ValueError("sync interval must be >= 1")

    def pull(self, r: int) -> bool:
        return r % self.sync_interval == 0

    def push(self, r: int) -> bool:
        return (r - 1) % self.sync_interval == 0

    def counts(self, epochs: int, levels: int):
        """(pulls, pushes) per worker over epochs 1..R for `levels` stored levels."""
        pulls = sum(self.pull(r) for r in range(1, epochs + 1)) * levels
        pushes = sum(self.push(r) for r in range(1, epochs + 1)) * levels
        return pulls, pushes


def broadcast_ids(make_id, count: int, rank: int, device="cpu"):
    """Rank 0 creates `count` 128-byte ids with make_id(); all ranks receive them."""
    out = []
    for _ in range(count):
        t = torch.zeros(128, dtype=torch.uint8, device=device)
        if rank == 0:
            t = torch.tensor(list(make_id()), dtype=torch.uint8, device=device)
        dist.broadcast(t, 0)
        out.append(bytes(t.cpu().tolist()))
    return out


def check_exchange_plan(send_count, recv_count, world: int, device="cpu"):
    """All-gather every rank's per-peer send/recv counts and check send[m][k] == recv[k][m].

    Returns the full (world x world) send matrix; raises RuntimeError on a mismatch."""
    s = torch.tensor([int(x) for x in send_count[:world]], dtype=torch.int64, device=device)
    r = torch.tensor([int(x) for x in recv_count[:world]], dtype=torch.int64, device=device)
    S = [torch.zeros_like(s) for _ in range(world)]
    R = [torch.zeros_like(r) for _ in range(world)]
    dist.all_gather(S, s)
    dist.all_gather(R, r)
    S = torch.stack(S).cpu()
    R = torch.stack(R).cpu()
    if not torch.equal(S, R.T):
        bad = (S != R.T).nonzero().tolist()
        raise RuntimeError(f"boundary exchange plan mismatch at (sender, receiver) {bad[:8]}")
    if torch.diagonal(S).any():
        raise RuntimeError("a rank plans to send boundary rows to itself")
    return S


def all_gather_bytes(blob: bytes, world: int):
    """Every rank's `blob`, rank order (any backend)."""
    out = [None] * world
    dist.all_gather_object(out, blob)
    return out


def grad_count(dims):
    """Floats in the flat weight/gradient buffer of a GCN with widths `dims`."""
    return sum(int(dims[l]) * int(dims[l + 1]) for l in range(len(dims) - 1))


def connect_peer_comm(world: int, rank: int, max_grad_count: int):
    """Create this rank's peer-memory window and map every peer's (collective).

    Every rank takes part in the handle exchange even if its own window failed, so a
    failure raises on the failing rank (and on the ranks that see its empty handle)
    instead of leaving the others blocked in the collective."""
    from . import capi as D
    comm, blob, err = None, b"", None
    try:
        comm = D.digest_comm_init_peer(world, rank, max_grad_count)
        blob = D.digest_comm_export(comm)
    except Exception as e:   # noqa: BLE001
        err = e
    blobs = all_gather_bytes(blob, world)
    if err is None and any(len(b) != D.IPC_HANDLE_BYTES for b in blobs):
        err = RuntimeError("a peer could not export its window")
    if err is None:
        try:
            D.digest_comm_connect(comm, blobs)
        except Exception as e:   # noqa: BLE001
            err = e
    if err is not None:
        if comm is not None:
            D.digest_comm_destroy(comm)
        raise err
    return comm


def connect_peer_store(store, world: int):
    """Map every rank's stale-store buffers into this rank's store (collective)."""
    from . import capi as D
    D.digest_store_connect(store, all_gather_bytes(D.digest_store_export(store), world))
