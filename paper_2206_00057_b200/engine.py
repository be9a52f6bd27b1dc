"""The DIGEST epoch driver (host logic only; every step runs in libdigest.so).

Implements Alg. 1 for one partition per worker:
  * PULL  at the start of epoch r if r % N == 0, levels l in [1, L-1];
  * layer l forward on [H^(l-1)_local ; front buffer of level l-1] (Eq. 5);
  * PUSH  right after level l is computed if (r-1) % N == 0 and l < L;
  * loss (Eq. 3), backward (Eq. 6), AGG as a gradient allreduce, update.
Reading A7: all pulls of an epoch happen before any push of that epoch, so pulls
only ever expose versions < r.  Torch provides memory, streams and process groups.

Two deployments:
  * DigestWorker with an NCCL or peer-memory communicator: one process per GPU
    (torchrun), or several processes sharing one GPU (peer transport, tests);
  * LoopbackGroup: M partitions in one process on one GPU, stores linked so a push
    writes the peers' back buffers directly (used by the single-GPU tests).
"""
import contextlib
from dataclasses import dataclass

import numpy as np
import torch

from . import capi as D
from .dist import Schedule


def _nvtx(name):
    """NVTX range around a phase of the epoch (visible to nsys/ncu timelines; a no-op
    without a profiler attached)."""
    if torch.cuda.is_available():
        return torch.cuda.nvtx.range(name)
    return contextlib.nullcontext()


@dataclass
class TrainConfig:
    dims: tuple                 # (d_0, ..., d_L), padded (multiples of 4)
    num_classes: int
    sync_interval: int = 1
    lr: float = 0.01
    optimizer: str = "sgd"      # 'sgd' (parity) or 'adam' (the paper's)
    order: int = D.ORDER_AUTO
    async_push: bool = False
    normalize_pushed: bool = False
    pull_mode: int = D.PULL_FLIP
    fresh: bool = False         # zero-staleness mode (the oracle's mode='fresh')
    cache_l1: bool = False      # aggregate the static layer-1 inputs once
    # SURVEY f2, the gradient returned to the owners of a part's halo rows:
    #   '' / False / 'none'   halo inputs are constants (Eq. 6; default)
    #   'prev_epoch'          the paper's DIGEST backward: P_out^T D~^(t-1) W~^(t)T
    #   'same_epoch' / True   the exact variant: P_out^T D~^(t) W~^(t)T in the same iteration
    halo_grad: object = ""
    transport: str = "nccl"     # multi-process exchange: 'nccl' or 'peer' (CUDA IPC windows)
    async_store: bool = False   # DIGEST-A on the peer transport: NOWAIT pushes, SNAPSHOT pulls
    store_bf16: bool = False    # bf16 stale store / transfers
    device_step: bool = False   # Adam step count on the device (CUDA-graph capturable epochs)
    fused_agg: bool = True      # peer transport: weight gradients written straight into the
                                # AGG window slot, one-kernel allreduce
    loss_rows: bool = True      # last layer's backward products over the training-row columns
                                # only (G_logits is zero elsewhere; exact)

    def __post_init__(self):
        hg = self.halo_grad
        hg = "same_epoch" if hg is True else ("" if hg in (False, None, "none") else hg)
        if hg not in ("", "same_epoch", "prev_epoch"):
            raise ValueError(f"halo_grad {self.halo_grad!r}")
        self.halo_grad = hg


class Partition:
    """A digest_part handle plus its info (host copy)."""

    def __init__(self, indptr, indices, part_of, num_parts, rank, stream=None):
        n = indptr.numel() - 1
        self.handle = D.digest_partition(n, indices.numel(), indptr, indices, part_of, num_parts,
                                         rank, 0, stream)
        self.info = D.digest_part_get_info(self.handle)
        self.num_parts, self.rank = num_parts, rank
        self.n_local, self.n_halo = self.info.n_local, self.info.n_halo

    def export(self, device="cuda"):
        i = self.info
        t = lambda n, dt: torch.empty(max(n, 0), dtype=dt, device=device)
        out = dict(local_ids=t(i.n_local, torch.int32), halo_ids=t(i.n_halo, torch.int32),
                   row_ptr=t(i.n_local + 1, torch.int64), col=t(i.nnz, torch.int32),
                   val=t(i.nnz, torch.float32), send_idx=t(i.n_send, torch.int32),
                   rh_ptr=t(i.n_halo + 1, torch.int64), rh_col=t(i.rh_nnz, torch.int32),
                   rh_val=t(i.rh_nnz, torch.float32))
        D.digest_part_export(self.handle, **out)
        M = self.num_parts
        out.update(send_count=np.array(i.send_count[:M]), send_off=np.array(i.send_off[:M]),
                   recv_count=np.array(i.recv_count[:M]), recv_off=np.array(i.recv_off[:M]))
        return out

    def close(self):
        if self.handle:
            D.digest_part_destroy(self.handle)
            self.handle = None


class DigestWorker:
    """Training state of one partition on the current CUDA device."""

    def __init__(self, part: Partition, cfg: TrainConfig, x_local, x_halo, labels, train_mask,
                 weights, w_loss, comm_grad=None, comm_halo=None):
        self.part, self.cfg = part, cfg
        self.L = len(cfg.dims) - 1
        dims = cfg.dims
        dev = x_local.device
        n, h = part.n_local, part.n_halo
        self.x_local, self.x_halo = x_local, (x_halo if h > 0 else None)
        self.labels, self.train_mask = labels, train_mask
        if cfg.loss_rows:   # the loss-row CSRs (the mask of the rows G_logits can be nonzero on)
            D.digest_part_set_loss_mask(part.handle, train_mask)
        self.w_loss = float(w_loss)
        self.comm_grad, self.comm_halo = comm_grad, comm_halo
        # weights: one flat buffer (AGG and the update are single launches)
        sizes = [dims[l] * dims[l + 1] for l in range(self.L)]
        self.W_flat = torch.empty(sum(sizes), dtype=torch.float32, device=dev)
        self.G_flat = torch.zeros_like(self.W_flat)
        self.W, self.GW, self.gw_off, off = [], [], [], 0
        for l, s in enumerate(sizes):
            self.W.append(self.W_flat[off:off + s].view(dims[l], dims[l + 1]))
            self.GW.append(self.G_flat[off:off + s].view(dims[l], dims[l + 1]))
            self.gw_off.append(off)
            off += s
        # fused AGG (peer transport, M > 1): this epoch's G_W outputs live in the window slot
        # (not in DIGEST-A, whose local step reads G_flat without an AGG)
        self.fused_agg = bool(cfg.fused_agg and cfg.transport == "peer" and comm_grad is not None
                              and part.num_parts > 1 and not cfg.async_store)
        self._gw_out = None
        for w, src in zip(self.W, weights):
            w.copy_(torch.as_tensor(src, dtype=torch.float32))
        self.adam_m = self.adam_v = None
        if cfg.optimizer == "adam":
            self.adam_m = torch.zeros_like(self.W_flat)
            self.adam_v = torch.zeros_like(self.W_flat)
        self.step_count = 0
        self.step_dev = torch.zeros(1, dtype=torch.int64, device=dev) if cfg.device_step else None
        # activations, saved state, gradients
        self.H = [None] + [torch.empty(n, dims[l], device=dev) for l in range(1, self.L + 1)]
        self.saved, scratch = [None], 0
        self._a1_ready = False
        for l in range(1, self.L + 1):
            sv, sc = D.digest_layer_workspace(part.handle, dims[l - 1], dims[l], self.layer_order(l))
            self.saved.append(torch.empty(max(sv, 256), dtype=torch.uint8, device=dev))
            scratch = max(scratch, sc)
        self.scratch = torch.empty(max(scratch, 256), dtype=torch.uint8, device=dev)
        # 1-bit ReLU masks the forward writes into saved
        self.mask_bits = [None] + [
            D.digest_layer_mask(part.handle, dims[l - 1], dims[l], self.layer_order(l),
                                self.saved[l]) for l in range(1, self.L + 1)]
        self.G = [None] + [torch.empty(n, dims[l], device=dev) for l in range(1, self.L + 1)]
        self.xent_scratch = torch.empty(max(D.digest_xent_workspace(n), 8), dtype=torch.uint8,
                                        device=dev)
        self.loss = torch.zeros(1, dtype=torch.float64, device=dev)
        # stale store: levels 1..L-1 (never L)
        self.store = D.digest_store_create(part.handle, comm_halo, list(dims[1:self.L]),
                                           D.STORE_BF16 if cfg.store_bf16 else 0)
        if cfg.transport == "peer" and comm_halo is not None and part.num_parts > 1:
            from .dist import connect_peer_store
            connect_peer_store(self.store, part.num_parts)   # collective over the process group
        self.pulls = self.pushes = 0
        # halo_grad='prev_epoch': S^(t-1) = P_out^T D~^(t-1) per layer l >= 2 (zero at t = 1)
        self.s_prev = {}
        if cfg.halo_grad == "prev_epoch" and h > 0:
            self.s_prev = {l: torch.zeros(h, dims[l], device=dev) for l in range(2, self.L + 1)}

    # --------------------------------------------------------------- schedule pieces
    def halo_input(self, l):
        """(pointer, ld) of the halo rows feeding layer l."""
        if l == 1:
            return (self.x_halo, self.cfg.dims[0]) if self.x_halo is not None else (None, 0)
        p, ld, _ = D.digest_store_front(self.store, l - 1)
        return (p if self.part.n_halo > 0 else None), ld

    def pull(self, epoch, stream=None):
        for l in range(1, self.L):
            D.digest_pull(self.store, l, epoch, self.cfg.pull_mode, stream)
            self.pulls += 1

    def layer_order(self, l):
        # with the layer-1 cache the first layer is always aggregate-first: A1 = P_m X_ext^(0)
        # depends only on static inputs, so it is aggregated once and reused every epoch
        return D.ORDER_AGG_FIRST if (l == 1 and self.cfg.cache_l1) else self.cfg.order

    def forward_layer(self, l, stream=None):
        dims, cfg = self.cfg.dims, self.cfg
        xl = self.x_local if l == 1 else self.H[l - 1]
        xh, ldh = self.halo_input(l)
        act = D.ACT_RELU if l < self.L else D.ACT_NONE
        flags = 0
        if l == 1 and cfg.cache_l1:
            flags = D.FWD_REUSE_SAVED if self._a1_ready else 0
            self._a1_ready = True
        D.digest_layer_fwd(self.part.handle, xl, xh, ldh, self.W[l - 1], dims[l - 1], dims[l],
                           act, self.layer_order(l), self.H[l], self.saved[l], self.scratch,
                           stream, flags=flags)

    def push(self, l, epoch, stream=None):
        cfg = self.cfg
        flags = ((D.PUSH_ASYNC if cfg.async_push else 0) | (D.PUSH_L2NORM if cfg.normalize_pushed else 0)
                 | (D.PUSH_NOWAIT if cfg.async_store else 0))
        D.digest_push_boundary(self.store, l, self.H[l], epoch, flags, stream)
        self.pushes += 1

    def forward(self, epoch, push: bool, stream=None):
        for l in range(1, self.L + 1):
            self.forward_layer(l, stream)
            if push and l < self.L:
                self.push(l, epoch, stream)

    def forward_fresh(self, epoch, stream=None):
        """Zero-staleness variant (the propagation-style exchange the paper
        compares against): after each level, push it and pull it back at
        once (epoch + 1 makes this epoch's push visible), so layer l+1 reads the
        current halo values.  Collective per level on every rank."""
        for l in range(1, self.L + 1):
            self.forward_layer(l, stream)
            if l < self.L:
                self.push(l, epoch, stream)
                D.digest_pull(self.store, l, epoch + 1, self.cfg.pull_mode, stream)
                self.pulls += 1

    def compute_loss(self, stream=None):
        cfg = self.cfg
        D.digest_xent(self.H[self.L], cfg.num_classes, self.labels, self.train_mask, self.w_loss,
                      self.G[self.L], self.loss, self.xent_scratch, stream)

    def backward_layer(self, l, stream=None):
        dims = self.cfg.dims
        xl = self.x_local if l == 1 else self.H[l - 1]
        xh, ldh = self.halo_input(l)
        act = D.ACT_RELU if l < self.L else D.ACT_NONE
        gh, ldgh, hflags = None, 0, 0
        if self.cfg.halo_grad and l >= 2 and self.part.n_halo > 0:
            gh, ldgh = D.digest_store_grad_buffer(self.store, l - 1)
            if self.cfg.halo_grad == "prev_epoch":
                # the rows returned now are S^(t-1) W^(t)T; this backward then
                # overwrites S with S^(t) = P_out^T D~^(t) (stream order: read, then write)
                S = self.s_prev[l]
                D.digest_gemm(S, self.W[l - 1], gh, bt=True, M=self.part.n_halo, ldc=ldgh,
                              stream=stream)
                gh, ldgh, hflags = S, 0, D.BWD_HALO_SAVE_S
        # G_in of layer l is produced already multiplied by 1[H^(l-1) > 0] (the 1-bit
        # mask of layer l-1), i.e. it is D^(l-1); layer l-1 then skips its own masking
        # pass (DIGEST_BWD_G_IS_D).
        gw = self.GW[l - 1] if self._gw_out is None else self._gw_out[l - 1]
        D.digest_layer_bwd(self.part.handle, xl, xh, ldh, self.W[l - 1], dims[l - 1], dims[l],
                           act, self.layer_order(l), self.saved[l], None, self.G[l],
                           gw, self.G[l - 1] if l >= 2 else None, self.scratch,
                           stream, flags=(D.BWD_G_IS_D if l < self.L else
                                          (D.BWD_LOSS_ROWS if self.cfg.loss_rows else 0)) | hflags,
                           gin_mask=self.mask_bits[l - 1] if l >= 2 else None, G_halo=gh,
                           ld_gh=ldgh)

    def return_halo_grad(self, l, stream=None):
        """Add the peers' G_halo rows for my nodes into D^(l-1)."""
        D.digest_return_halo_grad(self.store, l - 1, self.G[l - 1], self.H[l - 1], stream)

    def loss_and_backward(self, stream=None):
        if self.fused_agg:   # G_W of every layer -> the slot the next AGG call reduces
            slot = D.digest_grad_slot(self.comm_grad)
            self._gw_out = [slot + 4 * o for o in self.gw_off]
        self.compute_loss(stream)
        for l in range(self.L, 0, -1):
            self.backward_layer(l, stream)
            if self.cfg.halo_grad and l >= 2:
                self.return_halo_grad(l, stream)   # collective (NCCL) per level

    def allreduce(self, stream=None):
        if self._gw_out is not None:   # signal + rank-order sum, one kernel
            D.digest_grad_allreduce_ex(self.comm_grad, self.G_flat, 1.0, D.AR_IN_SLOT, stream)
            self._gw_out = None
        else:
            D.digest_grad_allreduce(self.comm_grad, self.G_flat, 1.0, stream)

    def update(self, stream=None):
        self.step_count += 1
        if self.cfg.optimizer == "sgd":
            D.digest_sgd_step(self.W_flat, self.G_flat, self.cfg.lr, stream)
        elif self.step_dev is not None:
            D.digest_adam_step_dev(self.W_flat, self.G_flat, self.adam_m, self.adam_v, self.cfg.lr,
                                   0.9, 0.999, 1e-8, self.step_dev, stream)
        else:
            D.digest_adam_step(self.W_flat, self.G_flat, self.adam_m, self.adam_v, self.cfg.lr,
                               0.9, 0.999, 1e-8, self.step_count, stream)

    def epoch(self, r, stream=None):
        """One full DIGEST epoch r (1-based) for a single worker (NCCL deployment)."""
        with _nvtx(f"epoch {r}"):
            if self.cfg.fresh:
                with _nvtx("forward (fresh)"):
                    self.forward_fresh(r, stream)
            else:
                sched = Schedule(self.cfg.sync_interval)
                if sched.pull(r):
                    with _nvtx("pull"):
                        self.pull(r, stream)
                with _nvtx("forward + push" if sched.push(r) else "forward"):
                    self.forward(r, sched.push(r), stream)
            with _nvtx("loss + backward"):
                self.loss_and_backward(stream)
            with _nvtx("AGG"):
                self.allreduce(stream)
            with _nvtx("update"):
                self.update(stream)

    def local_epoch(self, r, stream=None):
        """One DIGEST-A local epoch r (no AGG inside; the PS mixes afterwards):
        Alg. 1's pull/push guards on this worker's own counter, forward, loss, backward
        and the local optimizer step."""
        sched = Schedule(self.cfg.sync_interval)
        if sched.pull(r):
            self.pull(r, stream)
        self.forward(r, sched.push(r), stream)
        self.loss_and_backward(stream)
        self.update(stream)

    def close(self):
        if self.store:
            D.digest_store_destroy(self.store)
            self.store = None


class AsyncLoopbackGroup:
    """DIGEST-A for M partitions in one process.

    Asynchrony is an input: `event(m)` runs worker m's next local epoch -- download
    W_global, local epoch (pull/push keyed on its own counter), upload (PS mixing,
    digest_ps_mix) -- so a seeded event list (synth.async_sched: discrete-event clock
    with stragglers) fixes the interleaving and the run is comparable with the oracle.
    The stale store runs in COPY mode: a part's back buffer always holds every owner's
    latest pushed rows and a pull copies them (a flip could re-expose an owner's older
    rows when owners push at different rates)."""

    def __init__(self, workers, alpha=None):
        self.workers = workers
        M = len(workers)
        self.alpha = 1.0 / M if alpha is None else float(alpha)
        for w in workers:
            if w.cfg.pull_mode != D.PULL_COPY:
                raise ValueError("DIGEST-A needs pull_mode=PULL_COPY")
        if M > 1:
            D.digest_store_link([w.store for w in workers])
        self.W_global = workers[0].W_flat.clone()
        self.r = [0] * M
        self.ps_updates = 0

    def event(self, m, stream=None):
        w = self.workers[m]
        self.r[m] += 1
        D.digest_ps_download(self.W_global, w.W_flat, stream)
        w.local_epoch(self.r[m], stream)
        D.digest_ps_mix(self.W_global, w.W_flat, self.alpha, stream)
        self.ps_updates += 1

    def close(self):
        for w in self.workers:
            w.close()


def run_digest_a_peer(w, comm, epochs, alpha, delays_ns=None, stream=None):
    """DIGEST-A for one rank of a multi-process run on the peer transport:
    `epochs` local epochs of download (locked read of W_global in rank 0's window),
    optional straggler delay (digest_delay), local epoch, upload (locked mixing).
    No barrier and no AGG: ranks proceed at their own pace."""
    if not (w.cfg.async_store and w.cfg.pull_mode == D.PULL_SNAPSHOT):
        raise ValueError("DIGEST-A on the peer transport needs async_store and PULL_SNAPSHOT")
    for r in range(1, epochs + 1):
        D.digest_ps_download_peer(comm, w.W_flat, stream)
        if delays_ns is not None and delays_ns[r - 1] > 0:
            D.digest_delay(delays_ns[r - 1], stream)
        w.local_epoch(r, stream)
        D.digest_ps_upload_peer(comm, w.W_flat, alpha, stream)


class LoopbackGroup:
    """M partitions of one graph trained in one process (single GPU)."""

    def __init__(self, workers):
        self.workers = workers
        if len(workers) > 1:
            D.digest_store_link([w.store for w in workers])

    def epoch(self, r, stream=None):
        if self.workers[0].cfg.fresh:
            # zero staleness: layer-major, every level exchanged before the next layer
            for l in range(1, self.workers[0].L + 1):
                for w in self.workers:
                    w.forward_layer(l, stream)
                if l < self.workers[0].L:
                    for w in self.workers:
                        w.push(l, r, stream)
                    for w in self.workers:
                        D.digest_pull(w.store, l, r + 1, w.cfg.pull_mode, stream)
                        w.pulls += 1
        else:
            sched = Schedule(self.workers[0].cfg.sync_interval)
            if sched.pull(r):      # all pulls of epoch r precede any push of epoch r (A7)
                for w in self.workers:
                    w.pull(r, stream)
            for w in self.workers:
                w.forward(r, sched.push(r), stream)
        if self.workers[0].cfg.halo_grad:
            # layer-major: every part's G_halo of layer l exists before any owner adds it
            for w in self.workers:
                w.compute_loss(stream)
            for l in range(self.workers[0].L, 0, -1):
                for w in self.workers:
                    w.backward_layer(l, stream)
                if l >= 2:
                    for w in self.workers:
                        w.return_halo_grad(l, stream)
        else:
            for w in self.workers:
                w.loss_and_backward(stream)
        if len(self.workers) > 1:
            D.digest_grad_allreduce_local([w.G_flat for w in self.workers], 1.0, stream)
        for w in self.workers:
            w.update(stream)

    def close(self):
        for w in self.workers:
            w.close()


def build_workers(indptr, indices, x, y, train_mask, weights, part_of, num_parts, cfg: TrainConfig,
                  ranks=None, comm_grad=None, comm_halo=None, device="cuda",
                  loss_weighting="count"):
    """Partition on the device and set up workers for `ranks` (default: all parts).

    loss_weighting: 'count' = 1/#train over the whole graph (A12, the synchronous AGG of
    gradient sums); 'local' = 1/#train of the part (DIGEST-A's local objective, Eq. 3).

    indptr/indices/part_of/x/y/train_mask: host numpy arrays (the synthetic inputs).
    The layer-1 inputs X[V_m] and X[H_m] are gathered on the device by digest_gather_rows."""
    ranks = list(range(num_parts)) if ranks is None else ranks
    d_ip = torch.as_tensor(indptr, dtype=torch.int64).to(device)
    d_ix = torch.as_tensor(indices, dtype=torch.int32).to(device)
    d_po = torch.as_tensor(part_of, dtype=torch.int32).to(device)
    d_x = torch.as_tensor(x, dtype=torch.float32).to(device)
    d_y = torch.as_tensor(y, dtype=torch.int32).to(device)
    d_t = torch.as_tensor(train_mask, dtype=torch.uint8).to(device)
    tmask = np.asarray(train_mask).astype(bool)
    w_loss = 1.0 / max(1, int(tmask.sum()))   # count weighting (A12)
    workers = []
    for r in ranks:
        p = Partition(d_ip, d_ix, d_po, num_parts, r)
        ids = torch.empty(p.n_local, dtype=torch.int32, device=device)
        hids = torch.empty(max(p.n_halo, 0), dtype=torch.int32, device=device)
        D.digest_part_export(p.handle, local_ids=ids, halo_ids=hids)
        xl = torch.empty(p.n_local, cfg.dims[0], device=device)
        D.digest_gather_rows(d_x, ids, xl)
        xh = torch.empty(max(p.n_halo, 1), cfg.dims[0], device=device)
        if p.n_halo:
            D.digest_gather_rows(d_x, hids, xh)
        lab = d_y[ids.long()].contiguous()
        msk = d_t[ids.long()].contiguous()
        wl = w_loss
        if loss_weighting == "local":
            wl = 1.0 / max(1, int(tmask[np.asarray(part_of) == r].sum()))
        workers.append(DigestWorker(p, cfg, xl, xh, lab, msk, weights, wl,
                                    comm_grad, comm_halo))
    return workers
