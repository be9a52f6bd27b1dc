"""Thin ctypes binding of include/digest.h (argument marshalling only).

Every function here has the C name of the call it wraps, converts torch tensors to
device pointers, checks the status and raises DigestError with the library's
message.  All computation happens in libdigest.so; there is no Python or CPU
fallback: importing this module fails loudly if the library is missing.
"""
import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdigest.so")

DIGEST_MAX_PARTS = 64
ACT_NONE, ACT_RELU = 0, 1
ORDER_AUTO, ORDER_AGG_FIRST, ORDER_XFORM_FIRST = 0, 1, 2
PUSH_ASYNC, PUSH_L2NORM, PUSH_NOWAIT = 1, 2, 4
PULL_FLIP, PULL_COPY, PULL_SNAPSHOT = 0, 1, 2
IPC_HANDLE_BYTES = 64
STORE_BF16 = 1
PROF_SPMM, PROF_GEMM, PROF_PACK, PROF_OTHER = 0, 1, 2, 3
STATUS = {0: "OK", 1: "E_INVALID", 2: "E_SHAPE", 3: "E_STATE", 4: "E_CUDA", 5: "E_NCCL",
          6: "E_NOMEM", 7: "E_UNSUPPORTED"}


class DigestError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"digest {STATUS.get(status, status)}: {msg}")
        self.status = status


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2206_00057_b200.build` "
                      "(there is no CPU fallback)")
lib = C.CDLL(LIB_PATH)

_p, _i32, _i64, _u32, _f32, _sz = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_float, C.c_size_t


class PartInfo(C.Structure):
    _fields_ = [("num_nodes", _i64), ("n_local", _i64), ("n_halo", _i64), ("nnz", _i64),
                ("nnz_in", _i64), ("n_send", _i64), ("rh_nnz", _i64), ("num_parts", _i32),
                ("rank", _i32), ("send_count", _i64 * DIGEST_MAX_PARTS),
                ("send_off", _i64 * DIGEST_MAX_PARTS), ("recv_count", _i64 * DIGEST_MAX_PARTS),
                ("recv_off", _i64 * DIGEST_MAX_PARTS)]


_SIGS = {
    "digest_last_error": ([], C.c_char_p),
    "digest_launch_count": ([], C.c_uint64),
    "digest_prof_enable": ([_i32], _i32),
    "digest_prof_read": ([_p, _p, _p, _p], _i32),
    "digest_prof_read_detail": ([_i32, _p, _p, _p, _p, _p, _p, _p], _i32),
    "digest_comm_unique_id": ([_p], _i32),
    "digest_comm_init": ([_p, _i32, _i32, _p], _i32),
    "digest_comm_destroy": ([_p], _i32),
    "digest_comm_init_peer": ([_i32, _i32, _i64, _p], _i32),
    "digest_comm_export": ([_p, _p], _i32),
    "digest_comm_connect": ([_p, _p], _i32),
    "digest_store_export": ([_p, _p, _p], _i32),
    "digest_store_connect": ([_p, _p, _sz], _i32),
    "digest_partition": ([_i64, _i64, _p, _p, _p, _i32, _i32, _u32, _p, _p], _i32),
    "digest_part_get_info": ([_p, _p], _i32),
    "digest_part_export": ([_p] * 11, _i32),
    "digest_part_destroy": ([_p], _i32),
    "digest_part_set_loss_mask": ([_p, _p, _p], _i32),
    "digest_store_create": ([_p, _p, _i32, _p, _p], _i32),
    "digest_store_create_ex": ([_p, _p, _i32, _p, _u32, _p], _i32),
    "digest_store_link": ([_p, _i32], _i32),
    "digest_push_boundary": ([_p, _i32, _p, _i64, _i64, _u32, _p], _i32),
    "digest_pull": ([_p, _i32, _i64, _i32, _p, _p], _i32),
    "digest_gather_rows": ([_p, _i64, _p, _i64, _p, _i64, _i32, _p], _i32),
    "digest_store_front": ([_p, _i32, _p, _p, _p], _i32),
    "digest_store_destroy": ([_p], _i32),
    "digest_layer_workspace": ([_p, _i32, _i32, _i32, _p, _p], _i32),
    "digest_layer_fwd": ([_p, _p, _i64, _p, _i64, _p, _i32, _i32, _i32, _i32, _u32, _p, _i64, _p, _p,
                          _p], _i32),
    "digest_layer_bwd": ([_p, _p, _i64, _p, _i64, _p, _i32, _i32, _i32, _i32, _p, _p, _i64, _p, _i64,
                          _u32, _p, _p, _i64, _p, _i64, _p, _i64, _p, _p], _i32),
    "digest_layer_mask": ([_p, _i32, _i32, _i32, _p, _p, _p], _i32),
    "digest_store_grad_buffer": ([_p, _i32, _p, _p], _i32),
    "digest_return_halo_grad": ([_p, _i32, _p, _i64, _p, _i64, _p], _i32),
    "digest_propagate": ([_p, _i32, _p, _i64, _p, _i64, _i32, _p, _i64, _p], _i32),
    "digest_xent_workspace": ([_i64, _p], _i32),
    "digest_xent": ([_p, _i64, _i32, _i64, _p, _p, _f32, _p, _i64, _p, _p, _p], _i32),
    "digest_grad_allreduce": ([_p, _p, _i64, _f32, _p], _i32),
    "digest_grad_allreduce_ex": ([_p, _p, _i64, _f32, _u32, _p], _i32),
    "digest_grad_slot": ([_p, _p], _i32),
    "digest_comm_alltoallv": ([_p, _p, _p, _p, _p, _p], _i32),
    "digest_grad_allreduce_local": ([_p, _i32, _i64, _f32, _p], _i32),
    "digest_sgd_step": ([_p, _p, _i64, _f32, _p], _i32),
    "digest_ps_mix": ([_p, _p, _i64, _f32, _p], _i32),
    "digest_ps_download": ([_p, _p, _i64, _p], _i32),
    "digest_ps_init_peer": ([_p, _p, _i64, _p], _i32),
    "digest_ps_upload_peer": ([_p, _p, _i64, _f32, _p], _i32),
    "digest_ps_download_peer": ([_p, _p, _i64, _p], _i32),
    "digest_ps_updates_peer": ([_p, _p], _i32),
    "digest_delay": ([_i64, _p], _i32),
    "digest_adam_step_dev": ([_p, _p, _p, _p, _i64, _f32, _f32, _f32, _f32, _p, _p], _i32),
    "digest_adam_step": ([_p, _p, _p, _p, _i64, _f32, _f32, _f32, _f32, _i64, _p], _i32),
    "digest_gemm": ([_p, _i64, _p, _i64, _p, _i64, _i64, _i32, _i32, _u32, _p], _i32),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res


def _check(status):
    if status != 0:
        raise DigestError(status, lib.digest_last_error().decode(errors="replace"))


def ptr(x):
    """Device (or host) address of a tensor, an int, or None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, torch.Tensor):
        return x.data_ptr()
    if isinstance(x, (C.c_void_p,)):
        return x.value
    raise TypeError(f"cannot take the address of {type(x)}")


def stream_ptr(stream=None):
    if stream is None:
        if not torch.cuda.is_available():
            return None
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def ld_of(t: torch.Tensor) -> int:
    assert t.dim() == 2 and t.stride(1) == 1, "row-major 2-D tensor expected"
    return t.stride(0)


# ------------------------------------------------------------------ misc
def digest_last_error() -> str:
    return lib.digest_last_error().decode(errors="replace")


def digest_launch_count() -> int:
    return int(lib.digest_launch_count())


def digest_prof_enable(on: bool):
    _check(lib.digest_prof_enable(1 if on else 0))


def digest_prof_read():
    ms = (C.c_double * 4)()
    n = (C.c_int64 * 4)()
    b = (C.c_double * 4)()
    f = (C.c_double * 4)()
    _check(lib.digest_prof_read(ms, n, b, f))
    names = ["spmm", "gemm", "pack", "other"]
    return {names[i]: {"ms": ms[i], "launches": n[i], "bytes": b[i], "flops": f[i]} for i in range(4)}


def digest_prof_read_detail(max_groups=64):
    cls, tag = (C.c_int32 * max_groups)(), (C.c_int32 * max_groups)()
    ms, b, f = (C.c_double * max_groups)(), (C.c_double * max_groups)(), (C.c_double * max_groups)()
    n, cnt = (C.c_int64 * max_groups)(), C.c_int32()
    _check(lib.digest_prof_read_detail(max_groups, cls, tag, ms, n, b, f, C.byref(cnt)))
    names = ["spmm", "gemm", "pack", "other"]
    return [{"cls": names[cls[i]], "tag": tag[i], "ms": ms[i], "launches": n[i], "bytes": b[i],
             "flops": f[i]} for i in range(cnt.value)]


digest_prof_detail = digest_prof_read_detail


# ------------------------------------------------------------------ communicator
def digest_comm_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib.digest_comm_unique_id(buf))
    return bytes(buf)


def digest_comm_init(uid: bytes, nranks: int, rank: int):
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    out = C.c_void_p()
    _check(lib.digest_comm_init(buf, nranks, rank, C.byref(out)))
    return out.value


def digest_comm_destroy(comm):
    _check(lib.digest_comm_destroy(comm))


def digest_comm_init_peer(nranks: int, rank: int, max_grad_count: int):
    out = C.c_void_p()
    _check(lib.digest_comm_init_peer(nranks, rank, max_grad_count, C.byref(out)))
    return out.value


def digest_comm_export(comm) -> bytes:
    buf = (C.c_uint8 * IPC_HANDLE_BYTES)()
    _check(lib.digest_comm_export(comm, buf))
    return bytes(buf)


def digest_comm_connect(comm, handles):
    """handles: list of every rank's 64-byte export, rank order."""
    blob = b"".join(handles)
    buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
    _check(lib.digest_comm_connect(comm, buf))


# ------------------------------------------------------------------ partition
def digest_partition(num_nodes, nnz, indptr, indices, part_of, num_parts, rank, flags=0,
                     stream=None):
    out = C.c_void_p()
    _check(lib.digest_partition(num_nodes, nnz, ptr(indptr), ptr(indices), ptr(part_of),
                                num_parts, rank, flags, stream_ptr(stream), C.byref(out)))
    return out.value


def digest_part_get_info(part) -> PartInfo:
    info = PartInfo()
    _check(lib.digest_part_get_info(part, C.byref(info)))
    return info


def digest_part_export(part, local_ids=None, halo_ids=None, row_ptr=None, col=None, val=None,
                       send_idx=None, rh_ptr=None, rh_col=None, rh_val=None, stream=None):
    _check(lib.digest_part_export(part, ptr(local_ids), ptr(halo_ids), ptr(row_ptr), ptr(col),
                                  ptr(val), ptr(send_idx), ptr(rh_ptr), ptr(rh_col), ptr(rh_val),
                                  stream_ptr(stream)))


def digest_part_destroy(part):
    _check(lib.digest_part_destroy(part))


def digest_part_set_loss_mask(part, row_mask, stream=None):
    """row_mask: device uint8 [n_local] (the local training rows) or None to clear."""
    _check(lib.digest_part_set_loss_mask(part, ptr(row_mask), stream_ptr(stream)))


# ------------------------------------------------------------------ store
def digest_store_create_ex(part, comm, widths, flags=0):
    arr = (C.c_int32 * max(1, len(widths)))(*widths)
    out = C.c_void_p()
    _check(lib.digest_store_create_ex(part, comm, len(widths), arr, flags, C.byref(out)))
    return out.value


def digest_store_create(part, comm, widths, flags=0):
    if flags:
        return digest_store_create_ex(part, comm, widths, flags)
    arr = (C.c_int32 * max(1, len(widths)))(*widths)
    out = C.c_void_p()
    _check(lib.digest_store_create(part, comm, len(widths), arr, C.byref(out)))
    return out.value


def digest_store_link(stores):
    arr = (C.c_void_p * len(stores))(*stores)
    _check(lib.digest_store_link(arr, len(stores)))


def digest_push_boundary(store, level, H_local, version, flags=0, stream=None):
    _check(lib.digest_push_boundary(store, level, ptr(H_local), ld_of(H_local), version, flags,
                                    stream_ptr(stream)))


def digest_pull(store, level, epoch, mode=PULL_FLIP, stream=None) -> int:
    out = C.c_void_p()
    _check(lib.digest_pull(store, level, epoch, mode, stream_ptr(stream), C.byref(out)))
    return out.value


def digest_gather_rows(src, idx, dst, width=None, stream=None):
    n = idx.numel()
    _check(lib.digest_gather_rows(ptr(src), ld_of(src), ptr(idx), n, ptr(dst), ld_of(dst),
                                  width or dst.shape[1], stream_ptr(stream)))


def digest_store_front(store, level):
    p, ld, ver = C.c_void_p(), C.c_int64(), C.c_int64()
    _check(lib.digest_store_front(store, level, C.byref(p), C.byref(ld), C.byref(ver)))
    return p.value, ld.value, ver.value


def digest_store_destroy(store):
    _check(lib.digest_store_destroy(store))


def digest_store_export(store) -> bytes:
    n = C.c_size_t()
    _check(lib.digest_store_export(store, None, C.byref(n)))
    buf = (C.c_uint8 * n.value)()
    _check(lib.digest_store_export(store, buf, C.byref(n)))
    return bytes(buf)


def digest_store_connect(store, blobs):
    """blobs: every rank's digest_store_export, rank order."""
    size = len(blobs[0])
    assert all(len(b) == size for b in blobs)
    blob = b"".join(blobs)
    buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
    _check(lib.digest_store_connect(store, buf, size))


# ------------------------------------------------------------------ layer
def digest_layer_workspace(part, d_in, d_out, order=ORDER_AUTO):
    s, t = C.c_size_t(), C.c_size_t()
    _check(lib.digest_layer_workspace(part, d_in, d_out, order, C.byref(s), C.byref(t)))
    return s.value, t.value


FWD_REUSE_SAVED = 1


def digest_layer_fwd(part, X_local, X_halo, ld_xh, W, d_in, d_out, act, order, H_out, saved,
                     scratch, stream=None, flags=0):
    """X_halo may be a tensor, a raw device address (the store's front buffer) or None."""
    _check(lib.digest_layer_fwd(part, ptr(X_local), ld_of(X_local), ptr(X_halo), ld_xh, ptr(W),
                                d_in, d_out, act, order, flags, ptr(H_out), ld_of(H_out),
                                ptr(saved), ptr(scratch), stream_ptr(stream)))


def digest_layer_mask(part, d_in, d_out, order, saved):
    """(device address, words per row) of the 1-bit ReLU mask inside `saved`."""
    p, ld = C.c_void_p(), C.c_int64()
    _check(lib.digest_layer_mask(part, d_in, d_out, order, ptr(saved), C.byref(p), C.byref(ld)))
    return p.value, ld.value


BWD_G_IS_D = 1
BWD_GIN_MASK_BITS = 2
BWD_HALO_SAVE_S = 4
BWD_LOSS_ROWS = 8
GEMM_RELU = 1
GEMM_BT = 2


def digest_layer_bwd(part, X_local, X_halo, ld_xh, W, d_in, d_out, act, order, saved, H_out,
                     G_out, G_W, G_in, scratch, stream=None, flags=0, gin_mask=None,
                     G_halo=None, ld_gh=0):
    """G_halo may be a tensor or a raw device address (the store's gradient buffer).
    gin_mask: a float tensor, or (address, words per row) of a 1-bit mask
    (digest_layer_mask), which sets BWD_GIN_MASK_BITS."""
    if isinstance(G_halo, torch.Tensor):
        ld_gh = ld_of(G_halo)
    if isinstance(gin_mask, tuple):
        gm, ld_gm = gin_mask
        flags |= BWD_GIN_MASK_BITS
    else:
        gm, ld_gm = ptr(gin_mask), ld_of(gin_mask) if gin_mask is not None else 0
    _check(lib.digest_layer_bwd(part, ptr(X_local), ld_of(X_local), ptr(X_halo), ld_xh, ptr(W),
                                d_in, d_out, act, order, ptr(saved), ptr(H_out),
                                ld_of(H_out) if H_out is not None else 0, ptr(G_out),
                                ld_of(G_out), flags, ptr(G_W), ptr(G_in),
                                ld_of(G_in) if G_in is not None else 0, gm, ld_gm, ptr(G_halo),
                                ld_gh, ptr(scratch), stream_ptr(stream)))


def digest_store_grad_buffer(store, level):
    p, ld = C.c_void_p(), C.c_int64()
    _check(lib.digest_store_grad_buffer(store, level, C.byref(p), C.byref(ld)))
    return p.value, ld.value


def digest_return_halo_grad(store, level, G_local, mask=None, stream=None):
    _check(lib.digest_return_halo_grad(store, level, ptr(G_local), ld_of(G_local), ptr(mask),
                                       ld_of(mask) if mask is not None else 0,
                                       stream_ptr(stream)))


def digest_propagate(part, mode, X_local, X_halo, ld_xh, width, Y, stream=None):
    _check(lib.digest_propagate(part, mode, ptr(X_local), ld_of(X_local), ptr(X_halo), ld_xh,
                                width, ptr(Y), ld_of(Y), stream_ptr(stream)))


# ------------------------------------------------------------------ loss / AGG / update
def digest_xent_workspace(n):
    s = C.c_size_t()
    _check(lib.digest_xent_workspace(n, C.byref(s)))
    return s.value


def digest_xent(logits, C_, labels, train_mask, w_loss, G_logits, loss_out, scratch, stream=None):
    _check(lib.digest_xent(ptr(logits), logits.shape[0], C_, ld_of(logits), ptr(labels),
                           ptr(train_mask), w_loss, ptr(G_logits), ld_of(G_logits), ptr(loss_out),
                           ptr(scratch), stream_ptr(stream)))


def digest_grad_allreduce(comm, grads, scale=1.0, stream=None):
    _check(lib.digest_grad_allreduce(comm, ptr(grads), grads.numel(), scale, stream_ptr(stream)))


AR_IN_SLOT = 1


def digest_comm_alltoallv(comm, sends, recvs, stream=None):
    """sends / recvs: per-rank float tensors (or None); counts are their numel()."""
    n = len(sends)
    sp = (C.c_void_p * n)(*[ptr(t) for t in sends])
    rp = (C.c_void_p * n)(*[ptr(t) for t in recvs])
    cs = (C.c_int64 * n)(*[0 if t is None else t.numel() for t in sends])
    cr = (C.c_int64 * n)(*[0 if t is None else t.numel() for t in recvs])
    _check(lib.digest_comm_alltoallv(comm, sp, cs, rp, cr, stream_ptr(stream)))


def digest_grad_slot(comm) -> int:
    """Device address of the own peer-window slot the next allreduce_ex reduces."""
    p = C.c_void_p()
    _check(lib.digest_grad_slot(comm, C.byref(p)))
    return p.value


def digest_grad_allreduce_ex(comm, grads, scale=1.0, flags=0, stream=None):
    _check(lib.digest_grad_allreduce_ex(comm, ptr(grads), grads.numel(), scale, flags,
                                        stream_ptr(stream)))


def digest_grad_allreduce_local(bufs, scale=1.0, stream=None):
    arr = (C.c_void_p * len(bufs))(*[ptr(b) for b in bufs])
    _check(lib.digest_grad_allreduce_local(arr, len(bufs), bufs[0].numel(), scale,
                                           stream_ptr(stream)))


def digest_sgd_step(W, G, lr, stream=None):
    _check(lib.digest_sgd_step(ptr(W), ptr(G), W.numel(), lr, stream_ptr(stream)))


def digest_adam_step(W, G, m, v, lr, b1, b2, eps, step, stream=None):
    _check(lib.digest_adam_step(ptr(W), ptr(G), ptr(m), ptr(v), W.numel(), lr, b1, b2, eps, step,
                                stream_ptr(stream)))


def digest_gemm(A, B, Cm, relu=False, stream=None, bt=False, M=None, ldc=None):
    """C = A B (bt: C = A B^T, B given N x K).  Cm may be a tensor or a raw device address
    (then pass M rows and its ldc)."""
    Mr, K = A.shape
    M = Mr if M is None else M
    N = B.shape[0] if bt else B.shape[1]
    ldc = ld_of(Cm) if ldc is None else ldc
    _check(lib.digest_gemm(ptr(A), ld_of(A), ptr(B), ld_of(B), ptr(Cm), ldc, M, N, K,
                           (GEMM_RELU if relu else 0) | (GEMM_BT if bt else 0),
                           stream_ptr(stream)))


# ------------------------------------------------------------------ DIGEST-A parameter server
def digest_ps_mix(W_global, W_local, alpha, stream=None):
    _check(lib.digest_ps_mix(ptr(W_global), ptr(W_local), W_local.numel(), alpha,
                             stream_ptr(stream)))


def digest_ps_download(W_global, W_local, stream=None):
    _check(lib.digest_ps_download(ptr(W_global), ptr(W_local), W_local.numel(), stream_ptr(stream)))


def digest_ps_init_peer(comm, W0, stream=None):
    _check(lib.digest_ps_init_peer(comm, ptr(W0), W0.numel(), stream_ptr(stream)))


def digest_ps_upload_peer(comm, W_local, alpha, stream=None):
    _check(lib.digest_ps_upload_peer(comm, ptr(W_local), W_local.numel(), alpha,
                                     stream_ptr(stream)))


def digest_ps_download_peer(comm, W_local, stream=None):
    _check(lib.digest_ps_download_peer(comm, ptr(W_local), W_local.numel(), stream_ptr(stream)))


def digest_ps_updates_peer(comm) -> int:
    n = C.c_int64()
    _check(lib.digest_ps_updates_peer(comm, C.byref(n)))
    return n.value


def digest_delay(ns: int, stream=None):
    _check(lib.digest_delay(int(ns), stream_ptr(stream)))


def digest_adam_step_dev(W, G, m, v, lr, b1, b2, eps, step_dev, stream=None):
    _check(lib.digest_adam_step_dev(ptr(W), ptr(G), ptr(m), ptr(v), W.numel(), lr, b1, b2, eps,
                                    ptr(step_dev), stream_ptr(stream)))
