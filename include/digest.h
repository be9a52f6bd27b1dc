/*
 * digest.h -- C ABI of libdigest.so, the B200 (sm_100a) hot path of DIGEST
 * (arXiv 2206.00057): the per-subgraph GCN layer forward/backward over local and
 * stale out-of-subgraph ("halo") neighbours, the partition build, the periodic
 * boundary push into the stale store and the weight-gradient allreduce.
 *
 * Citations: P:n = PAPER.md line n (section / equation), S:n = SPEC.md line n.
 *
 * Conventions (apply to every call unless stated):
 *  - Pointers are DEVICE memory unless the parameter name ends in `_h` (host).
 *    The caller owns every numeric buffer; the library owns the opaque handles
 *    (digest_part, digest_store, digest_comm) and the device memory inside them.
 *  - Matrices are row-major fp32.  A leading dimension `ld*` is in floats and must
 *    be a multiple of 4 (16-byte rows, float4 / TMA rule) and >= the row width;
 *    device pointers of matrices must be 16-byte aligned.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    All work is enqueued on it; nothing but digest_partition and the *_info /
 *    *_export calls synchronises the host.  fwd/bwd/push/pull/xent/allreduce/step
 *    never allocate, so an epoch is CUDA-graph capturable (pull in COPY mode).
 *  - Errors: argument checks run before anything is enqueued; a non-OK status
 *    means nothing was launched.  digest_last_error() returns a thread-local text
 *    for the last non-OK status.  DIGEST_E_CUDA / DIGEST_E_NCCL report runtime
 *    failures (asynchronous device faults surface at the next sync).  No C++
 *    exception or abort crosses this ABI.
 */
#ifndef DIGEST_H
#define DIGEST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DIGEST_OK = 0,
  DIGEST_E_INVALID = 1,     /* bad argument value (range, alignment, empty part, ...) */
  DIGEST_E_SHAPE = 2,       /* dimension mismatch */
  DIGEST_E_STATE = 3,       /* call out of protocol order (e.g. pull of an unpushed level) */
  DIGEST_E_CUDA = 4,        /* CUDA runtime error */
  DIGEST_E_NCCL = 5,        /* NCCL error */
  DIGEST_E_NOMEM = 6,       /* device allocation failed */
  DIGEST_E_UNSUPPORTED = 7  /* valid but not implemented on this build/device */
} digest_status;

#define DIGEST_MAX_PARTS 64

const char* digest_last_error(void);
/* Number of kernels this library has launched in this process (all streams). */
uint64_t digest_launch_count(void);

/* ------------------------------------------------------------------ profiling
 * Live per-kernel-class timing with CUDA events recorded on the stream each
 * kernel is launched on.  Classes: 0 spmm, 1 gemm, 2 pack, 3 other.
 * digest_prof_read synchronises on the recorded events and returns, per class,
 * the summed milliseconds, the launch count and the algorithmic bytes/flops the
 * launches declared (SURVEY §8.d.4 models). */
enum { DIGEST_PROF_SPMM = 0, DIGEST_PROF_GEMM = 1, DIGEST_PROF_PACK = 2, DIGEST_PROF_OTHER = 3,
       DIGEST_PROF_CLASSES = 4 };
digest_status digest_prof_enable(int32_t on);
digest_status digest_prof_read(double* ms_h, int64_t* launches_h, double* alg_bytes_h,
                               double* alg_flops_h);
/* The same, grouped by (class, tag) where tag is the SpMM width (0 for other
 * kernels); writes up to max_groups groups and their count to *count_h. */
digest_status digest_prof_read_detail(int32_t max_groups, int32_t* cls_h, int32_t* tag_h,
                                      double* ms_h, int64_t* launches_h, double* alg_bytes_h,
                                      double* alg_flops_h, int32_t* count_h);

/* ------------------------------------------------------------------ communicator
 * A library-owned NCCL communicator.  The 128-byte id is produced on rank 0 by
 * digest_comm_unique_id and carried to the other ranks by the caller's process
 * group (torch.distributed broadcast).  Used by the boundary exchange (C1) and the
 * gradient allreduce (C2); the halo exchange gets its own side stream. */
typedef struct digest_comm digest_comm;
digest_status digest_comm_unique_id(uint8_t id_h[128]);
digest_status digest_comm_init(const uint8_t id_h[128], int32_t nranks, int32_t rank,
                               digest_comm** out_h);
digest_status digest_comm_destroy(digest_comm* comm);

/* Peer-memory transport (the alternative to NCCL for C1/C2; the
 * exchange as loads/stores of the library's own kernels through NVLink/NVSwitch
 * peer mappings).  Every rank allocates a window (flag words + two gradient slots
 * of max_grad_count floats) with digest_comm_init_peer, exports its 64-byte CUDA
 * IPC handle with digest_comm_export, the caller all-gathers the handles over its
 * process group (rank order) and passes them to digest_comm_connect, which maps
 * every peer's window.  Works between processes on different GPUs (peer access is
 * enabled lazily) and between processes sharing one GPU.  A peer communicator may
 * serve both the store (digest_store_create) and digest_grad_allreduce; its calls
 * never synchronise the host: producers raise flags with a system-scope release,
 * consumers spin on them inside their kernels (a wait longer than 30 s traps the
 * kernel: a CUDA error instead of a hang).  Every rank must issue the same sequence
 * of collective calls (push/pull/return per level, allreduce). */
/* The boundary exchange primitive of the NCCL transport (push; halo-gradient
 * return): grouped ncclSend/ncclRecv, send_h[k] (count_s_h[k] floats, device) to rank
 * k and recv_h[k] (count_r_h[k] floats, device) from rank k, for every k with a
 * non-zero count -- the own rank included (a self transfer), so a 1-rank communicator
 * runs the same NCCL calls as a multi-rank one.  Host arrays have nranks entries.
 * DIGEST_E_INVALID for a peer-memory communicator; DIGEST_E_NCCL on NCCL errors. */
digest_status digest_comm_alltoallv(digest_comm* comm, const float* const* send_h,
                                    const int64_t* count_s_h, float* const* recv_h,
                                    const int64_t* count_r_h, void* stream);
#define DIGEST_IPC_HANDLE_BYTES 64
digest_status digest_comm_init_peer(int32_t nranks, int32_t rank, int64_t max_grad_count,
                                    digest_comm** out_h);
digest_status digest_comm_export(const digest_comm* comm,
                                 uint8_t handle_h[DIGEST_IPC_HANDLE_BYTES]);
/* handles_h: nranks x DIGEST_IPC_HANDLE_BYTES, rank order (own entry ignored). */
digest_status digest_comm_connect(digest_comm* comm, const uint8_t* handles_h);

/* ------------------------------------------------------------------ partition
 * north_star call #1.  Builds, for partition `rank` of `num_parts`, the split of
 * the GCN propagation matrix of Eq. 5 (P_m = P_in + P_out),
 * the halo index (N(v)\V_m over v in V_m) and the boundary send lists.
 *
 *  indptr  int64[num_nodes+1], indices int32[nnz]: a symmetric adjacency, rows
 *          sorted ascending, no duplicates, no self loops (checked: E_INVALID).
 *  part_of int32[num_nodes] in [0, num_parts); every part non-empty.
 *
 * Result (bit-exact with the oracle):
 *  local_ids : V_m ascending;  halo_ids : H_m ordered by (part_of, id);
 *  extended column space [0, n_local) local, [n_local, n_local+n_halo) halo;
 *  row i = loc(v) holds {(ext(u), P_vu) : u in N(v)} U {(i, P_vv)} sorted by
 *  column (in-block entries first); P_vu = fp32(1/sqrt(double(deg v+1)*double(deg u+1)))
 *  with global degrees (Kipf normalisation, "following GCN's definition").
 *  send list to k: {u in V_m : N(u) meets V_k} ascending, concatenated over k;
 *  recv_count[k] = #{u in H_m : part_of[u] = k}; offsets are exclusive prefixes.
 *  The reverse-halo CSR (P_out^T: halo row j -> local columns) is always built.
 * Synchronises `stream` (sizes are data-dependent).  The input arrays may be
 * freed after return. */
typedef struct digest_part digest_part;
typedef struct {
  int64_t num_nodes, n_local, n_halo, nnz, nnz_in, n_send, rh_nnz;
  int32_t num_parts, rank;
  int64_t send_count[DIGEST_MAX_PARTS], send_off[DIGEST_MAX_PARTS];
  int64_t recv_count[DIGEST_MAX_PARTS], recv_off[DIGEST_MAX_PARTS];
} digest_part_info;

digest_status digest_partition(int64_t num_nodes, int64_t nnz, const int64_t* indptr,
                               const int32_t* indices, const int32_t* part_of,
                               int32_t num_parts, int32_t rank, uint32_t flags,
                               void* stream, digest_part** out_h);
digest_status digest_part_get_info(const digest_part* part, digest_part_info* info_h);
/* Copies the partition arrays into caller buffers (device); any NULL is skipped.
 * Sizes: local_ids[n_local], halo_ids[n_halo], row_ptr[n_local+1], col/val[nnz],
 * send_idx[n_send], rh_ptr[n_halo+1], rh_col/rh_val[rh_nnz]. */
digest_status digest_part_export(const digest_part* part, int32_t* local_ids,
                                 int32_t* halo_ids, int64_t* row_ptr, int32_t* col,
                                 float* val, int32_t* send_idx, int64_t* rh_ptr,
                                 int32_t* rh_col, float* rh_val, void* stream);
digest_status digest_part_destroy(digest_part* part);

/* Loss rows of the partition (Eq. 3: the loss sums over the training nodes only, so
 * the last layer's gradient G_logits -- and every operand derived from it row by row, D and
 * U = D W^T -- is zero on the other local rows).  row_mask: device uint8[n_local], nonzero =
 * the row may be nonzero (the local training rows); NULL clears.  Builds, inside the
 * handle, P_in and P_out^T restricted to the columns whose row_mask is set (entries kept in
 * their order, so the products equal the full ones exactly: the dropped terms are products
 * with zero rows).  digest_layer_bwd(..., DIGEST_BWD_LOSS_ROWS) then runs its P_in / P_out^T
 * products over them; the caller guarantees G_out's rows outside the mask are zero.
 * Synchronises `stream` (sizes are data-dependent).  Errors: DIGEST_E_INVALID (NULL
 * partition), DIGEST_E_NOMEM, DIGEST_E_CUDA. */
digest_status digest_part_set_loss_mask(digest_part* part, const uint8_t* row_mask, void* stream);

/* ------------------------------------------------------------------ stale store
 * The stale representation store H~^(l), l in [1, L-1] (levels never
 * equal L).  Per level: a front buffer (read by the layer that
 * consumes level l) and a back buffer (written by pushes), each n_halo x ld_l
 * with ld_l = round_up(width_l, 4), zero at creation (cold start).
 * comm == NULL: single-process store; several stores of one process (the M
 * partitions of a loopback run) are linked with digest_store_link so a push
 * writes straight into the peers' back buffers (a fused gather + put). */
typedef struct digest_store digest_store;
enum { DIGEST_PUSH_ASYNC = 1u, DIGEST_PUSH_L2NORM = 2u, DIGEST_PUSH_NOWAIT = 4u };
enum { DIGEST_PULL_FLIP = 0, DIGEST_PULL_COPY = 1, DIGEST_PULL_SNAPSHOT = 2 };
/* DIGEST-A on the peer transport ("pulls/pushes stale representations of other
 * subgraphs from the shared KVS ... without blindly waiting"): a push with
 * DIGEST_PUSH_NOWAIT does not wait for the receiver; it brackets its rows with a
 * per-(level, owner) sequence word (odd while writing, even when complete), and a pull
 * in DIGEST_PULL_SNAPSHOT mode copies every owner's segment back -> front, retrying a
 * segment whose sequence word changed or was odd during the copy -- each owner's rows
 * are taken from one push (key atomicity, SPEC "Concurrency Model").  Every rank of a
 * store must use the same mode.  On a single-process (linked) store both behave like
 * the plain push and DIGEST_PULL_COPY. */

digest_status digest_store_create(const digest_part* part, digest_comm* comm,
                                  int32_t num_levels, const int32_t* width_h,
                                  digest_store** out_h);
/* The same with flags.  DIGEST_STORE_BF16: the back buffers, the send
 * buffers and every transfer (loopback, NCCL, peer) hold bf16 copies of the pushed rows
 * (round to nearest even), half the exchange bytes; the front buffer stays fp32 and a
 * pull widens back -> front exactly (FLIP pulls become this copy).  The halo inputs then
 * carry bf16 precision (relative 2^-9), so parity with the oracle holds only with the
 * oracle's matching store_dtype='bf16' and a looser tolerance. */
enum { DIGEST_STORE_BF16 = 1u };
digest_status digest_store_create_ex(const digest_part* part, digest_comm* comm,
                                     int32_t num_levels, const int32_t* width_h, uint32_t flags,
                                     digest_store** out_h);
/* Link the stores of all partitions of one process, index = rank (loopback). */
digest_status digest_store_link(digest_store* const* stores_h, int32_t count);
/* north_star call #4 ("push", Alg. 1 PUSH P:220-221).  Packs the boundary
 * rows H_local[send_idx] of level `level` (optionally row-L2-normalised, Alg. 1
 * P:226) and delivers them into every peer's back buffer at the
 * (owner, id) segment of its halo.  `version` = epoch r.  With DIGEST_PUSH_ASYNC
 * the NCCL exchange runs on the store's side stream behind an event (overlap with the
 * next layer); on the peer transport the push is one fused gather + put
 * kernel on `stream` (the put is the gather's own stores; ASYNC is accepted and has
 * nothing to defer).  Collective: every rank pushes the same (level, version). */
digest_status digest_push_boundary(digest_store* store, int32_t level, const float* H_local,
                                   int64_t ld, int64_t version, uint32_t flags,
                                   void* stream);
/* Alg. 1 PULL: make the last pushed version of `level` the front
 * buffer.  Requires the back version < epoch (pushes become visible only to later
 * epochs); if no push happened since the last pull this is a no-op.  Mode FLIP
 * swaps pointers; COPY copies back -> a fixed front (graph-safe).  Makes `stream`
 * wait for an in-flight async exchange.  *front_h receives the front pointer. */
digest_status digest_pull(digest_store* store, int32_t level, int64_t epoch, int32_t mode,
                          void* stream, const float** front_h);
/* Row gather dst[i, 0:width] = src[idx[i], 0:width], i < n (e.g. the static layer-1
 * inputs X[V_m] and X[H_m] of X_ext^(0)).  width % 4 == 0. */
digest_status digest_gather_rows(const float* src, int64_t ld_src, const int32_t* idx, int64_t n,
                                 float* dst, int64_t ld_dst, int32_t width, void* stream);
/* Halo-gradient return (the appendix's P_out^T D W^T term):
 * digest_store_grad_buffer gives the store-owned n_halo x ld buffer of `level` that
 * digest_layer_bwd fills (its G_halo output) with the gradient this part computes for
 * its halo rows; digest_return_halo_grad then delivers every halo segment to its owner
 * and adds it, masked by 1[mask > 0] (the owner's ReLU', NULL = unmasked), into the
 * owner's local gradient rows G_local[send_idx] -- peer by peer in ascending order, so
 * the result is deterministic.  Collective over the parts (loopback: linked stores). */
digest_status digest_store_grad_buffer(digest_store* store, int32_t level, float** buf_h,
                                       int64_t* ld_h);
digest_status digest_return_halo_grad(digest_store* store, int32_t level, float* G_local,
                                      int64_t ld_g, const float* mask, int64_t ld_m,
                                      void* stream);
/* Current front buffer, its leading dimension and the version it holds. */
digest_status digest_store_front(const digest_store* store, int32_t level,
                                 const float** front_h, int64_t* ld_h, int64_t* version_h);
/* Peer transport only: after digest_store_create with a peer communicator, every
 * rank exports a blob (its halo buffers' IPC handles and its receive offsets; query
 * the size with blob_h = NULL), the caller all-gathers the blobs in rank order and
 * passes them to digest_store_connect.  A push then writes straight into the
 * receivers' back buffers (one fused gather + put + signal kernel, which first waits
 * for the receiver's pull of the previous exchange); a pull waits for the arrival
 * flags of the version it exposes; digest_return_halo_grad reads the peers'
 * gradient slots in place.  digest_store_grad_buffer alternates between two slots on
 * this transport (each call returns the next one). */
digest_status digest_store_export(const digest_store* store, uint8_t* blob_h, size_t* bytes_h);
digest_status digest_store_connect(digest_store* store, const uint8_t* blobs_h, size_t blob_bytes);
digest_status digest_store_destroy(digest_store* store);

/* ------------------------------------------------------------------ one GCN layer
 * north_star calls #2/#3.  Eq. 5: H = sigma(P_in X_in W + P_out X~_out W)
 * and Eq. 6 / P:783-794 backward with the halo block constant.
 * X_local: n_local x d_in (ld_x); X_halo: n_halo x d_in (ld_xh; NULL iff n_halo==0);
 * W: d_in x d_out row-major (ld = d_out).
 * order: AGG_FIRST computes A = P_m X_ext then Z = A W; XFORM_FIRST computes
 * T = X_ext W then Z = P_m T; AUTO picks AGG_FIRST iff d_in <= d_out (the SpMM runs
 * at width min(d_in, d_out)).  act RELU: H = max(Z, 0); NONE: H = Z (output layer).
 * `saved` (size from digest_layer_workspace) keeps what backward needs: A for
 * AGG_FIRST and, for act RELU, the 1-bit activation mask 1[H > 0] (
 * n_local rows of ld_words 32-bit words, bit j%32 of word j/32 = column j, words
 * past (d_out+31)/32 are unspecified padding; see digest_layer_mask).  The caller keeps X_local/X_halo alive until backward.
 * scratch is per-call temporary memory. */
typedef enum { DIGEST_ACT_NONE = 0, DIGEST_ACT_RELU = 1 } digest_act;
typedef enum { DIGEST_ORDER_AUTO = 0, DIGEST_ORDER_AGG_FIRST = 1,
               DIGEST_ORDER_XFORM_FIRST = 2 } digest_order;

digest_status digest_layer_workspace(const digest_part* part, int32_t d_in, int32_t d_out,
                                     int32_t order, size_t* saved_bytes_h,
                                     size_t* scratch_bytes_h);
/* flags DIGEST_FWD_REUSE_SAVED (AGG_FIRST only): `saved` already holds A = P_m X_ext
 * from an earlier call on the same inputs -- the layer-1 aggregation of the static
 * features X_ext^(0) is the same every epoch -- so only the GEMM and
 * the activation run. */
enum { DIGEST_FWD_REUSE_SAVED = 1u };
digest_status digest_layer_fwd(const digest_part* part, const float* X_local, int64_t ld_x,
                               const float* X_halo, int64_t ld_xh, const float* W,
                               int32_t d_in, int32_t d_out, int32_t act, int32_t order,
                               uint32_t flags, float* H_out, int64_t ld_h, void* saved,
                               void* scratch, void* stream);
/* The 1-bit ReLU mask digest_layer_fwd (act RELU) left inside `saved`: *bits_h points
 * into saved (device memory, caller-owned through saved), *ld_words_h words per row.
 * Pass it as the next layer's backward gin_mask with DIGEST_BWD_GIN_MASK_BITS. */
digest_status digest_layer_mask(const digest_part* part, int32_t d_in, int32_t d_out,
                                int32_t order, const void* saved, const uint32_t** bits_h,
                                int64_t* ld_words_h);
/* G_out: n_local x d_out gradient of the layer output (ld_g).  sigma'(Z) for act RELU
 * (ReLU'(0) := 0) is read from the 1-bit mask in `saved`; H_out (the forward output,
 * its sign) is consulted only when saved is NULL (XFORM_FIRST); ignored for ACT_NONE.
 * flags DIGEST_BWD_G_IS_D: G_out already is D = G o sigma'(Z).
 * G_W (d_in x d_out, overwritten) = (P_m X_ext)^T D with D = G_out o sigma'(Z).
 * G_in (n_local x d_in, ld_gi; NULL = skip, first layer) = P_in^T D W^T, multiplied
 * by the previous layer's ReLU' when gin_mask != NULL, which emits that layer's D
 * directly (then call it with DIGEST_BWD_G_IS_D).  gin_mask is either a float
 * n_local x d_in tensor (ld_gm floats; factor 1[gin_mask > 0], e.g. the previous H)
 * or, with flags DIGEST_BWD_GIN_MASK_BITS, a 1-bit mask (ld_gm 32-bit words per row,
 * e.g. digest_layer_mask of the previous layer). */
enum { DIGEST_BWD_G_IS_D = 1u, DIGEST_BWD_GIN_MASK_BITS = 2u, DIGEST_BWD_HALO_SAVE_S = 4u,
       DIGEST_BWD_LOSS_ROWS = 8u };
digest_status digest_layer_bwd(const digest_part* part, const float* X_local, int64_t ld_x,
                               const float* X_halo, int64_t ld_xh, const float* W,
                               int32_t d_in, int32_t d_out, int32_t act, int32_t order,
                               const void* saved, const float* H_out, int64_t ld_h,
                               const float* G_out, int64_t ld_g, uint32_t flags, float* G_W,
                               float* G_in, int64_t ld_gi, const void* gin_mask,
                               int64_t ld_gm, float* G_halo, int64_t ld_gh, void* scratch,
                               void* stream);
/* G_halo (n_halo x d_in, ld_gh; NULL = skip) = P_out^T D W^T: the gradient of this
 * part's halo rows, unmasked, for digest_return_halo_grad, returned in the SAME
 * iteration (the exact / zero-staleness variant of the appendix term).
 * With flags DIGEST_BWD_HALO_SAVE_S, G_halo (n_halo x d_out, ld_gh >= d_out) instead
 * receives S = P_out^T D~^(t), the part of the term the paper's DIGEST backward returns
 * ONE iteration later (G~_H^(t) = P_in^T D~^(t) W~^(t)T + P_out^T D~^(t-1)
 * W~^(t)T); the caller keeps it and forms next iteration's rows with
 * digest_gemm(S, W, G, DIGEST_GEMM_BT) = S W^T at the then-current W.
 * With flags DIGEST_BWD_LOSS_ROWS (the last layer, after digest_part_set_loss_mask): the
 * P_in / P_out^T products run over the loss-row CSRs; identical results when G_out is zero
 * outside the mask (DIGEST_E_STATE if no mask was set). */

/* The propagation product alone (the aggregation of Eq. 5 / its transposes):
 *   mode 0: Y = P_m X_ext      (n_local rows; X_ext = [X_local ; X_halo], width w)
 *   mode 1: Y = P_in^T X_local (= P_in X_local, n_local rows; the in-block part)
 *   mode 2: Y = P_out^T X_local (n_halo rows; reverse-halo CSR)
 * w % 4 == 0.  Used by the layer; exported for tests, benchmarks and aggregation
 * caches (e.g. the static layer-1 aggregation). */
digest_status digest_propagate(const digest_part* part, int32_t mode, const float* X_local,
                               int64_t ld_x, const float* X_halo, int64_t ld_xh, int32_t width,
                               float* Y, int64_t ld_y, void* stream);

/* ------------------------------------------------------------------ loss
 * Eq. 3 on training rows: for v with train_mask[v] != 0,
 * l_v = logsumexp(z_v[0:C]) - z_v[y_v]; G_logits[v,0:C] = w_loss*(softmax - e_y),
 * 0 on other rows and on padded columns >= C.  loss_out[0] (device double) =
 * w_loss * sum_v l_v, reduced in a fixed order (deterministic).  scratch: see
 * digest_xent_workspace. */
digest_status digest_xent_workspace(int64_t n, size_t* scratch_bytes_h);
digest_status digest_xent(const float* logits, int64_t n, int32_t C, int64_t ld,
                          const int32_t* labels, const uint8_t* train_mask, float w_loss,
                          float* G_logits, int64_t ld_g, double* loss_out, void* scratch,
                          void* stream);

/* ------------------------------------------------------------------ AGG and update
 * north_star call #5 (Alg. 1 AGG; update rule P:896): grads <- scale *
 * sum over ranks of grads, in place (ncclAllReduce sum, then a scale kernel; on a
 * peer communicator: publish into the own window, then every rank sums all ranks'
 * slots in rank order with the scale fused -- bit-identical to
 * digest_grad_allreduce_local on the same buffers; count <= max_grad_count).
 * comm == NULL or a 1-rank peer comm: only the scale is applied (a 1-rank NCCL comm
 * still runs ncclAllReduce, a copy, so that path is exercised on one GPU). */
digest_status digest_grad_allreduce(digest_comm* comm, float* grads, int64_t count,
                                    float scale, void* stream);
/* Fused weight-gradient + AGG on the peer transport (Alg. 1 line 13,
 * P:233): digest_grad_slot returns the own window slot (count <= max_grad_count floats,
 * device memory owned by the communicator) that the NEXT digest_grad_allreduce_ex call
 * reduces; the caller makes it the G_W output of its digest_layer_bwd calls, so the
 * split-K weight-gradient reduction writes the peer-visible slot directly (no publish
 * copy).  digest_grad_allreduce_ex with DIGEST_AR_IN_SLOT then runs ONE kernel: signal
 * this rank's slot ready to every peer, wait for theirs, grads <- scale * (slot_0 + ...
 * + slot_{M-1}) in rank order (bit-identical to digest_grad_allreduce).  Without the
 * flag it is digest_grad_allreduce.  Both: DIGEST_E_UNSUPPORTED unless `comm` is a
 * connected peer communicator with more than one rank; DIGEST_E_SHAPE if count >
 * max_grad_count. */
enum { DIGEST_AR_IN_SLOT = 1u };
digest_status digest_grad_slot(digest_comm* comm, float** slot_h);
digest_status digest_grad_allreduce_ex(digest_comm* comm, float* grads, int64_t count,
                                       float scale, uint32_t flags, void* stream);
/* Loopback AGG for M partitions of one process: every buffer receives
 * scale * (bufs[0] + ... + bufs[n-1]) summed in index order. */
digest_status digest_grad_allreduce_local(float* const* bufs_h, int32_t n, int64_t count,
                                          float scale, void* stream);
/* DIGEST-A parameter server ("downloads/uploads parameters from the PS without
 * blindly waiting for the slowest subgraph"; P:243 aggregation moved into the subgraph
 * loop).  Upload = mixing W_global <- (1 - alpha) W_global + alpha W_local (reading R1,
 * S:383/S:426; alpha in (0, 1], 1/M by default), download = W_local <- W_global.
 * digest_ps_mix / digest_ps_download: W_global is a caller device buffer (one process;
 * the caller orders the uploads).  digest_ps_*_peer: W_global lives in rank 0's
 * peer-memory window (count <= the window's max_grad_count); each call is one kernel
 * that holds a system-scope lock in that window, so uploads from independent processes
 * are atomic and no rank ever waits for another's epoch.  digest_ps_init_peer (rank 0
 * only) sets W_global; digest_ps_updates_peer reads the upload count (synchronous). */
digest_status digest_ps_mix(float* W_global, const float* W_local, int64_t count, float alpha,
                            void* stream);
digest_status digest_ps_download(const float* W_global, float* W_local, int64_t count,
                                 void* stream);
digest_status digest_ps_init_peer(digest_comm* comm, const float* W0, int64_t count,
                                  void* stream);
digest_status digest_ps_upload_peer(digest_comm* comm, const float* W_local, int64_t count,
                                    float alpha, void* stream);
digest_status digest_ps_download_peer(digest_comm* comm, float* W_local, int64_t count,
                                      void* stream);
digest_status digest_ps_updates_peer(digest_comm* comm, int64_t* updates_h);
/* Straggler injection ("a random delay ... added to the chosen straggler"; SPEC
 * inject_delay): a one-thread kernel that spins for `ns` nanoseconds on `stream`. */
digest_status digest_delay(int64_t ns, void* stream);
/* Alg. 1 local update W <- W - lr*G. */
digest_status digest_sgd_step(float* W, const float* G, int64_t count, float lr, void* stream);
/* Adam, bias-corrected, step >= 1. */
digest_status digest_adam_step(float* W, const float* G, float* m, float* v, int64_t count,
                               float lr, float b1, float b2, float eps, int64_t step,
                               void* stream);

/* The same with the step count in device memory (*step_dev = updates done so far; this
 * call uses step *step_dev + 1 and then increments it), so an epoch captured in a CUDA
 * graph replays with the right bias correction. */
digest_status digest_adam_step_dev(float* W, const float* G, float* m, float* v, int64_t count,
                                   float lr, float b1, float b2, float eps, int64_t* step_dev,
                                   void* stream);

/* ------------------------------------------------------------------ dense helper
 * C[M x N] = op(A[M x K] B[K x N]) in fp32 on the path the layer uses (exposed for
 * tests, the GEMM roofline and the stale halo-gradient term).  flags bit0
 * (DIGEST_GEMM_RELU): ReLU epilogue; bit1 (DIGEST_GEMM_BT): B is given transposed, as
 * an N x K row-major matrix (ldb >= K), so C = A B^T -- e.g. S W^T with W d_in x d_out. */
enum { DIGEST_GEMM_RELU = 1u, DIGEST_GEMM_BT = 2u };
digest_status digest_gemm(const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                          int64_t ldc, int64_t M, int32_t N, int32_t K, uint32_t flags,
                          void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DIGEST_H */
