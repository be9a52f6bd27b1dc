// digest_layer_fwd / digest_layer_bwd: one GCN layer of DIGEST on partition m.
//
// Forward, Eq. 5:  H = sigma(P_in X_in W + P_out X~_out W) = sigma(P_m X_ext W)
//   AGG_FIRST:   A = P_m X_ext (SpMM, width d_in)       -> saved
//                H = sigma(A W) (GEMM + ReLU epilogue)
//   XFORM_FIRST: T = X_ext W    (GEMM over n_local + n_halo rows, width d_out)
//                H = sigma(P_m T) (SpMM + ReLU epilogue)
// Backward, Eq. 6 and P:783-794, halo constant:
//   D = G o 1[H > 0]
//   AGG_FIRST:   G_W = A^T D;  G_in = P_in^T (D W^T) = P_in (D W^T)      (P_in symmetric)
//   XFORM_FIRST: S_loc = P_in^T D = P_in D,  S_halo = P_out^T D (reverse-halo CSR)
//                G_W = X_loc^T S_loc + X_halo^T S_halo;  G_in = S_loc W^T
// P_in is the principal block P[V_m, V_m] of the symmetric P, so P_in^T = P_in and
// the in-block part of each forward CSR row (its first in_len entries) serves the
// transposed product without a second copy; only P_out^T needs the reverse CSR.
#include "kernels.cuh"
#include "part_internal.cuh"

namespace dg {

digest_status gemm(const GemmArgs& g, cudaStream_t s) {
  if (g.M == 0 || g.N == 0) return DIGEST_OK;
  return gemm_tc_eligible(g) ? gemm_tc(g, s) : gemm_simt(g, s);
}

}  // namespace dg

namespace {

using dg::round_up;

struct Plan {
  bool agg_first;
  int64_t n, h;
  int64_t ldi, ldo;   // padded widths of d_in / d_out scratch rows
  int64_t ldmb;       // 32-bit words per row of the 1-bit ReLU mask (multiple of 4)
  size_t bits_off;    // byte offset of the mask inside `saved`
  size_t saved, scratch;
};

digest_status make_plan(const digest_part* p, int32_t d_in, int32_t d_out, int32_t order,
                        Plan* pl) {
  DG_ARG(p, DIGEST_E_INVALID, "NULL partition");
  DG_ARG(d_in > 0 && d_out > 0, DIGEST_E_SHAPE, "d_in/d_out must be positive");
  DG_ARG(d_in % 4 == 0 && d_out % 4 == 0, DIGEST_E_SHAPE,
         "d_in (%d) and d_out (%d) must be multiples of 4 (pad features/classes)", d_in, d_out);
  DG_ARG(order >= 0 && order <= 2, DIGEST_E_INVALID, "bad order");
  pl->agg_first = order == DIGEST_ORDER_AUTO ? d_in <= d_out : order == DIGEST_ORDER_AGG_FIRST;
  pl->n = p->n_local;
  pl->h = p->n_halo;
  pl->ldi = round_up(d_in, 4);
  pl->ldo = round_up(d_out, 4);
  const size_t f = sizeof(float);
  // every scratch sub-buffer is carved with the same 256-byte rounding as carve()
  auto r = [](size_t b) { return (size_t)round_up((int64_t)b, 256); };
  size_t wg = dg::wgrad_scratch_bytes(pl->n + pl->h, d_in, d_out);
  pl->ldmb = round_up((d_out + 31) / 32, 4);
  if (pl->agg_first) {
    pl->saved = f * pl->n * pl->ldi;
    size_t bwd = r(f * pl->n * pl->ldo) + r(f * pl->n * pl->ldi) + wg;
    pl->scratch = bwd;
  } else {
    pl->saved = 0;
    size_t fwd = r(f * (pl->n + pl->h) * pl->ldo);
    size_t bwd = r(f * pl->n * pl->ldo) + r(f * (pl->n + pl->h) * pl->ldo) + wg;
    pl->scratch = fwd > bwd ? fwd : bwd;
  }
  // saved = [A (AGG_FIRST) | 1-bit ReLU mask of H, n x ldmb words]
  pl->bits_off = round_up(pl->saved, 256);
  pl->saved = pl->bits_off + sizeof(uint32_t) * pl->n * pl->ldmb;
  pl->saved = round_up(pl->saved, 256);
  pl->scratch = round_up(pl->scratch, 256);
  return DIGEST_OK;
}

digest_status check_mat(const void* p, int64_t ld, int32_t w, const char* name) {
  DG_ARG(p, DIGEST_E_INVALID, "%s is NULL", name);
  DG_ARG(ld >= w && ld % 4 == 0, DIGEST_E_INVALID, "%s: ld %lld must be >= %d and a multiple of 4",
         name, (long long)ld, w);
  DG_ARG(((uintptr_t)p & 15) == 0, DIGEST_E_INVALID, "%s must be 16-byte aligned", name);
  return DIGEST_OK;
}

float* carve(void* base, size_t& off, size_t bytes) {
  float* p = reinterpret_cast<float*>(reinterpret_cast<char*>(base) + off);
  off += round_up(bytes, 256);
  return p;
}

dg::SpmmArgs spmm_full(const digest_part* p, const float* X0, int64_t ld0, const float* X1,
                       int64_t ld1, float* Y, int64_t ldy, int32_t w, int relu) {
  dg::SpmmArgs a{};
  a.row_ptr = p->row_ptr;
  a.in_len = nullptr;
  a.col = p->col;
  a.val = p->val;
  a.n_rows = p->n_local;
  a.nnz = p->nnz;
  a.X0 = X0;
  a.ld0 = ld0;
  a.split = p->n_local;
  a.x0_rows = p->n_local;
  a.csr_len = p->nnz;
  a.X1 = p->n_halo > 0 ? X1 : nullptr;   // no halo columns: a single-source product
  a.ld1 = ld1;
  a.Y = Y;
  a.ldy = ldy;
  a.width = w;
  a.relu = relu;
  a.order = p->ord_full;
  return a;
}

dg::SpmmArgs spmm_in(const digest_part* p, const float* X, int64_t ld, float* Y, int64_t ldy,
                     int32_t w) {
  dg::SpmmArgs a = spmm_full(p, X, ld, X, ld, Y, ldy, w, 0);
  a.in_len = p->in_len;
  a.nnz = p->nnz_in;
  a.order = p->ord_in;
  return a;
}

// The loss-row forms (digest_part_set_loss_mask): the same products over the CSRs that keep
// only the columns whose operand row can be nonzero (the training rows of the last layer's
// gradient), in the same entry order -- the dropped terms are exact zeros.
dg::SpmmArgs spmm_lm(const digest_part* p, const float* X, int64_t ld, float* Y, int64_t ldy,
                     int32_t w) {
  dg::SpmmArgs a{};
  a.row_ptr = p->lm_ptr;
  a.order = p->ord_lm;
  a.col = p->lm_col;
  a.val = p->lm_val;
  a.n_rows = p->n_local;
  a.nnz = p->lm_nnz;
  a.csr_len = p->lm_nnz;
  a.X0 = X;
  a.ld0 = ld;
  a.split = INT64_MAX;
  a.x0_rows = p->n_local;
  a.X1 = X;
  a.ld1 = ld;
  a.Y = Y;
  a.ldy = ldy;
  a.width = w;
  return a;
}
dg::SpmmArgs spmm_lmh(const digest_part* p, const float* X, int64_t ld, float* Y, int64_t ldy,
                      int32_t w) {
  dg::SpmmArgs a = spmm_lm(p, X, ld, Y, ldy, w);
  a.row_ptr = p->lmh_ptr;
  a.order = p->ord_lmh;
  a.col = p->lmh_col;
  a.val = p->lmh_val;
  a.n_rows = p->n_halo;
  a.nnz = p->lmh_nnz;
  a.csr_len = p->lmh_nnz;
  return a;
}

// Y (n_halo rows) = P_out^T X over the reverse-halo CSR (halo row j -> local columns).
dg::SpmmArgs spmm_rh(const digest_part* p, const float* X, int64_t ld, float* Y, int64_t ldy,
                     int32_t w) {
  dg::SpmmArgs a{};
  a.row_ptr = p->rh_ptr;
  a.in_len = nullptr;
  a.order = p->ord_rh;
  a.col = p->rh_col;
  a.val = p->rh_val;
  a.n_rows = p->n_halo;
  a.nnz = p->rh_nnz;
  a.csr_len = p->rh_nnz;
  a.X0 = X;
  a.ld0 = ld;
  a.split = INT64_MAX;
  a.x0_rows = p->n_local;
  a.X1 = X;
  a.ld1 = ld;
  a.Y = Y;
  a.ldy = ldy;
  a.width = w;
  return a;
}

dg::GemmArgs gemm_rm(const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                     int64_t ldc, int64_t M, int32_t N, int64_t K, int relu) {
  dg::GemmArgs g{};
  g.A = A;
  g.sAi = lda;
  g.sAk = 1;
  g.B = B;
  g.sBk = ldb;
  g.sBj = 1;
  g.C = C;
  g.ldc = ldc;
  g.M = M;
  g.N = N;
  g.K = K;
  g.relu = relu;
  return g;
}

}  // namespace

extern "C" {

digest_status digest_layer_workspace(const digest_part* part, int32_t d_in, int32_t d_out,
                                     int32_t order, size_t* saved_bytes_h,
                                     size_t* scratch_bytes_h) {
  Plan pl;
  DG_TRY(make_plan(part, d_in, d_out, order, &pl));
  if (saved_bytes_h) *saved_bytes_h = pl.saved;
  if (scratch_bytes_h) *scratch_bytes_h = pl.scratch;
  return DIGEST_OK;
}

digest_status digest_layer_fwd(const digest_part* p, const float* X_local, int64_t ld_x,
                               const float* X_halo, int64_t ld_xh, const float* W, int32_t d_in,
                               int32_t d_out, int32_t act, int32_t order, uint32_t flags,
                               float* H_out, int64_t ld_h, void* saved, void* scratch,
                               void* stream) {
  Plan pl;
  DG_TRY(make_plan(p, d_in, d_out, order, &pl));
  const bool reuse = (flags & DIGEST_FWD_REUSE_SAVED) != 0;
  DG_ARG(!reuse || pl.agg_first, DIGEST_E_INVALID,
         "DIGEST_FWD_REUSE_SAVED needs the aggregate-first order (saved holds A = P_m X_ext)");
  DG_ARG(act == DIGEST_ACT_NONE || act == DIGEST_ACT_RELU, DIGEST_E_INVALID, "bad act");
  DG_TRY(check_mat(X_local, ld_x, d_in, "X_local"));
  if (pl.h > 0) DG_TRY(check_mat(X_halo, ld_xh, d_in, "X_halo"));
  DG_TRY(check_mat(H_out, ld_h, d_out, "H_out"));
  DG_ARG(W, DIGEST_E_INVALID, "W is NULL");
  const int relu = act == DIGEST_ACT_RELU;
  DG_ARG(saved || !(pl.agg_first || relu), DIGEST_E_INVALID, "saved is NULL");
  DG_ARG(pl.agg_first || scratch, DIGEST_E_INVALID, "scratch is NULL");
  cudaStream_t s = dg::as_stream(stream);
  // ReLU layers also emit the 1-bit mask 1[H > 0] into saved: the
  // backward's sigma' reads 1/32 of the bytes of H.
  uint32_t* bits = relu ? reinterpret_cast<uint32_t*>(static_cast<char*>(saved) + pl.bits_off)
                        : nullptr;
  if (pl.agg_first) {
    float* A = reinterpret_cast<float*>(saved);
    if (!reuse)   // A = P_m X_ext; with REUSE_SAVED the caller's static inputs were aggregated before
      DG_TRY(dg::spmm(spmm_full(p, X_local, ld_x, X_halo, ld_xh, A, pl.ldi, d_in, 0), s));
    dg::GemmArgs g = gemm_rm(A, pl.ldi, W, d_out, H_out, ld_h, pl.n, d_out, d_in, relu);
    g.obits = bits;
    g.ldob = pl.ldmb;
    DG_TRY(dg::gemm(g, s));
  } else {
    size_t off = 0;
    float* T = carve(scratch, off, sizeof(float) * (pl.n + pl.h) * pl.ldo);
    DG_TRY(dg::gemm(gemm_rm(X_local, ld_x, W, d_out, T, pl.ldo, pl.n, d_out, d_in, 0), s));
    if (pl.h > 0)
      DG_TRY(dg::gemm(gemm_rm(X_halo, ld_xh, W, d_out, T + pl.n * pl.ldo, pl.ldo, pl.h, d_out,
                              d_in, 0), s));
    dg::SpmmArgs a = spmm_full(p, T, pl.ldo, T + pl.n * pl.ldo, pl.ldo, H_out, ld_h, d_out, relu);
    a.obits = bits;
    a.ldob = pl.ldmb;
    DG_TRY(dg::spmm(a, s));
  }
  return DIGEST_OK;
}

digest_status digest_layer_mask(const digest_part* p, int32_t d_in, int32_t d_out, int32_t order,
                                const void* saved, const uint32_t** bits_h,
                                int64_t* ld_words_h) {
  Plan pl;
  DG_TRY(make_plan(p, d_in, d_out, order, &pl));
  DG_ARG(saved && bits_h && ld_words_h, DIGEST_E_INVALID, "NULL argument");
  *bits_h = reinterpret_cast<const uint32_t*>(static_cast<const char*>(saved) + pl.bits_off);
  *ld_words_h = pl.ldmb;
  return DIGEST_OK;
}

digest_status digest_layer_bwd(const digest_part* p, const float* X_local, int64_t ld_x,
                               const float* X_halo, int64_t ld_xh, const float* W, int32_t d_in,
                               int32_t d_out, int32_t act, int32_t order, const void* saved,
                               const float* H_out, int64_t ld_h, const float* G_out, int64_t ld_g,
                               uint32_t flags, float* G_W, float* G_in, int64_t ld_gi,
                               const void* gin_mask, int64_t ld_gm, float* G_halo,
                               int64_t ld_gh, void* scratch, void* stream) {
  Plan pl;
  DG_TRY(make_plan(p, d_in, d_out, order, &pl));
  DG_ARG(act == DIGEST_ACT_NONE || act == DIGEST_ACT_RELU, DIGEST_E_INVALID, "bad act");
  DG_TRY(check_mat(G_out, ld_g, d_out, "G_out"));
  const bool g_is_d = (flags & DIGEST_BWD_G_IS_D) != 0;
  const bool gm_bits = (flags & DIGEST_BWD_GIN_MASK_BITS) != 0;
  // sigma' of this layer: the 1-bit mask the forward left in saved; H_out only if
  // saved is NULL (transform-first layers may be called without it)
  const bool d_from_bits = act == DIGEST_ACT_RELU && !g_is_d && saved != nullptr;
  if (act == DIGEST_ACT_RELU && !g_is_d && !saved) DG_TRY(check_mat(H_out, ld_h, d_out, "H_out"));
  if (G_in) DG_TRY(check_mat(G_in, ld_gi, d_in, "G_in"));
  if (G_in && gin_mask && !gm_bits) DG_TRY(check_mat(gin_mask, ld_gm, d_in, "gin_mask"));
  if (G_in && gin_mask && gm_bits)
    DG_ARG(ld_gm >= (d_in + 31) / 32, DIGEST_E_INVALID, "gin_mask (bits): ld %lld words < %d",
           (long long)ld_gm, (d_in + 31) / 32);
  const float* gm_f = gm_bits ? nullptr : static_cast<const float*>(gin_mask);
  const uint32_t* gm_b = gm_bits ? static_cast<const uint32_t*>(gin_mask) : nullptr;
  const bool save_s = (flags & DIGEST_BWD_HALO_SAVE_S) != 0;   // G_halo <- P_out^T D
  // DIGEST_BWD_LOSS_ROWS: G_out's rows outside the loss mask are zero, so the P_in / P_out^T
  // products of D (and of U = D W^T) run over the loss-row CSRs
  const bool lrows = (flags & DIGEST_BWD_LOSS_ROWS) != 0;
  DG_ARG(!lrows || p->lm_nnz >= 0, DIGEST_E_STATE,
         "DIGEST_BWD_LOSS_ROWS without digest_part_set_loss_mask");
  auto p_in = [&](const float* X, int64_t ld, float* Y, int64_t ldy, int32_t w) {
    return lrows ? spmm_lm(p, X, ld, Y, ldy, w) : spmm_in(p, X, ld, Y, ldy, w);
  };
  auto p_rh = [&](const float* X, int64_t ld, float* Y, int64_t ldy, int32_t w) {
    return lrows ? spmm_lmh(p, X, ld, Y, ldy, w) : spmm_rh(p, X, ld, Y, ldy, w);
  };
  if (G_halo && pl.h > 0) DG_TRY(check_mat(G_halo, ld_gh, save_s ? d_out : d_in, "G_halo"));
  const bool want_halo = G_halo && pl.h > 0;
  DG_ARG(W && G_W && scratch, DIGEST_E_INVALID, "W, G_W and scratch must be non-NULL");
  cudaStream_t s = dg::as_stream(stream);
  size_t off = 0;
  // D = G o sigma'(Z)   (sigma'(Z) = 1[H > 0] for ReLU, ReLU'(0) := 0); with
  // DIGEST_BWD_G_IS_D the producer of G_out already applied it (gin_mask of the
  // next layer's backward), so no separate masking pass runs.
  const float* D = G_out;
  int64_t ldd = ld_g;
  if (act == DIGEST_ACT_RELU && !g_is_d) {
    float* Dm = carve(scratch, off, sizeof(float) * pl.n * pl.ldo);
    if (d_from_bits)
      DG_TRY(dg::relu_mask_bits(G_out, ld_g,
                                reinterpret_cast<const uint32_t*>(
                                    static_cast<const char*>(saved) + pl.bits_off),
                                pl.ldmb, Dm, pl.ldo, pl.n, d_out, s));
    else
      DG_TRY(dg::relu_mask(G_out, ld_g, H_out, ld_h, Dm, pl.ldo, pl.n, d_out, s));
    D = Dm;
    ldd = pl.ldo;
  } else {
    carve(scratch, off, sizeof(float) * pl.n * pl.ldo);
  }
  if (pl.agg_first) {
    DG_ARG(saved, DIGEST_E_INVALID, "saved is NULL");
    const float* A = reinterpret_cast<const float*>(saved);
    float* U = carve(scratch, off, sizeof(float) * pl.n * pl.ldi);
    void* wsc = carve(scratch, off, 0);
    dg::WgradSeg seg{A, pl.ldi, D, ldd, nullptr, 0, pl.n};
    DG_TRY(dg::wgrad(&seg, 1, d_in, d_out, G_W, wsc, s));
    if (G_in || (want_halo && !save_s)) {
      // U = D W^T : B(k, j) = W[j, k]
      dg::GemmArgs g = gemm_rm(D, ldd, W, d_out, U, pl.ldi, pl.n, d_in, d_out, 0);
      g.sBk = 1;
      g.sBj = d_out;
      DG_TRY(dg::gemm(g, s));
    }
    if (G_in) {
      dg::SpmmArgs a = p_in(U, pl.ldi, G_in, ld_gi, d_in);
      a.mask = gm_f;
      a.ldm = ld_gm;
      a.mbits = gm_b;
      a.ldmb = ld_gm;
      DG_TRY(dg::spmm(a, s));
    }
    if (want_halo && save_s)   // S = P_out^T D~^(t), returned next iteration
      DG_TRY(dg::spmm(p_rh(D, ldd, G_halo, ld_gh, d_out), s));
    else if (want_halo)        // same-iteration return: G_halo = P_out^T U
      DG_TRY(dg::spmm(p_rh(U, pl.ldi, G_halo, ld_gh, d_in), s));
  } else {
    DG_TRY(check_mat(X_local, ld_x, d_in, "X_local"));
    if (pl.h > 0) DG_TRY(check_mat(X_halo, ld_xh, d_in, "X_halo"));
    float* S = carve(scratch, off, sizeof(float) * (pl.n + pl.h) * pl.ldo);
    void* wsc = carve(scratch, off, 0);
    DG_TRY(dg::spmm(p_in(D, ldd, S, pl.ldo, d_out), s));
    // S_halo = P_out^T D (reverse-halo CSR, no atomics); with HALO_SAVE_S written
    // straight into the caller's G_halo, which also feeds the weight gradient
    float* Sh = want_halo && save_s ? G_halo : S + pl.n * pl.ldo;
    const int64_t ldsh = want_halo && save_s ? ld_gh : pl.ldo;
    if (pl.h > 0) DG_TRY(dg::spmm(p_rh(D, ldd, Sh, ldsh, d_out), s));
    dg::WgradSeg segs[2] = {{X_local, ld_x, S, pl.ldo, nullptr, 0, pl.n},
                            {X_halo, ld_xh, Sh, ldsh, nullptr, 0, pl.h}};
    DG_TRY(dg::wgrad(segs, pl.h > 0 ? 2 : 1, d_in, d_out, G_W, wsc, s));
    if (G_in) {
      dg::GemmArgs g = gemm_rm(S, pl.ldo, W, d_out, G_in, ld_gi, pl.n, d_in, d_out, 0);
      g.sBk = 1;
      g.sBj = d_out;
      g.mask = gm_f;
      g.ldm = ld_gm;
      g.mbits = gm_b;
      g.ldmb = ld_gm;
      DG_TRY(dg::gemm(g, s));
    }
    if (want_halo && !save_s) {   // same-iteration return: G_halo = S_halo W^T
      dg::GemmArgs g = gemm_rm(S + pl.n * pl.ldo, pl.ldo, W, d_out, G_halo, ld_gh, pl.h, d_in,
                               d_out, 0);
      g.sBk = 1;
      g.sBj = d_out;
      DG_TRY(dg::gemm(g, s));
    }
  }
  return DIGEST_OK;
}

digest_status digest_propagate(const digest_part* p, int32_t mode, const float* X_local,
                               int64_t ld_x, const float* X_halo, int64_t ld_xh, int32_t width,
                               float* Y, int64_t ld_y, void* stream) {
  DG_ARG(p, DIGEST_E_INVALID, "NULL partition");
  DG_ARG(mode >= 0 && mode <= 2, DIGEST_E_INVALID, "bad mode");
  DG_ARG(width > 0 && width % 4 == 0, DIGEST_E_SHAPE, "width must be a positive multiple of 4");
  DG_TRY(check_mat(X_local, ld_x, width, "X_local"));
  if (mode == 0 && p->n_halo > 0) DG_TRY(check_mat(X_halo, ld_xh, width, "X_halo"));
  if (mode != 2 || p->n_halo > 0) DG_TRY(check_mat(Y, ld_y, width, "Y"));
  cudaStream_t s = dg::as_stream(stream);
  if (mode == 0) return dg::spmm(spmm_full(p, X_local, ld_x, X_halo, ld_xh, Y, ld_y, width, 0), s);
  if (mode == 1) return dg::spmm(spmm_in(p, X_local, ld_x, Y, ld_y, width), s);
  return dg::spmm(spmm_rh(p, X_local, ld_x, Y, ld_y, width), s);
}

digest_status digest_gemm(const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                          int64_t ldc, int64_t M, int32_t N, int32_t K, uint32_t flags,
                          void* stream) {
  DG_ARG(A && B && C, DIGEST_E_INVALID, "NULL matrix");
  const bool bt = (flags & DIGEST_GEMM_BT) != 0;
  DG_ARG(M >= 0 && N > 0 && K > 0 && lda >= K && ldb >= (bt ? K : N) && ldc >= N,
         DIGEST_E_SHAPE, "bad GEMM shape");
  dg::GemmArgs g = gemm_rm(A, lda, B, ldb, C, ldc, M, N, K, (int)(flags & DIGEST_GEMM_RELU));
  if (bt) {   // B(k, j) = B_given[j, k]
    g.sBk = 1;
    g.sBj = ldb;
  }
  return dg::gemm(g, dg::as_stream(stream));
}

}  // extern "C"
