// Internal layout of the partition handle.
#pragma once
#include <vector>

#include "common.cuh"

struct digest_part {
  int64_t num_nodes = 0, n_local = 0, n_halo = 0, nnz = 0, nnz_in = 0, n_send = 0, rh_nnz = 0;
  int32_t num_parts = 0, rank = 0;
  int64_t max_row = 0, max_rh_row = 0;
  int64_t hot_rows = 0;          // extended columns flagged (bit 31 of col/rh_col) as L2-hot
  std::vector<int64_t> send_count, send_off, recv_count, recv_off;
  // device arrays, owned
  int32_t* local_ids = nullptr;  // [n_local]
  int32_t* halo_ids = nullptr;   // [n_halo]
  int64_t* row_ptr = nullptr;    // [n_local+1]
  int32_t* col = nullptr;        // [nnz] extended column | bit 31: L2-hot source row
  float* val = nullptr;          // [nnz]
  int32_t* in_len = nullptr;     // [n_local] entries with col < n_local (they come first)
  int32_t* send_idx = nullptr;   // [n_send]
  int64_t* rh_ptr = nullptr;     // [n_halo+1]
  int32_t* rh_col = nullptr;     // [rh_nnz]
  float* rh_val = nullptr;       // [rh_nnz]
  // row orders for the grouped narrow SpMM (internal): rows grouped by length bin within
  // windows of consecutive rows, for P (full rows), P_in (in_len) and P_out^T (rh rows)
  int32_t* ord_full = nullptr;   // [n_local]
  int32_t* ord_in = nullptr;     // [n_local]
  int32_t* ord_rh = nullptr;     // [n_halo]
  // loss-row products (digest_part_set_loss_mask): P_in and P_out^T restricted to the
  // columns (local rows) whose mask is set -- the only rows of the last layer's gradient
  // operand that can be nonzero.  Same entry order as col / rh_col; empty when unset.
  int64_t lm_nnz = -1, lmh_nnz = 0;   // lm_nnz < 0: no loss mask set
  int64_t* lm_ptr = nullptr;     // [n_local+1]
  int32_t* lm_col = nullptr;     // [lm_nnz]
  float* lm_val = nullptr;
  int32_t* ord_lm = nullptr;     // [n_local]
  int64_t* lmh_ptr = nullptr;    // [n_halo+1]
  int32_t* lmh_col = nullptr;    // [lmh_nnz]
  float* lmh_val = nullptr;
  int32_t* ord_lmh = nullptr;    // [n_halo]
};
