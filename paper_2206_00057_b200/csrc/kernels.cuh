// Internal kernel entry points shared by the layer, store and ABI files.
#pragma once
#include "common.cuh"

namespace dg {

// Y[i, 0:w] = act( sum_{e in row i} val[e] * Xsrc(col[e])[0:w] ),
// Xsrc(c) = X0 + c*ld0 if c < split else X1 + (c - split)*ld1.
// row range of row i: [row_ptr[i], row_ptr[i] + in_len[i]) if in_len != NULL
// (the in-block P_in part, whose entries come first), else [row_ptr[i], row_ptr[i+1]).
struct SpmmArgs {
  const int64_t* row_ptr;
  const int32_t* in_len;
  const int32_t* col;
  const float* val;
  int64_t n_rows;
  int64_t nnz;   // entries the call traverses (for the byte model / GTEPS)
  const float* X0;
  int64_t ld0;
  int64_t split;
  const float* X1;
  int64_t ld1;
  float* Y;
  int64_t ldy;
  int32_t width;
  int32_t relu;
  const float* mask;   // optional: Y *= 1[mask > 0] (fused ReLU' of the consumer layer)
  int64_t ldm;
  const uint32_t* mbits;   // optional: Y *= bit(mbits, row, col) (the 1-bit form of `mask`)
  int64_t ldmb;            // words per mbits row
  uint32_t* obits;         // optional: write bit(obits, row, col) = Y[row, col] > 0
  int64_t ldob;
  int32_t hints;       // L2 evict_last on gathers / evict_first on CSR streams
  int32_t full_width;  // column-slab launches: width of the whole product (accounting; 0 = width)
  int32_t stream_out;  // 1: evict-first (st.global.cs) stores of the output rows
  int64_t x0_rows;     // rows of X0 (0 = unknown); the TMA row-gather kernel needs it
  int64_t csr_len;     // entries of col/val (0 = unknown); bounds the CSR-tile staging
  const int32_t* order;  // optional: the rows grouped by length within windows (partition-built;
                         // the grouped narrow kernel processes rows in this order)
};
// 1-bit activation masks: bit (col & 31) of word row * ld + (col >> 5).
__device__ __forceinline__ bool mask_bit(const uint32_t* bits, int64_t ld, int64_t row, int col) {
  return (__ldg(bits + row * ld + (col >> 5)) >> (col & 31)) & 1u;
}
digest_status spmm(const SpmmArgs& a, cudaStream_t s);
// Allocates (once) the work counters of the grouped SpMM; called at partition build, so no
// allocation happens inside a launch that may be stream-captured.  false on failure.
bool spmm_counters_init();

// C = A * B (+ optional ReLU) with generic strides:
//   A(i,k) = A[i*sAi + k*sAk],  B(k,j) = B[k*sBk + j*sBj],  C[i*ldc + j].
struct GemmArgs {
  const float* A;
  int64_t sAi, sAk;
  const float* B;
  int64_t sBk, sBj;
  float* C;
  int64_t ldc;
  int64_t M;
  int32_t N;
  int64_t K;
  int32_t relu;
  const float* mask;   // optional: C *= 1[mask > 0] (fused ReLU' of the consumer layer)
  int64_t ldm;
  const uint32_t* mbits;   // optional: C *= bit(mbits, i, j)
  int64_t ldmb;
  uint32_t* obits;         // optional: bit(obits, i, j) = C[i, j] > 0
  int64_t ldob;
};
digest_status gemm(const GemmArgs& g, cudaStream_t s);        // dispatch (tensor core if eligible)
digest_status gemm_simt(const GemmArgs& g, cudaStream_t s);   // CUDA-core fp32
bool gemm_tc_eligible(const GemmArgs& g);                      // 3xTF32 tcgen05 path applies
digest_status gemm_tc(const GemmArgs& g, cudaStream_t s);     // 3xTF32 on tcgen05 (sm_100a)

// Weight gradient over a very long K: C[M x N] (dense, ld = N) = sum over segments of
// A_seg^T B_seg with A_seg [K_seg x M] (ld lda), B_seg [K_seg x N] (ld ldb).
// Split-K with a fixed-order second pass (deterministic).  `mask` (optional, per
// segment) multiplies B by 1[mask > 0] elementwise (ReLU' from the layer output).
struct WgradSeg {
  const float* A;
  int64_t lda;
  const float* B;
  int64_t ldb;
  const float* mask;
  int64_t ldm;
  int64_t K;
};
size_t wgrad_scratch_bytes(int64_t K_total, int32_t M, int32_t N);
digest_status wgrad(const WgradSeg* segs, int nseg, int32_t M, int32_t N, float* C,
                    void* scratch, cudaStream_t s);       // dispatch (tensor core if eligible)
digest_status wgrad_simt(const WgradSeg* segs, int nseg, int32_t M, int32_t N, float* C,
                         void* scratch, cudaStream_t s);

// D = G o 1[H > 0] (n x w)
digest_status relu_mask(const float* G, int64_t ldg, const float* H, int64_t ldh, float* D,
                        int64_t ldd, int64_t n, int32_t w, cudaStream_t s);
// D = G o bit(mbits) (n x w)
digest_status relu_mask_bits(const float* G, int64_t ldg, const uint32_t* mbits, int64_t ldmb,
                             float* D, int64_t ldd, int64_t n, int32_t w, cudaStream_t s);
// bits(i, j) = C[i, j] > 0 for j < w; the pad bits of each row's last word are 0
digest_status sign_bits(const float* C, int64_t ldc, int64_t n, int32_t w, uint32_t* bits,
                        int64_t ldb, cudaStream_t s);

}  // namespace dg
