// FP64 / complex128 tensor-core GEMM on sm_100a.
//
// FP64 has no tcgen05 kind on sm_100a (ptxas rejects kind::f64), so the
// tensor-core path for double is the warp-level DMMA: mma.sync m16n8k4 f64
// (SASS DMMA.8x8x4).  Operands are staged global->shared with 8-byte (real)
// or 16-byte (complex) cp.async in a multi-stage pipeline; RFP blocks with an
// odd leading dimension (real TRANSR='N', ldar odd) are only 8-byte aligned,
// which rules out TMA tensor maps and 16-byte vectors for them.
//
// C <- alpha * op(A) * op(B) + beta * C, where A (M x K) and B (K x N) are
// strided views that are either contiguous along M/N ("MN-major") or along
// K ("K-major"), and C is column-major.  TRI_LOWER / TRI_UPPER restrict the
// update to one triangle of a square C (SYRK/HERK), launching only the tiles
// that intersect it and masking the diagonal tiles, so the other triangle --
// which in RFP storage physically holds the other diagonal block -- is never
// written (reference: kernels.py:341-351 `_blend_tri`).
#pragma once
#include "common.cuh"

namespace rfpk {

template <typename T> struct GemmArgs {
  int M, N, K;
  const T* A;
  i64 lda;
  const T* B;
  i64 ldb;
  T* C;
  i64 ldc;
  T alpha, beta;
  int conjA, conjB;   // complex only
  int herm_diag;      // complex TRI modes: force Im(C_ii) = 0
  const int* skip;    // device flag: nonzero -> do nothing (failed factorization)
  int tiles_m;        // tiles along M (for the triangular mapping)
  int a_tri;          // A operand mask: 0 none, 1 lower, 2 upper, 3 strict lower, 4 strict upper, 5 upper band
  int b_tri;          // same mask applied to B (k, n) as if it were A (n, k) (transposed problems)
  long long ntiles;   // tiles of the launch (CTAs stride over them)
  int band;           // TRI square tiles: rows per band of the rasterised order (0: row by row)
};


// A-operand triangle masks (for triangular-times-matrix leaves)
// A_UBAND: upper-triangular operand whose lower part is already zero in
// memory -- only the K band is narrowed, no per-element mask
enum ATri : int { A_FULL = 0, A_LOWER = 1, A_UPPER = 2, A_SLOWER = 3, A_SUPPER = 4, A_UBAND = 5 };


template <typename T>
int gemm(int tri_mode, T alpha, View<T> A, bool conjA, View<T> B, bool conjB, T beta,
         View<T> C, bool herm_diag, const int* skip, cudaStream_t st, int a_tri = A_FULL,
         bool inplace_leaf = false);
// inplace_leaf: C aliases B and M <= 64; the launch uses one CTA row (BM >= M) so
// every CTA reads its whole B column block before writing it back.

// in-place complex conjugation of a view (no-op for real)
template <typename T> int conj_view(View<T> C, const int* skip, cudaStream_t st);

// scale/zero a (possibly triangular) view: C <- beta*C (beta == 0 writes zeros)
template <typename T>
int scale_view(View<T> C, T beta, int tri_mode, bool herm_diag, const int* skip, cudaStream_t st);

}  // namespace rfpk
