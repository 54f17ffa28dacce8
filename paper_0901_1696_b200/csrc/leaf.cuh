// Shared-memory / register building blocks for the 64 x 64 diagonal leaves.
//
// A leaf is split 2 x 2 into 32 x 32 blocks.  The 32 x 32 Cholesky and the
// 32 x 32 triangular inverse each run on ONE warp over shared memory (lane i
// owns row i for the Cholesky, column i for the inverse; only __syncwarp, no
// CTA barriers); the 32 x 32 off-diagonal products use all four warps.
// Leaves are stored column-major in shared memory with a 65-element stride
// (conflict-free columns).  Loops are kept rolled on purpose: a fully
// unrolled register version compiled to ~36k SASS instructions and ran
// 10x slower from instruction-cache misses.
#pragma once
#include "common.cuh"

namespace rfpk {

constexpr int LD64 = 65;

__device__ __forceinline__ double shfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ Z shfl(Z v, int src) {
  return Z{__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src)};
}

template <typename T> __device__ __forceinline__ T zero_() { return sc_from<T>(0.0); }
template <typename T> __device__ __forceinline__ T one_() { return sc_from<T>(1.0); }

// Load the lower triangle of an n x n view (n <= 64) into S (col-major, LD64);
// the strict upper part is zeroed and rows/cols >= n are padded with the
// identity, so the padded leaf factors / inverts to the identity.
template <typename T>
__device__ void leaf_load_lower(T* S, const View<T> A, int n) {
  const int nt = blockDim.x;
  if (A.rs == 1 || A.n == 1) {
    for (int e = threadIdx.x; e < 64 * 64; e += nt) {
      const int i = e & 63, j = e >> 6;
      T v = (i == j) ? one_<T>() : zero_<T>();
      if (i < n && j < n && i >= j) v = *A.at(i, j);
      S[i + j * LD64] = v;
    }
  } else {
    for (int e = threadIdx.x; e < 64 * 64; e += nt) {
      const int j = e & 63, i = e >> 6;
      T v = (i == j) ? one_<T>() : zero_<T>();
      if (i < n && j < n && i >= j) v = *A.at(i, j);
      S[i + j * LD64] = v;
    }
  }
}

// Store the lower triangle (optionally without the diagonal) of S into A.
template <typename T>
__device__ void leaf_store_lower(const T* S, View<T> A, int n, bool skip_diag) {
  const int nt = blockDim.x;
  if (A.rs == 1 || A.n == 1) {
    for (int e = threadIdx.x; e < n * n; e += nt) {
      const int i = e % n, j = e / n;
      if (i > j || (i == j && !skip_diag)) *A.at(i, j) = S[i + j * LD64];
    }
  } else {
    for (int e = threadIdx.x; e < n * n; e += nt) {
      const int j = e % n, i = e / n;
      if (i > j || (i == j && !skip_diag)) *A.at(i, j) = S[i + j * LD64];
    }
  }
}

// One warp: in-place Cholesky (A = L L^H) of the 32 x 32 lower block of S at
// (off, off), right-looking, lane i owning row i.  Loops stay rolled (the
// leaf kernels must fit the instruction cache).  Returns 0 or the 1-based
// failing pivot (warp-uniform); `not d > 0` catches NaN (kernels.py:441).
template <typename T>
__device__ int chol32_warp(T* S, int off) {
  const int i = threadIdx.x & 31;
  T* B = S + off + off * LD64;
  for (int k = 0; k < 32; ++k) {
    const double dkk = sc_re(B[k + k * LD64]);
    if (!(dkk > 0.0)) return k + 1;
    const double d = sqrt(dkk);
    T lik = zero_<T>();
    if (i > k) {
      lik = B[i + k * LD64] / d;
      B[i + k * LD64] = lik;
    }
    __syncwarp();
    if (i == k) B[k + k * LD64] = sc_from<T>(d);
    if (i > k) {
#pragma unroll 4
      for (int j = k + 1; j <= i; ++j) B[i + j * LD64] = fnmac(lik, conj_(B[j + k * LD64]), B[i + j * LD64]);
    }
    __syncwarp();
  }
  return 0;
}

// One warp: W(offw.., offw..) = inverse of the 32 x 32 lower block of S at
// (off, off); lane j computes column j (zeros above the diagonal).
template <typename T>
__device__ void inv32_warp(const T* S, int off, T* W, int offw, bool unit) {
  const int j = threadIdx.x & 31;
  const T* L = S + off + off * LD64;
  T* w = W + offw + (offw + j) * LD64;
  for (int i = 0; i < 32; ++i) {
    if (i < j) {
      w[i] = zero_<T>();
      continue;
    }
    T s0 = (i == j) ? one_<T>() : zero_<T>(), s1 = zero_<T>();
    int k = j;
    for (; k + 1 < i; k += 2) {
      s0 = fnmac(L[i + k * LD64], w[k], s0);
      s1 = fnmac(L[i + (k + 1) * LD64], w[k + 1], s1);
    }
    if (k < i) s0 = fnmac(L[i + k * LD64], w[k], s0);
    const T s = s0 + s1;
    w[i] = unit ? s : s / L[i + i * LD64];
  }
  __syncwarp();
}

// 128 threads: R(32x32) = op(X) * op(Y) over 32 x 32 blocks of LD64 smem
// tiles.  Thread t computes rows (t & 31), columns 8*(t>>5) .. +7, returned
// in `acc`; X is read as X[i][k] and Y as Y[k][j] (Ytrans: Y[j][k], with
// optional conjugation).
template <typename T, bool YT, bool YC>
__device__ __forceinline__ void mm32(const T* X, int xr, int xc, const T* Y, int yr, int yc,
                                     T acc[8]) {
  const int i = threadIdx.x & 31, jg = (threadIdx.x >> 5) * 8;
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = zero_<T>();
#pragma unroll 8
  for (int k = 0; k < 32; ++k) {
    const T x = X[(xr + i) + (xc + k) * LD64];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int j = jg + q;
      T y = YT ? Y[(yr + j) + (yc + k) * LD64] : Y[(yr + k) + (yc + j) * LD64];
      if (YC) y = conj_(y);
      acc[q] = fmac(x, y, acc[q]);
    }
  }
}

// Full inverse of the 64 x 64 lower leaf in S into W (zeros above the
// diagonal).  Needs 128 threads; S's upper-right 32 x 32 block is used as
// scratch.  Caller syncs before (S ready) and after.
template <typename T>
__device__ void inv64_block(T* S, T* W, bool unit, bool both_diag_done) {
  const int warp = threadIdx.x >> 5;
  if (!both_diag_done) {
    if (warp == 0) inv32_warp(S, 0, W, 0, unit);
    if (warp == 1) inv32_warp(S, 32, W, 32, unit);
    __syncthreads();
  }
  // Y = L21 * W11  (scratch: S rows 0..31, cols 32..63)
  T acc[8];
  mm32<T, false, false>(S, 32, 0, W, 0, 0, acc);
  const int i = threadIdx.x & 31, jg = (threadIdx.x >> 5) * 8;
#pragma unroll
  for (int q = 0; q < 8; ++q) S[i + (32 + jg + q) * LD64] = acc[q];
  __syncthreads();
  // W21 = -W22 * Y ; W12 = 0
  mm32<T, false, false>(W, 32, 32, S, 0, 32, acc);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    W[(32 + i) + (jg + q) * LD64] = zero_<T>() - acc[q];
    W[i + (32 + jg + q) * LD64] = zero_<T>();
  }
}

}  // namespace rfpk
