// Shared-memory / register building blocks for the 64 x 64 diagonal leaves.
//
// A leaf is split 2 x 2 into 32 x 32 blocks.  The 32 x 32 Cholesky and the
// 32 x 32 triangular inverse each run on ONE warp with the block in registers
// (lane i owns row i for the Cholesky, column i for the inverse; shuffles and
// shared-memory broadcasts, no CTA barriers); the 32 x 32 off-diagonal
// products use all four warps.  Leaves are stored column-major in shared
// memory with a 65-element stride (conflict-free columns).  The unrolled
// 32-blocks are __noinline__ so each kernel holds ONE copy: inlining every
// call site (and per-element divisions) produced ~36k SASS instructions per
// kernel and a 10x slowdown from instruction-cache misses.
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

// 1/sqrt(x) for x > 0: MUFU seed + Newton steps (relative error ~1 ulp).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y = rsqrt(x);
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  return y;
}

// One warp: in-place Cholesky (A = L L^H) of the 32 x 32 lower block of S at
// (off, off), right-looking, lane i holding row i in registers.  Column k is
// broadcast through a 32-entry shared-memory vector (one LDS per update, no
// shuffles); the trailing update runs unpredicated on every lane -- values
// that land above the diagonal are never read back or stored, so lower
// entries only ever combine valid factor entries.  Not inlined: one copy of
// the unrolled body serves both diagonal blocks.  Returns 0 or the 1-based
// failing pivot (warp-uniform); `not d > 0` catches NaN (kernels.py:441).
template <typename T>
__device__ __noinline__ int chol32_warp(T* S, int off, T* colk) {
  const int lane = threadIdx.x & 31;
  T r[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) r[j] = S[(off + lane) + (off + j) * LD64];
  int fail = 0;
  double dkk = shfl(sc_re(r[0]), 0);
  double rd = rsqrt(dkk);
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (!(dkk > 0.0)) fail = fail ? fail : k + 1;
    const T lk = (lane == k) ? sc_from<T>(dkk * rd) : rd * r[k];
    r[k] = lk;
    // the next pivot straight from lane k+1's own registers (its update with
    // its own lk); its rsqrt is issued before this step's trailing update so
    // the two overlap -- the serial chain per step is mul -> fma -> shfl ->
    // rsqrt, everything else runs beside it
    double dnext = 1.0;
    if (k + 1 < 32) dnext = shfl(sc_re(fnmac(lk, conj_(lk), r[k + 1])), k + 1);
    T* cb = colk + (k & 1) * 32;  // double-buffered column broadcast
    cb[lane] = conj_(lk);
    __syncwarp();
    const double rd_next = rsqrt(dnext);
#pragma unroll
    for (int j = k + 1; j < 32; ++j) r[j] = fnmac(lk, cb[j], r[j]);
    dkk = dnext;
    rd = rd_next;
  }
  if (fail) return fail;
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if (j <= lane) S[(off + lane) + (off + j) * LD64] = r[j];
  return 0;
}

// One warp: W(offw.., offw..) = inverse of the 32 x 32 lower block of S at
// (off, off); lane j holds column j of W in registers (rows above j are 0).
// Row i of L is read with shared-memory broadcasts; reciprocals of the
// diagonal are computed once per lane into `rdiag`.
template <typename T>
__device__ __noinline__ void inv32_warp(const T* S, int off, T* W, int offw, bool unit, T* rdiag) {
  const int j = threadIdx.x & 31;
  const T* L = S + off + off * LD64;
  rdiag[j] = unit ? one_<T>() : one_<T>() / L[j + j * LD64];
  __syncwarp();
  T w[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    T s0 = (i == j) ? one_<T>() : zero_<T>(), s1 = zero_<T>();
#pragma unroll
    for (int k = 0; k < i; ++k) {
      if (k & 1) s1 = fnmac(L[i + k * LD64], w[k], s1);
      else s0 = fnmac(L[i + k * LD64], w[k], s0);
    }
    w[i] = (s0 + s1) * rdiag[i];
  }
  T* wc = W + offw + (offw + j) * LD64;
#pragma unroll
  for (int i = 0; i < 32; ++i) wc[i] = (i >= j) ? w[i] : zero_<T>();
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
__device__ void inv64_block(T* S, T* W, bool unit, bool both_diag_done, T* scratch) {
  const int warp = threadIdx.x >> 5;
  if (!both_diag_done) {
    if (warp == 0) inv32_warp(S, 0, W, 0, unit, scratch);
    if (warp == 1) inv32_warp(S, 32, W, 32, unit, scratch + 32);
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

// The whole 64-leaf on 128 threads: S (lower, LD64, identity-padded) is
// factored in place (S = L, upper part scratch) and, when Ws is given, its
// inverse formed in Ws (zeros above the diagonal).  Returns 0 or the 1-based
// failing pivot, uniform over the CTA (s_fail: a __shared__ int).  Callers
// sync before (S ready) and after.
template <typename T>
__device__ int leaf_factor_inv64(T* S, T* Ws, T* scratch, int* s_fail) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) *s_fail = 0;
  __syncthreads();
  if (warp == 0) {
    const int f = chol32_warp(S, 0, scratch);
    if (lane == 0 && f) *s_fail = f;
  }
  __syncthreads();
  if (*s_fail) return *s_fail;
  if (warp == 0) inv32_warp(S, 0, Ws, 0, false, scratch);
  __syncthreads();
  const int i = threadIdx.x & 31, jg = (threadIdx.x >> 5) * 8;
  T acc[8];
  mm32<T, true, true>(S, 32, 0, Ws, 0, 0, acc);  // L21 = A21 W11^H
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 8; ++q) S[(32 + i) + (jg + q) * LD64] = acc[q];
  __syncthreads();
  mm32<T, true, true>(S, 32, 0, S, 32, 0, acc);  // L21 L21^H
#pragma unroll
  for (int q = 0; q < 8; ++q)
    if (jg + q <= i) S[(32 + i) + (32 + jg + q) * LD64] = S[(32 + i) + (32 + jg + q) * LD64] - acc[q];
  __syncthreads();
  if (warp == 0) {
    const int f = chol32_warp(S, 32, scratch);
    if (lane == 0 && f) *s_fail = 32 + f;
  }
  __syncthreads();
  if (*s_fail) return *s_fail;
  if (warp == 1) inv32_warp(S, 32, Ws, 32, false, scratch + 32);
  __syncthreads();
  inv64_block(S, Ws, false, true, scratch);
  return 0;
}

}  // namespace rfpk
