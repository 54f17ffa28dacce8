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
#include "dmma.cuh"

#ifndef LEAF_MARK
#define LEAF_MARK(d, ev)
#endif

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

// One warp: C(16 x 16) = A(16 x 16) * op(B) on FP64 DMMA (m16n8k4, two n8
// tiles), A(i, k) = A[i + k*LD64], B(k, n) = B[k*bk + n*bn] (BC: conjugated).
// c[q][ni][r]: q = re / im plane; element (g + 8(r>>1), 8ni + 2t + (r&1)).
template <typename T> struct Frag16 {
  double c[is_cplx<T>::value ? 2 : 1][2][4];
};

template <typename T, bool BC, bool ACC = false>
__device__ __forceinline__ void mm16_warp(const T* A, const T* B, int bk, int bn, Frag16<T>& f) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  constexpr bool CPLX = is_cplx<T>::value;
  __syncwarp();  // mma.sync.aligned needs the converged warp
  if constexpr (!ACC) {
#pragma unroll
    for (int q = 0; q < (CPLX ? 2 : 1); ++q)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni)
#pragma unroll
        for (int r = 0; r < 4; ++r) f.c[q][ni][r] = 0.0;
  }
#pragma unroll
  for (int k0 = 0; k0 < 16; k0 += 4) {
    const int k = k0 + t;
    const T a0 = A[g + k * LD64], a1 = A[g + 8 + k * LD64];
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      T b = B[k * bk + (8 * ni + g) * bn];
      if (BC) b = conj_(b);
      if constexpr (!CPLX) {
        dmma16x8x4(f.c[0][ni], a0, a1, b);
      } else {
        dmma16x8x4(f.c[0][ni], a0.x, a1.x, b.x);
        dmma16x8x4(f.c[0][ni], -a0.y, -a1.y, b.y);
        dmma16x8x4(f.c[1][ni], a0.x, a1.x, b.y);
        dmma16x8x4(f.c[1][ni], a0.y, a1.y, b.x);
      }
    }
  }
}

template <typename T, class F>
__device__ __forceinline__ void frag16_each(const Frag16<T>& f, F fn) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int ni = 0; ni < 2; ++ni)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = g + ((r & 2) ? 8 : 0), j = 8 * ni + 2 * t + (r & 1);
      if constexpr (is_cplx<T>::value) fn(i, j, Z{f.c[0][ni][r], f.c[1][ni][r]});
      else fn(i, j, f.c[0][ni][r]);
    }
}

// One warp: right-looking Cholesky of the 16 columns [c0, c0 + 16) of the
// 32 x 32 lower block of S at (off, off), rows c0 .. 31 (lane i holds row i's
// 16 panel entries; lanes below c0 idle).  The pivot column is broadcast
// through colk (double-buffered); the next pivot is taken straight from lane
// p+1's registers and its rsqrt issued before the trailing update, so the
// serial chain per step is mul -> fma -> shfl -> rsqrt.  16-wide rows keep the
// per-step update short enough that this chain, not the warp's in-order
// issue of the update, sets the pace.  Returns 0 or the failing pivot
// (1-based within the 32-block; `not d > 0` catches NaN, kernels.py:441).
template <typename T>
__device__ __noinline__ int chol_panel16(T* S, int off, int c0, T* colk) {
  const int lane = threadIdx.x & 31;
  const bool act = lane >= c0;
  T* prow = S + (off + lane) + (off + c0) * LD64;
  T r[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) r[j] = act ? prow[j * LD64] : zero_<T>();
  int fail = 0;
  double dkk = shfl(sc_re(r[0]), c0);
  double rd = rsqrt_pivot(dkk);
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int p = c0 + k;
    if (!(dkk > 0.0)) fail = fail ? fail : p + 1;
    const T lk = (lane == p) ? sc_from<T>(dkk * rd) : rd * r[k];
    r[k] = lk;
    double dnext = 1.0;
    if (k + 1 < 16) dnext = shfl(sc_re(fnmac(lk, conj_(lk), r[k + 1])), p + 1);
    T* cb = colk + (k & 1) * 32;
    cb[lane] = conj_(lk);
    __syncwarp();
    const double rd_next = rsqrt_pivot(dnext);
    if constexpr (is_cplx<T>::value) {
#pragma unroll
      for (int j = k + 1; j < 16; ++j) r[j] = fnmac(lk, cb[c0 + j], r[j]);
    } else {
#pragma unroll
      for (int jj = (k + 1) & ~1; jj < 16; jj += 2) {
        const double2 c2 = *reinterpret_cast<const double2*>(cb + c0 + jj);
        if (jj >= k + 1) r[jj] = fnmac(lk, c2.x, r[jj]);
        r[jj + 1] = fnmac(lk, c2.y, r[jj + 1]);
      }
    }
    dkk = dnext;
    rd = rd_next;
  }
  if (fail) return fail;
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (act && c0 + j <= lane) prow[j * LD64] = r[j];
  __syncwarp();
  return 0;
}

// One warp: in-place Cholesky (A = L L^H) of the 32 x 32 lower block of S at
// (off, off): panel [0, 16) (L11 and L21), A22 -= L21 L21^H on DMMA, panel
// [16, 32).  Returns 0 or the 1-based failing pivot (warp-uniform).
template <typename T>
__device__ __noinline__ int chol32_warp(T* S, int off, T* colk) {
  int f = chol_panel16(S, off, 0, colk);
  if (f) return f;
  const T* L21 = S + (off + 16) + off * LD64;
  Frag16<T> fr;
  mm16_warp<T, true>(L21, L21, LD64, 1, fr);  // B(k, n) = conj(L21(n, k))
  T* A22 = S + (off + 16) + (off + 16) * LD64;
  frag16_each(fr, [&](int i, int j, T v) {
    if (j <= i) A22[i + j * LD64] = A22[i + j * LD64] - v;
  });
  __syncwarp();
  return chol_panel16(S, off, 16, colk);
}

// The same panel over the 64 x 32 block [A11; A21] of the leaf (S at 0, 0):
// lane i also carries row 32 + i, which the pivot column broadcasts update
// too, so L21 = A21 L11^-H comes out of the factorization's own broadcasts
// (no inverse of L11 on the critical path).  Returns 0 or the failing pivot.
template <typename T>
__device__ __noinline__ int chol_panel16x2(T* S, int c0, T* colk) {
  const int lane = threadIdx.x & 31;
  const bool act = lane >= c0;
  T* prow = S + lane + c0 * LD64;
  T* qrow = prow + 32;
  T r[16], q[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    r[j] = act ? prow[j * LD64] : zero_<T>();
    q[j] = qrow[j * LD64];
  }
  int fail = 0;
  double dkk = shfl(sc_re(r[0]), c0);
  double rd = rsqrt_pivot(dkk);
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int p = c0 + k;
    if (!(dkk > 0.0)) fail = fail ? fail : p + 1;
    const T lk = (lane == p) ? sc_from<T>(dkk * rd) : rd * r[k];
    const T mk = rd * q[k];
    r[k] = lk;
    q[k] = mk;
    double dnext = 1.0;
    if (k + 1 < 16) dnext = shfl(sc_re(fnmac(lk, conj_(lk), r[k + 1])), p + 1);
    T* cb = colk + (k & 1) * 32;
    cb[lane] = conj_(lk);
    __syncwarp();
    const double rd_next = rsqrt_pivot(dnext);
    if constexpr (is_cplx<T>::value) {
#pragma unroll
      for (int j = k + 1; j < 16; ++j) {
        const T c = cb[c0 + j];
        r[j] = fnmac(lk, c, r[j]);
        q[j] = fnmac(mk, c, q[j]);
      }
    } else {
#pragma unroll
      for (int jj = (k + 1) & ~1; jj < 16; jj += 2) {
        const double2 c2 = *reinterpret_cast<const double2*>(cb + c0 + jj);
        if (jj >= k + 1) {
          r[jj] = fnmac(lk, c2.x, r[jj]);
          q[jj] = fnmac(mk, c2.x, q[jj]);
        }
        r[jj + 1] = fnmac(lk, c2.y, r[jj + 1]);
        q[jj + 1] = fnmac(mk, c2.y, q[jj + 1]);
      }
    }
    dkk = dnext;
    rd = rd_next;
  }
  if (fail) return fail;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (act && c0 + j <= lane) prow[j * LD64] = r[j];
    qrow[j * LD64] = q[j];
  }
  __syncwarp();
  return 0;
}

// One warp: L11 and L21 of the leaf's first 32 columns, [A11; A21] =
// [L11; L21] L11^H: panel [0, 16) over 64 rows, rows 16..63 of columns
// [16, 32) -= (their first 16 columns) L(16..31, 0..15)^H on DMMA, panel
// [16, 32) over rows 16..63.  Returns 0 or the 1-based failing pivot.
template <typename T>
__device__ __noinline__ int chol64x32_warp(T* S, T* colk) {
  int f = chol_panel16x2(S, 0, colk);
  if (f) return f;
  const T* Lb = S + 16;  // B(k, n) = conj(L(16 + n, k))
#pragma unroll 1
  for (int rb = 16; rb < 64; rb += 16) {
    Frag16<T> fr;
    mm16_warp<T, true>(S + rb, Lb, LD64, 1, fr);
    T* C = S + rb + 16 * LD64;
    const bool diag = rb == 16;
    frag16_each(fr, [&](int i, int j, T v) {
      if (!diag || j <= i) C[i + j * LD64] = C[i + j * LD64] - v;
    });
  }
  __syncwarp();
  return chol_panel16x2(S, 16, colk);
}

// One warp: Y = L21 W11 (32 x 32, W11 lower) into Y (LD64 smem), as four
// 16 x 16 blocks (the block above W11's diagonal skipped)
template <typename T>
__device__ __noinline__ void mm_l21_w11_warp(const T* L21, const T* W11, T* Y) {
#pragma unroll 1
  for (int bi = 0; bi < 2; ++bi)
#pragma unroll 1
    for (int bj = 0; bj < 2; ++bj) {
      Frag16<T> fr;
      // sum over kb >= bj (W11(kb, bj) = 0 for kb < bj)
      mm16_warp<T, false>(L21 + 16 * bi + 16 * bj * LD64, W11 + 16 * bj + 16 * bj * LD64, 1,
                          LD64, fr);
      if (bj == 0)
        mm16_warp<T, false, true>(L21 + 16 * bi + 16 * LD64, W11 + 16, 1, LD64, fr);
      T* Yb = Y + 16 * bi + 16 * bj * LD64;
      frag16_each(fr, [&](int i, int j, T v) { Yb[i + j * LD64] = v; });
    }
  __syncwarp();
}

// One warp: W(offw.., offw..) = inverse of the 32 x 32 lower block of S at
// (off, off), zeros above the diagonal.  The two 16 x 16 diagonal inverses
// run side by side (lane j < 16: column j of W11; lane 16 + j: of W22),
// right-looking (w_k = s_k / L_kk, s_i -= L(i, k) w_k: the chain per step is
// one multiply and one FMA); then W21 = -W22 (L21 W11) on DMMA, with L21 W11
// staged in W's upper-right block (zeroed afterwards).
template <typename T>
__device__ __noinline__ void inv32_warp(const T* S, int off, T* W, int offw, bool unit, T* rdiag) {
  const int lane = threadIdx.x & 31, h = lane >> 4, j = lane & 15;
  const T* L = S + (off + 16 * h) + (off + 16 * h) * LD64;
  rdiag[lane] = unit ? one_<T>() : one_<T>() / L[j + j * LD64];
  __syncwarp();
  T sv[16], w[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) sv[i] = (i == j) ? one_<T>() : zero_<T>();
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    w[k] = sv[k] * rdiag[16 * h + k];
#pragma unroll
    for (int i = k + 1; i < 16; ++i) sv[i] = fnmac(L[i + k * LD64], w[k], sv[i]);
  }
  T* wc = W + (offw + 16 * h) + (offw + 16 * h + j) * LD64;
#pragma unroll
  for (int i = 0; i < 16; ++i) wc[i] = (i >= j) ? w[i] : zero_<T>();
  __syncwarp();
  T* W11 = W + offw + offw * LD64;
  T* W12 = W11 + 16 * LD64;
  T* W21 = W11 + 16;
  T* W22 = W12 + 16;
  Frag16<T> fr;
  mm16_warp<T, false>(S + (off + 16) + off * LD64, W11, 1, LD64, fr);  // L21 W11
  frag16_each(fr, [&](int i, int c, T v) { W12[i + c * LD64] = v; });
  __syncwarp();
  mm16_warp<T, false>(W22, W12, 1, LD64, fr);  // W22 (L21 W11)
  __syncwarp();
  frag16_each(fr, [&](int i, int c, T v) {
    W21[i + c * LD64] = zero_<T>() - v;
    W12[i + c * LD64] = zero_<T>();
  });
  __syncwarp();
}

// 128 threads: R(32x32) = X * op(Y) over 32 x 32 blocks of LD64 smem tiles on
// FP64 DMMA; warp w owns the two 16 x 8 tiles of columns 8w .. 8w+7.  X is
// read as X[i][k], Y as Y[k][j] (YT: Y[j][k], YC: conjugated).
template <typename T> struct Frag32 {
  double c[is_cplx<T>::value ? 2 : 1][2][4];
};

template <typename T, bool YT, bool YC>
__device__ __forceinline__ void mm32_mma(const T* X, int xr, int xc, const T* Y, int yr, int yc,
                                         Frag32<T>& f) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  constexpr bool CPLX = is_cplx<T>::value;
  __syncwarp();  // mma.sync.aligned needs the converged warp (lane-0 fail flags precede)
#pragma unroll
  for (int q = 0; q < (CPLX ? 2 : 1); ++q)
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int r = 0; r < 4; ++r) f.c[q][mi][r] = 0.0;
  const int nj = 8 * w + g;
#pragma unroll
  for (int k0 = 0; k0 < 32; k0 += 4) {
    const int k = k0 + t;
    T b = YT ? Y[(yr + nj) + (yc + k) * LD64] : Y[(yr + k) + (yc + nj) * LD64];
    if (YC) b = conj_(b);
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const T a0 = X[(xr + mi * 16 + g) + (xc + k) * LD64];
      const T a1 = X[(xr + mi * 16 + g + 8) + (xc + k) * LD64];
      if constexpr (!CPLX) {
        dmma16x8x4(f.c[0][mi], a0, a1, b);
      } else {
        dmma16x8x4(f.c[0][mi], a0.x, a1.x, b.x);
        dmma16x8x4(f.c[0][mi], -a0.y, -a1.y, b.y);
        dmma16x8x4(f.c[1][mi], a0.x, a1.x, b.y);
        dmma16x8x4(f.c[1][mi], a0.y, a1.y, b.x);
      }
    }
  }
}

// fn(i, j, v) for every element of the warp's fragments
template <typename T, class F>
__device__ __forceinline__ void frag32_each(const Frag32<T>& f, F fn) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = mi * 16 + g + ((r & 2) ? 8 : 0), j = 8 * w + 2 * t + (r & 1);
      if constexpr (is_cplx<T>::value) fn(i, j, Z{f.c[0][mi][r], f.c[1][mi][r]});
      else fn(i, j, f.c[0][mi][r]);
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
    cta_sync();
  }
  // Y = L21 * W11  (scratch: S rows 0..31, cols 32..63)
  Frag32<T> f;
  mm32_mma<T, false, false>(S, 32, 0, W, 0, 0, f);
  frag32_each(f, [&](int i, int j, T v) { S[i + (32 + j) * LD64] = v; });
  cta_sync();
  // W21 = -W22 * Y ; W12 = 0
  mm32_mma<T, false, false>(W, 32, 32, S, 0, 32, f);
  frag32_each(f, [&](int i, int j, T v) {
    W[(32 + i) + j * LD64] = zero_<T>() - v;
    W[i + (32 + j) * LD64] = zero_<T>();
  });
}

// The whole 64-leaf on 128 threads: S (lower, LD64, identity-padded) is
// factored in place (S = L, upper part scratch) and, when Ws is given, its
// inverse formed in Ws (zeros above the diagonal).  Returns 0 or the 1-based
// failing pivot, uniform over the CTA (s_fail: a __shared__ int).  Callers
// sync before (S ready) and after.
template <typename T>
__device__ int leaf_factor_inv64(T* S, T* Ws, T* scratch, int* s_fail, int trace_id = -1) {
  // warp 0 carries the pivot chain: [L11; L21] in one 64-row panel, then
  // L22 after the 4-warp update A22 -= L21 L21^H; meanwhile warp 1 inverts
  // L11 and forms Y = L21 W11 (staged in S's unused upper-right block), so
  // only L22's inverse and W21 = -W22 Y follow the chain
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) *s_fail = 0;
  cta_sync();
  if (warp == 0) {
    const int f = chol64x32_warp(S, scratch);
    if (lane == 0 && f) *s_fail = f;
  }
  cta_sync();
  LEAF_MARK(trace_id, 8);
  if (*s_fail) return *s_fail;
  Frag32<T> f;
  mm32_mma<T, true, true>(S, 32, 0, S, 32, 0, f);  // L21 L21^H
  frag32_each(f, [&](int i, int j, T v) {
    if (j <= i) S[(32 + i) + (32 + j) * LD64] = S[(32 + i) + (32 + j) * LD64] - v;
  });
  cta_sync();
  LEAF_MARK(trace_id, 9);
  if (warp == 0) {
    const int fl = chol32_warp(S, 32, scratch);
    if (lane == 0 && fl) *s_fail = 32 + fl;
  } else if (warp == 1) {
    inv32_warp(S, 0, Ws, 0, false, scratch + 64);
    mm_l21_w11_warp(S + 32, Ws, S + 32 * LD64);
  }
  cta_sync();
  LEAF_MARK(trace_id, 10);
  if (*s_fail) return *s_fail;
  if (warp == 0) inv32_warp(S, 32, Ws, 32, false, scratch);
  cta_sync();
  LEAF_MARK(trace_id, 11);
  // W21 = -W22 Y ; W12 = 0
  mm32_mma<T, false, false>(Ws, 32, 32, S, 0, 32, f);
  frag32_each(f, [&](int i, int j, T v) {
    Ws[(32 + i) + j * LD64] = zero_<T>() - v;
    Ws[i + (32 + j) * LD64] = zero_<T>();
  });
  LEAF_MARK(trace_id, 12);
  return 0;
}

}  // namespace rfpk
