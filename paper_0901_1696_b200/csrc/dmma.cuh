// Device building blocks of the DMMA GEMM shared by gemm.cu and the tiled
// dataflow Cholesky (tile_potrf.cu): cp.async helpers, the m16n8k4 FP64 MMA,
// conflict-free shared-memory stage layouts and the hoisted tile loader.
#pragma once
#include "gemm.cuh"

namespace rfpk {

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
// D += A(16x4, row) * B(4x8, col); fragments per the PTX m16n8k4 f64 layout
// (verified on the B200 by tools/probe_mma.cu): a0=(g,t) a1=(g+8,t), b=(t,g),
// c0..c3 = (g,2t) (g,2t+1) (g+8,2t) (g+8,2t+1) with g = lane/4, t = lane%4.
__device__ __forceinline__ void dmma16x8x4(double* c, double a0, double a1, double b) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

__device__ __forceinline__ bool a_keep(int a_tri, int m, int k) {
  switch (a_tri) {
    case A_LOWER: return m >= k;
    case A_UPPER: return m <= k;
    case A_SLOWER: return m > k;
    case A_SUPPER: return m < k;
    default: return true;
  }
}

// ------------------------------------------------------------ tile loader
// Global -> shared copy of one operand tile (R rows along M or N, BK along K)
// with all addressing hoisted out of the K loop: each thread owns EPT
// elements at a fixed stride, so a stage costs one 64-bit add + one cp.async
// per element.  The K tail and the triangular masks (a_tri / b_tri, used only
// by the in-place triangular leaves) take a separate predicated path.
// Shared-memory layout of one operand stage.  MN-major operands are stored
// [k][r] with pitch R + 4 (complex R + 2), K-major ones [r][k] with pitch
// BK + 4, so both the cp.async stores (contiguous along the global fast
// dimension) and the m16n8k4 fragment loads are bank-conflict free.
template <typename T, int R, int BK, bool KM>
struct SmemLayout {
  static constexpr int P = KM ? BK + 4 : R + (is_cplx<T>::value ? 2 : 4);
  static constexpr int SIZE = KM ? R * P : BK * P;  // elements per stage
  static constexpr int RS = KM ? P : 1;             // stride between rows r
  static constexpr int KS = KM ? 1 : P;             // stride between k
};

template <typename T, int R, int BK, int NT, bool KMAJOR>
struct TileLoader {
  using L = SmemLayout<T, R, BK, KMAJOR>;
  static constexpr int EPT = R * BK / NT;
  static_assert(R * BK % NT == 0, "tile must divide evenly");
  static constexpr int RE = KMAJOR ? NT / BK : 0;   // row delta per element
  static constexpr int KE = KMAJOR ? 0 : NT / R;    // k delta per element
  static constexpr int SSTEP = RE * L::RS + KE * L::KS;
  const T* ptr;     // element 0 at the current k0
  i64 step;         // global delta between consecutive elements
  i64 kstep;        // global delta per stage
  int r0, k_0;      // tile coords of element 0
  int soff;         // smem offset of element 0
  unsigned rowok;   // bit e: row of element e inside the matrix

  __device__ __forceinline__ void init(const T* base, i64 ld, int tile0, int rows, int tid) {
    if (KMAJOR) { k_0 = tid % BK; r0 = tid / BK; }
    else { r0 = tid % R; k_0 = tid / R; }
    // element (r, k) at base + r*ld + k (KMAJOR) or base + r + k*ld
    ptr = KMAJOR ? base + (i64)(tile0 + r0) * ld + k_0 : base + (tile0 + r0) + (i64)k_0 * ld;
    step = KMAJOR ? (i64)RE * ld : (i64)KE * ld;
    kstep = KMAJOR ? (i64)BK : (i64)BK * ld;
    soff = r0 * L::RS + k_0 * L::KS;
    rowok = 0;
#pragma unroll
    for (int e = 0; e < EPT; ++e)
      if (tile0 + r0 + e * RE < rows) rowok |= 1u << e;
  }

  // fast path: full K range, no mask
  __device__ __forceinline__ void load(T* s) const {
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      if (rowok & (1u << e)) {
        cp_async_t(s + soff + e * SSTEP, ptr + e * step, true);
      } else {
        cp_async_t(s + soff + e * SSTEP, ptr, false);
      }
    }
  }
  // tail / masked path: K bound and triangle mask (tri on (row, k) coords)
  __device__ __forceinline__ void load_pred(T* s, int k0, int K, int tile0, int tri) const {
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const int r = tile0 + r0 + e * RE, k = k0 + k_0 + e * KE;
      const bool ok = (rowok & (1u << e)) && k < K && a_keep(tri, r, k);
      cp_async_t(s + soff + e * SSTEP, ok ? ptr + e * step : ptr, ok);
    }
  }
  __device__ __forceinline__ void advance() { ptr += kstep; }
  __device__ __forceinline__ void skip(int stages) { ptr += (i64)stages * kstep; }

  __device__ __forceinline__ static void cp_async_t(T* s, const T* g, bool ok) {
    if constexpr (sizeof(T) == 8) cp_async8(s, g, ok);
    else cp_async16(s, g, ok);
  }
};

}  // namespace rfpk
