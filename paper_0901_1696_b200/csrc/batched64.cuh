// Batched n = 64 RFP Cholesky factor + solve, ONE WARP PER MATRIX
// (BASELINE config 4: 65,536 x n = 64, TRANSR='N', UPLO='U', nrhs = 8).
//
// The matrix never leaves the RFP layout: the 65 x 32 normal rectangle of the
// 16,640-byte RFP buffer is copied into shared memory and the reference's
// SRPA composition (rfp.py:55-136) runs on the T1 / T2 / S1 views of that
// rectangle *inside shared memory*:
//
//   chol(T1) -> W1 = L1^-1 -> S <- S W1^T  -> T2 -= S S^T (its lower view)
//   -> chol(T2) -> W2
//   solve:  b1 = W1 b1; b2 -= S b1; b2 = W2 b2;  b2 = W2^T b2; b1 -= S^T b2;
//           b1 = W1^T b1
//
// with S = S1 for UPLO 'L' and S = S1^T for 'U' (the two compositions of
// rfp.py:70-89 / 118-136 are the same algebra on a transposed S1), the 32x32
// Cholesky and inverse on the warp's registers and every product on FP64 DMMA
// (mma.m16n8k4) fragments read from shared memory.  Only __syncwarp is needed,
// so twelve matrices (warps) are resident per SM.
//
// Shared-memory layout.  The kernel is bound by shared-memory wavefronts
// (ncu, profiles/r01_prof_batched_v3: LSU data pipe 89% busy), and a
// verbatim copy of the rectangle (ld 65) serves three access patterns that no
// single pitch makes conflict-free: column segments (lanes along r), row
// segments (lanes along c: transposed views) and the 4x4 (g, t) blocks of the
// DMMA operand fragments (odd pitch -> 4-way conflicts).  Column c therefore
// starts at colstart(c) = 1088*(c>>4) + 273*((c>>2)&3) + 68*(c&3): within
// every aligned group of 16 columns the starts are a permutation of the 16
// 8-byte banks, and within every aligned group of 4 they share one residue
// mod 4 -- which makes all three patterns conflict-free -- for 2176 doubles
// (17 KB) instead of 2080.
#pragma once
#include "common.cuh"

namespace rfpk {
namespace b64 {

constexpr int N = 64, H = 32, NT = N * (N + 1) / 2;  // 2080
constexpr int RECT = 2176;                             // swizzled 65 x 32 rectangle

__host__ __device__ constexpr int colstart(int c) {
  return 1088 * (c >> 4) + 273 * ((c >> 2) & 3) + 68 * (c & 3);
}

__device__ __forceinline__ double shfl(double v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

__device__ __forceinline__ void mma(double* c, double a0, double a1, double b) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

// Per-lane parts of the swizzled addresses of the fragment patterns
// (g = lane / 4, t = lane % 4); colstart is additive over aligned bit fields,
// colstart(8m + x) = colstart(8m) + colstart(x) for x < 8.
struct LaneOff {
  int o1;  // g + colstart(t)          (row R+g, column K+t)
  int o2;  // t + colstart(g)          (row K+t, column N+g)
  int o3;  // g + colstart(2t)         accumulator (R+g, N+2t), normal view
  int o4;  // 2t + colstart(g)         accumulator, transposed view
  __device__ __forceinline__ LaneOff() {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    o1 = g + colstart(t);
    o2 = t + colstart(g);
    o3 = g + colstart(2 * t);
    o4 = 2 * t + colstart(g);
  }
};

// A 32 x 32 view of the rectangle starting at row r0: element (i, j) is
// rect(r0 + i, j) (T = false) or rect(r0 + j, i) (T = true, a transposed
// block); p = smem base + r0.
template <bool T> struct RV {
  double* p;
  __device__ __forceinline__ double& operator()(int i, int j) const {
    return T ? p[j + colstart(i)] : p[i + colstart(j)];
  }
  // element (R + g, K + t); R a multiple of 8, K of 4 (compile-time)
  __device__ __forceinline__ double& gt(const LaneOff& o, int R, int K) const {
    return T ? p[o.o2 + K + colstart(R)] : p[o.o1 + R + colstart(K)];
  }
  // element (K + t, Nc + g)
  __device__ __forceinline__ double& tg(const LaneOff& o, int K, int Nc) const {
    return T ? p[o.o1 + Nc + colstart(K)] : p[o.o2 + K + colstart(Nc)];
  }
  // accumulator element (R + g, Nc + 2t + e)
  __device__ __forceinline__ double& acc(const LaneOff& o, int R, int Nc, int e) const {
    return T ? p[o.o4 + Nc + e + colstart(R)] : p[o.o3 + R + colstart(Nc) + colstart(e)];
  }
  __device__ __forceinline__ RV<!T> t() const { return RV<!T>{p}; }
};

// 32x32 lower Cholesky of the view in place (lower triangle only; the slots
// above it belong to the other RFP block) by one warp.  Lane i holds row i in
// registers; 32 right-looking steps, the pivot column broadcast through colk
// (64 entries, double-buffered).  Returns 0 or the 1-based failing pivot
// (warp-uniform; NaN fails like the reference's `not d > 0`, kernels.py:436).
template <bool T>
__device__ __noinline__ int factor32(double* p, double* colk) {
  __builtin_assume(__isShared(p));
  __builtin_assume(__isShared(colk));
  const int lane = threadIdx.x & 31;
  // row `lane`: element j at prow[T ? j : colstart(j)]
  double* prow = p + (T ? colstart(lane) : lane);
  double r[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) r[j] = (j <= lane) ? prow[T ? j : colstart(j)] : 0.0;
  int fail = 0;
  double dkk = shfl(r[0], 0);
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (!(dkk > 0.0)) fail = fail ? fail : k + 1;
    const double rd = rsqrt(dkk);
    const double lk = (lane == k) ? dkk * rd : rd * r[k];
    r[k] = lk;
    double dnext = 0.0;
    if (k + 1 < 32) dnext = shfl(fma(-lk, lk, r[k + 1]), k + 1);  // lane k+1's new pivot
    double* cb = colk + (k & 1) * 32;
    cb[lane] = lk;
    __syncwarp();
#pragma unroll
    for (int jj = (k + 1) & ~1; jj < 32; jj += 2) {
      const double2 c = *reinterpret_cast<const double2*>(cb + jj);
      if (jj >= k + 1) r[jj] = fma(-lk, c.x, r[jj]);
      r[jj + 1] = fma(-lk, c.y, r[jj + 1]);
    }
    dkk = dnext;
  }
  if (fail) return fail;
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if (j <= lane) prow[T ? j : colstart(j)] = r[j];
  __syncwarp();
  return 0;
}

// In-place inverse of the lower 32x32 view L (only the lower triangle is read
// or written).  Lane j computes column j; rdiag is a 32-entry scratch.  The
// substitution runs along L's unit-stride direction so that L is read two
// entries per 16-byte broadcast LDS: right-looking (column k of L per step)
// for a normal view, left-looking (row i per step) for a transposed one.  PAR
// is the parity of p's element offset from the 16-byte-aligned smem base, so
// the pairing is resolved at compile time.
template <bool T, int PAR>
__device__ __noinline__ void inv32(double* p, double* rdiag) {
  __builtin_assume(__isShared(p));
  __builtin_assume(__isShared(rdiag));
  const RV<T> L{p};
  const int j = threadIdx.x & 31;
  rdiag[j] = 1.0 / p[j + colstart(j)];
  __syncwarp();
  double w[32];
  if constexpr (!T) {
    // right-looking: s <- e_j; for k: w_k = s_k / L_kk; s_i -= L(i, k) w_k
    double sv[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) sv[i] = (i == j) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      w[k] = sv[k] * rdiag[k];
      int i = k + 1;
      if (i < 32 && ((PAR + i + colstart(k)) & 1)) {  // odd start: single load
        sv[i] = fma(-L(i, k), w[k], sv[i]);
        ++i;
      }
#pragma unroll
      for (; i + 1 < 32; i += 2) {
        const double2 q = *reinterpret_cast<const double2*>(&L(i, k));
        sv[i] = fma(-q.x, w[k], sv[i]);
        sv[i + 1] = fma(-q.y, w[k], sv[i + 1]);
      }
      if (i < 32) sv[i] = fma(-L(i, k), w[k], sv[i]);
    }
  } else {
    // left-looking along rows: w_i = (e_j(i) - sum_k L(i, k) w_k) / L_ii
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      double s0 = (i == j) ? 1.0 : 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int k = 0;
      if (i > 0 && ((PAR + colstart(i)) & 1)) {
        s0 = fma(-L(i, 0), w[0], s0);
        k = 1;
      }
#pragma unroll
      for (; k + 1 < i; k += 2) {
        const double2 q = *reinterpret_cast<const double2*>(&L(i, k));
        if ((k & 2) == 0) { s0 = fma(-q.x, w[k], s0); s1 = fma(-q.y, w[k + 1], s1); }
        else { s2 = fma(-q.x, w[k], s2); s3 = fma(-q.y, w[k + 1], s3); }
      }
      if (k < i) s1 = fma(-L(i, k), w[k], s1);
      w[i] = ((s0 + s1) + (s2 + s3)) * rdiag[i];
    }
  }
  __syncwarp();  // every lane has finished reading L
  // column j: element i at pcol[T ? colstart(i) : i]
  double* pcol = p + (T ? j : colstart(j));
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i >= j) pcol[T ? colstart(i) : i] = w[i];
  __syncwarp();
}

// acc(32 x NC) += A(32x32) * B(32 x NC), A and B views; fragment layout of
// m16n8k4.  acc[mi][ni][4].  TA / TB select a triangular operand whose other
// triangle holds unrelated data and reads as zero: TA 1 = A lower (k <= i),
// 2 = A upper (k >= i); TB 2 = B upper (k <= n).  SKIPU skips the output
// tiles strictly above the diagonal (rows 0-15 x columns 16-31).
template <int NC, int TA, int TB, bool SKIPU, class VA, class VB>
__device__ __forceinline__ void mm32(const LaneOff& o, VA A, VB B, double acc[2][NC / 8][4]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int k0 = 0; k0 < 32; k0 += 4) {
    const int kk = k0 + t;
    double a[2][2], b[NC / 8];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const int r0 = mi * 16 + g, r1 = r0 + 8;
      a[mi][0] = (TA == 1 && kk > r0) || (TA == 2 && kk < r0) ? 0.0 : A.gt(o, mi * 16, k0);
      a[mi][1] = (TA == 1 && kk > r1) || (TA == 2 && kk < r1) ? 0.0 : A.gt(o, mi * 16 + 8, k0);
    }
#pragma unroll
    for (int ni = 0; ni < NC / 8; ++ni) {
      const int nn = ni * 8 + g;
      b[ni] = (TB == 2 && kk > nn) ? 0.0 : B.tg(o, k0, ni * 8);
    }
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      // whole 16-row strips that the triangle zeroes are skipped
      if (TA == 1 && mi == 0 && k0 >= 16) continue;
      if (TA == 2 && mi == 1 && k0 < 16) continue;
#pragma unroll
      for (int ni = 0; ni < NC / 8; ++ni) {
        if (TB == 2 && k0 >= (ni + 1) * 8) continue;
        if (SKIPU && mi == 0 && ni >= 2) continue;
        mma(acc[mi][ni], a[mi][0], a[mi][1], b[ni]);
      }
    }
  }
}

// C = alpha*acc + beta*C on a 32 x 32 view; LOWER keeps i >= j only.
template <bool LOWER, bool BETA, class VC>
__device__ __forceinline__ void store_acc(const LaneOff& o, VC C, double acc[2][4][4],
                                          double alpha) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      if (LOWER && mi == 0 && ni >= 2) continue;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int R = mi * 16 + ((r & 2) ? 8 : 0), e = r & 1;
        const int i = R + g, j = ni * 8 + 2 * t + e;
        if (LOWER && i < j) continue;
        double& cref = C.acc(o, R, ni * 8, e);
        double v = alpha * acc[mi][ni][r];
        if (BETA) v += cref;
        cref = v;
      }
    }
}

// ---- the right-hand side in registers
// A 32 x 8 block X is held as the m16n8k4 B operand: lane (g, t) owns
// xb[s] = X(4s + t, g), s = 0..7.  Products land in the accumulator layout
// c[mi][r] = C(16 mi + g + 8 (r >> 1), 2t + (r & 1)).

// c (32 x 8) += A (32 x 32 view, triangle mask TA) * X (registers)
template <int TA, class VA>
__device__ __forceinline__ void mm32r(const LaneOff& o, VA A, const double (&xb)[8],
                                      double (&c)[2][4]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int kk = 4 * s + t;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      if (TA == 1 && mi == 0 && s >= 4) continue;  // strip above the lower triangle
      if (TA == 2 && mi == 1 && s < 4) continue;   // strip below the upper triangle
      const int r0 = mi * 16 + g, r1 = r0 + 8;
      const double a0 =
          (TA == 1 && kk > r0) || (TA == 2 && kk < r0) ? 0.0 : A.gt(o, mi * 16, 4 * s);
      const double a1 =
          (TA == 1 && kk > r1) || (TA == 2 && kk < r1) ? 0.0 : A.gt(o, mi * 16 + 8, 4 * s);
      mma(c[mi], a0, a1, xb[s]);
    }
  }
}

// accumulator layout -> B-operand layout (16 shuffles)
__device__ __forceinline__ void c2b(const double (&c)[2][4], double (&xb)[8]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int mi = s >> 2, half = (s & 3) >> 1;
    const int src = (4 * (s & 1) + t) * 4 + (g >> 1);
    const double v0 = __shfl_sync(0xffffffffu, c[mi][half * 2], src);
    const double v1 = __shfl_sync(0xffffffffu, c[mi][half * 2 + 1], src);
    xb[s] = (g & 1) ? v1 : v0;
  }
}

__device__ __forceinline__ void zero_c(double (&c)[2][4]) {
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int r = 0; r < 4; ++r) c[mi][r] = 0.0;
}

template <int NC>
__device__ __forceinline__ void zero_acc(double acc[2][NC / 8][4]) {
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < NC / 8; ++ni)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[mi][ni][r] = 0.0;
}

// ---- HBM <-> shared memory.  Global image of the normal rectangle:
// (r, c) at 65 c + r (TRANSR 'N') or 32 r + c ('T'/'C').  Both directions
// keep lanes on the unit-stride global dimension (coalesced), and both smem
// patterns (lanes along r, or along c) are conflict-free in the swizzle.

template <int TRANS>
__device__ __forceinline__ void load_rect(double* R, const double* g) {
  const int lane = threadIdx.x & 31;
  auto cp8 = [](double* dst, const double* src) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src));
  };
  if (TRANS) {
    double* d = R + colstart(lane);
    const double* s = g + lane;
#pragma unroll 5
    for (int r = 0; r < 65; ++r) cp8(d + r, s + 32 * r);
  } else {
#pragma unroll 4
    for (int c = 0; c < 32; ++c) {
      double* d = R + colstart(c) + lane;
      const double* s = g + 65 * c + lane;
      cp8(d, s);
      cp8(d + 32, s + 32);
      if (lane == 0) cp8(d + 64, s + 64);
    }
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  __syncwarp();
}

// rows r0 .. r0+31 of the rectangle -> HBM.  MASK 0: all 32 columns;
// 1: c <= r - r0 (a normal lower view); 2: c >= r - r0 (a transposed lower view)
template <int TRANS, int MASK>
__device__ __forceinline__ void store_band(const double* R, double* g, int r0) {
  const int lane = threadIdx.x & 31;
  if (TRANS) {
    const double* s = R + r0 + colstart(lane);
    double* d = g + 32 * r0 + lane;
#pragma unroll 4
    for (int i = 0; i < 32; ++i)
      if (MASK == 0 || (MASK == 1 ? lane <= i : lane >= i)) d[32 * i] = s[i];
  } else {
#pragma unroll 4
    for (int c = 0; c < 32; ++c)
      if (MASK == 0 || (MASK == 1 ? lane >= c : lane <= c))
        g[65 * c + r0 + lane] = R[r0 + lane + colstart(c)];
  }
}

}  // namespace b64
}  // namespace rfpk
