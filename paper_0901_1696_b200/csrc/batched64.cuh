// Batched n = 64 RFP Cholesky factor + solve, ONE WARP PER MATRIX
// (BASELINE config 4: 65,536 x n = 64, TRANSR='N', UPLO='U', nrhs = 8).
//
// The matrix never leaves the RFP layout: the 16,640-byte RFP buffer is
// copied into shared memory with 16-byte cp.async, and the reference's SRPA
// composition (rfp.py:55-136) runs on the T1 / T2 / S1 views *inside shared
// memory* (ld 65 for TRANSR='N', 32 for 'T'):
//
//   chol(T1) -> W1 = L1^-1 -> S1 <- S1 W1^T (L) | W1 S1 (U)
//   -> T2 -= S1 S1^T (L) | S1^T S1 (U)  (upper part)  -> chol(T2^T) -> W2
//   solve:  b1 = W1 b1; b2 -= S1 b1 | S1^T b1; b2 = W2 b2;          (forward)
//           b2 = W2^T b2; b1 -= S1^T b2 | S1 b2; b1 = W1^T b1       (back)
//
// with the 32x32 Cholesky and inverse on the warp's registers and every
// product (S1 update, T2 update, all six solve steps) on FP64 DMMA
// (mma.m16n8k4) fragments read from shared memory.  Only __syncwarp is
// needed, so up to six matrices (warps) are resident per SM and their
// loads/compute overlap.  The factor is written back in the RFP layout,
// coalesced; HBM traffic is the algorithmic 2*nt*8 (+ 2*n*nrhs*8) bytes.
#pragma once
#include "common.cuh"

namespace rfpk {
namespace b64 {

constexpr int N = 64, H = 32, NT = N * (N + 1) / 2;  // 2080

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

// shared-memory view with compile-time strides: element (i, j) at p[i*RS + j*CS]
template <int RS, int CS> struct SV {
  double* p;
  __device__ __forceinline__ double& operator()(int i, int j) const { return p[i * RS + j * CS]; }
  __device__ __forceinline__ SV<CS, RS> t() const { return SV<CS, RS>{p}; }
};

// 32x32 lower Cholesky and/or in-place inverse of the smem view
// p[i*rs + j*cs] (lower triangle only; the slots above it belong to the other
// RFP block) by one warp.  One non-inlined body serves every view and layout
// (strides are runtime values touched only at load / store), which keeps the
// per-SM instruction footprint small with ten matrices in flight.
//   FACTOR: lane i holds row i in registers; 32 right-looking steps, the
//           pivot column broadcast through colk (64 entries, double-buffered).
//           The factor is written back, and to gout (the global image of p)
//           when given, with lanes along the unit-stride dimension.
//   INVERT: lane j forms column j of L^-1 by forward substitution, reading
//           L(i, k) from lane i's registers with shuffles; written in place.
// Returns 0 or the 1-based failing pivot (warp-uniform).
enum { F32_FACTOR = 1, F32_INVERT = 2 };
__device__ __noinline__ int factor_inv32(double* p, int rs, int cs, double* colk, double* gout,
                                         int mode) {
  __builtin_assume(__isShared(p));
  __builtin_assume(__isShared(colk));
  const int lane = threadIdx.x & 31;
  double* prow = p + lane * rs;
  double r[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) r[j] = (j <= lane) ? prow[j * cs] : 0.0;
  double myrd;  // 1 / L(lane, lane)
  if (mode & F32_FACTOR) {
    int fail = 0;
    double dkk = shfl(r[0], 0);
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (!(dkk > 0.0)) fail = fail ? fail : k + 1;
      const double rd = rsqrt(dkk);
      const double lk = (lane == k) ? dkk * rd : rd * r[k];
      if (lane == k) myrd = rd;
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
      if (j <= lane) prow[j * cs] = r[j];
    if (gout) {
      if (rs == 1) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j <= lane) gout[lane + j * cs] = r[j];
      } else {
        __syncwarp();
        // cs == 1: lane j stores column j
#pragma unroll 4
        for (int i = 0; i < 32; ++i)
          if (i >= lane) gout[i * rs + lane] = p[i * rs + lane];
      }
    }
  } else {
    myrd = 1.0 / prow[lane * cs];
  }
  if (mode & F32_INVERT) {
    const int j = lane;
    double w[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      double s0 = (i == j) ? 1.0 : 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int k = 0; k < i; ++k) {
        const double l = shfl(r[k], i);
        if ((k & 3) == 0) s0 = fma(-l, w[k], s0);
        else if ((k & 3) == 1) s1 = fma(-l, w[k], s1);
        else if ((k & 3) == 2) s2 = fma(-l, w[k], s2);
        else s3 = fma(-l, w[k], s3);
      }
      w[i] = ((s0 + s1) + (s2 + s3)) * shfl(myrd, i);
    }
    __syncwarp();  // every lane is done reading p
    double* pcol = p + j * cs;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i >= j) pcol[i * rs] = w[i];
  }
  __syncwarp();
  return 0;
}

// In-place inverse of the lower 32x32 view L (only the lower triangle is read
// or written: the slots above it belong to the other RFP block).  Lane j
// computes column j; rdiag is a 32-entry scratch.  The substitution runs
// along L's unit-stride direction so that L is read two entries per 16-byte
// LDS: right-looking (column k of L per step) when columns are contiguous
// (RS == 1), left-looking (row i per step) when rows are (CS == 1).  PAR is
// the parity of L.p's element offset from the 16-byte-aligned smem base, so
// the pairing is resolved at compile time.
template <int RS, int CS, int PAR>
__device__ __forceinline__ double2 ld_pair(SV<RS, CS> L, int i, int k) {
  // L(i, k) and its unit-stride neighbour (i+1, k) [RS == 1] / (i, k+1) [CS == 1]
  return *reinterpret_cast<const double2*>(&L(i, k));
}
template <int RS, int CS, int PAR>
__device__ __noinline__ void inv32(SV<RS, CS> L, double* rdiag) {
  __builtin_assume(__isShared(L.p));
  __builtin_assume(__isShared(rdiag));
  const int j = threadIdx.x & 31;
  rdiag[j] = 1.0 / L(j, j);
  __syncwarp();
  double w[32];
  if constexpr (RS == 1) {
    // right-looking: s <- e_j; for k: w_k = s_k / L_kk; s_i -= L(i, k) w_k
    double sv[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) sv[i] = (i == j) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      w[k] = sv[k] * rdiag[k];
      int i = k + 1;
      if (i < 32 && ((PAR + i + k * CS) & 1)) {  // odd start: single load
        sv[i] = fma(-L(i, k), w[k], sv[i]);
        ++i;
      }
#pragma unroll
      for (; i + 1 < 32; i += 2) {
        const double2 q = ld_pair<RS, CS, PAR>(L, i, k);
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
      if (i > 0 && ((PAR + i * RS) & 1)) {
        s0 = fma(-L(i, 0), w[0], s0);
        k = 1;
      }
#pragma unroll
      for (; k + 1 < i; k += 2) {
        const double2 q = ld_pair<RS, CS, PAR>(L, i, k);
        if ((k & 2) == 0) { s0 = fma(-q.x, w[k], s0); s1 = fma(-q.y, w[k + 1], s1); }
        else { s2 = fma(-q.x, w[k], s2); s3 = fma(-q.y, w[k + 1], s3); }
      }
      if (k < i) s1 = fma(-L(i, k), w[k], s1);
      w[i] = ((s0 + s1) + (s2 + s3)) * rdiag[i];
    }
  }
  __syncwarp();  // every lane has finished reading L
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i >= j) L(i, j) = w[i];
  __syncwarp();
}

// acc(32 x NC) += A(32x32) * B(32 x NC), A and B smem views; fragment layout of
// m16n8k4 (g = lane/4, t = lane%4).  acc[mi][ni][4].  TA / TB select a
// triangular operand whose other triangle holds unrelated data and reads as
// zero: TA 1 = A lower (k <= i), 2 = A upper (k >= i); TB 2 = B upper (k <= n).
template <int NC, int TA, int TB, class VA, class VB>
__device__ __forceinline__ void mm32(VA A, VB B, double acc[2][NC / 8][4]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int k0 = 0; k0 < 32; k0 += 4) {
    const int kk = k0 + t;
    double a[2][2], b[NC / 8];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const int r0 = mi * 16 + g, r1 = r0 + 8;
      a[mi][0] = (TA == 1 && kk > r0) || (TA == 2 && kk < r0) ? 0.0 : A(r0, kk);
      a[mi][1] = (TA == 1 && kk > r1) || (TA == 2 && kk < r1) ? 0.0 : A(r1, kk);
    }
#pragma unroll
    for (int ni = 0; ni < NC / 8; ++ni) {
      const int nn = ni * 8 + g;
      b[ni] = (TB == 2 && kk > nn) ? 0.0 : B(kk, nn);
    }
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      // whole 16-row strips that the triangle zeroes are skipped
      if (TA == 1 && mi == 0 && k0 >= 16) continue;
      if (TA == 2 && mi == 1 && k0 < 16) continue;
#pragma unroll
      for (int ni = 0; ni < NC / 8; ++ni) {
        if (TB == 2 && k0 >= (ni + 1) * 8) continue;
        mma(acc[mi][ni], a[mi][0], a[mi][1], b[ni]);
      }
    }
  }
}

// global <- smem for the part of view V selected by MASK (0 all, 1 lower incl.
// diagonal); g is the global image of the smem buffer R.  Lanes run along
// the unit-stride dimension so every store instruction is coalesced.
template <int MASK, int RS, int CS>
__device__ __forceinline__ void put_view(SV<RS, CS> V, const double* R, double* g) {
  const int lane = threadIdx.x & 31;
  double* gv = g + (V.p - R);
  if (RS == 1) {
#pragma unroll 4
    for (int j = 0; j < 32; ++j)
      if (MASK == 0 || lane >= j) gv[lane + j * CS] = V(lane, j);
  } else {
#pragma unroll 4
    for (int i = 0; i < 32; ++i)
      if (MASK == 0 || i >= lane) gv[i * RS + lane] = V(i, lane);
  }
}

// ---- the right-hand side in registers (frees 4 KB of smem per matrix)
// A 32 x 8 block X is held as the m16n8k4 B operand: lane (g, t) owns
// xb[s] = X(4s + t, g), s = 0..7.  Products land in the accumulator layout
// c[mi][r] = C(16 mi + g + 8 (r >> 1), 2t + (r & 1)).

// c (32 x 8) += A (32 x 32 smem view, triangle mask TA) * X (registers)
template <int TA, class VA>
__device__ __forceinline__ void mm32r(VA A, const double (&xb)[8], double (&c)[2][4]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int kk = 4 * s + t;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      if (TA == 1 && mi == 0 && s >= 4) continue;  // strip above the lower triangle
      if (TA == 2 && mi == 1 && s < 4) continue;   // strip below the upper triangle
      const int r0 = mi * 16 + g, r1 = r0 + 8;
      const double a0 = (TA == 1 && kk > r0) || (TA == 2 && kk < r0) ? 0.0 : A(r0, kk);
      const double a1 = (TA == 1 && kk > r1) || (TA == 2 && kk < r1) ? 0.0 : A(r1, kk);
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

// C = alpha*acc + beta*C on a 32 x NC view (mask: 0 all, 2 upper incl diag)
template <int NC, class VC>
__device__ __forceinline__ void store_acc(VC C, double acc[2][NC / 8][4], double alpha,
                                          double beta, int mask) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < NC / 8; ++ni)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int i = mi * 16 + g + ((r & 2) ? 8 : 0), j = ni * 8 + 2 * t + (r & 1);
        if (mask == 2 && i > j) continue;
        double v = alpha * acc[mi][ni][r];
        if (beta != 0.0) v = fma(beta, C(i, j), v);
        C(i, j) = v;
      }
}

}  // namespace b64
}  // namespace rfpk
