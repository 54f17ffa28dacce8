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
// fragments read from shared memory (mma.m16n8k4 for the factorization's
// products; the solve runs transposed on mma.m8n8k4 with the right-hand side
// in accumulator-layout registers, so its six products chain without a
// shuffle, see vmm).  Only __syncwarp is needed,
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

// One warp: right-looking Cholesky of the 16 columns [C0, C0 + 16) of the
// lower 32x32 view at p, rows C0 .. 31 (lane i holds row i's 16 panel
// entries).  The pivot column is broadcast through colk (double-buffered,
// 16-byte pairs); the next pivot comes straight from lane p+1's registers.
// 16-wide rows halve the broadcast volume of a 32-wide right-looking sweep.
// The view orientation T is compile-time, so every row slot is an immediate
// offset from the lane's row pointer; the panel C0 (0 or 16) is a run-time
// argument -- two instantiations instead of four shrink the fused kernel from
// 73 to 56 KB of straight-line code, which its three warps per scheduler
// fetch at different places (ncu: no_instruction 13% of the stall cycles;
// 59.9 -> 61.0 M matrices/s).  Lanes whose row
// lies above the panel (and the slots of a row above its diagonal, which
// belong to the other RFP block) load and update garbage that is never
// broadcast or stored.  Returns 0 or the failing pivot (1-based in the view;
// NaN fails like the reference's `not d > 0`, kernels.py:436).
template <bool T>
__device__ __noinline__ int panel16(double* p, double* colk, int C0) {
  __builtin_assume(__isShared(p));
  __builtin_assume(__isShared(colk));
  const int lane = threadIdx.x & 31;
  double* prow = p + (T ? colstart(lane) + C0 : lane + colstart(C0));
  double r[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) r[j] = prow[T ? j : colstart(j)];
  unsigned bad = 0;
  double dkk = shfl(r[0], C0);
  const double* cbase = colk + C0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int pv = C0 + k;
    bad |= (dkk > 0.0) ? 0u : (1u << k);
    const double rd = rsqrt_pivot(dkk);
    const double lk = (lane == pv) ? dkk * rd : rd * r[k];
    r[k] = lk;
    double dnext = 0.0;
    if (k + 1 < 16) dnext = shfl(fma(-lk, lk, r[k + 1]), pv + 1);  // lane pv+1's new pivot
    const int buf = (k & 1) * 32;
    colk[buf + lane] = lk;
    __syncwarp();
#pragma unroll
    for (int jj = (k + 1) & ~1; jj < 16; jj += 2) {
      const double2 c = *reinterpret_cast<const double2*>(cbase + buf + jj);
      if (jj >= k + 1) r[jj] = fma(-lk, c.x, r[jj]);
      r[jj + 1] = fma(-lk, c.y, r[jj + 1]);
    }
    dkk = dnext;
  }
  if (bad) return C0 + __ffs(bad);
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (C0 + j <= lane) prow[T ? j : colstart(j)] = r[j];
  __syncwarp();
  return 0;
}

// 32x32 lower Cholesky of the view in place (lower triangle only; the slots
// above it belong to the other RFP block) by one warp: panel [0, 16) (L11 and
// L21), V22 -= L21 L21^T on DMMA (m16n8k4, lower tiles), panel [16, 32).
template <bool T>
__device__ __forceinline__ int factor32(const LaneOff& o, double* p, double* colk) {
  int f = panel16<T>(p, colk, 0);
  if (f) return f;
  const RV<T> V{p};
  double acc[2][4];
#pragma unroll
  for (int ni = 0; ni < 2; ++ni)
#pragma unroll
    for (int r = 0; r < 4; ++r) acc[ni][r] = 0.0;
#pragma unroll
  for (int k0 = 0; k0 < 16; k0 += 4) {
    const double a0 = V.gt(o, 16, k0), a1 = V.gt(o, 24, k0);   // L21(g (+8), k0 + t)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
      mma(acc[ni], a0, a1, V.t().tg(o, k0, 16 + 8 * ni));      // L21(8ni + g, k0 + t)
  }
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int ni = 0; ni < 2; ++ni)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = g + ((r & 2) ? 8 : 0), j = 8 * ni + 2 * t + (r & 1);
      if (j <= i) {
        double& c = V.acc(o, 16 + ((r & 2) ? 8 : 0), 16 + 8 * ni, r & 1);
        c -= acc[ni][r];
      }
    }
  __syncwarp();
  return panel16<T>(p, colk, 16);
}

// In-place inverse of the lower 32x32 view (only its lower triangle is read
// or written) by one warp.  The two 16x16 diagonal blocks are inverted side
// by side: lane (h, j) = (lane / 16, lane % 16) forms column j of W_hh by
// right-looking substitution (w_k = s_k / L_kk, s_i -= L(i, k) w_k: chain of
// one multiply + one FMA per step), reading column k of its block by
// broadcast (16-byte pairs along a contiguous column, PAR = parity of p's
// element offset).  Then W21 = -W22 (L21 W11) on DMMA, the product L21 W11
// moved from accumulator to B-operand layout by shuffles.
template <bool T, int PAR>
__device__ __noinline__ void inv32(double* p, double* rdiag) {
  __builtin_assume(__isShared(p));
  __builtin_assume(__isShared(rdiag));
  const int lane = threadIdx.x & 31, h = lane >> 4, j = lane & 15;
  const RV<T> V{p};
  // block h at pb: element (i, k) at pb[T ? k + colstart(i) : i + colstart(k)]
  // (colstart additive over the 16-aligned 16h; 16 + colstart(16) is even)
  const double* pb = p + 16 * h + colstart(16 * h);
  rdiag[lane] = 1.0 / pb[j + colstart(j)];
  __syncwarp();
  double sv[16], w[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) sv[i] = (i == j) ? 1.0 : 0.0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    w[k] = sv[k] * rdiag[16 * h + k];
    if constexpr (!T) {
      int i = k + 1;
      if (i < 16 && ((PAR + i + colstart(k)) & 1)) {
        sv[i] = fma(-pb[i + colstart(k)], w[k], sv[i]);
        ++i;
      }
#pragma unroll
      for (; i + 1 < 16; i += 2) {
        const double2 q = *reinterpret_cast<const double2*>(pb + i + colstart(k));
        sv[i] = fma(-q.x, w[k], sv[i]);
        sv[i + 1] = fma(-q.y, w[k], sv[i + 1]);
      }
      if (i < 16) sv[i] = fma(-pb[i + colstart(k)], w[k], sv[i]);
    } else {
#pragma unroll
      for (int i = k + 1; i < 16; ++i) sv[i] = fma(-pb[k + colstart(i)], w[k], sv[i]);
    }
  }
  __syncwarp();  // every lane has finished reading its block
  double* pw = const_cast<double*>(pb);
#pragma unroll
  for (int i = 0; i < 16; ++i)
    if (i >= j) pw[T ? j + colstart(i) : i + colstart(j)] = w[i];
  __syncwarp();
  // T1 = L21 W11 (16 x 16, W11 lower: its upper slots hold the other block)
  const LaneOff o;
  const int g = lane >> 2, t = lane & 3;
  double c1[2][4];
#pragma unroll
  for (int ni = 0; ni < 2; ++ni)
#pragma unroll
    for (int r = 0; r < 4; ++r) c1[ni][r] = 0.0;
#pragma unroll
  for (int k0 = 0; k0 < 16; k0 += 4) {
    const double a0 = V.gt(o, 16, k0), a1 = V.gt(o, 24, k0);
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      if (k0 + 4 <= 8 * ni) continue;  // rows k < 8ni: W11 above its diagonal
      const double bv = (k0 + t < 8 * ni + g) ? 0.0 : V.tg(o, k0, 8 * ni);
      mma(c1[ni], a0, a1, bv);
    }
  }
  // accumulator -> B operand: xb[ni][s] = T1(4s + t, 8ni + g)
  double xb[2][4];
#pragma unroll
  for (int ni = 0; ni < 2; ++ni)
#pragma unroll
    for (int s4 = 0; s4 < 4; ++s4) {
      const int half = s4 >> 1, src = (4 * (s4 & 1) + t) * 4 + (g >> 1);
      const double v0 = __shfl_sync(0xffffffffu, c1[ni][half * 2], src);
      const double v1 = __shfl_sync(0xffffffffu, c1[ni][half * 2 + 1], src);
      xb[ni][s4] = (g & 1) ? v1 : v0;
    }
  // W21 = -W22 T1 (W22 lower)
  double c2[2][4];
#pragma unroll
  for (int ni = 0; ni < 2; ++ni)
#pragma unroll
    for (int r = 0; r < 4; ++r) c2[ni][r] = 0.0;
#pragma unroll
  for (int s4 = 0; s4 < 4; ++s4) {
    const int kk = 4 * s4 + t;
    const double a0 = (kk > g) ? 0.0 : V.gt(o, 16, 16 + 4 * s4);
    const double a1 = (kk > g + 8) ? 0.0 : V.gt(o, 24, 16 + 4 * s4);
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) mma(c2[ni], a0, a1, xb[ni][s4]);
  }
  __syncwarp();  // L21 fully read (T1) before W21 overwrites it
#pragma unroll
  for (int ni = 0; ni < 2; ++ni)
#pragma unroll
    for (int r = 0; r < 4; ++r) V.acc(o, 16 + ((r & 2) ? 8 : 0), 8 * ni, r & 1) = -c2[ni][r];
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

// ---- the right-hand side TRANSPOSED in registers (the solve of the fused
// kernel).  Y = X^T is 8 x 32 (row g = right-hand side g) and lives in the
// m8n8k4 accumulator layout: lane (g, t) holds y[j][e] = Y(g, 8j + 2t + e).
// The same registers ARE the A operand of the next product when its k-step
// (j, e) takes the four k = 8j + 2t + e of lanes t = 0..3 -- a permutation of
// the summation order only -- so the six products of the solve chain hand
// their results on without any shuffle.  The B operand of that k-step is
// M(8jp + g, 8j + 2t + e): exactly the accumulator access pattern of the view
// (conflict-free in the swizzle for both orientations).
__device__ __forceinline__ void mma8(double (&c)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// out (8 x 32) += Y (8 x 32) M^T for a 32 x 32 view M indexed (n, k).
// TRI 1: M lower (k <= n), 2: M upper (k >= n); the other triangle holds
// unrelated data and reads as zero.
template <int TRI, class VM>
__device__ __forceinline__ void vmm(const LaneOff& o, VM M, const double (&y)[4][2],
                                    double (&out)[4][2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) {
        if (TRI == 1 && j > jp) continue;
        if (TRI == 2 && j < jp) continue;
        const int k = 2 * t + e;
        const bool off = j == jp && ((TRI == 1 && k > g) || (TRI == 2 && k < g));
        const double b = off ? 0.0 : M.acc(o, 8 * jp, 8 * j, e);
        mma8(out[jp], y[j][e], b);
      }
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
    }
    cp8(R + 64 + colstart(lane), g + 65 * lane + 64);  // row 64 of every column
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
