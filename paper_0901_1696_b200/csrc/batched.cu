// Batched small-n RFP Cholesky (BASELINE config 4: 65,536 x n = 64).
//
// One CTA per matrix.  The whole RFP buffer (nt doubles, 16,640 B at n = 64)
// is read from HBM once with coalesced loads into shared memory, factored
// (and, for the fused entry point, the n x nrhs right-hand side solved) in
// shared memory, and written back once -- so HBM traffic is the algorithmic
// 2*nt*8 (+2*n*nrhs*8) bytes per matrix.  Inside shared memory the factor is
// computed on the logical lower triangle (for uplo 'U' the stored upper
// triangle is its transpose, U = L^T, the identity used by blas_potrf), so
// all eight RFP layouts share one code path; the index map is the RFP cell
// map of SURVEY Appendix B (layout.py:127-163).
#include "../../include/rfpk_b200.h"
#include "rfp.cuh"
#include "batched64.cuh"

#include <cstdint>
#include <cstdlib>
#include <type_traits>

namespace rfpk {

constexpr int BMAX = 64;       // largest order handled by the batched kernels
constexpr int BLD = BMAX + 1;  // smem column stride of the expanded triangle

__device__ __forceinline__ i64 rfp_off(const RfpDesc& r, int i, int j) {
  // (i, j) of the *stored* triangle (i >= j for 'L', i <= j for 'U')
  i64 row, col;
  if (r.lower) {
    if (j < r.n1) { row = i + r.d; col = j; }
    else { row = j - r.n1; col = i - r.n1 + 1 - r.d; }
  } else {
    if (j >= r.n2) { row = i; col = j - r.n2; }
    else { row = j + r.n2 + 1; col = i; }
  }
  return r.trans ? row * r.n1 + col : col * r.ldar + row;
}

template <int NT>
__device__ void batched_body(const RfpDesc r, double* __restrict__ arf, int nrhs,
                             double* __restrict__ b, i64 ldb, int* info_out, bool factor,
                             bool solve) {
  __shared__ double L[BMAX * BLD];
  __shared__ double X[BMAX * 8];
  __shared__ int fail;
  const int n = (int)r.n, tid = threadIdx.x;
  if (tid == 0) fail = 0;
  // expand: L(i, j) for i >= j of the logical lower triangle
  for (int e = tid; e < n * n; e += NT) {
    int i = e % n, j = e / n;
    if (i >= j) L[i + j * BLD] = r.lower ? arf[rfp_off(r, i, j)] : arf[rfp_off(r, j, i)];
  }
  cta_sync();
  if (factor) {
    for (int k = 0; k < n; ++k) {
      double d = L[k + k * BLD];
      if (!(d > 0.0)) {
        if (tid == 0) fail = k + 1;
        break;
      }
      d = sqrt(d);
      for (int i = k + 1 + tid; i < n; i += NT) L[i + k * BLD] /= d;
      cta_sync();
      const int m = n - k - 1;
      for (int e = tid; e < m * m; e += NT) {
        int i = k + 1 + e % m, j = k + 1 + e / m;
        if (j <= i) L[i + j * BLD] = fma(-L[i + k * BLD], L[j + k * BLD], L[i + j * BLD]);
      }
      if (tid == 0) L[k + k * BLD] = d;
      cta_sync();
    }
    cta_sync();
    if (tid == 0) *info_out = fail;
    if (fail) return;
    // compress the factor back into the RFP buffer
    for (int e = tid; e < n * n; e += NT) {
      int i = e % n, j = e / n;
      if (i >= j) {
        if (r.lower) arf[rfp_off(r, i, j)] = L[i + j * BLD];
        else arf[rfp_off(r, j, i)] = L[i + j * BLD];
      }
    }
  }
  if (!solve || nrhs == 0) return;
  // X = B (n x nrhs, column-major); L L^T X = B, one column per thread group
  for (int c0 = 0; c0 < nrhs; c0 += 8) {
    const int cw = nrhs - c0 < 8 ? nrhs - c0 : 8;
    for (int e = tid; e < n * cw; e += NT) {
      int i = e % n, c = e / n;
      X[i + c * BMAX] = b[i + (i64)(c0 + c) * ldb];
    }
    cta_sync();
    // forward substitution L y = b: rows processed in order, columns in parallel
    for (int i = 0; i < n; ++i) {
      if (tid < cw) X[i + tid * BMAX] /= L[i + i * BLD];
      cta_sync();
      for (int e = tid; e < (n - i - 1) * cw; e += NT) {
        int rr = i + 1 + e % (n - i - 1), c = e / (n - i - 1);
        X[rr + c * BMAX] = fma(-L[rr + i * BLD], X[i + c * BMAX], X[rr + c * BMAX]);
      }
      cta_sync();
    }
    // back substitution L^T x = y
    for (int i = n - 1; i >= 0; --i) {
      if (tid < cw) X[i + tid * BMAX] /= L[i + i * BLD];
      cta_sync();
      for (int e = tid; e < i * cw; e += NT) {
        int rr = e % i, c = e / i;
        X[rr + c * BMAX] = fma(-L[i + rr * BLD], X[i + c * BMAX], X[rr + c * BMAX]);
      }
      cta_sync();
    }
    for (int e = tid; e < n * cw; e += NT) {
      int i = e % n, c = e / n;
      b[i + (i64)(c0 + c) * ldb] = X[i + c * BMAX];
    }
    cta_sync();
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) batched_kernel(RfpDesc r, double* arf, i64 stride_arf,
                                                     int nrhs, double* b, i64 ldb, i64 stride_b,
                                                     int* info, int factor, int solve) {
  const i64 k = blockIdx.x;
  int* inf = info + k;
  batched_body<NT>(r, arf + k * stride_arf, nrhs, b ? b + k * stride_b : nullptr, ldb, inf,
                   factor != 0, solve != 0);
}


// ---------------------------------------------------------------- n == 64
// One warp per matrix; see batched64.cuh for the algorithm and the swizzled
// shared-memory rectangle.  Shared memory: rectangle (2176) + pivot column
// (64) + reciprocal diagonal (32) doubles = 17.8 KB, so twelve matrices
// (warps) are resident per SM.  W1 = L1^-1 and W2 = L2^-1 are formed IN PLACE
// of the factor blocks once those are safely in HBM.
constexpr int B64_SMEM_DOUBLES = b64::RECT + 96;

template <bool LOWER, int TRANS, bool FACTOR, bool SOLVE>
__global__ void __launch_bounds__(32, 12) batched64_kernel(double* arf, i64 stride_arf, int nrhs,
                                                       double* b, i64 ldb, i64 stride_b,
                                                       int* info) {
  using namespace b64;
  extern __shared__ __align__(16) double sm[];
  double* R = sm;
  double* colk = R + RECT;    // 64 entries (factor32)
  double* rdiag = colk + 64;  // 32 entries (inv32)
  const int lane = threadIdx.x;
  const i64 k = blockIdx.x;
  double* g = arf + k * stride_arf;
  load_rect<TRANS>(R, g);
  // the first 8-column chunk of the right-hand side goes into its registers
  // now (transposed accumulator layout, see vmm: right-hand side g8, rows
  // 8j + 2 t4 + e of b1 / b2): the load latency then hides under the
  // factorization instead of sitting between the inverses and the solve
  double y1p[4][2], y2p[4][2];
  if (SOLVE) {
    const int g8 = lane >> 2, t4 = lane & 3;
    const int cw = nrhs < 8 ? nrhs : 8;
    const double* bc = b + k * stride_b + (i64)g8 * ldb + 2 * t4;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        y1p[j][e] = g8 < cw ? bc[8 * j + e] : 0.0;
        y2p[j][e] = g8 < cw ? bc[32 + 8 * j + e] : 0.0;
      }
  }
  // T1 / T2 / S1 of the normal 65 x 32 rectangle (convert.py:142-153, d = 1):
  // V1 = T1 (L1, lower), V2 = T2^T (L2, lower), S = S1 ('L') | S1^T ('U')
  constexpr int r1 = LOWER ? 1 : 33, r2 = LOWER ? 0 : 32, rs = LOWER ? 33 : 0;
  const RV<false> V1{R + r1};
  const RV<true> V2{R + r2};
  const RV<!LOWER> S{R + rs};
  const LaneOff o;
  if (FACTOR) {
    int f = factor32<false>(o, V1.p, colk);
    if (f) {
      if (lane == 0) info[k] = f;
      return;
    }
    store_band<TRANS, 1>(R, g, r1);
    inv32<false, r1 & 1>(V1.p, rdiag);
    double acc[2][4][4];
    zero_acc<32>(acc);
    mm32<32, 0, 2, false>(o, S, V1.t(), acc);  // S <- S W1^T
    __syncwarp();
    store_acc<false, false>(o, S, acc, 1.0);
    __syncwarp();
    zero_acc<32>(acc);
    mm32<32, 0, 0, true>(o, S, S.t(), acc);    // T2 -= S S^T (its lower view V2)
    store_acc<true, true>(o, V2, acc, -1.0);
    __syncwarp();
    store_band<TRANS, 0>(R, g, rs);
    f = factor32<true>(o, V2.p, colk);
    if (lane == 0) info[k] = f ? 32 + f : 0;
    if (f) return;
    store_band<TRANS, 2>(R, g, r2);
    if (SOLVE) inv32<true, r2 & 1>(V2.p, rdiag);
  } else {
    inv32<false, r1 & 1>(V1.p, rdiag);
    inv32<true, r2 & 1>(V2.p, rdiag);
  }
  if (!SOLVE) return;
  double* bk = b + k * stride_b;
  const auto W1 = V1;
  const auto W2 = V2;
  const int g8 = lane >> 2, t4 = lane & 3;
  for (int c0 = 0; c0 < nrhs; c0 += 8) {
    const int cw = nrhs - c0 < 8 ? nrhs - c0 : 8;
    // b1^T / b2^T (8 x 32 each) in the transposed accumulator layout
    double y1[4][2], y2[4][2], z[4][2];
    if (c0 == 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          y1[j][e] = y1p[j][e];
          y2[j][e] = y2p[j][e];
        }
    } else {
      const double* bc = bk + (i64)(c0 + g8) * ldb + 2 * t4;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          y1[j][e] = g8 < cw ? bc[8 * j + e] : 0.0;
          y2[j][e] = g8 < cw ? bc[32 + 8 * j + e] : 0.0;
        }
    }
    auto zero = [](double (&v)[4][2]) {
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j][0] = v[j][1] = 0.0;
    };
    auto negate = [](double (&v)[4][2]) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        v[j][0] = -v[j][0];
        v[j][1] = -v[j][1];
      }
    };
    zero(z);
    vmm<1>(o, W1, y1, z);       // z = (W1 b1)^T
    negate(z);
    vmm<0>(o, S, z, y2);        // b2 -= S (W1 b1)
    zero(y1);
    vmm<1>(o, W2, y2, y1);      // y1 <- (W2 b2)^T
    zero(y2);
    vmm<2>(o, W2.t(), y1, y2);  // y2 = x2^T = (W2^T W2 b2)^T: final
    double* bc = bk + (i64)(c0 + g8) * ldb + 2 * t4;
    if (g8 < cw) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        bc[32 + 8 * j] = y2[j][0];
        bc[32 + 8 * j + 1] = y2[j][1];
      }
    }
    // z = -(W1 b1)^T; b1' = W1 b1 - S^T x2 = -(z + S^T x2)
    vmm<0>(o, S.t(), y2, z);
    negate(z);
    zero(y1);
    vmm<2>(o, W1.t(), z, y1);   // x1^T = (W1^T b1')^T
    if (g8 < cw) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        bc[8 * j] = y1[j][0];
        bc[8 * j + 1] = y1[j][1];
      }
    }
  }
}

int batched64_launch(const RfpDesc& r, double* arf, i64 stride_arf, i64 batch, int nrhs,
                     double* b, i64 ldb, i64 stride_b, int* info, bool factor, bool solve,
                     cudaStream_t st) {
  const size_t sm = B64_SMEM_DOUBLES * sizeof(double);
  auto launch = [&](auto kern) {
    kernel_setup(kern, 32, sm);
    kern<<<(unsigned)batch, 32, sm, st>>>(arf, stride_arf, nrhs, b, ldb, stride_b, info);
  };
  auto pick = [&](auto lower_tag, auto trans_tag) {
    constexpr bool L = decltype(lower_tag)::value;
    constexpr int T = decltype(trans_tag)::value;
    if (factor && solve) launch(batched64_kernel<L, T, true, true>);
    else if (factor) launch(batched64_kernel<L, T, true, false>);
    else launch(batched64_kernel<L, T, false, true>);
  };
  using F = std::false_type;
  using Tr = std::true_type;
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;
  KernelClock kc(st);
  if (r.lower) {
    if (r.trans) pick(Tr{}, I1{});
    else pick(Tr{}, I0{});
  } else {
    if (r.trans) pick(F{}, I1{});
    else pick(F{}, I0{});
  }
  RFPK_CHECK_LAUNCH();
  kc.stop("batched64", batch, nrhs);
  return 0;
}

int batched_launch(const RfpDesc& r, double* arf, i64 stride_arf, i64 batch, int nrhs, double* b,
                   i64 ldb, i64 stride_b, int* info, bool factor, bool solve, cudaStream_t st) {
  if (batch == 0) return 0;
  cudaError_t e = cudaMemsetAsync(info, 0, sizeof(int) * batch, st);
  if (e != cudaSuccess) return (int)e;
  if (r.n == 0) return 0;
  if (r.n == 64 && !tune(TK_BATCHED_GENERIC))
    return batched64_launch(r, arf, stride_arf, batch, nrhs, b, ldb, stride_b, info, factor, solve,
                            st);
  batched_kernel<128><<<(unsigned)batch, 128, 0, st>>>(r, arf, stride_arf, nrhs, b, ldb, stride_b,
                                                       info, factor, solve);
  RFPK_CHECK_LAUNCH();
  return 0;
}

}  // namespace rfpk

using namespace rfpk;

namespace {
char upc(char c) { return (c >= 'a' && c <= 'z') ? (char)(c - 32) : c; }
int check(char& transr, char& uplo, int64_t n) {
  transr = upc(transr);
  uplo = upc(uplo);
  if (!(transr == 'N' || transr == 'T' || transr == 'C')) return -1;
  if (!(uplo == 'L' || uplo == 'U')) return -2;
  if (n < 0 || n > BMAX) return -3;
  return 0;
}
}  // namespace

extern "C" {

int rfpk_dpftrf_batched(char transr, char uplo, int64_t n, double* arf, int64_t stride_arf,
                        int64_t batch, int* info, rfpk_stream_t s) {
  StreamDevice dg_(s);
  if (int rc = check(transr, uplo, n)) return rc;
  if (stride_arf < n * (n + 1) / 2) return -5;
  if (batch < 0) return -6;
  if (!info) return -7;
  return batched_launch(rfp_desc(n, uplo, transr), arf, stride_arf, batch, 0, nullptr, 1, 0, info,
                        true, false, reinterpret_cast<cudaStream_t>(s));
}

int rfpk_dpftrs_batched(char transr, char uplo, int64_t n, int64_t nrhs, const double* arf,
                        int64_t stride_arf, double* b, int64_t ldb, int64_t stride_b,
                        int64_t batch, int* info, rfpk_stream_t s) {
  StreamDevice dg_(s);
  if (int rc = check(transr, uplo, n)) return rc;
  if (nrhs < 0) return -4;
  if (stride_arf < n * (n + 1) / 2) return -6;
  if (ldb < (n > 1 ? n : 1)) return -8;
  if (batch < 0) return -10;
  if (!info) return -11;
  return batched_launch(rfp_desc(n, uplo, transr), const_cast<double*>(arf), stride_arf, batch,
                        (int)nrhs, b, ldb, stride_b, info, false, true,
                        reinterpret_cast<cudaStream_t>(s));
}

int rfpk_dpftrf_pftrs_batched(char transr, char uplo, int64_t n, int64_t nrhs, double* arf,
                              int64_t stride_arf, double* b, int64_t ldb, int64_t stride_b,
                              int64_t batch, int* info, rfpk_stream_t s) {
  StreamDevice dg_(s);
  if (int rc = check(transr, uplo, n)) return rc;
  if (nrhs < 0) return -4;
  if (stride_arf < n * (n + 1) / 2) return -6;
  if (ldb < (n > 1 ? n : 1)) return -8;
  if (batch < 0) return -10;
  if (!info) return -11;
  return batched_launch(rfp_desc(n, uplo, transr), arf, stride_arf, batch, (int)nrhs, b, ldb,
                        stride_b, info, true, true, reinterpret_cast<cudaStream_t>(s));
}

}  // extern "C"
