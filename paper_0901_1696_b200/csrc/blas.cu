// Recursive full-format kernels (potrf / trsm / trmm / trtri / lauum / herk)
// built on the DMMA GEMM, with one-CTA shared-memory leaf kernels for the
// <= LEAF diagonal blocks.
//
// Reference semantics (kernels.py) are kept; the *algorithm* is B200-first:
// instead of the reference's blocked loops with per-row Python updates
// (kernels.py:152-174, 245-264, 430-465), each operation is a 2x2 recursive
// split whose off-diagonal work is one large tensor-core GEMM/SYRK launch,
// so > 95% of the flops at large n run in the DMMA GEMM.
//
// Canonical forms: every call is reduced to a *left* operation with a
// triangular matrix T that is lower or upper *in its view*, plus a
// conjugation flag -- the same reductions as kernels.py:78-84, 198-213,
// 290-304, but expressed with transposed views and conj flags instead of
// conjugating B in place.  potrf/trtri/lauum with uplo 'U' are run as the
// lower algorithm on the transposed view (exact identities, see blas_potrf).
#include "blas.cuh"

namespace rfpk {

// ============================================================ leaf kernels

// Load an m x n view into column-major shared memory s[i + j*ld].
// tri: 0 = all, 1 = lower (i >= j), 2 = upper (i <= j); others are zeroed.
template <typename T>
__device__ void smem_load(T* s, int ld, const View<T> v, int m, int n, int tri) {
  const int nt = blockDim.x;
  const int total = m * n;
  if (v.rs == 1 || v.n == 1) {
    for (int e = threadIdx.x; e < total; e += nt) {
      int i = e % m, j = e / m;
      bool keep = tri == 0 || (tri == 1 ? i >= j : i <= j);
      s[i + j * ld] = keep ? *v.at(i, j) : sc_from<T>(0.0);
    }
  } else {
    for (int e = threadIdx.x; e < total; e += nt) {
      int j = e % n, i = e / n;
      bool keep = tri == 0 || (tri == 1 ? i >= j : i <= j);
      s[i + j * ld] = keep ? *v.at(i, j) : sc_from<T>(0.0);
    }
  }
}

template <typename T>
__device__ void smem_store(const T* s, int ld, View<T> v, int m, int n, int tri, bool unit_skip) {
  const int nt = blockDim.x;
  const int total = m * n;
  if (v.rs == 1 || v.n == 1) {
    for (int e = threadIdx.x; e < total; e += nt) {
      int i = e % m, j = e / m;
      bool keep = tri == 0 || (tri == 1 ? i >= j : i <= j);
      if (unit_skip && i == j) keep = false;
      if (keep) *v.at(i, j) = s[i + j * ld];
    }
  } else {
    for (int e = threadIdx.x; e < total; e += nt) {
      int j = e % n, i = e / n;
      bool keep = tri == 0 || (tri == 1 ? i >= j : i <= j);
      if (unit_skip && i == j) keep = false;
      if (keep) *v.at(i, j) = s[i + j * ld];
    }
  }
}

template <typename T> __device__ __forceinline__ T real_part_as(T v);
template <> __device__ __forceinline__ double real_part_as(double v) { return v; }
template <> __device__ __forceinline__ Z real_part_as(Z v) { return Z{v.x, 0.0}; }

// Lower Cholesky of an n x n (n <= LEAF) block in shared memory: right-looking,
// two barriers per pivot.  `not d > 0` (catches NaN) -> info = base + k + 1
// (kernels.py:441-442).  Only the lower triangle is read or written.
template <typename T>
__global__ void __launch_bounds__(256) potf2_kernel(View<T> A, int* info, int base) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* S = reinterpret_cast<T*>(smem_raw);
  if (*info) return;
  const int n = (int)A.m;
  constexpr int LD = LEAF + 1;
  smem_load(S, LD, A, n, n, 1);
  __syncthreads();
  int fail = 0;
  for (int k = 0; k < n; ++k) {
    double d = sc_re(S[k + k * LD]);
    if (!(d > 0.0)) { fail = k + 1; break; }
    d = sqrt(d);
    const double rd = 1.0 / d;
    (void)rd;
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) S[i + k * LD] = S[i + k * LD] / d;
    __syncthreads();
    const int r = n - k - 1;
    for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
      int i = k + 1 + e % r, j = k + 1 + e / r;
      if (j <= i) S[i + j * LD] = fnmac(S[i + k * LD], conj_(S[j + k * LD]), S[i + j * LD]);
    }
    if (threadIdx.x == 0) S[k + k * LD] = sc_from<T>(d);
    __syncthreads();
  }
  if (fail) {
    if (threadIdx.x == 0) *info = base + fail;
    return;
  }
  smem_store(S, LD, A, n, n, 1, false);
}

// In-place inverse of an n x n lower triangle (n <= LEAF): thread j owns
// column j of W = L^{-1} and runs the row recurrence with no barriers.
template <typename T>
__global__ void __launch_bounds__(LEAF) trtri_leaf_kernel(View<T> A, int unit, const int* skip) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* L = reinterpret_cast<T*>(smem_raw);
  constexpr int LD = LEAF + 1;
  T* W = L + LD * LEAF;
  if (skip && *skip) return;
  const int n = (int)A.m;
  smem_load(L, LD, A, n, n, 1);
  __syncthreads();
  const int j = threadIdx.x;
  if (j < n) {
    for (int i = j; i < n; ++i) {
      T s = sc_from<T>(i == j ? 1.0 : 0.0);
      for (int k = j; k < i; ++k) s = fnmac(L[i + k * LD], W[k + j * LD], s);
      W[i + j * LD] = unit ? s : s / L[i + i * LD];
    }
  }
  __syncthreads();
  smem_store(W, LD, A, n, n, 1, unit != 0);
}

// In-place A <- L^H L on an n x n lower triangle (n <= LEAF)  (kernels.py:554-572)
template <typename T>
__global__ void __launch_bounds__(256) lauum_leaf_kernel(View<T> A, const int* skip) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* L = reinterpret_cast<T*>(smem_raw);
  constexpr int LD = LEAF + 1;
  T* X = L + LD * LEAF;
  if (skip && *skip) return;
  const int n = (int)A.m;
  smem_load(L, LD, A, n, n, 1);
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    int i = e % n, j = e / n;
    if (j > i) continue;
    T s = sc_from<T>(0.0);
    for (int k = i; k < n; ++k) s = fmac(conj_(L[k + i * LD]), L[k + j * LD], s);
    if (i == j) s = real_part_as(s);
    X[i + j * LD] = s;
  }
  __syncthreads();
  smem_store(X, LD, A, n, n, 1, false);
}

// Triangular solve conj?(T) X = B for an n x n (n <= LEAF) triangle against a
// chunk of CW columns of B; one thread per column.
constexpr int TRSM_CW = 64;
template <typename T>
__global__ void __launch_bounds__(TRSM_CW)
    trsm_leaf_kernel(View<T> Tm, View<T> B, int lower, int conj, int unit, const int* skip) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* S = reinterpret_cast<T*>(smem_raw);
  constexpr int LD = LEAF + 1;
  T* X = S + LD * LEAF;  // X[i + c*LD]
  if (skip && *skip) return;
  const int n = (int)Tm.m;
  const i64 c0 = (i64)blockIdx.x * TRSM_CW;
  const int cw = (int)((B.n - c0) < TRSM_CW ? (B.n - c0) : TRSM_CW);
  View<T> Bc = B.sub(0, c0, B.m, cw);
  smem_load(S, LD, Tm, n, n, lower ? 1 : 2);
  smem_load(X, LD, Bc, n, cw, 0);
  __syncthreads();
  const int c = threadIdx.x;
  if (c < cw) {
    T* x = X + c * LD;
    if (lower) {
      for (int i = 0; i < n; ++i) {
        T s = x[i];
        for (int k = 0; k < i; ++k) s = fnmac(cj(S[i + k * LD], conj), x[k], s);
        x[i] = unit ? s : s / cj(S[i + i * LD], conj);
      }
    } else {
      for (int i = n - 1; i >= 0; --i) {
        T s = x[i];
        for (int k = i + 1; k < n; ++k) s = fnmac(cj(S[i + k * LD], conj), x[k], s);
        x[i] = unit ? s : s / cj(S[i + i * LD], conj);
      }
    }
  }
  __syncthreads();
  smem_store(X, LD, Bc, n, cw, 0, false);
}

// B <- alpha conj?(T) B for an n x n triangle against CW columns of B.
template <typename T>
__global__ void __launch_bounds__(TRSM_CW) trmm_leaf_kernel(View<T> Tm, View<T> B, int lower,
                                                            int conj, int unit, T alpha,
                                                            const int* skip) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* S = reinterpret_cast<T*>(smem_raw);
  constexpr int LD = LEAF + 1;
  T* X = S + LD * LEAF;
  if (skip && *skip) return;
  const int n = (int)Tm.m;
  const i64 c0 = (i64)blockIdx.x * TRSM_CW;
  const int cw = (int)((B.n - c0) < TRSM_CW ? (B.n - c0) : TRSM_CW);
  View<T> Bc = B.sub(0, c0, B.m, cw);
  smem_load(S, LD, Tm, n, n, lower ? 1 : 2);
  smem_load(X, LD, Bc, n, cw, 0);
  __syncthreads();
  const int c = threadIdx.x;
  if (c < cw) {
    T* x = X + c * LD;
    if (lower) {
      for (int i = n - 1; i >= 0; --i) {
        T s = unit ? x[i] : cj(S[i + i * LD], conj) * x[i];
        for (int k = 0; k < i; ++k) s = fmac(cj(S[i + k * LD], conj), x[k], s);
        x[i] = alpha * s;
      }
    } else {
      for (int i = 0; i < n; ++i) {
        T s = unit ? x[i] : cj(S[i + i * LD], conj) * x[i];
        for (int k = i + 1; k < n; ++k) s = fmac(cj(S[i + k * LD], conj), x[k], s);
        x[i] = alpha * s;
      }
    }
  }
  __syncthreads();
  smem_store(X, LD, Bc, n, cw, 0, false);
}

// Zero-diagonal scan: first (lowest, mode 0) or last (highest, mode 1)
// 1-based index with A_ii == 0, written to *info if *info is still 0.
template <typename T>
__global__ void diag_scan_kernel(View<T> A, int* info, int base, int highest) {
  __shared__ int best;
  if (threadIdx.x == 0) best = highest ? 0 : 0x7fffffff;
  __syncthreads();
  if (*info) return;
  const int n = (int)A.m;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (is_zero(*A.at(i, i))) {
      if (highest) atomicMax(&best, i + 1);
      else atomicMin(&best, i + 1);
    }
  __syncthreads();
  if (threadIdx.x == 0) {
    int b = best;
    if (highest ? b > 0 : b != 0x7fffffff) *info = base + b;
  }
}

// ============================================================ launch helpers
namespace {

template <typename T> size_t leaf_smem(int tiles) {
  return (size_t)tiles * (LEAF + 1) * LEAF * sizeof(T);
}

template <typename K> void allow_smem(K kern, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)bytes);
}

i64 split_point(i64 n) {
  const i64 q = n > 512 ? 128 : (n > 128 ? 64 : 32);
  i64 n1 = ((n / 2 + q - 1) / q) * q;
  if (n1 >= n) n1 = n / 2;
  return n1;
}

template <typename T> T one() { return sc_from<T>(1.0); }
template <typename T> T neg_one() { return sc_from<T>(-1.0); }
template <typename T> bool is_one(T v) {
  if constexpr (is_cplx<T>::value) return v.x == 1.0 && v.y == 0.0;
  else return v == 1.0;
}

// ----------------------------------------------------------- canonical ops
// herk/syrk on the `tri` triangle of C: C <- alpha G op(G) + beta C where
// G = conj?(Gv) (n x k) and op(G) = G^H (herm) or G^T.
template <typename T>
int herk_core(Ctx c, int tri, double alpha, View<T> Gv, bool gconj, double beta, View<T> C,
              bool herm) {
  const bool cplx = is_cplx<T>::value;
  const bool bconj = cplx ? (herm ? !gconj : gconj) : false;
  return gemm<T>(tri, sc_from<T>(alpha), Gv, cplx && gconj, Gv.t(), bconj, sc_from<T>(beta), C,
                 cplx && herm, c.info, c.st);
}

template <typename T>
int trsm_rec(Ctx c, bool lower, bool conj, bool unit, View<T> Tm, View<T> B) {
  const i64 n = Tm.m;
  if (n == 0 || B.n == 0) return 0;
  if (n <= LEAF) {
    const size_t sm = leaf_smem<T>(2);
    auto k = trsm_leaf_kernel<T>;
    allow_smem(k, sm);
    unsigned grid = (unsigned)((B.n + TRSM_CW - 1) / TRSM_CW);
    k<<<grid, TRSM_CW, sm, c.st>>>(Tm, B, lower, conj, unit, c.info);
    RFPK_CHECK_LAUNCH();
    return 0;
  }
  const i64 n1 = split_point(n), n2 = n - n1;
  View<T> B1 = B.sub(0, 0, n1, B.n), B2 = B.sub(n1, 0, n2, B.n);
  int rc;
  if (lower) {
    if ((rc = trsm_rec(c, lower, conj, unit, Tm.sub(0, 0, n1, n1), B1))) return rc;
    if ((rc = gemm<T>(TRI_FULL, neg_one<T>(), Tm.sub(n1, 0, n2, n1), conj, B1, false, one<T>(), B2,
                      false, c.info, c.st)))
      return rc;
    return trsm_rec(c, lower, conj, unit, Tm.sub(n1, n1, n2, n2), B2);
  }
  if ((rc = trsm_rec(c, lower, conj, unit, Tm.sub(n1, n1, n2, n2), B2))) return rc;
  if ((rc = gemm<T>(TRI_FULL, neg_one<T>(), Tm.sub(0, n1, n1, n2), conj, B2, false, one<T>(), B1,
                    false, c.info, c.st)))
    return rc;
  return trsm_rec(c, lower, conj, unit, Tm.sub(0, 0, n1, n1), B1);
}

template <typename T>
int trsm_left(Ctx c, bool lower, bool conj, bool unit, T alpha, View<T> Tm, View<T> B) {
  if (B.empty()) return 0;
  if (!is_one(alpha)) {
    int rc = scale_view<T>(B, alpha, TRI_FULL, false, c.info, c.st);
    if (rc || is_zero(alpha)) return rc;
  }
  return trsm_rec(c, lower, conj, unit, Tm, B);
}

template <typename T>
int trmm_rec(Ctx c, bool lower, bool conj, bool unit, T alpha, View<T> Tm, View<T> B) {
  const i64 n = Tm.m;
  if (n == 0 || B.n == 0) return 0;
  if (n <= LEAF) {
    const size_t sm = leaf_smem<T>(2);
    auto k = trmm_leaf_kernel<T>;
    allow_smem(k, sm);
    unsigned grid = (unsigned)((B.n + TRSM_CW - 1) / TRSM_CW);
    k<<<grid, TRSM_CW, sm, c.st>>>(Tm, B, lower, conj, unit, alpha, c.info);
    RFPK_CHECK_LAUNCH();
    return 0;
  }
  const i64 n1 = split_point(n), n2 = n - n1;
  View<T> B1 = B.sub(0, 0, n1, B.n), B2 = B.sub(n1, 0, n2, B.n);
  int rc;
  if (lower) {
    if ((rc = trmm_rec(c, lower, conj, unit, alpha, Tm.sub(n1, n1, n2, n2), B2))) return rc;
    if ((rc = gemm<T>(TRI_FULL, alpha, Tm.sub(n1, 0, n2, n1), conj, B1, false, one<T>(), B2,
                      false, c.info, c.st)))
      return rc;
    return trmm_rec(c, lower, conj, unit, alpha, Tm.sub(0, 0, n1, n1), B1);
  }
  if ((rc = trmm_rec(c, lower, conj, unit, alpha, Tm.sub(0, 0, n1, n1), B1))) return rc;
  if ((rc = gemm<T>(TRI_FULL, alpha, Tm.sub(0, n1, n1, n2), conj, B2, false, one<T>(), B1, false,
                    c.info, c.st)))
    return rc;
  return trmm_rec(c, lower, conj, unit, alpha, Tm.sub(n1, n1, n2, n2), B2);
}

template <typename T>
int trmm_left(Ctx c, bool lower, bool conj, bool unit, T alpha, View<T> Tm, View<T> B) {
  if (B.empty()) return 0;
  if (is_zero(alpha)) return scale_view<T>(B, alpha, TRI_FULL, false, c.info, c.st);
  return trmm_rec(c, lower, conj, unit, alpha, Tm, B);
}

// A = L L^H, lower triangle of the view (recursive; leaves in one CTA)
template <typename T> int potrf_lower(Ctx c, View<T> A, int base) {
  const i64 n = A.m;
  if (n == 0) return 0;
  if (n <= LEAF) {
    const size_t sm = leaf_smem<T>(1);
    auto k = potf2_kernel<T>;
    allow_smem(k, sm);
    k<<<1, 256, sm, c.st>>>(A, c.info, base);
    RFPK_CHECK_LAUNCH();
    return 0;
  }
  const i64 n1 = split_point(n), n2 = n - n1;
  View<T> A11 = A.sub(0, 0, n1, n1), A21 = A.sub(n1, 0, n2, n1), A22 = A.sub(n1, n1, n2, n2);
  int rc;
  if ((rc = potrf_lower(c, A11, base))) return rc;
  // A21 <- A21 L11^{-H}  <=>  conj(L11) A21^T = A21^T
  if ((rc = trsm_rec(c, true, is_cplx<T>::value, false, A11, A21.t()))) return rc;
  // A22 <- A22 - A21 A21^H (lower triangle)
  if ((rc = herk_core(c, TRI_LOWER, -1.0, A21, false, 1.0, A22, true))) return rc;
  return potrf_lower(c, A22, base + (int)n1);
}

// A <- L^{-1} in place, lower triangle
template <typename T> int trtri_lower(Ctx c, bool unit, View<T> A) {
  const i64 n = A.m;
  if (n == 0) return 0;
  if (n <= LEAF) {
    const size_t sm = leaf_smem<T>(2);
    auto k = trtri_leaf_kernel<T>;
    allow_smem(k, sm);
    k<<<1, LEAF, sm, c.st>>>(A, unit ? 1 : 0, c.info);
    RFPK_CHECK_LAUNCH();
    return 0;
  }
  const i64 n1 = split_point(n), n2 = n - n1;
  View<T> A11 = A.sub(0, 0, n1, n1), A21 = A.sub(n1, 0, n2, n1), A22 = A.sub(n1, n1, n2, n2);
  int rc;
  if ((rc = trtri_lower(c, unit, A11))) return rc;
  // A21 <- A21 W11   <=>  A21^T <- W11^T A21^T (W11^T upper in its view)
  if ((rc = trmm_rec(c, false, false, unit, one<T>(), A11.t(), A21.t()))) return rc;
  // A21 <- -L22^{-1} A21
  if ((rc = trsm_left(c, true, false, unit, neg_one<T>(), A22, A21))) return rc;
  return trtri_lower(c, unit, A22);
}

// A <- L^H L in place, lower triangle
template <typename T> int lauum_lower(Ctx c, View<T> A) {
  const i64 n = A.m;
  if (n == 0) return 0;
  if (n <= LEAF) {
    const size_t sm = leaf_smem<T>(2);
    auto k = lauum_leaf_kernel<T>;
    allow_smem(k, sm);
    k<<<1, 256, sm, c.st>>>(A, c.info);
    RFPK_CHECK_LAUNCH();
    return 0;
  }
  const i64 n1 = split_point(n), n2 = n - n1;
  View<T> A11 = A.sub(0, 0, n1, n1), A21 = A.sub(n1, 0, n2, n1), A22 = A.sub(n1, n1, n2, n2);
  const bool cplx = is_cplx<T>::value;
  int rc;
  if ((rc = lauum_lower(c, A11))) return rc;
  // A11 += A21^H A21 : G = conj(A21^T)
  if ((rc = herk_core(c, TRI_LOWER, 1.0, A21.t(), cplx, 1.0, A11, true))) return rc;
  // A21 <- L22^H A21 : T = conj(A22^T), upper in its view
  if ((rc = trmm_rec(c, false, cplx, false, one<T>(), A22.t(), A21))) return rc;
  return lauum_lower(c, A22);
}

template <typename T> int diag_scan(Ctx c, View<T> A, int base, bool highest) {
  if (A.m == 0) return 0;
  diag_scan_kernel<T><<<1, 256, 0, c.st>>>(A, c.info, base, highest ? 1 : 0);
  RFPK_CHECK_LAUNCH();
  return 0;
}

// op(A) as a triangle in its own view: (view, lower?, conj?)   (kernels.py:78-84)
template <typename T> void effective(View<T> A, char uplo, char trans, View<T>& v, bool& lower,
                                     bool& conj) {
  if (trans == 'N') {
    v = A; lower = uplo == 'L'; conj = false;
  } else {
    v = A.t(); lower = uplo != 'L'; conj = trans == 'C' && is_cplx<T>::value;
  }
}

}  // namespace

// ============================================================ reference API

template <typename T>
int blas_gemm(Ctx c, char transa, char transb, T alpha, View<T> A, View<T> B, T beta, View<T> C) {
  const bool cplx = is_cplx<T>::value;
  View<T> a = transa == 'N' ? A : A.t();
  View<T> b = transb == 'N' ? B : B.t();
  return gemm<T>(TRI_FULL, alpha, a, cplx && transa == 'C', b, cplx && transb == 'C', beta, C,
                 false, c.info, c.st);
}

template <typename T>
int blas_trsm(Ctx c, char side, char uplo, char trans, char diag, T alpha, View<T> A, View<T> B,
              bool scan) {
  if (B.empty() || A.m == 0) return 0;
  View<T> v, b = B;
  bool lower, conj;
  if (side == 'R') {
    // X op(A) = alpha B  <=>  op(A)^T X^T = alpha B^T        (kernels.py:200-207)
    b = B.t();
    if (trans == 'N') { v = A.t(); lower = uplo != 'L'; conj = false; }
    else { v = A; lower = uplo == 'L'; conj = trans == 'C' && is_cplx<T>::value; }
  } else {
    effective(A, uplo, trans, v, lower, conj);
  }
  if (diag == 'N' && scan) {
    // the reference raises at the first zero pivot in its solve order
    int rc = diag_scan(c, v, 0, !lower);
    if (rc) return rc;
  }
  return trsm_left(c, lower, conj, diag == 'U', alpha, v, b);
}

template <typename T>
int blas_trmm(Ctx c, char side, char uplo, char trans, char diag, T alpha, View<T> A, View<T> B) {
  if (B.empty() || A.m == 0) return 0;
  View<T> v, b = B;
  bool lower, conj;
  if (side == 'R') {
    b = B.t();
    if (trans == 'N') { v = A.t(); lower = uplo != 'L'; conj = false; }
    else { v = A; lower = uplo == 'L'; conj = trans == 'C' && is_cplx<T>::value; }
  } else {
    effective(A, uplo, trans, v, lower, conj);
  }
  return trmm_left(c, lower, conj, diag == 'U', alpha, v, b);
}

template <typename T>
int blas_syrk(Ctx c, char uplo, char trans, double alpha, View<T> A, double beta, View<T> C,
              bool herm) {
  const bool cplx = is_cplx<T>::value;
  // G = A (trans 'N') or A^H / A^T (trans 'T'/'C')              (kernels.py:328-338)
  View<T> g = trans == 'N' ? A : A.t();
  const bool gconj = trans != 'N' && cplx && herm;
  return herk_core(c, uplo == 'L' ? TRI_LOWER : TRI_UPPER, alpha, g, gconj, beta, C, herm);
}

// potrf('U', A) == potrf('L', A^T view): with V = A^T, V's lower triangle holds
// conj(H); conj(H) = L L^H gives H = conj(L) L^T = U^H U for U = L^T, which
// is stored exactly where the reference stores U.  Same pivots, same info.
template <typename T> int blas_potrf(Ctx c, char uplo, View<T> A, int base) {
  return potrf_lower(c, uplo == 'L' ? A : A.t(), base);
}

template <typename T> int blas_trtri(Ctx c, char uplo, char diag, View<T> A, int base) {
  View<T> v = uplo == 'L' ? A : A.t();
  if (diag == 'N') {
    int rc = diag_scan(c, v, base, false);   // pre-scan, matrix untouched (kernels.py:526-529)
    if (rc) return rc;
  }
  return trtri_lower(c, diag == 'U', v);
}

// lauum('U', A) == lauum('L', A^T): V^H V at V(c, r) equals (U U^H)(r, c).
template <typename T> int blas_lauum(Ctx c, char uplo, View<T> A) {
  return lauum_lower(c, uplo == 'L' ? A : A.t());
}

#define RFPK_INST(T)                                                                           \
  template int blas_gemm<T>(Ctx, char, char, T, View<T>, View<T>, T, View<T>);                 \
  template int blas_trsm<T>(Ctx, char, char, char, char, T, View<T>, View<T>, bool);                 \
  template int blas_trmm<T>(Ctx, char, char, char, char, T, View<T>, View<T>);                 \
  template int blas_syrk<T>(Ctx, char, char, double, View<T>, double, View<T>, bool);          \
  template int blas_potrf<T>(Ctx, char, View<T>, int);                                         \
  template int blas_trtri<T>(Ctx, char, char, View<T>, int);                                   \
  template int blas_lauum<T>(Ctx, char, View<T>);
RFPK_INST(double)
RFPK_INST(Z)

}  // namespace rfpk
