// Full-format drivers (potrf / trsm / trmm / trtri / lauum / herk).
//
// potrf (every n > 64) and real trsm (n >= 512) dispatch to the dataflow tile
// kernels of tile_potrf.cu.  Everything else -- trmm, trtri, lauum, complex
// trsm, small orders -- is the recursive form below, built on the DMMA GEMM
// with one-CTA shared-memory leaf kernels for the <= LEAF diagonal blocks.
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
#include "leaf.cuh"

#include <cstdlib>

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

// 64-leaf Cholesky + inverse: L (lower, in place) and W = L^{-1} (64 x 64,
// zero upper part, column-major ld 64) for the in-place GEMM trsm leaves.
// info <- base + first failing pivot (kernels.py:441-442); on failure
// nothing is written back.
template <typename T>
__global__ void __launch_bounds__(128) potf2_inv64_kernel(View<T> A, T* W, int* info, int base) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* S = reinterpret_cast<T*>(smem_raw);
  T* Ws = S + 64 * LD64;
  T* scratch = Ws + 64 * LD64;  // 128 entries: column broadcast (2 x 64) / reciprocals
  __shared__ int fail;
  if (*info) return;
  const int n = (int)A.m;
  leaf_load_lower(S, A, n);
  cta_sync();
  const int f = leaf_factor_inv64(S, Ws, scratch, &fail);
  if (f) {
    if (threadIdx.x == 0) *info = base + f;
    return;
  }
  cta_sync();
  leaf_store_lower(S, A, n, false);
  if (W)
    for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) W[e] = Ws[(e & 63) + (e >> 6) * LD64];
}

// Inverses of all 64-leaves of a lower-triangular view (one CTA per leaf):
// into the W slabs (W != null, slab b at W + 64*64*b) or in place.
template <typename T>
__global__ void __launch_bounds__(128) trtri_leaves_kernel(View<T> A, T* W, int unit,
                                                           const int* skip) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* S = reinterpret_cast<T*>(smem_raw);
  T* Ws = S + 64 * LD64;
  T* scratch = Ws + 64 * LD64;
  if (skip && *skip) return;
  const i64 r0 = (i64)blockIdx.x * 64;
  const int len = (int)((A.m - r0) < 64 ? (A.m - r0) : 64);
  View<T> blk = A.sub(r0, r0, len, len);
  leaf_load_lower(S, blk, len);
  cta_sync();
  inv64_block(S, Ws, unit != 0, false, scratch);
  cta_sync();
  if (W) {
    T* dst = W + r0 * 64;
    for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) dst[e] = Ws[(e & 63) + (e >> 6) * LD64];
  } else {
    leaf_store_lower(Ws, blk, len, unit != 0);
  }
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
  cta_sync();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    int i = e % n, j = e / n;
    if (j > i) continue;
    T s = sc_from<T>(0.0);
    for (int k = i; k < n; ++k) s = fmac(conj_(L[k + i * LD]), L[k + j * LD], s);
    if (i == j) s = real_part_as(s);
    X[i + j * LD] = s;
  }
  cta_sync();
  smem_store(X, LD, A, n, n, 1, false);
}

// Zero-diagonal scan: first (lowest, mode 0) or last (highest, mode 1)
// 1-based index with A_ii == 0, written to *info if *info is still 0.
template <typename T>
__global__ void diag_scan_kernel(View<T> A, int* info, int base, int highest) {
  __shared__ int best;
  if (threadIdx.x == 0) best = highest ? 0 : 0x7fffffff;
  cta_sync();
  if (*info) return;
  const int n = (int)A.m;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (is_zero(*A.at(i, i))) {
      if (highest) atomicMax(&best, i + 1);
      else atomicMin(&best, i + 1);
    }
  cta_sync();
  if (threadIdx.x == 0) {
    int b = best;
    if (highest ? b > 0 : b != 0x7fffffff) *info = base + b;
  }
}

// ============================================================ launch helpers
namespace {

template <typename T> size_t leaf_smem(int tiles) {
  return ((size_t)tiles * (LEAF + 1) * LEAF + 128) * sizeof(T);
}

template <typename K> void allow_smem(K kern, size_t bytes) {
  kernel_setup(kern, 128, bytes);  // per device, once
}

// Recursive split: n1 is a multiple of 64 (128 for large n), so every leaf
// starts at a multiple of 64 and all leaves but the last are exactly 64 wide.
// potrf, trsm, trmm, trtri and lauum split identically, which lets a trsm
// reuse the leaf inverses its potrf produced (W slab b <-> rows 64b..64b+63).
i64 split_point(i64 n) {
  const i64 q = n > 512 ? 128 : 64;
  i64 n1 = ((n / 2 + q - 1) / q) * q;
  if (n1 >= n) n1 = ((n - 1) / 64) * 64;
  return n1;
}

template <typename T> T one() { return sc_from<T>(1.0); }
template <typename T> T neg_one() { return sc_from<T>(-1.0); }
template <typename T> bool is_one(T v) {
  if constexpr (is_cplx<T>::value) return v.x == 1.0 && v.y == 0.0;
  else return v == 1.0;
}

}  // namespace

// workspace for the leaf inverses of an order-n triangle (64 x 64 per leaf)
template <typename T> size_t leaf_ws_elems(i64 n) { return (size_t)((n + 63) / 64) * 64 * 64; }

// The device's default memory pool keeps freed blocks (release threshold =
// max), so the per-call workspace is a cheap stream-ordered suballocation.
static void keep_pool_memory() {
  static std::atomic<bool> done[MAX_DEVICES];
  const int dev = cur_device();
  if (done[dev & (MAX_DEVICES - 1)].exchange(true)) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    unsigned long long thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

template <typename T> int ws_alloc(T** p, i64 n, cudaStream_t st) {
  *p = nullptr;
  if (n <= 0) return 0;
  keep_pool_memory();
  cudaError_t e = cudaMallocAsync((void**)p, leaf_ws_elems<T>(n) * sizeof(T), st);
  return e == cudaSuccess ? 0 : (int)e;
}
template <typename T> void ws_free(T* p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
}

namespace {

// ----------------------------------------------------------- canonical ops
// herk/syrk on the `tri` triangle of C: C <- alpha G op(G) + beta C where
// G = conj?(Gv) (n x k) and op(G) = G^H (herm) or G^T.
template <typename T>
int herk_core(Ctx c, int tri, double alpha, View<T> Gv, bool gconj, double beta, View<T> C,
              bool herm, int g_tri = A_FULL) {
  const bool cplx = is_cplx<T>::value;
  const bool bconj = cplx ? (herm ? !gconj : gconj) : false;
  return gemm<T>(tri, sc_from<T>(alpha), Gv, cplx && gconj, Gv.t(), bconj, sc_from<T>(beta), C,
                 cplx && herm, c.info, c.st, g_tri);
}

// Inverses of all 64-leaves of the lower-in-view triangle L into W slabs.
// ---------------------------------------------------------------- one-launch forms
// For small and medium orders the in-place recursions (trmm / trtri / lauum)
// are chains of small launches; these out-of-place forms are one parallel
// GEMM-shaped launch each (plus O(n^2) copies), at the price of an n x n (or
// m x n) workspace.  Measured crossover in rfpk_oop_max (tools/perf.py).
enum CopyMode : int { CP_ALL = 0, CP_LOWER0 = 1, CP_LOWER_ONLY = 2, CP_EYE = 3, CP_SLOWER_ONLY = 4 };

template <typename T>
__global__ void tri_copy_kernel(View<T> src, View<T> dst, int mode, const int* skip) {
  if (skip && *skip) return;
  const i64 total = dst.m * dst.n;
  // the fast index runs along dst's contiguous dimension (the workspaces
  // take the orientation of the view they shadow, so src matches it too)
  const bool ifast = dst.rs == 1;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total;
       e += (i64)gridDim.x * blockDim.x) {
    const i64 i = ifast ? e % dst.m : e / dst.n, j = ifast ? e / dst.m : e % dst.n;
    switch (mode) {
      case CP_ALL: *dst.at(i, j) = *src.at(i, j); break;
      case CP_LOWER0: *dst.at(i, j) = i >= j ? *src.at(i, j) : sc_from<T>(0.0); break;
      case CP_LOWER_ONLY: if (i >= j) *dst.at(i, j) = *src.at(i, j); break;
      case CP_SLOWER_ONLY: if (i > j) *dst.at(i, j) = *src.at(i, j); break;
      default: *dst.at(i, j) = sc_from<T>(i == j ? 1.0 : 0.0);
    }
  }
}

template <typename T> int tri_copy(Ctx c, View<T> src, View<T> dst, int mode) {
  if (dst.empty()) return 0;
  const i64 total = dst.m * dst.n;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 8 * num_sms()) blocks = 8 * num_sms();
  tri_copy_kernel<T><<<blocks, 256, 0, c.st>>>(src, dst, mode, c.info);
  RFPK_CHECK_LAUNCH();
  return 0;
}

// m x n workspace view, column-major or (rowmajor) row-major -- callers take
// the orientation of the view the workspace shadows, so copies are coalesced
// on both sides (the RFP blocks of TRANSR='T'/'C' are row-major)
template <typename T> int ws_matrix(Ctx c, i64 m, i64 n, View<T>& v, bool rowmajor = false) {
  T* p = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&p, (size_t)(m > 0 ? m : 1) * (n > 0 ? n : 1) * sizeof(T),
                                  c.st);
  v = rowmajor ? View<T>{p, m, n, n, 1} : View<T>{p, m, n, 1, m};
  return e == cudaSuccess ? 0 : (int)e;
}
template <typename T> bool is_rowmajor(const View<T>& v) { return v.rs != 1 && v.cs == 1; }

inline i64 oop_max() { return tune(TK_OOP_MAX); }

template <typename T> int leaf_inverses(Ctx c, View<T> L, bool unit, T* W) {
  if (L.m == 0) return 0;
  const size_t sm = leaf_smem<T>(2);
  auto k = trtri_leaves_kernel<T>;
  allow_smem(k, sm);
  k<<<(unsigned)((L.m + 63) / 64), 128, sm, c.st>>>(L, W, unit ? 1 : 0, c.info);
  RFPK_CHECK_LAUNCH();
  return 0;
}

// ---------------------------------------------------------------- look-ahead
// Library-owned streams for the recursive look-ahead: the critical path of a
// factorization runs on a high-priority stream, and the bulk trailing update
// of each level is forked to a low-priority side stream (one per nesting
// depth) so it overlaps the latency-bound factorization of the next diagonal
// block.  Fork/join are event record/wait, which also work under CUDA-graph
// stream capture (the forked streams join the capture).
// Per host thread and device (thread_local): two threads never record or
// wait on each other's events, and their look-ahead forks never share a
// stream -- the library is re-entrant for callers on distinct streams.
struct LaStreams {
  cudaStream_t hi = nullptr;
  cudaStream_t side[24] = {};
  cudaEvent_t ev[128] = {};
  int next = 0;
  bool ok = false;
  ~LaStreams() {  // thread exit (errors after runtime teardown are ignored)
    if (!ok) return;
    cudaStreamDestroy(hi);
    for (auto x : side) cudaStreamDestroy(x);
    for (auto e : ev) cudaEventDestroy(e);
  }
};

static LaStreams& la_streams() {
  static thread_local LaStreams s[MAX_DEVICES];
  LaStreams& L = s[cur_device() & (MAX_DEVICES - 1)];
  if (!L.ok) {
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    cudaStreamCreateWithPriority(&L.hi, cudaStreamNonBlocking, greatest);
    for (auto& x : L.side) cudaStreamCreateWithPriority(&x, cudaStreamNonBlocking, least);
    for (auto& e : L.ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    L.ok = true;
  }
  return L;
}

// make `to` wait for everything issued so far on `from`
static int la_link(cudaStream_t from, cudaStream_t to) {
  LaStreams& L = la_streams();
  cudaEvent_t e = L.ev[L.next++ % 128];
  cudaError_t r = cudaEventRecord(e, from);
  if (r == cudaSuccess) r = cudaStreamWaitEvent(to, e, 0);
  return r == cudaSuccess ? 0 : (int)r;
}

// run `body` on the high-priority library stream, ordered after / before the
// caller's stream
template <typename F> int on_hi_stream(Ctx c, F&& body) {
  cudaStream_t hi = la_streams().hi;
  int rc = la_link(c.st, hi);
  if (rc) return rc;
  rc = body(Ctx{hi, c.info});
  int rc2 = la_link(hi, c.st);
  return rc ? rc : rc2;
}

// levels whose trailing block is at least this large use the look-ahead
constexpr i64 LA_MIN = 512;

// Solve conj?(T) X = B (T lower or upper in its view) with the leaf inverses
// W: W slab b holds inv(leaf b) of T (wtrans == false) or of T^T (wtrans).
// Leaves are in-place 64-row GEMMs X_b = W_b B_b; updates are GEMMs.
template <typename T>
int trsm_plain(Ctx c, bool lower, bool conj, View<T> Tm, View<T> B, T* W, bool wtrans) {
  const i64 n = Tm.m;
  if (n == 0 || B.n == 0) return 0;
  if (n <= LEAF) {
    View<T> Wv{W, n, n, 1, 64};
    if (wtrans) Wv = Wv.t();
    return gemm<T>(TRI_FULL, one<T>(), Wv, conj, B, false, sc_from<T>(0.0), B, false, c.info,
                   c.st, A_FULL, true);
  }
  const i64 n1 = split_point(n), n2 = n - n1;
  View<T> B1 = B.sub(0, 0, n1, B.n), B2 = B.sub(n1, 0, n2, B.n);
  T* W2 = W + n1 * 64;
  int rc;
  if (lower) {
    if ((rc = trsm_plain(c, lower, conj, Tm.sub(0, 0, n1, n1), B1, W, wtrans))) return rc;
    if ((rc = gemm<T>(TRI_FULL, neg_one<T>(), Tm.sub(n1, 0, n2, n1), conj, B1, false, one<T>(), B2,
                      false, c.info, c.st)))
      return rc;
    return trsm_plain(c, lower, conj, Tm.sub(n1, n1, n2, n2), B2, W2, wtrans);
  }
  if ((rc = trsm_plain(c, lower, conj, Tm.sub(n1, n1, n2, n2), B2, W2, wtrans))) return rc;
  if ((rc = gemm<T>(TRI_FULL, neg_one<T>(), Tm.sub(0, n1, n1, n2), conj, B2, false, one<T>(), B1,
                    false, c.info, c.st)))
    return rc;
  return trsm_plain(c, lower, conj, Tm.sub(0, 0, n1, n1), B1, W, wtrans);
}


// Look-ahead trsm (SURVEY 7 "hard part": small solves on the critical path).
// After a block of rows is solved, the update of the remaining rows is split:
// the rows of the next diagonal child are updated on the critical stream and
// solved immediately, while the update of the other rows runs on a side
// stream.  Same splits and leaf inverses as trsm_plain.
template <typename T>
int trsm_rest_lower(Ctx c, bool conj, View<T> Tm, View<T> B, i64 n1, T* W, bool wtrans, int depth);
template <typename T>
int trsm_rest_upper(Ctx c, bool conj, View<T> Tm, View<T> B, i64 n1, T* W, bool wtrans, int depth);

template <typename T>
int trsm_rec(Ctx c, bool lower, bool conj, View<T> Tm, View<T> B, T* W, bool wtrans,
             int depth = 0) {
  const i64 n = Tm.m;
  if (n < LA_MIN || depth >= 8 || B.n == 0) return trsm_plain(c, lower, conj, Tm, B, W, wtrans);
  const i64 n1 = split_point(n), n2 = n - n1;
  int rc;
  if (lower) {
    if ((rc = trsm_rec(c, true, conj, Tm.sub(0, 0, n1, n1), B.sub(0, 0, n1, B.n), W, wtrans,
                       depth)))
      return rc;
    return trsm_rest_lower(c, conj, Tm, B, n1, W, wtrans, depth);
  }
  if ((rc = trsm_rec(c, false, conj, Tm.sub(n1, n1, n2, n2), B.sub(n1, 0, n2, B.n), W + n1 * 64,
                     wtrans, depth)))
    return rc;
  return trsm_rest_upper(c, conj, Tm, B, n1, W, wtrans, depth);
}

// rows [0, n1) of B solved; finish rows [n1, n): T22^{-1} (B2 - T21 X1)
template <typename T>
int trsm_rest_lower(Ctx c, bool conj, View<T> Tm, View<T> B, i64 n1, T* W, bool wtrans, int depth) {
  const i64 n = Tm.m, n2 = n - n1, N = B.n;
  View<T> T21 = Tm.sub(n1, 0, n2, n1), T22 = Tm.sub(n1, n1, n2, n2);
  View<T> X1 = B.sub(0, 0, n1, N), B2 = B.sub(n1, 0, n2, N);
  T* W2 = W + n1 * 64;
  int rc;
  if (n2 < LA_MIN || depth >= 8) {
    if ((rc = gemm<T>(TRI_FULL, neg_one<T>(), T21, conj, X1, false, one<T>(), B2, false, c.info,
                      c.st)))
      return rc;
    return trsm_plain(c, true, conj, T22, B2, W2, wtrans);
  }
  const i64 m1 = split_point(n2), m2 = n2 - m1;
  if ((rc = gemm<T>(TRI_FULL, neg_one<T>(), T21.sub(0, 0, m1, n1), conj, X1, false, one<T>(),
                    B2.sub(0, 0, m1, N), false, c.info, c.st)))
    return rc;
  cudaStream_t side = la_streams().side[12 + depth];
  if ((rc = la_link(c.st, side))) return rc;
  if ((rc = gemm<T>(TRI_FULL, neg_one<T>(), T21.sub(m1, 0, m2, n1), conj, X1, false, one<T>(),
                    B2.sub(m1, 0, m2, N), false, c.info, side)))
    return rc;
  if ((rc = trsm_rec(c, true, conj, T22.sub(0, 0, m1, m1), B2.sub(0, 0, m1, N), W2, wtrans,
                     depth + 1)))
    return rc;
  if ((rc = la_link(side, c.st))) return rc;
  return trsm_rest_lower(c, conj, T22, B2, m1, W2, wtrans, depth);
}

// rows [n1, n) of B solved; finish rows [0, n1): T11^{-1} (B1 - T12 X2), T upper
template <typename T>
int trsm_rest_upper(Ctx c, bool conj, View<T> Tm, View<T> B, i64 n1, T* W, bool wtrans, int depth) {
  const i64 n = Tm.m, n2 = n - n1, N = B.n;
  View<T> T12 = Tm.sub(0, n1, n1, n2), T11 = Tm.sub(0, 0, n1, n1);
  View<T> X2 = B.sub(n1, 0, n2, N), B1 = B.sub(0, 0, n1, N);
  int rc;
  if (n1 < LA_MIN || depth >= 8) {
    if ((rc = gemm<T>(TRI_FULL, neg_one<T>(), T12, conj, X2, false, one<T>(), B1, false, c.info,
                      c.st)))
      return rc;
    return trsm_plain(c, false, conj, T11, B1, W, wtrans);
  }
  const i64 m1 = split_point(n1), m2 = n1 - m1;  // T11's children [0,m1), [m1,n1)
  if ((rc = gemm<T>(TRI_FULL, neg_one<T>(), T12.sub(m1, 0, m2, n2), conj, X2, false, one<T>(),
                    B1.sub(m1, 0, m2, N), false, c.info, c.st)))
    return rc;
  cudaStream_t side = la_streams().side[12 + depth];
  if ((rc = la_link(c.st, side))) return rc;
  if ((rc = gemm<T>(TRI_FULL, neg_one<T>(), T12.sub(0, 0, m1, n2), conj, X2, false, one<T>(),
                    B1.sub(0, 0, m1, N), false, c.info, side)))
    return rc;
  if ((rc = trsm_rec(c, false, conj, T11.sub(m1, m1, m2, m2), B1.sub(m1, 0, m2, N), W + m1 * 64,
                     wtrans, depth + 1)))
    return rc;
  if ((rc = la_link(side, c.st))) return rc;
  return trsm_rest_upper(c, conj, T11, B1, m1, W, wtrans, depth);
}

// conj?(T) X = alpha B.  If W is null the leaf inverses are computed here.
template <typename T>
int trsm_left(Ctx c, bool lower, bool conj, bool unit, T alpha, View<T> Tm, View<T> B, T* W) {
  if (B.empty() || Tm.m == 0) return 0;
  if (!is_one(alpha)) {
    int rc = scale_view<T>(B, alpha, TRI_FULL, false, c.info, c.st);
    if (rc || is_zero(alpha)) return rc;
  }
  T* own = nullptr;
  int rc;
  if (!W) {
    if ((rc = ws_alloc(&own, Tm.m, c.st))) return rc;
    if ((rc = leaf_inverses(c, lower ? Tm : Tm.t(), unit, own))) return rc;
    W = own;
  }
  // the dataflow trsm for real data (complex tiles need 133 KB of smem -> one
  // CTA per SM, where the recursive GEMM form measured faster: 65 vs 78 ms on
  // config 5's S1 solve at n = 16000)
  // (narrow right-hand sides run 64 x 16 tiles, which win from two tiles up)
  constexpr i64 tile_min = 512, tile_min_narrow = 128, narrow = 256;
  const i64 tasks64 = ((Tm.m + 63) / 64) * ((B.n + 63) / 64);
  const i64 tmin = (B.n <= narrow || tasks64 <= 10 * (i64)num_sms()) ? tile_min_narrow : tile_min;
  if (!is_cplx<T>::value && Tm.m >= tmin &&
      (rc = trsm_tiles(c, lower, conj, Tm, B, (const T*)W, !lower)) != -100) {
    ws_free(own, c.st);
    return rc;
  }
  if (Tm.m >= LA_MIN)
    rc = on_hi_stream(c, [&](Ctx h) { return trsm_rec(h, lower, conj, Tm, B, W, !lower); });
  else rc = trsm_rec(c, lower, conj, Tm, B, W, !lower);
  ws_free(own, c.st);
  return rc;
}

// B <- alpha conj?(T) B; leaves are in-place 64-row GEMMs with a masked
// (triangular) A operand; unit diagonal = strict mask + beta = alpha.
template <typename T>
int trmm_rec(Ctx c, bool lower, bool conj, bool unit, T alpha, View<T> Tm, View<T> B) {
  const i64 n = Tm.m;
  if (n == 0 || B.n == 0) return 0;
  if (n <= LEAF) {
    const int mask = lower ? (unit ? A_SLOWER : A_LOWER) : (unit ? A_SUPPER : A_UPPER);
    return gemm<T>(TRI_FULL, alpha, Tm, conj, B, false, unit ? alpha : sc_from<T>(0.0), B, false,
                   c.info, c.st, mask, true);
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

// B <- alpha conj?(T) B as ONE masked GEMM from a copy of B: C = B is read
// by the epilogue only (unit diagonal: strict mask + beta = alpha)
template <typename T>
int trmm_oop(Ctx c, bool lower, bool conj, bool unit, T alpha, View<T> Tm, View<T> B) {
  View<T> Bc;
  int rc = ws_matrix(c, B.m, B.n, Bc, is_rowmajor(B));
  if (!rc) rc = tri_copy(c, B, Bc, CP_ALL);
  const int mask = lower ? (unit ? A_SLOWER : A_LOWER) : (unit ? A_SUPPER : A_UPPER);
  if (!rc)
    rc = gemm<T>(TRI_FULL, alpha, Tm, conj, Bc, false, unit ? alpha : sc_from<T>(0.0), B, false,
                 c.info, c.st, mask, false);
  if (Bc.p) cudaFreeAsync(Bc.p, c.st);
  return rc;
}

template <typename T>
int trmm_left(Ctx c, bool lower, bool conj, bool unit, T alpha, View<T> Tm, View<T> B) {
  if (B.empty()) return 0;
  if (is_zero(alpha)) return scale_view<T>(B, alpha, TRI_FULL, false, c.info, c.st);
  if (Tm.m > LEAF && Tm.m <= oop_max() && B.n <= oop_max()) {
    const int rc = trmm_oop(c, lower, conj, unit, alpha, Tm, B);
    if (rc != -100) return rc;
  }
  return trmm_rec(c, lower, conj, unit, alpha, Tm, B);
}

template <typename T> int potrf_node(Ctx c, View<T> A, int base, T* W, int depth);

// A22 <- A22 - G G^H, then factor A22 (lower).  With look-ahead the update is
// split: B11 (the first diagonal child of A22) is updated on the critical
// stream and factored right away, while B21/B22 are updated on a side stream.
template <typename T>
int update_and_factor(Ctx c, View<T> A22, View<T> G, int base, T* W, int depth) {
  const i64 n2 = A22.m, k = G.n;
  int rc;
  if (n2 < LA_MIN || depth >= 24) {
    if ((rc = herk_core(c, TRI_LOWER, -1.0, G, false, 1.0, A22, true))) return rc;
    return potrf_node(c, A22, base, W, depth);
  }
  const i64 m1 = split_point(n2), m2 = n2 - m1;
  View<T> G1 = G.sub(0, 0, m1, k), G2 = G.sub(m1, 0, m2, k);
  View<T> B11 = A22.sub(0, 0, m1, m1), B21 = A22.sub(m1, 0, m2, m1), B22 = A22.sub(m1, m1, m2, m2);
  if ((rc = herk_core(c, TRI_LOWER, -1.0, G1, false, 1.0, B11, true))) return rc;
  cudaStream_t side = la_streams().side[depth];
  if ((rc = la_link(c.st, side))) return rc;
  Ctx cs{side, c.info};
  const bool cplx = is_cplx<T>::value;
  if ((rc = gemm<T>(TRI_FULL, sc_from<T>(-1.0), G2, false, G1.t(), cplx, sc_from<T>(1.0), B21,
                    false, c.info, side)))
    return rc;
  if ((rc = herk_core(cs, TRI_LOWER, -1.0, G2, false, 1.0, B22, true))) return rc;
  if ((rc = potrf_node(c, B11, base, W, depth + 1))) return rc;
  if ((rc = la_link(side, c.st))) return rc;
  if ((rc = trsm_rec(c, true, cplx, B11, B21.t(), W, false))) return rc;
  return update_and_factor(c, B22, B21, base + (int)m1, W + m1 * 64, depth);
}

// A = L L^H, lower triangle of the view; W receives the leaf inverses (slab
// b <-> rows 64b..), reused by the trsm steps of this recursion and by the
// caller (pftrf's S1 solve).
template <typename T> int potrf_node(Ctx c, View<T> A, int base, T* W, int depth) {
  const i64 n = A.m;
  if (n == 0) return 0;
  if (n <= LEAF) {
    const size_t sm = leaf_smem<T>(2);
    auto k = potf2_inv64_kernel<T>;
    allow_smem(k, sm);
    k<<<1, 128, sm, c.st>>>(A, W, c.info, base);
    RFPK_CHECK_LAUNCH();
    return 0;
  }
  const i64 n1 = split_point(n), n2 = n - n1;
  View<T> A11 = A.sub(0, 0, n1, n1), A21 = A.sub(n1, 0, n2, n1), A22 = A.sub(n1, n1, n2, n2);
  int rc;
  if ((rc = potrf_node(c, A11, base, W, depth))) return rc;
  // A21 <- A21 L11^{-H}  <=>  conj(L11) A21^T = A21^T
  if ((rc = trsm_rec(c, true, is_cplx<T>::value, A11, A21.t(), W, false))) return rc;
  // A22 <- A22 - A21 A21^H, then factor (with look-ahead)
  return update_and_factor(c, A22, A21, base + (int)n1, W + n1 * 64, depth);
}


template <typename T> int potrf_lower(Ctx c, View<T> A, int base, T* W) {
  // the dataflow tile kernel (tile_potrf.cu) at every order above one leaf
  // (measured faster than the recursion everywhere)
  if (A.m > LEAF && W) {
    // complex, large: one split level, the halves on the tile kernel and the
    // panel solve / update on the GEMM kernel (34 TFLOP/s against the complex
    // tile kernel's 26 at n = 12000, one CTA per SM: zpotrf 12000 88.7 ms
    // whole; real orders stay whole -- potrf 8192 6.9 ms vs ~8.2 split)
    if (is_cplx<T>::value && A.m >= tune(TK_ZPOTRF_SPLIT_MIN)) {
      const i64 n1 = split_point(A.m), n2 = A.m - n1;
      View<T> A11 = A.sub(0, 0, n1, n1), A21 = A.sub(n1, 0, n2, n1), A22 = A.sub(n1, n1, n2, n2);
      int rc;
      if ((rc = potrf_tiles(c, A11, base, W))) return rc;
      if ((rc = trsm_rec(c, true, true, A11, A21.t(), W, false))) return rc;
      if ((rc = herk_core(c, TRI_LOWER, -1.0, A21, false, 1.0, A22, true))) return rc;
      return potrf_tiles(c, A22, base + (int)n1, W + n1 * 64);
    }
    return potrf_tiles(c, A, base, W);
  }
  // (fallback / n <= 64: the recursive driver with look-ahead streams)
  if (A.m < LA_MIN) return potrf_node(c, A, base, W, 0);
  return on_hi_stream(c, [&](Ctx h) { return potrf_node(h, A, base, W, 0); });
}

// A <- L^{-1} in place (lower): all 64-leaves are inverted in one launch,
// then each recursion node forms A21 <- -W22 A21 W11 with two trmms.
template <typename T> int trtri_rec(Ctx c, bool unit, View<T> A) {
  const i64 n = A.m;
  if (n <= LEAF) return 0;
  const i64 n1 = split_point(n), n2 = n - n1;
  View<T> A11 = A.sub(0, 0, n1, n1), A21 = A.sub(n1, 0, n2, n1), A22 = A.sub(n1, n1, n2, n2);
  int rc;
  if ((rc = trtri_rec(c, unit, A11))) return rc;
  if ((rc = trtri_rec(c, unit, A22))) return rc;
  // A21 <- A21 W11  <=>  A21^T <- W11^T A21^T (upper in its view)
  if ((rc = trmm_rec(c, false, false, unit, one<T>(), A11.t(), A21.t()))) return rc;
  return trmm_rec(c, true, false, unit, neg_one<T>(), A22, A21);
}

// A <- L^{-1} by the dataflow tile trsm on an identity workspace (every column
// chain of the inverse in parallel), then the lower triangle copied back
template <typename T> int trtri_oop(Ctx c, bool unit, View<T> A) {
  const i64 n = A.m;
  T* W = nullptr;
  View<T> X{nullptr, 0, 0, 1, 1};
  int rc = ws_alloc(&W, n, c.st);
  if (!rc) rc = leaf_inverses(c, A, unit, W);
  if (!rc) rc = ws_matrix(c, n, n, X, is_rowmajor(A));
  if (!rc) rc = tri_copy(c, X, X, CP_EYE);
  if (!rc) rc = trsm_tiles(c, true, false, A, X, (const T*)W, false, nullptr, 0, nullptr, true);
  // (unit diagonal: the stored diagonal is never referenced nor written)
  if (!rc) rc = tri_copy(c, X, A, unit ? CP_SLOWER_ONLY : CP_LOWER_ONLY);
  if (X.p) cudaFreeAsync(X.p, c.st);
  ws_free(W, c.st);
  return rc;
}

template <typename T> int trtri_lower_rec(Ctx c, bool unit, View<T> A);

// Above the one-launch size: the top levels of the trmm recursion, with every
// sub-block <= oop_max inverted by trtri_oop from the original L (config 5's
// complex trtri at 12000: children 3000 on the tile trsm instead of a chain
// of leaf inverses and small trmms)
template <typename T> int trtri_hyb(Ctx c, bool unit, View<T> A) {
  const i64 n = A.m;
  if (n <= oop_max()) return n > LEAF ? trtri_oop(c, unit, A) : trtri_lower_rec(c, unit, A);
  const i64 n1 = split_point(n), n2 = n - n1;
  View<T> A11 = A.sub(0, 0, n1, n1), A21 = A.sub(n1, 0, n2, n1), A22 = A.sub(n1, n1, n2, n2);
  int rc;
  if ((rc = trtri_hyb(c, unit, A11))) return rc;
  if ((rc = trtri_hyb(c, unit, A22))) return rc;
  if ((rc = trmm_rec(c, false, false, unit, one<T>(), A11.t(), A21.t()))) return rc;
  return trmm_rec(c, true, false, unit, neg_one<T>(), A22, A21);
}

template <typename T> int trtri_lower_rec(Ctx c, bool unit, View<T> A) {
  int rc = leaf_inverses<T>(c, A, unit, nullptr);
  if (rc) return rc;
  return trtri_rec(c, unit, A);
}

template <typename T> int trtri_lower(Ctx c, bool unit, View<T> A) {
  if (A.m == 0) return 0;
  if (A.m > LEAF) return trtri_hyb(c, unit, A);
  return trtri_lower_rec(c, unit, A);
}

// A <- L^H L (lower triangle) as ONE herk launch from a zero-padded copy of L
template <typename T> int lauum_oop(Ctx c, View<T> A) {
  View<T> Lw;
  int rc = ws_matrix(c, A.m, A.m, Lw, is_rowmajor(A));
  if (!rc) rc = tri_copy(c, A, Lw, CP_LOWER0);
  // L^H L = G G^H with G = conj(L^T), upper triangular with its zeros in Lw:
  // the lower output tile (i, j) only needs K from row i on (1/3 the flops)
  if (!rc) rc = herk_core(c, TRI_LOWER, 1.0, Lw.t(), is_cplx<T>::value, 0.0, A, true, A_UBAND);
  if (Lw.p) cudaFreeAsync(Lw.p, c.st);
  return rc;
}

// A <- L^H L in place, lower triangle
template <typename T> int lauum_lower(Ctx c, View<T> A) {
  const i64 n = A.m;
  if (n == 0) return 0;
  if (n > LEAF && n <= oop_max()) {
    const int rc = lauum_oop(c, A);
    if (rc != -100) return rc;
  }
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
              bool scan, T* W, int base) {
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
    int rc = diag_scan(c, v, base, !lower);
    if (rc) return rc;
  }
  return trsm_left(c, lower, conj, diag == 'U', alpha, v, b, W);
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
template <typename T> int blas_potrf(Ctx c, char uplo, View<T> A, int base, T* W) {
  View<T> v = uplo == 'L' ? A : A.t();
  T* own = nullptr;
  int rc;
  if (!W) {
    if ((rc = ws_alloc(&own, v.m, c.st))) return rc;
    W = own;
  }
  rc = potrf_lower(c, v, base, W);
  ws_free(own, c.st);
  return rc;
}

template <typename T> int blas_leaf_inverses(Ctx c, View<T> L, T* W) {
  return leaf_inverses(c, L, false, W);
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
  template int blas_trsm<T>(Ctx, char, char, char, char, T, View<T>, View<T>, bool, T*, int);       \
  template int blas_trmm<T>(Ctx, char, char, char, char, T, View<T>, View<T>);                 \
  template int blas_syrk<T>(Ctx, char, char, double, View<T>, double, View<T>, bool);          \
  template int blas_potrf<T>(Ctx, char, View<T>, int, T*);                                     \
  template int blas_trtri<T>(Ctx, char, char, View<T>, int);                                   \
  template int blas_leaf_inverses<T>(Ctx, View<T>, T*);                                        \
  template int blas_lauum<T>(Ctx, char, View<T>);                                              \
  template int ws_alloc<T>(T**, i64, cudaStream_t);                                            \
  template void ws_free<T>(T*, cudaStream_t);
RFPK_INST(double)
RFPK_INST(Z)

}  // namespace rfpk
