// Full-format FP64/complex128 kernels on strided device views, with the
// reference's flag semantics (kernels.py).  Everything is stream-ordered and
// asynchronous; failures are reported through a device int (`info`), which
// also acts as a skip flag for every later kernel of the same chain, so a
// host never synchronises inside a factorisation.
#pragma once
#include "common.cuh"
#include "gemm.cuh"

namespace rfpk {

struct Ctx {
  cudaStream_t st;
  int* info;  // device int: 0 = ok; >0 = 1-based failure index (also skips work)
};

// Leaf size of the recursive drivers (diagonal blocks factored in one CTA).
constexpr int LEAF = 64;

// --- reference-API level (flags as characters, like kernels.py) ---------
// gemm: C <- alpha op(A) op(B) + beta C                       (kernels.py:129)
template <typename T>
int blas_gemm(Ctx c, char transa, char transb, T alpha, View<T> A, View<T> B, T beta, View<T> C);
// trsm: op(A) X = alpha B (side L) / X op(A) = alpha B (side R) (kernels.py:218)
//       zero diagonal -> *info = 1-based index, B untouched
template <typename T>
int blas_trsm(Ctx c, char side, char uplo, char trans, char diag, T alpha, View<T> A, View<T> B,
              bool scan = true, T* W = nullptr, int base = 0);
// (W: optional leaf inverses of the effective triangle, as produced by
//  blas_potrf on the same view -- pftrf reuses T1's.)
// trmm: B <- alpha op(A) B / alpha B op(A)                     (kernels.py:307)
template <typename T>
int blas_trmm(Ctx c, char side, char uplo, char trans, char diag, T alpha, View<T> A, View<T> B);
// syrk/herk on the uplo triangle of C (real alpha/beta)        (kernels.py:405)
template <typename T>
int blas_syrk(Ctx c, char uplo, char trans, double alpha, View<T> A, double beta, View<T> C,
              bool herm);
// potrf: L L^H (uplo L) / U^H U (uplo U); *info = base + first failing pivot
template <typename T> int blas_potrf(Ctx c, char uplo, View<T> A, int base, T* W = nullptr);
// Input gate for the dataflow kernels (host->device streaming): while an
// InputGate is alive on this host thread, the next tile potrf waits for
// flags[j] before reading any original tile of column block j, and the next
// tile trsm waits for flags[mode == 0 ? i : c] before reading B's original
// block (i, c).  The flags are set by the copy stream after each 64-column
// chunk of the input has landed (rfpk_?pftrf_host / rfpk_?pfsv_host).
struct InputGate {
  const int* prev_flags;
  int prev_mode;
  InputGate(const int* flags, int mode);
  ~InputGate();
  static const int* flags();
  static int mode();
};

// Row-completion hook for the host-buffer drivers (rfpk_?pfsv_host): while a
// RowHook is installed on this host thread, the NEXT tile trsm launch counts,
// per 64-row block i of its right-hand side, the finished column tasks in
// rowcnt[i] (released after the block's stores), records `launched` on its
// stream just before the launch and fills nb / nc / forward; the caller can
// then copy each row block back as soon as rowcnt[i] reaches nc (a
// stream-ordered wait on device memory) instead of after the whole solve.
struct RowDoneHook {
  int* rowcnt = nullptr;   // >= ceil(rows / 64) ints, device memory
  cudaEvent_t launched = nullptr;
  int nb = 0, nc = 0;
  bool forward = true;     // row blocks finish in ascending order
  bool used = false;
};
struct RowHook {
  RowDoneHook* prev;
  explicit RowHook(RowDoneHook* h);
  ~RowHook();
  static RowDoneHook* current();
  static void consumed();  // the hook applies to one launch only
};

// dataflow tile Cholesky of a lower view (tile_potrf.cu); W required
template <typename T> int potrf_tiles(Ctx c, View<T> A, int base, T* W);
// the same on a tall panel P (m x n): potrf of its n x n head + solve of the
// rows below (pftrf's potrf(T1) and S1 <- S1 T1^-H in one launch); -100 if
// the layout is not supported
template <typename T>
int potrf_panel_tiles(Ctx c, View<T> P, i64 n, int base, T* W, int** keep_sync = nullptr);
// the whole SRPA pftrf of an RFP (rfp.py:70-89) as ONE dataflow launch: P =
// [T1; S] (n x n1 tall panel, T1 lower), V = lower view of T2^T (n2 x n2);
// global info = base + first failing pivot of the n x n chain.  Real only;
// W = ws_alloc(n + 64).  -100 if not applicable.
template <typename T> int potrf_rfp_tiles(Ctx c, View<T> P, View<T> V, int base, T* W);
// dataflow tile trsm: conj?(Tm) X = B in place (tile_potrf.cu); W = lower-form
// 64-block inverses, wtrans when Tm is upper; -100 = unsupported strides
// agate: row block i of Tm (and W_i) readable once agate[i * agate_stride]
// is set by a concurrent producer (aabort != 0: it failed)
// tri_rhs: B is lower-triangular (a forward solve's identity in trtri): the
// zero blocks of X above its diagonal are neither summed nor solved
template <typename T>
int trsm_tiles(Ctx c, bool lower, bool conj, View<T> Tm, View<T> B, const T* W, bool wtrans,
               const int* agate = nullptr, int agate_stride = 0, const int* aabort = nullptr,
               bool tri_rhs = false);
// per-device streams for concurrent launches: hi = greatest priority (the
// critical-path kernel), lo = least; ev = scratch fork/join events
// Per host thread and device (thread_local; see tile_potrf.cu)
struct OverlapStreams {
  cudaStream_t hi = nullptr, lo = nullptr;
  cudaEvent_t ev[6] = {};
  bool ok = false;
  ~OverlapStreams();
};
OverlapStreams& overlap_streams();
// potrf('L', T) -> trsm with T's factor, overlapped: the tile potrf on the
// high-priority stream, the tile trsm conj?(T) X = B (lower, W from the
// potrf) on a side stream gated row block by row block on the potrf's
// diagonal flags; -100 = not applicable (the caller runs them in sequence)
template <typename T>
int potrf_trsm_overlap(Ctx c, View<T> A, T* W, bool conj, View<T> B, const int* pgate = nullptr,
                       const int* bgate = nullptr, int bgate_mode = 0);
// stream-ordered workspace for leaf inverses of an order-n triangle
template <typename T> int ws_alloc(T** p, i64 n, cudaStream_t st);
template <typename T> void ws_free(T* p, cudaStream_t st);
// the 64-block inverses of a lower view into W (ws_alloc(n)): what trsm computes
// when called without W, so a caller solving twice with one triangle shares it
template <typename T> int blas_leaf_inverses(Ctx c, View<T> L, T* W);
// trtri: in-place inverse; zero diagonal -> *info (matrix untouched) (kernels.py:515)
template <typename T> int blas_trtri(Ctx c, char uplo, char diag, View<T> A, int base);
// lauum: L^H L (uplo L) / U U^H (uplo U)                        (kernels.py:575)
template <typename T> int blas_lauum(Ctx c, char uplo, View<T> A);

}  // namespace rfpk
