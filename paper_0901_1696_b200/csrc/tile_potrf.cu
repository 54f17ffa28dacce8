// Dataflow tile Cholesky: ONE persistent kernel factors a lower view
// A = L L^H tile by tile (64 x 64 tiles = the 64-leaves of the recursive
// drivers), with the dependencies tracked on the device instead of by host
// streams and events.
//
// Task (i, j), i >= j, owns tile (i, j).  Tasks are handed out in column-major
// order (j, then i) by an atomic counter to whichever CTA is free, and each
// task is left-looking:
//
//   acc = sum_{k < j} L(i, k) L(j, k)^H         64-wide chunks, DMMA, 3-stage
//                                               cp.async pipeline; chunk k is
//                                               loaded only once done(i, k)
//                                               and done(j, k) are published
//   i == j:  L(j, j), W_j = L(j, j)^-1  <- leaf(A(j, j) - acc)     (one CTA)
//   i >  j:  wait done(j, j);  L(i, j) = (A(i, j) - acc) W_j^H     (DMMA)
//   publish done(i, j)
//
// A task only ever waits on tasks handed out before it, and those are held
// by running CTAs, so progress never depends on co-residency (no deadlock
// whatever the grid size or other work on the GPU).  Publication: the CTA's
// stores, __syncthreads, then one thread's st.release.gpu of
// the flag; consumption: one thread's ld.acquire.gpu spin, __syncthreads,
// then the tile reads (cp.async / ld.global.cg from L2).
//
// Compared with the stream-scheduled right-looking driver, the critical path
// per column shrinks to one 64-chunk update + the leaf + one 64x64x64
// product (no kernel launches, no event round trips), and all other tiles'
// updates overlap it.  The W_j slabs are those every other driver produces
// (slab j at W + 64*64*j), so the trsm that follows in pftrf reuses them.
// Failure: the failing diagonal task writes info = base + pivot and raises
// an abort flag that every waiting CTA checks (kernels.py:441-442 semantics:
// the first failing pivot; later tiles are never factored).
#include <cuda_runtime.h>

namespace rfpk {
// Developer timeline of the diagonal chain (build variant with
// -DRFPK_CHAIN_TRACE, read by tools/chain_trace.py through
// rfpk_chain_trace_read): per diagonal tile d, %globaltimer stamps of the
// SUPER task that produces it.
#ifdef RFPK_CHAIN_TRACE
constexpr int CT_EV = 16, CT_MAX = 1024;
__device__ unsigned long long g_chain_trace[CT_MAX * CT_EV];
__device__ __forceinline__ void ct_mark(int d, int ev) {
  if (threadIdx.x == 0 && d >= 0 && d < CT_MAX) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_chain_trace[d * CT_EV + ev] = t;
  }
  // (without reconverging here the tile potrf computed wrong factors: the
  // warp stayed split after the thread-0 store -- see cta_sync)
  __syncwarp();
}
#define LEAF_MARK(d, ev) ::rfpk::ct_mark(d, ev)
// per-task start / end stamps of the tile trsm (task index t < TT_MAX)
constexpr int TT_MAX = 1 << 16;
__device__ unsigned long long g_task_trace[2 * TT_MAX];
__device__ __forceinline__ void tt_mark(long long t, int ev) {
  if (threadIdx.x == 0 && t >= 0 && t < TT_MAX) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    g_task_trace[2 * t + ev] = v;
  }
  __syncwarp();
}
#else
__device__ __forceinline__ void ct_mark(int, int) {}
__device__ __forceinline__ void tt_mark(long long, int) {}
#endif

}  // namespace rfpk

#include "blas.cuh"
#include "dmma.cuh"
#include "leaf.cuh"

#include <cstdlib>
#include <mutex>

namespace rfpk {

namespace {
thread_local const int* tl_gate = nullptr;
thread_local int tl_gate_mode = 0;
}  // namespace
InputGate::InputGate(const int* f, int m) : prev_flags(tl_gate), prev_mode(tl_gate_mode) {
  tl_gate = f;
  tl_gate_mode = m;
}
InputGate::~InputGate() {
  tl_gate = prev_flags;
  tl_gate_mode = prev_mode;
}
const int* InputGate::flags() { return tl_gate; }
int InputGate::mode() { return tl_gate_mode; }

namespace {
thread_local RowDoneHook* tl_rowhook = nullptr;
}  // namespace
RowHook::RowHook(RowDoneHook* h) : prev(tl_rowhook) { tl_rowhook = h; }
RowHook::~RowHook() { tl_rowhook = prev; }
RowDoneHook* RowHook::current() { return tl_rowhook; }
void RowHook::consumed() { tl_rowhook = nullptr; }

namespace {

constexpr int TP = 64;    // tile order (== LEAF)
constexpr int TPT = 128;  // threads per CTA (4 warps, 2 x 2 of 32 x 32)
constexpr int STAGES = 3;
constexpr int SYNC_HDR = 32;  // ints before the flag array: [0] counter, [1] abort

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// acquire side of the flag protocol: relaxed polls (no L1 invalidation per
// poll), then ONE acquire fence once the flags are seen set
__device__ __forceinline__ void fence_acquire() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// one thread: wait for *f != 0 with acquire loads (the tile trsm's chain
// wait: measured faster there than relaxed polling + a fence)
__device__ void spin_wait_acquire(const int* f) {
  unsigned ns = 32;
  while (!ld_acquire(f)) {
    __nanosleep(ns);
    if (ns < 256) ns *= 2;
  }
}
// one thread: wait for *f != 0 (true) or an abort (false; abort may be null);
// the caller issues fence_acquire() before trusting data guarded by *f.
__device__ bool spin_wait(const int* f, const int* abort) {
  unsigned ns = 32;
  for (;;) {
    if (ld_relaxed(f)) return true;
    if (abort && ld_relaxed(abort)) return false;
    __nanosleep(ns);
    if (ns < 256) ns *= 2;
  }
}

template <typename T> struct TileCfg {
  static constexpr bool CPLX = is_cplx<T>::value;
  static constexpr int BK = CPLX ? 8 : 16;
  static constexpr int NACC = CPLX ? 2 : 1;
};

// Cholesky K-loop pipeline per operand orientation.  Row-major (K-major)
// operands from RFP blocks have an odd leading dimension, so a 16-wide k
// slice of a row (128 B real) straddles 5 sectors instead of 4; 32-wide
// slices (256 B: 9 instead of 8) with two stages keep three CTAs per SM and
// measured 9.1 -> ~7.8 ms on potrf(8192) with ld 8193.
// Column-major (MN-major) real operands of the single-region kernel (the
// large orders): four stages of 8 k instead of three of 16, as in the GEMM
// kernel -- alone the potrf does not change (8192: 6.93 vs 6.94 ms), beside
// the gated S1 solve and beside pftrs part 1 it does (config 3: 23.8 -> 23.2
// and 13.9 -> 13.2 ms).  The two-region chain of the mid orders keeps 16 x 3
// (config 2 measured +-1% either way).
template <typename T, bool KM, bool TWO> struct PipeCfg {
  static constexpr bool CPLX = is_cplx<T>::value;
  static constexpr bool FINE = !KM && !CPLX && !TWO;
  static constexpr int BK = KM ? (CPLX ? 16 : 32) : (CPLX || FINE ? 8 : 16);
  static constexpr int ST = (KM && !CPLX) ? 2 : (FINE ? 4 : 3);
  static constexpr int SPC = TP / BK;
};

template <typename T, bool KM, bool TWO> size_t pipe_smem_elems() {
  using P = PipeCfg<T, KM, TWO>;
  return (size_t)P::ST * 2 * SmemLayout<T, TP, P::BK, KM>::SIZE;
}
template <typename T, bool KM0, bool KM1, bool TWO> size_t tile_smem_bytes() {
  const size_t p0 = pipe_smem_elems<T, KM0, TWO>(), p1 = pipe_smem_elems<T, KM1, TWO>();
  const size_t pipe = p0 > p1 ? p0 : p1;
  const size_t leaf = (size_t)2 * TP * LD64 + 128;
  return (pipe > leaf ? pipe : leaf) * sizeof(T);
}

template <typename T>
__device__ __forceinline__ T frag(const double (&acc)[TileCfg<T>::NACC][2][4][4], int mi, int ni,
                                  int r) {
  if constexpr (is_cplx<T>::value) return Z{acc[0][mi][ni][r], acc[1][mi][ni][r]};
  else return acc[0][mi][ni][r];
}
// the same for any fragment grid (re / im planes passed separately)
template <typename T, int MI, int NI>
__device__ __forceinline__ T fragn(const double (&re)[MI][NI][4], const double (&im)[MI][NI][4],
                                   int mi, int ni, int r) {
  if constexpr (is_cplx<T>::value) return Z{re[mi][ni][r], im[mi][ni][r]};
  else return re[mi][ni][r];
}

// acc += X Y^H for 64-wide K from two LD64 shared tiles (rows of X and of Y
// along M / N): the off-diagonal solve L(i, j) = C W_j^H.
template <typename T>
__device__ __forceinline__ void smem_mm_yh(const T* X, const T* Y,
                                           double (&acc)[TileCfg<T>::NACC][2][4][4]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp & 1, wn = warp >> 1, g = lane >> 2, t = lane & 3;
  __syncwarp();  // mma.sync.aligned needs the converged warp (see publish)
#pragma unroll 4
  for (int k = 0; k < TP; k += 4) {
    if constexpr (!is_cplx<T>::value) {
      double a[2][2], b[4];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        a[mi][0] = X[(wm * 32 + mi * 16 + g) + (k + t) * LD64];
        a[mi][1] = X[(wm * 32 + mi * 16 + g + 8) + (k + t) * LD64];
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[ni] = Y[(wn * 32 + ni * 8 + g) + (k + t) * LD64];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma16x8x4(acc[0][mi][ni], a[mi][0], a[mi][1], b[ni]);
    } else {
      double ar[2][2], ai[2][2], nai[2][2], br[4], bi[4];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const Z v0 = X[(wm * 32 + mi * 16 + g) + (k + t) * LD64];
        const Z v1 = X[(wm * 32 + mi * 16 + g + 8) + (k + t) * LD64];
        ar[mi][0] = v0.x; ai[mi][0] = v0.y; nai[mi][0] = -v0.y;
        ar[mi][1] = v1.x; ai[mi][1] = v1.y; nai[mi][1] = -v1.y;
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const Z w = Y[(wn * 32 + ni * 8 + g) + (k + t) * LD64];
        br[ni] = w.x; bi[ni] = -w.y;  // conj
      }
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
          dmma16x8x4(acc[0][mi][ni], ar[mi][0], ar[mi][1], br[ni]);
          dmma16x8x4(acc[0][mi][ni], nai[mi][0], nai[mi][1], bi[ni]);
          dmma16x8x4(acc[1][mi][ni], ar[mi][0], ar[mi][1], bi[ni]);
          dmma16x8x4(acc[1][mi][ni], ai[mi][0], ai[mi][1], br[ni]);
        }
    }
  }
}

// ---------------------------------------------------------- task helpers
// Task kinds of the Cholesky DAG (see potrf_tiles): the chain of diagonal
// tiles is carried by "super" tasks -- ST(j) finishes tile (j+1, j) AND
// factors diagonal tile j+1 straight from its own result, so the critical
// path per column is one 64^3 solve + one 64^3 rank-64 update + the leaf,
// with no flag round trip between the sub-diagonal tile and the next leaf.
enum TaskKind : int { TK_DIAG0 = 0, TK_SUPER = 1, TK_NORMAL = 2, TK_PARTIAL = 3 };

// The factored matrix is one or two REGIONS of the global lower triangle:
// region 0 = columns [0, n1) of view A (all m rows: for a tall panel the
// rows below n1 are solved, not factored), region 1 = the trailing
// (n - n1) x (n - n1) lower block at global offset (n1, n1), its own view B
// (an RFP's T2^T beside the [T1; S] panel: pftrf's whole SRPA chain in one
// launch).  Row and column tiles restart at n1, so the last tile of region
// 0 may be ragged; off / sz give every tile's global offset and order.
template <typename T, bool TWO = false> struct CholCtx {
  View<T> A, B;
  T* W;
  int* info;
  int* done;    // mt x nt tile flags
  int* pready;  // nt flags: diagonal partial sums written
  int* abort;
  int base, n, nt;  // columns (the factored order) and their tiles
  int m, mt;        // rows and row tiles (m >= n: a tall panel [L11; L21])
  int n1, nt1;      // region 0's columns and column tiles (n1 == n: one region)
  const int* ext;   // optional input gate: column block j readable once ext[j]
  // (TWO = false: one region, tiles on the plain 64-grid -- the kernel's
  // code stays small, which the latency-bound chain measurably needs)
  __device__ __forceinline__ int off(int I) const {
    if constexpr (!TWO) return I * TP;
    return I < nt1 ? I * TP : n1 + (I - nt1) * TP;
  }
  __device__ __forceinline__ int sz(int I) const {
    const int e = (TWO && I >= nt1 ? m : (I < nt1 ? n1 : m)) - off(I);
    return e < TP ? e : TP;
  }
  // tile (I, J) as a view (origin, order sz(I) x sz(J), the region's strides)
  __device__ __forceinline__ View<T> tile(int I, int J) const {
    const int r = off(I), c = off(J);
    if (!TWO || J < nt1) return View<T>{A.p + (i64)r * A.rs + (i64)c * A.cs, sz(I), sz(J), A.rs, A.cs};
    return View<T>{B.p + (i64)(r - n1) * B.rs + (i64)(c - n1) * B.cs, sz(I), sz(J), B.rs, B.cs};
  }
  // the tile's view is row-major (loads with lanes along columns)
  __device__ __forceinline__ bool rowmajor(int J) const {
    return ((!TWO || J < nt1) ? A.rs : B.rs) != 1;
  }
};

template <typename T>
__device__ __forceinline__ void zero_acc(double (&acc)[TileCfg<T>::NACC][2][4][4]) {
#pragma unroll
  for (int c = 0; c < TileCfg<T>::NACC; ++c)
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[c][mi][ni][r] = 0.0;
}

// fragment (mi, ni, r) -> tile coordinates
__device__ __forceinline__ void frag_rc(int mi, int ni, int r, int& row, int& col) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  row = (warp & 1) * 32 + mi * 16 + (lane >> 2) + ((r & 2) ? 8 : 0);
  col = (warp >> 1) * 32 + ni * 8 + 2 * (lane & 3) + (r & 1);
}

// Convergence: the flag protocol runs in thread 0 (spins, atomics, the
// release) while the other threads wait at the barrier; every barrier here
// is cta_sync() (common.cuh: reconverge, then bar.sync) and every warp-wide
// DMMA sequence (mma.sync.aligned) starts with __syncwarp().
//
// one thread publishes a flag after the whole CTA's stores: the barrier
// orders every thread's stores before thread 0's release, and a release is
// cumulative over what its thread has observed, so ONE gpu-scope fence (the
// release's own) publishes the whole tile (an extra __threadfence before it
// cost ~0.5 us per diagonal step on the chain)
__device__ __forceinline__ void publish(int* f) {
  cta_sync();
#ifdef RFPK_PUBLISH_FENCE
  if (threadIdx.x == 0) __threadfence();
#endif
  if (threadIdx.x == 0) st_release(f, 1);
}
__device__ __forceinline__ bool wait_flag(int* f, int* abort, int* s_ok, bool hot = false) {
  if (threadIdx.x == 0) {
    if (hot) {
      // the chain's wait: acquire polls (no separate fence after the flag)
      int ok;
      for (;;) {
        if (ld_acquire(f)) { ok = 1; break; }
        if (ld_relaxed(abort)) { ok = 0; break; }
      }
      *s_ok = ok;
    } else {
      *s_ok = spin_wait(f, abort);
      fence_acquire();
    }
  }
  cta_sync();
  return *s_ok != 0;
}

// acc += sum_{kb <= k < ke} L(i, k) L(j, k)^H over the chunks of ONE region
// (view V, global offset roff), chunk k loaded only once tiles (i, k) and
// (j, k) are published.  Pipelined cp.async; a ragged chunk (region 0's last
// tile) is zero-filled past its width.  Returns false on abort.  Leaves the
// pipeline drained and the CTA synchronised.
template <typename T, bool KM, bool TWO>
__device__ bool acc_range(const CholCtx<T, TWO>& X, const View<T>& V, int roff, int i, int j, int kb,
                          int ke, T* sm, int* s_ok, double (&acc)[TileCfg<T>::NACC][2][4][4]) {
  using C = TileCfg<T>;
  using P = PipeCfg<T, KM, TWO>;
  using LA = SmemLayout<T, TP, P::BK, KM>;
  constexpr int BK = P::BK, SPC = P::SPC, STAGES = P::ST;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1, gq = lane >> 2, tq = lane & 3;
  T* As = sm;
  T* Bs = sm + STAGES * LA::SIZE;
  const i64 ld = KM ? V.rs : V.cs;
  // element (r, k) of the region in GLOBAL coordinates, k from chunk kb
  const T* base = V.p - (i64)roff * V.rs + (i64)(X.off(kb) - roff) * V.cs;
  TileLoader<T, TP, BK, TPT, KM> la, lb;
  const int ri = X.off(i), rj = X.off(j);
  la.init(base, ld, ri, ri + X.sz(i), tid);
  lb.init(base, ld, rj, rj + X.sz(j), tid);
  // chunk kc's tiles are final.  Thread 0 also scans ahead over chunks that
  // are already published, so a task whose inputs are all done pays ONE
  // barrier instead of one per chunk.  *s_ok = 1 + last verified chunk, or 0
  // on abort (read by all threads before the loop's next barrier).
  int known = kb - 1;
  auto ready = [&](int kc) -> bool {
    if (kc <= known) return true;
    if (tid == 0) {
      bool ok = spin_wait(X.done + (i64)i * X.nt + kc, X.abort);
      if (ok && i != j) ok = spin_wait(X.done + (i64)j * X.nt + kc, X.abort);
      int k2 = kc;
      if (ok)
        while (k2 + 1 < ke && ld_relaxed(X.done + (i64)i * X.nt + k2 + 1) &&
               (i == j || ld_relaxed(X.done + (i64)j * X.nt + k2 + 1)))
          ++k2;
      fence_acquire();
      *s_ok = ok ? k2 + 1 : 0;
    }
    cta_sync();
    known = *s_ok - 1;
    return known >= kc;
  };
  auto load_stage = [&](int stage, int q) {
    const int kw = TWO ? X.sz(kb + q / SPC) : TP;
    if (kw == TP) {
      la.load(As + stage * LA::SIZE);
      lb.load(Bs + stage * LA::SIZE);
    } else {
      la.load_pred(As + stage * LA::SIZE, (q % SPC) * BK, kw, ri, 0);
      lb.load_pred(Bs + stage * LA::SIZE, (q % SPC) * BK, kw, rj, 0);
    }
    la.advance();
    lb.advance();
  };
  const int KT = (ke - kb) * SPC;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) {
      if (s % SPC == 0 && !ready(kb + s / SPC)) {
        cp_async_wait<0>();
        return false;
      }
      load_stage(s, s);
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    cta_sync();
    const int nk = kt + STAGES - 1;
    if (nk < KT) {
      if (nk % SPC == 0 && !ready(kb + nk / SPC)) {
        cp_async_wait<0>();
        return false;
      }
      load_stage(nk % STAGES, nk);
    }
    cp_async_commit();
    __syncwarp();  // (a thread-0 flag wait may have left the warp split)
    const T* as = As + (kt % STAGES) * LA::SIZE + (wm * 32 + gq) * LA::RS + tq * LA::KS;
    const T* bs = Bs + (kt % STAGES) * LA::SIZE + (wn * 32 + gq) * LA::RS + tq * LA::KS;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      if constexpr (!C::CPLX) {
        double af[2][2], bf[4];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
          af[mi][0] = as[kk * LA::KS + (mi * 16) * LA::RS];
          af[mi][1] = as[kk * LA::KS + (mi * 16 + 8) * LA::RS];
        }
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) bf[ni] = bs[kk * LA::KS + (ni * 8) * LA::RS];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma16x8x4(acc[0][mi][ni], af[mi][0], af[mi][1], bf[ni]);
      } else {
        double ar[2][2], ai[2][2], nai[2][2], br[4], bi[4];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
          const Z v0 = as[kk * LA::KS + (mi * 16) * LA::RS];
          const Z v1 = as[kk * LA::KS + (mi * 16 + 8) * LA::RS];
          ar[mi][0] = v0.x; ai[mi][0] = v0.y; nai[mi][0] = -v0.y;
          ar[mi][1] = v1.x; ai[mi][1] = v1.y; nai[mi][1] = -v1.y;
        }
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
          const Z w = bs[kk * LA::KS + (ni * 8) * LA::RS];
          br[ni] = w.x; bi[ni] = -w.y;  // L(j, k)^H
        }
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) {
            dmma16x8x4(acc[0][mi][ni], ar[mi][0], ar[mi][1], br[ni]);
            dmma16x8x4(acc[0][mi][ni], nai[mi][0], nai[mi][1], bi[ni]);
            dmma16x8x4(acc[1][mi][ni], ar[mi][0], ar[mi][1], bi[ni]);
            dmma16x8x4(acc[1][mi][ni], ai[mi][0], ai[mi][1], br[ni]);
          }
      }
    }
  }
  cp_async_wait<0>();
  cta_sync();  // pipeline buffers are reused by the caller
  return true;
}

template <typename T, bool KM0, bool KM1, bool TWO>
__device__ bool accumulate(const CholCtx<T, TWO>& X, int i, int j, int kend, T* sm, int* s_ok,
                           double (&acc)[TileCfg<T>::NACC][2][4][4]) {
  if constexpr (!TWO) {
    return acc_range<T, KM0, TWO>(X, X.A, 0, i, j, 0, kend, sm, s_ok, acc);
  } else if constexpr (KM0 == KM1) {
    // one copy of the pipeline for both regions (a second inlined copy grew
    // the kernel by a third and slowed the latency-bound chain)
#pragma unroll 1
    for (int rg = 0; rg < 2; ++rg) {
      const int kb = rg ? X.nt1 : 0, ke = rg ? kend : (kend < X.nt1 ? kend : X.nt1);
      if (ke <= kb) continue;
      if (!acc_range<T, KM0, TWO>(X, rg ? X.B : X.A, rg ? X.n1 : 0, i, j, kb, ke, sm, s_ok, acc))
        return false;
    }
    return true;
  } else {
    const int k0 = kend < X.nt1 ? kend : X.nt1;
    if (k0 > 0 && !acc_range<T, KM0, TWO>(X, X.A, 0, i, j, 0, k0, sm, s_ok, acc)) return false;
    if (kend > X.nt1 && !acc_range<T, KM1, TWO>(X, X.B, X.n1, i, j, X.nt1, kend, sm, s_ok, acc))
      return false;
    return true;
  }
}

// Off-diagonal tile (i, j) in two halves so that everything not needing W_j
// happens before the wait for it:
//   build_c: S = A(i, j) - acc (rows past the matrix zeroed)
//   apply_w: Ws = W_j, x = S W_j^H; X written to A(i, j) and to smem tile Xs
template <typename T, bool TWO>
__device__ void build_c(const CholCtx<T, TWO>& X, int i, int j,
                        const double (&acc)[TileCfg<T>::NACC][2][4][4], T* S) {
  const View<T> tv = X.tile(i, j);
  const int mrows = (int)tv.m, ncols = (int)tv.n;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        int row, col;
        frag_rc(mi, ni, r, row, col);
        S[row + col * LD64] = row < mrows && col < ncols
                                  ? *tv.at(row, col) - frag<T>(acc, mi, ni, r)
                                  : zero_<T>();
      }
}
template <typename T, bool TWO>
__device__ void apply_w(const CholCtx<T, TWO>& X, int i, int j, T* S, T* Ws,
                        double (&x)[TileCfg<T>::NACC][2][4][4], T* Xs) {
  const int tid = threadIdx.x;
  const View<T> tv = X.tile(i, j);
  const int mrows = (int)tv.m, ncols = (int)tv.n;
  const T* w = X.W + (i64)j * TP * TP;
  // W_j (32 KB, L2-resident: just written by the diagonal task) with every
  // load in flight at once (cp.async.cg bypasses L1: written by another CTA)
#ifdef RFPK_W_LDCG
  if constexpr (!is_cplx<T>::value) {
#pragma unroll 8
    for (int e = tid; e < TP * TP; e += TPT) Ws[(e & 63) + (e >> 6) * LD64] = __ldcg(w + e);
  }
  if (is_cplx<T>::value)
#endif
#pragma unroll 8
  for (int e = tid; e < TP * TP; e += TPT) {
    if constexpr (is_cplx<T>::value) {
      cp_async16(Ws + (e & 63) + (e >> 6) * LD64, w + e, true);
    } else {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(Ws + (e & 63) + (e >> 6) * LD64);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(w + e));
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  cta_sync();
  zero_acc<T>(x);
  smem_mm_yh<T>(S, Ws, x);
  cta_sync();  // S and Ws fully read
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        int row, col;
        frag_rc(mi, ni, r, row, col);
        const T v = frag<T>(x, mi, ni, r);
        // (columns past a ragged tile come out exactly 0: S is zero there and
        // W_j identity-padded)
        Xs[row + col * LD64] = row < mrows ? v : zero_<T>();
        if (row < mrows && col < ncols) *tv.at(row, col) = v;
      }
}

// Diagonal tile d from S (lower, identity-padded, ready): leaf -> L(d, d)
// into A and W_d into its slab, then publish done(d, d).  false = failure.
template <typename T, bool TWO>
__device__ bool finish_diag(const CholCtx<T, TWO>& X, int d, T* S, T* Ws, T* scr, int* s_ok) {
  const int tid = threadIdx.x;
  const View<T> tv = X.tile(d, d);
  const int d0 = X.off(d), m = (int)tv.m;
  ct_mark(d, 4);
  const int f = leaf_factor_inv64(S, Ws, scr, s_ok, d);
  ct_mark(d, 5);
  if (f) {
    if (tid == 0) {
      *X.info = X.base + d0 + f;
      __threadfence();
      st_release(X.abort, 1);
    }
    return false;
  }
  cta_sync();
  const bool km = X.rowmajor(d);
  for (int e = tid; e < TP * TP; e += TPT) {
    int r, c;
    if (km) { c = e & 63; r = e >> 6; }  // lanes along the unit-stride dimension
    else { r = e & 63; c = e >> 6; }
    if (r < m && c <= r) *tv.at(r, c) = S[r + c * LD64];
  }
  T* w = X.W + (i64)d * TP * TP;
  for (int e = tid; e < TP * TP; e += TPT) w[e] = Ws[(e & 63) + (e >> 6) * LD64];
  ct_mark(d, 6);
  publish(X.done + (i64)d * X.nt + d);
  ct_mark(d, 7);
  return true;
}

// S <- identity-padded lower part of A(d, d) (read from L2: it may have been
// written by another CTA)
template <typename T, bool TWO> __device__ void load_diag(const CholCtx<T, TWO>& X, int d, T* S) {
  const View<T> tv = X.tile(d, d);
  const int m = (int)tv.m;
  const bool km = X.rowmajor(d);
  for (int e = threadIdx.x; e < TP * TP; e += TPT) {
    int r, c;
    if (km) { c = e & 63; r = e >> 6; }
    else { r = e & 63; c = e >> 6; }
    T v = (r == c) ? one_<T>() : zero_<T>();
    if (r < m && c < m && c <= r) {
      const T* src = tv.at(r, c);
      if constexpr (is_cplx<T>::value) {
        const double2 q = __ldcg(reinterpret_cast<const double2*>(src));
        v = Z{q.x, q.y};
      } else {
        v = __ldcg(src);
      }
    }
    S[r + c * LD64] = v;
  }
}

// the input gate (if any): column block j of A's original data has landed
template <typename T, bool TWO>
__device__ __forceinline__ bool wait_input(const CholCtx<T, TWO>& X, int j, int* s_ok) {
  if (!X.ext) return true;
  return wait_flag(const_cast<int*>(X.ext) + j, X.abort, s_ok);
}

template <typename T, bool KM0, bool KM1, bool TWO>
__device__ bool run_task(const CholCtx<T, TWO>& X, int kind, int a, int b, T* sm, int* s_ok) {
  using C = TileCfg<T>;
  T* S = sm;
  T* Ws = S + TP * LD64;
  T* scr = Ws + TP * LD64;
  double acc[C::NACC][2][4][4];
  zero_acc<T>(acc);
  if (kind == TK_DIAG0) {
    if (!wait_input(X, 0, s_ok)) return false;
    load_diag(X, 0, S);
    cta_sync();
    const bool ok = finish_diag(X, 0, S, Ws, scr, s_ok);
    return ok;
  }
  if (kind == TK_PARTIAL) {
    // A(d, d) <- A(d, d) - sum_{k < d-1} L(d, k) L(d, k)^H  (lower part)
    const int d = a;
    if (!accumulate<T, KM0, KM1, TWO>(X, d, d, d - 1, sm, s_ok, acc)) return false;
    if (!wait_input(X, d, s_ok)) return false;
    const View<T> tv = X.tile(d, d);
    const int m = (int)tv.m;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          int row, col;
          frag_rc(mi, ni, r, row, col);
          if (row < m && col <= row) {
            T* p = tv.at(row, col);
            *p = *p - frag<T>(acc, mi, ni, r);
          }
        }
    publish(X.pready + d);
    return true;
  }
  // TK_NORMAL (i, j) and TK_SUPER (j + 1, j)
  const int i = a, j = b;
  if (kind == TK_SUPER) ct_mark(i, 0);
  if (!accumulate<T, KM0, KM1, TWO>(X, i, j, j, sm, s_ok, acc)) return false;
  if (kind == TK_SUPER) ct_mark(i, 1);
  if (!wait_input(X, j, s_ok)) return false;
  // (diag 1 has no partial task: its original tile is read below)
  if (kind == TK_SUPER && i == 1 && !wait_input(X, 1, s_ok)) return false;
  build_c(X, i, j, acc, S);
  const int d = i;  // super: the diagonal tile factored next
  const int m = X.sz(d);
  // real: prefetch the diagonal partial sum into acc (fragment layout, lower
  // part, identity padding) while W_j is still being produced; complex (no
  // spare registers) reloads it after the solve instead
  if (kind == TK_SUPER && !C::CPLX) {
    if (d >= 2 && !wait_flag(X.pready + d, X.abort, s_ok)) return false;
    const View<T> tv = X.tile(d, d);
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          int row, col;
          frag_rc(mi, ni, r, row, col);
          T v = (row == col) ? one_<T>() : zero_<T>();
          if (row < m && col < m && col <= row) {
            const T* src = tv.at(row, col);
            if constexpr (is_cplx<T>::value) {
              const double2 q = __ldcg(reinterpret_cast<const double2*>(src));
              v = Z{q.x, q.y};
            } else {
              v = __ldcg(src);
            }
          }
          if constexpr (is_cplx<T>::value) { acc[0][mi][ni][r] = v.x; acc[1][mi][ni][r] = v.y; }
          else acc[0][mi][ni][r] = v;
        }
  }
  if (!wait_flag(X.done + (i64)j * X.nt + j, X.abort, s_ok, kind == TK_SUPER)) return false;
  if (kind == TK_SUPER) ct_mark(i, 2);
  double x[C::NACC][2][4][4];
  apply_w(X, i, j, S, Ws, x, kind == TK_SUPER ? Ws : S);
  if (kind == TK_SUPER) ct_mark(i, 3);
  publish(X.done + (i64)i * X.nt + j);
  if (kind == TK_NORMAL) {
    return true;
  }
  // super: diag d = partial - L(d, j) L(d, j)^H, then the leaf (X is in Ws)
  if constexpr (C::CPLX) {
    if (d >= 2 && !wait_flag(X.pready + d, X.abort, s_ok)) return false;
    load_diag(X, d, S);
    cta_sync();
  }
  zero_acc<T>(x);
  smem_mm_yh<T>(Ws, Ws, x);
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        int row, col;
        frag_rc(mi, ni, r, row, col);
        if constexpr (C::CPLX) {
          if (row < m && col <= row) S[row + col * LD64] = S[row + col * LD64] - frag<T>(x, mi, ni, r);
        } else {
          T v = (row == col) ? one_<T>() : zero_<T>();
          if (row < m && col < m && col <= row) v = frag<T>(acc, mi, ni, r) - frag<T>(x, mi, ni, r);
          S[row + col * LD64] = v;
        }
      }
  cta_sync();
  const bool ok = finish_diag(X, d, S, Ws, scr, s_ok);
  return ok;
}

// Task list: DIAG0, then for every column block g = 0 .. nt-1 the group
//   [ SUPER(g) = tile (g+1, g) + diag g+1          (if g+1 < nt),
//     NORMAL (i, g) for i = g+2 .. mt-1 (g+1 .. mt-1 when there is no SUPER),
//     PARTIAL(g+2) = diag g+2 over chunks k <= g  (if g+2 < nt) ]
// Every task depends only on tasks listed before it.  mt > nt: a tall panel
// whose rows below the last diagonal tile are solved like any other tile.
__host__ __device__ inline long long chol_group_size(int g, int nt, int mt) {
  const int sup = g + 1 < nt ? 1 : 0;
  const int first = g + 1 + sup;  // first NORMAL row tile
  return sup + (mt > first ? mt - first : 0) + (g + 2 < nt ? 1 : 0);
}
__host__ __device__ inline long long chol_task_count(int nt, int mt) {
  long long t = nt > 0 ? 1 : 0;
  for (int g = 0; g < nt; ++g) t += chol_group_size(g, nt, mt);
  return t;
}

template <typename T, bool KM0, bool KM1, bool TWO>
__global__ void __launch_bounds__(TPT, is_cplx<T>::value ? 1 : 3)
    tile_potrf_kernel(View<T> A, View<T> B, int n1, int nt1, int ncols, T* W, int* info, int base,
                      int* sync, int nt, int mt, const int* ext) {
  extern __shared__ __align__(16) double smem_d[];
  T* sm = reinterpret_cast<T*>(smem_d);
  __shared__ int s_task, s_ok;
  if (*info) return;  // an earlier step of the chain failed
  CholCtx<T, TWO> X;
  X.A = A;
  X.B = B;
  X.W = W;
  X.info = info;
  X.abort = sync + 1;
  X.done = sync + SYNC_HDR;
  X.pready = X.done + (i64)mt * nt;
  X.base = base;
  X.n = ncols;
  X.nt = nt;
  X.m = nt1 < nt ? ncols : (int)A.m;
  X.mt = mt;
  X.n1 = n1;
  X.nt1 = nt1;
  X.ext = ext;
  const long long total = chol_task_count(nt, mt);
  int g = 0;
  long long gbase = 1;  // first task of group g
  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(sync, 1);
    cta_sync();
    const long long t = s_task;
    cta_sync();
    if (t >= total) return;
    int kind, a, b;
    if (t == 0) {
      kind = TK_DIAG0; a = 0; b = 0;
    } else {
      for (;;) {
        const long long gs = chol_group_size(g, nt, mt);
        if (t < gbase + gs) break;
        gbase += gs;
        ++g;
      }
      int o = (int)(t - gbase);
      const int sup = g + 1 < nt ? 1 : 0;
      const int first = g + 1 + sup;
      const int nnorm = mt > first ? mt - first : 0;
      if (sup && o == 0) { kind = TK_SUPER; a = g + 1; b = g; }
      else if ((o -= sup) < nnorm) { kind = TK_NORMAL; a = first + o; b = g; }
      else { kind = TK_PARTIAL; a = g + 2; b = 0; }
    }
    if (!run_task<T, KM0, KM1, TWO>(X, kind, a, b, sm, &s_ok)) return;
  }
}

template <typename T, bool KM0, bool KM1, bool TWO>
int tile_launch(View<T> A, View<T> B, int n1, int nt1, int ncols, T* W, Ctx c, int base, int* sync,
                int nt, int mt) {
  auto kern = tile_potrf_kernel<T, KM0, KM1, TWO>;
  const size_t smem = tile_smem_bytes<T, KM0, KM1, TWO>();
  const int per_sm = kernel_setup(kern, TPT, smem);
  const long long tasks = chol_task_count(nt, mt);
  // two CTAs per SM up to ~12k columns: the diagonal chain's CTA then shares
  // its SM with one other task instead of two (measured: potrf 8192 7.69 ->
  // 7.22 ms, 4000 2.22 -> 2.13); the bulk-bound larger orders keep three
  const int ps = per_sm > 2 && nt <= 192 ? 2 : per_sm;
  long long grid = (long long)ps * num_sms();
  if (grid > tasks) grid = tasks;
  KernelClock kc(c.st);
  kern<<<(unsigned)grid, TPT, smem, c.st>>>(A, B, n1, nt1, ncols, W, c.info, base, sync, nt, mt,
                                            InputGate::flags());
  RFPK_CHECK_LAUNCH();
  kc.stop("tile_potrf", A.m, ncols);
  return 0;
}

// ============================================================ tile trsm
// conj?(Tm) X = B in place, Tm lower (forward) or upper (backward) in its
// view, with the 64-block inverses W (lower form; wtrans: the diagonal block
// of Tm is the TRANSPOSE of slab i, i.e. Tm upper).  Same dataflow scheme:
// task (i, c) owns the 64 x 64 block X(i, c) (c: 64-column block of B);
//   acc = sum_{k solved before i} Tm(i, k) X(k, c)   (waits done(k, c))
//   X(i, c) = W'_i (B(i, c) - acc)                    (DMMA from smem)
// Tasks go out step-major (forward: i ascending; backward: descending), so
// every column block's chain of row blocks advances in parallel and all
// off-chain accumulation overlaps it.

// Warp layout of a 64 x TN trsm tile: TN = 64 -> 2 x 2 warps of 32 x 32,
// TN = 16 (narrow right-hand sides) -> 4 x 1 warps of 16 x 16.
template <int TN> struct TrsmTile {
  static constexpr int WN = TN >= 64 ? 2 : 1;   // warps along N
  static constexpr int WMW = 4 / WN;            // warps along M
  static constexpr int RW = TP / WMW;           // rows per warp
  static constexpr int CW = TN / WN;            // columns per warp
  static constexpr int MI = RW / 16, NI = CW / 8;
};

// acc += A B for LD64 shared tiles, A 64 x 64 (A(r, k) = A[r + k*LD64]) and
// B 64 x TN (B(k, n) = B[k + n*LD64]).
template <typename T, int TN>
__device__ __forceinline__ void smem_mm_ab(
    const T* As, const T* Bs,
    double (&acc)[TileCfg<T>::NACC][TrsmTile<TN>::MI][TrsmTile<TN>::NI][4]) {
  using W = TrsmTile<TN>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp % W::WMW, wn = warp / W::WMW, g = lane >> 2, t = lane & 3;
  __syncwarp();  // mma.sync.aligned needs the converged warp
#pragma unroll 4
  for (int k = 0; k < TP; k += 4) {
    if constexpr (!is_cplx<T>::value) {
      double a[W::MI][2], b[W::NI];
#pragma unroll
      for (int mi = 0; mi < W::MI; ++mi) {
        a[mi][0] = As[(wm * W::RW + mi * 16 + g) + (k + t) * LD64];
        a[mi][1] = As[(wm * W::RW + mi * 16 + g + 8) + (k + t) * LD64];
      }
#pragma unroll
      for (int ni = 0; ni < W::NI; ++ni) b[ni] = Bs[(k + t) + (wn * W::CW + ni * 8 + g) * LD64];
#pragma unroll
      for (int mi = 0; mi < W::MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < W::NI; ++ni) dmma16x8x4(acc[0][mi][ni], a[mi][0], a[mi][1], b[ni]);
    } else {
      double ar[W::MI][2], ai[W::MI][2], nai[W::MI][2], br[W::NI], bi[W::NI];
#pragma unroll
      for (int mi = 0; mi < W::MI; ++mi) {
        const Z v0 = As[(wm * W::RW + mi * 16 + g) + (k + t) * LD64];
        const Z v1 = As[(wm * W::RW + mi * 16 + g + 8) + (k + t) * LD64];
        ar[mi][0] = v0.x; ai[mi][0] = v0.y; nai[mi][0] = -v0.y;
        ar[mi][1] = v1.x; ai[mi][1] = v1.y; nai[mi][1] = -v1.y;
      }
#pragma unroll
      for (int ni = 0; ni < W::NI; ++ni) {
        const Z w = Bs[(k + t) + (wn * W::CW + ni * 8 + g) * LD64];
        br[ni] = w.x; bi[ni] = w.y;
      }
#pragma unroll
      for (int mi = 0; mi < W::MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < W::NI; ++ni) {
          dmma16x8x4(acc[0][mi][ni], ar[mi][0], ar[mi][1], br[ni]);
          dmma16x8x4(acc[0][mi][ni], nai[mi][0], nai[mi][1], bi[ni]);
          dmma16x8x4(acc[1][mi][ni], ar[mi][0], ar[mi][1], bi[ni]);
          dmma16x8x4(acc[1][mi][ni], ai[mi][0], ai[mi][1], br[ni]);
        }
    }
  }
}

// prefetch W'_i into its own smem tile at the task start: only where the
// register budget already limits the kernel to two CTAs per SM (the
// column-major-B variants), so the extra 33 KB costs no occupancy
template <typename T, bool BKM> constexpr bool trsm_prew() { return BKM && !is_cplx<T>::value; }
// the solve's cp.async pipeline: real wide tiles take four stages of 8 k
// (S1 solve of config 3 alone 17.51 -> 17.19 ms, pftrs's 8192 x 1024 solves
// 2.59 -> 2.54 ms); the narrow, chain-bound tiles keep three of 16 (pftrs at
// n = 4000, nrhs = 64: 0.716 vs 0.750 ms)
template <typename T, int TN> struct TrsmPipe {
  static constexpr bool FINE = !is_cplx<T>::value && TN >= TP;
  static constexpr int BK = FINE ? 8 : TileCfg<T>::BK;
  static constexpr int ST = FINE ? 4 : STAGES;
  static constexpr int SPC = TP / BK;
};

struct TrsmArgs {
  int n, nrhs, nb, nc;
  int lower, conj, wtrans;
  const int* ext;  // input gate (see InputGate): B(i, c) readable once ext[ext_mode ? c : i]
  int ext_mode;
  // triangle gate (potrf_trsm_overlap): row block i of Tm and W_i are
  // readable once agate[i * agate_stride] is set; aabort != 0 = the producer
  // failed (every task then exits without touching B)
  const int* agate;
  int agate_stride;
  const int* aabort;
  // dispatch guard: a CTA at blockIdx >= aguard_keep that finds *aguard == 0
  // (the producer has not started) exits at once, so a solve whose CTAs got
  // dispatched first can never hold every slot the producer needs
  const int* aguard;
  int aguard_keep;
  int scan;  // scan-ahead chunk waits (see trsm_task's open_chunk)
  int* rowcnt;  // RowHook: finished column tasks per row block (or null)
  // forward solve whose right-hand side is lower-triangular (B(r, j) = 0 for
  // r < j: trtri's identity): X(r, j) = 0 for r < j too, so task (i, c)
  // sums only chunks k >= c TN / 64 and the tasks above that are no-ops
  int tri_rhs;
  // split tasks (shorter tail): the task of solve position p >= split_from
  // sums only its last split_m chunks; a PRE task handed out split_m + 1
  // steps earlier (its chunks are all handed out by then) sums the chunks
  // before that and subtracts them from B(i, c) in place, then sets
  // pre[i * nc + c].  0 = off.
  int split_m, split_from;
  int* pre;
};

template <typename T, bool AK, bool BKM, int TN>
__device__ bool trsm_task(const View<T>& Tm, const View<T>& B, const T* W, const TrsmArgs& a,
                          int* done, int i, int c, T* sm, int* s_ok, int kind = 0) {
  // kind 0: the whole task; 1: the task of a split position (its last
  // split_m chunks, then B(i, c) once the PRE task has updated it); 2: PRE
  if (a.agate) {  // Tm's row block i and W_i come from a concurrent tile potrf
    if (threadIdx.x == 0) {
      const int* f = a.agate + (i64)i * a.agate_stride;
      unsigned ns = 32;
      int ok;
      while (!(ok = ld_acquire(f)) && !ld_relaxed(a.aabort)) {
        __nanosleep(ns);
        if (ns < 256) ns *= 2;
      }
      *s_ok = ok;
    }
    cta_sync();
    if (!*s_ok) return false;
  }
  using C = TileCfg<T>;
  using PP = TrsmPipe<T, TN>;
  constexpr int STAGES = PP::ST;  // (shadows the file-wide default)
  using LA = SmemLayout<T, TP, PP::BK, AK>;
  using LB = SmemLayout<T, TN, PP::BK, BKM>;
  using WL = TrsmTile<TN>;
  constexpr int MI = WL::MI, NI = WL::NI;
  constexpr int NACC = C::NACC, BK = PP::BK, SPC = PP::SPC;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WL::WMW, wn = warp / WL::WMW, gq = lane >> 2, tq = lane & 3;
  T* As = sm;
  T* Bs = sm + STAGES * LA::SIZE;
  const i64 lda = AK ? Tm.rs : Tm.cs, ldb = BKM ? B.cs : B.rs;
  const int nprev = a.lower ? i : a.nb - 1 - i;  // chunks solved before block i
  // (triangular right-hand side: chunks before q0 hold zeros of X)
  const int q0 = kind == 1 ? nprev - a.split_m
                           : ((a.tri_rhs && a.lower) ? (c * TN) / TP : 0);
  const int qend = kind == 2 ? nprev - a.split_m : nprev;  // chunks [q0, qend)
  if (nprev < q0) return true;  // X(i, c) = 0: the workspace already holds it
  // (wide tiles only: the narrow, chain-bound solves measured slower with
  // the extra scan on their critical wait -- pftrs n = 4000 0.73 -> 0.755 ms)
  const bool scan_ahead = TN == TP && a.scan != 0;
  __shared__ int s_ready_sh;
  constexpr bool PREW = trsm_prew<T, BKM>();
  constexpr int PIPE = STAGES * (LA::SIZE + LB::SIZE);
  constexpr int STILE = (TN > TP ? TN : TP) * LD64;  // the S tile (64 x TN, LD64 columns)
  T* const Wpre = sm + (PIPE > STILE ? PIPE : STILE);  // PREW only
  if (PREW && kind != 2) {
    // W'_i does not depend on any task: fetch it now (oldest cp.async group,
    // complete before the first pipeline wait returns)
    const T* w = W + (i64)i * TP * TP;
    for (int e = tid; e < TP * TP; e += TPT) {
      const int r = e & 63, k = e >> 6;
      T* dst = a.wtrans ? Wpre + (k + r * LD64) : Wpre + (r + k * LD64);
      cp_async8(dst, w + e, true);
    }
    cp_async_commit();
  }
  auto chunk = [&](int q) { return a.lower ? q : a.nb - 1 - q; };

  TileLoader<T, TP, BK, TPT, AK> la;
  TileLoader<T, TN, BK, TPT, BKM> lb;
  double acc[NACC][MI][NI][4];
#pragma unroll
  for (int q = 0; q < NACC; ++q)
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[q][mi][ni][r] = 0.0;

  int kvalid = TP;  // valid k of the chunk being loaded
  // chunks q < ready (in solve order) are known published: a chunk beyond
  // waits for its flag with acquire polls (the chain's critical wait), then
  // warp 0 scans ahead 32 flags per round trip and one acquire fence covers
  // every further chunk found published -- one barrier for the long run of
  // chunks solved well before this task instead of one per chunk
  int ready = q0;
  auto open_chunk = [&](int kk) -> bool {
    const int q = a.lower ? kk : a.nb - 1 - kk;  // position in solve order
    if (!scan_ahead) {
      if (tid == 0) spin_wait_acquire(done + (i64)kk * a.nc + c);
      cta_sync();
    } else if (q >= ready) {
      if (warp == 0) {
        if (lane == 0) spin_wait_acquire(done + (i64)kk * a.nc + c);
        __syncwarp();
        int rr = q + 1;
        for (;;) {
          const int qq = rr + lane;
          const int k2 = a.lower ? qq : a.nb - 1 - qq;
          const bool ok = qq < qend && ld_relaxed(done + (i64)k2 * a.nc + c);
          const unsigned m = __ballot_sync(0xffffffffu, ok);
          if (m == 0xffffffffu) { rr += 32; continue; }
          rr += __ffs(~m) - 1;
          break;
        }
        // every lane that did a relaxed load of a flag orders it before the
        // barrier with its own fence (rr is warp-uniform; one MEMBAR per warp)
        if (rr > q + 1) fence_acquire();
        if (lane == 0) s_ready_sh = rr;
      }
      cta_sync();
      ready = s_ready_sh;
    }
    const T* ta = AK ? Tm.p + (i64)kk * TP : Tm.p + (i64)kk * TP * Tm.cs;
    la.init(ta, lda, i * TP, a.n, tid);
    const T* tb = BKM ? B.p + (i64)kk * TP : B.p + (i64)kk * TP * B.rs;
    lb.init(tb, ldb, c * TN, a.nrhs, tid);
    kvalid = a.n - kk * TP < TP ? a.n - kk * TP : TP;
    return true;  // (the solve never aborts: trsm inputs cannot fail)
  };
  auto load_stage = [&](int stage, int q) {
    const int k0 = (q % SPC) * BK;
    if (kvalid == TP) {
      la.load(As + stage * LA::SIZE);
      lb.load(Bs + stage * LB::SIZE);
    } else {
      la.load_pred(As + stage * LA::SIZE, k0, kvalid, 0, A_FULL);
      lb.load_pred(Bs + stage * LB::SIZE, k0, kvalid, 0, A_FULL);
    }
    la.advance();
    lb.advance();
  };

  // narrow tiles: B(i, c) does not depend on the chain -- read it into
  // registers now so the S build after the last chunk waits on nothing but
  // the accumulation (not under the host-streaming gate, which must be
  // waited first)
  constexpr bool BPRE = TN < TP;
  T bpre[BPRE ? MI : 1][BPRE ? NI : 1][4];
  const bool bpre_ok = BPRE && !a.ext;
  if constexpr (BPRE) {
    if (bpre_ok) {
      const i64 i0p = (i64)i * TP, c0p = (i64)c * TN;
      const int mr = a.n - (int)i0p < TP ? a.n - (int)i0p : TP;
      const int nc = a.nrhs - (int)c0p < TN ? a.nrhs - (int)c0p : TN;
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int row = wm * WL::RW + mi * 16 + gq + ((r & 2) ? 8 : 0);
            const int col = wn * WL::CW + ni * 8 + 2 * tq + (r & 1);
            bpre[mi][ni][r] = (row < mr && col < nc) ? *B.at(i0p + row, c0p + col) : zero_<T>();
          }
    }
  }
  const int KT = (qend - q0) * SPC;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) {
      if (s % SPC == 0) open_chunk(chunk(q0 + s / SPC));
      load_stage(s, s);
    }
    cp_async_commit();
  }
  const double sa = (C::CPLX && a.conj) ? -1.0 : 1.0;
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    cta_sync();
    const int nk = kt + STAGES - 1;
    if (nk < KT) {
      if (nk % SPC == 0) open_chunk(chunk(q0 + nk / SPC));
      load_stage(nk % STAGES, nk);
    }
    cp_async_commit();
    __syncwarp();  // (a thread-0 flag wait may have left the warp split)
    const T* as = As + (kt % STAGES) * LA::SIZE + (wm * WL::RW + gq) * LA::RS + tq * LA::KS;
    const T* bs = Bs + (kt % STAGES) * LB::SIZE + (wn * WL::CW + gq) * LB::RS + tq * LB::KS;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      if constexpr (!C::CPLX) {
        double af[MI][2], bf[NI];
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
          af[mi][0] = as[kk * LA::KS + (mi * 16) * LA::RS];
          af[mi][1] = as[kk * LA::KS + (mi * 16 + 8) * LA::RS];
        }
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) bf[ni] = bs[kk * LB::KS + (ni * 8) * LB::RS];
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) dmma16x8x4(acc[0][mi][ni], af[mi][0], af[mi][1], bf[ni]);
      } else {
        double ar[MI][2], ai[MI][2], nai[MI][2], br[NI], bi[NI];
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
          const Z v0 = as[kk * LA::KS + (mi * 16) * LA::RS];
          const Z v1 = as[kk * LA::KS + (mi * 16 + 8) * LA::RS];
          ar[mi][0] = v0.x; ai[mi][0] = sa * v0.y; nai[mi][0] = -ai[mi][0];
          ar[mi][1] = v1.x; ai[mi][1] = sa * v1.y; nai[mi][1] = -ai[mi][1];
        }
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          const Z w = bs[kk * LB::KS + (ni * 8) * LB::RS];
          br[ni] = w.x; bi[ni] = w.y;
        }
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) {
            dmma16x8x4(acc[0][mi][ni], ar[mi][0], ar[mi][1], br[ni]);
            dmma16x8x4(acc[0][mi][ni], nai[mi][0], nai[mi][1], bi[ni]);
            dmma16x8x4(acc[1][mi][ni], ar[mi][0], ar[mi][1], bi[ni]);
            dmma16x8x4(acc[1][mi][ni], ai[mi][0], ai[mi][1], br[ni]);
          }
      }
    }
  }
  cp_async_wait<0>();
  cta_sync();
  if (nprev > 0 && !*s_ok) return false;

  if (kind == 2) {  // PRE: B(i, c) -= the partial sum, in place
    const i64 pi0 = (i64)i * TP, pc0 = (i64)c * TN;
    const int pm = a.n - (int)pi0 < TP ? a.n - (int)pi0 : TP;
    const int pn = a.nrhs - (int)pc0 < TN ? a.nrhs - (int)pc0 : TN;
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int row = wm * WL::RW + mi * 16 + gq + ((r & 2) ? 8 : 0);
          const int col = wn * WL::CW + ni * 8 + 2 * tq + (r & 1);
          if (row < pm && col < pn) {
            T* bp = B.at(pi0 + row, pc0 + col);
            *bp = *bp - fragn<T>(acc[0], acc[NACC - 1], mi, ni, r);
          }
        }
    cta_sync();
    if (tid == 0) st_release(a.pre + (i64)i * a.nc + c, 1);
    return true;
  }
  if (kind == 1) {  // B(i, c) as the PRE task left it
    // (release/acquire through thread 0 and the CTA barriers on both sides,
    // as for the done flags: the PRE task's stores happen before every
    // thread's loads of the tile below.  Reading the tile with ld.global.cg
    // instead was measured: the changed register allocation costs 2.7%.)
    if (tid == 0) spin_wait_acquire(a.pre + (i64)i * a.nc + c);
    cta_sync();
  }

  if (a.ext) {  // B's original block (i, c) streamed in by the copy engine
    // (the gate's flags cover 64-column chunks; c counts TN-wide blocks)
    // (a TN-wide block may span several chunks: wait for its last one; the
    // copy stream publishes the chunks in order)
    if (tid == 0) {
      const int last = (c * TN + TN - 1 < a.nrhs - 1 ? c * TN + TN - 1 : a.nrhs - 1) / TP;
      spin_wait_acquire(a.ext + (a.ext_mode ? last : i));
    }
    cta_sync();
  }
  // S = B(i, c) - acc (zero outside the matrix), Ws = W'_i, X = Ws S
  T* S = sm;
  T* Ws = PREW ? Wpre : S + STILE;
  const i64 i0 = (i64)i * TP, c0 = (i64)c * TN;
  const int mrows = a.n - (int)i0 < TP ? a.n - (int)i0 : TP;
  const int ncols = a.nrhs - (int)c0 < TN ? a.nrhs - (int)c0 : TN;
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int row = wm * WL::RW + mi * 16 + gq + ((r & 2) ? 8 : 0);
        const int col = wn * WL::CW + ni * 8 + 2 * tq + (r & 1);
        T bv;
        if constexpr (BPRE) bv = bpre_ok ? bpre[mi][ni][r] : zero_<T>();
        if (!bpre_ok) bv = (row < mrows && col < ncols) ? *B.at(i0 + row, c0 + col) : zero_<T>();
        S[row + col * LD64] = (row < mrows && col < ncols)
                                  ? bv - fragn<T>(acc[0], acc[NACC - 1], mi, ni, r)
                                  : zero_<T>();
      }
  const T* w = W + (i64)i * TP * TP;
  for (int e = tid; e < (PREW ? 0 : TP * TP); e += TPT) {
    const int r = e & 63, k = e >> 6;
    T v;
    if constexpr (is_cplx<T>::value) {
      const double2 d = __ldcg(reinterpret_cast<const double2*>(w + e));
      v = Z{d.x, d.y};
    } else {
      v = __ldcg(w + e);
    }
    if (a.conj) v = conj_(v);
    if (a.wtrans) Ws[k + r * LD64] = v;  // W'(k, r) = W(r, k)
    else Ws[r + k * LD64] = v;
  }
  cta_sync();
  double x[NACC][MI][NI][4];
#pragma unroll
  for (int q = 0; q < NACC; ++q)
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni)
#pragma unroll
        for (int r = 0; r < 4; ++r) x[q][mi][ni][r] = 0.0;
  smem_mm_ab<T, TN>(Ws, S, x);
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int row = wm * WL::RW + mi * 16 + gq + ((r & 2) ? 8 : 0);
        const int col = wn * WL::CW + ni * 8 + 2 * tq + (r & 1);
        if (row < mrows && col < ncols) *B.at(i0 + row, c0 + col) = fragn<T>(x[0], x[NACC - 1], mi, ni, r);
      }
  cta_sync();
  if (tid == 0) {
    st_release(done + (i64)i * a.nc + c, 1);
    if (a.rowcnt)  // (a release of its own: ordered after this task's stores)
      asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(a.rowcnt + i) : "memory");
  }
  return true;
}

// row-major-B variants: 175 registers would round to two CTAs per SM; capped
// at 168 they fit three (the column-major-B ones need ~250 and run two)
template <typename T, bool AK, bool BKM, int TN>
__global__ void __launch_bounds__(TPT, TN < TP ? 3 : (TN > TP ? 2 : ((BKM || is_cplx<T>::value) ? 1 : 3)))
    tile_trsm_kernel(View<T> Tm, View<T> B, const T* W,
                                                        TrsmArgs a, int* sync, const int* info) {
  extern __shared__ __align__(16) double smem_d[];
  T* sm = reinterpret_cast<T*>(smem_d);
  __shared__ int s_task, s_ok;
  if (info && *info) {
    // skipped (an earlier step failed): a row-completion watcher must not
    // wait forever -- report every row block as done (b stays untouched)
    if (a.rowcnt && blockIdx.x == 0)
      for (int r = threadIdx.x; r < a.nb; r += blockDim.x) atomicExch(a.rowcnt + r, a.nc);
    return;
  }
  if (threadIdx.x == 0) s_ok = 1;  // cleared only by a failed triangle gate
  if (a.aguard && (int)blockIdx.x >= a.aguard_keep) {
    if (threadIdx.x == 0) s_task = ld_relaxed(a.aguard);
    cta_sync();
    if (s_task == 0) return;
  }
  int* counter = sync;
  int* done = sync + SYNC_HDR;
  const int npre = a.split_m ? a.nb - a.split_from : 0;
  const long long total = (long long)(a.nb + npre) * a.nc;
  // hand-out order: step by step the tasks of solve position `step`, and
  // (split solves) behind them the PRE tasks of position step + split_m + 1
  const int s1 = a.split_from - a.split_m - 1;
  const long long t1 = (long long)s1 * a.nc, span = (long long)npre * 2 * a.nc;
  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(counter, 1);
    cta_sync();
    const long long t = s_task;
    cta_sync();
    if (t >= total) return;
    int step, c, kind = 0;
    if (TN != TP || !a.split_m || t < t1) {
      step = (int)(t / a.nc), c = (int)(t % a.nc);
    } else if (t - t1 < span) {
      const long long u = t - t1;
      step = s1 + (int)(u / (2 * a.nc));
      c = (int)(u % (2 * a.nc));
      if (c >= a.nc) {
        c -= a.nc;
        step += a.split_m + 1;
        kind = 2;
      }
    } else {
      const long long u = t - t1 - span;
      step = s1 + npre + (int)(u / a.nc), c = (int)(u % a.nc);
    }
    if (TN == TP && a.split_m && kind == 0 && step >= a.split_from) kind = 1;
    const int i = a.lower ? step : a.nb - 1 - step;
    tt_mark(t, 0);
    if (!trsm_task<T, AK, BKM, TN>(Tm, B, W, a, done, i, c, sm, &s_ok, TN == TP ? kind : 0))
      return;
    tt_mark(t, 1);
  }
}

template <typename T, bool AK, bool BKM, int TN> size_t trsm_smem_bytes() {
  using C = TileCfg<T>;
  using PP = TrsmPipe<T, TN>;
  const size_t pipe = (size_t)PP::ST * (SmemLayout<T, TP, PP::BK, AK>::SIZE +
                                        SmemLayout<T, TN, PP::BK, BKM>::SIZE);
  const size_t stile = (size_t)(TN > TP ? TN : TP) * LD64, one = (size_t)TP * LD64;
  if (trsm_prew<T, BKM>()) return ((pipe > stile ? pipe : stile) + one) * sizeof(T);
  const size_t tiles = stile + one;  // S and W'_i
  return (pipe > tiles ? pipe : tiles) * sizeof(T);
}

template <typename T, bool AK, bool BKM, int TN>
int trsm_launch(View<T> Tm, View<T> B, const T* W, const TrsmArgs& a, int* sync, Ctx c) {
  auto kern = tile_trsm_kernel<T, AK, BKM, TN>;
  const size_t smem = trsm_smem_bytes<T, AK, BKM, TN>();
  const int per_sm = kernel_setup(kern, TPT, smem);
  const long long tasks = (long long)a.nb * a.nc;
  long long grid = (long long)per_sm * num_sms();
  if (grid > tasks) grid = tasks;
  KernelClock kc(c.st);
  kern<<<(unsigned)grid, TPT, smem, c.st>>>(Tm, B, W, a, sync, c.info);
  RFPK_CHECK_LAUNCH();
  kc.stop("tile_trsm", Tm.m, B.n);
  return 0;
}

}  // namespace

// conj?(Tm) X = B in place with the dataflow kernel (W: lower-form 64-block
// inverses; wtrans for Tm upper).  Returns -100 for unsupported strides.
template <typename T>
int trsm_tiles(Ctx c, bool lower, bool conj, View<T> Tm, View<T> B, const T* W, bool wtrans,
               const int* agate, int agate_stride, const int* aabort, bool tri_rhs) {
  const i64 n = Tm.m;
  if (n == 0 || B.n == 0) return 0;
  const bool ak = !(Tm.rs == 1);
  if (ak && Tm.cs != 1) return -100;
  if (!(B.rs == 1 || B.cs == 1 || B.n == 1)) return -100;
  TrsmArgs a;
  a.n = (int)n;
  a.nrhs = (int)B.n;
  a.nb = (int)((n + TP - 1) / TP);
  // 64 x 16 tiles give four times the chains and a four times shorter step
  // on each: used for narrow right-hand sides (pftrs at n = 4000, nrhs = 64:
  // 1.63 -> 0.74 ms) and whenever the 64-wide tiles would be few (<= ~10 per
  // SM: pftrf's S1 solve at n = 4000 0.72 -> 0.52 ms, n = 1000 0.16 ->
  // 0.07 ms); measured slower with more tasks (S1 at n = 6000 1.48 vs 1.31
  // ms, 16384 26.8 vs 17.6 ms; pftrs 16384 x 1024 3.4 vs 2.7 ms per solve)
  constexpr int narrow_max = 256;
  // (a 64 x 128 tile with 2 x 2 warps of 32 x 64 measured slower on the S1
  // solve of config 3: 255 registers with spills, two CTAs per SM, 18.4 vs
  // 17.7 ms)
  const long long tasks64 = (long long)a.nb * ((B.n + TP - 1) / TP);
  const int tn = (!is_cplx<T>::value &&
                  (B.n <= narrow_max || tasks64 <= 10LL * num_sms())) ? 16 : TP;
  a.nc = (int)((B.n + tn - 1) / tn);
  a.lower = lower ? 1 : 0;
  a.conj = conj ? 1 : 0;
  a.wtrans = wtrans ? 1 : 0;
  a.ext = InputGate::flags();
  a.ext_mode = InputGate::mode();
  a.agate = agate;
  a.agate_stride = agate_stride;
  a.aabort = aabort;
  a.aguard = agate ? aabort - 1 : nullptr;  // the producer's task counter (sync[0])
  a.aguard_keep = num_sms();
  a.scan = 1;
  a.rowcnt = nullptr;
  a.tri_rhs = tri_rhs && lower ? 1 : 0;
  // split tasks: plain wide-tile solves only (a PRE task of row block i would
  // sit on the triangle gate of a concurrent potrf, or on the input gate, long
  // before its turn), and only where the tail is a few long tasks per CTA
  a.split_m = a.split_from = 0;
  a.pre = nullptr;
  {
    // tuning "trsm_split": 0 off, 1 automatic, > 1 the kept chunks.  The tail
    // of a solve is its last tasks (nb chunks each) running out one by one:
    // about 2 grid / (nb nc) of the run, so it only matters for few columns
    // (config 3's pftrs solves, 128 x 16 tasks: 2.76 -> 2.60 ms; kept chunks
    // 16 / 24 / 32: 2.70 / 2.60 / 2.64 ms)
    const long long v = tune(TK_TRSM_SPLIT);
    int m = (int)v;
    if (v == 1) {
      m = (a.nb * 3 / 16) & ~7;
      if (m < 16) m = 16;
      if (m > 64) m = 64;
      if ((long long)a.nb * a.nc > 48LL * num_sms()) m = 0;
    }
    if (m > 0 && tn == TP && !agate && !a.ext && !a.tri_rhs && a.nb >= (v == 1 ? 4 : 3) * m) {
      a.split_m = m;
      a.split_from = 2 * m;
    }
  }
  RowDoneHook* hook = RowHook::current();
  const size_t ints = SYNC_HDR + (size_t)a.nb * a.nc * (a.split_m ? 2 : 1);
  int* sync = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&sync, ints * sizeof(int), c.st);
  if (e != cudaSuccess) return (int)e;
  if ((e = cudaMemsetAsync(sync, 0, ints * sizeof(int), c.st)) != cudaSuccess) return (int)e;
  if (hook && hook->rowcnt && !(tn == 16 && is_cplx<T>::value)) {
    if ((e = cudaMemsetAsync(hook->rowcnt, 0, (size_t)a.nb * sizeof(int), c.st)) != cudaSuccess)
      return (int)e;
    a.rowcnt = hook->rowcnt;
    hook->nb = a.nb;
    hook->nc = a.nc;
    hook->forward = lower;
    hook->used = true;
    cudaEventRecord(hook->launched, c.st);
    RowHook::consumed();
  }
  if (a.split_m) a.pre = sync + SYNC_HDR + (size_t)a.nb * a.nc;
  // B operand = X^T (nrhs x K): K-major when B is column-major
  const bool bkm = B.rs == 1;
  int rc;
  if (tn == 16) {
    if constexpr (!is_cplx<T>::value) {
      if (ak) rc = bkm ? trsm_launch<T, true, true, 16>(Tm, B, W, a, sync, c)
                       : trsm_launch<T, true, false, 16>(Tm, B, W, a, sync, c);
      else rc = bkm ? trsm_launch<T, false, true, 16>(Tm, B, W, a, sync, c)
                    : trsm_launch<T, false, false, 16>(Tm, B, W, a, sync, c);
    } else {
      rc = -100;
    }
  } else if (ak) {
    rc = bkm ? trsm_launch<T, true, true, TP>(Tm, B, W, a, sync, c)
             : trsm_launch<T, true, false, TP>(Tm, B, W, a, sync, c);
  } else {
    rc = bkm ? trsm_launch<T, false, true, TP>(Tm, B, W, a, sync, c)
             : trsm_launch<T, false, false, TP>(Tm, B, W, a, sync, c);
  }
  cudaFreeAsync(sync, c.st);
  return rc;
}

template int trsm_tiles<double>(Ctx, bool, bool, View<double>, View<double>, const double*, bool,
                                const int*, int, const int*, bool);
template int trsm_tiles<Z>(Ctx, bool, bool, View<Z>, View<Z>, const Z*, bool, const int*, int,
                           const int*, bool);

size_t potrf_sync_ints(int nt, int mt) { return SYNC_HDR + (size_t)mt * nt + nt; }

// Factor the tall lower panel P (m x n, m >= n, col- or row-major): the
// Cholesky of its leading n x n block and the solve of the rows below it,
// P = [L11; L21] with L21 = P21 L11^-H, in one dataflow launch.  m == n is
// potrf.  W (leaf-inverse slabs for the column tiles) is required; the row
// tiles restart at n, so n need not be a multiple of 64.
template <typename T>
int potrf_panel_tiles(Ctx c, View<T> P, i64 n, int base, T* W, int** keep_sync) {
  const i64 m = P.m;
  if (n == 0) return 0;
  if (!W || m < n) return -100;
  const bool km = !(P.rs == 1);
  if (km && P.cs != 1) return -100;
  const int nt = (int)((n + TP - 1) / TP), mt = nt + (int)((m - n + TP - 1) / TP);
  const size_t ints = potrf_sync_ints(nt, mt);
  int* sync = keep_sync ? *keep_sync : nullptr;  // a caller-provided, zeroed array
  if (!sync) {
    cudaError_t e = cudaMallocAsync((void**)&sync, ints * sizeof(int), c.st);
    if (e != cudaSuccess) return (int)e;
    if ((e = cudaMemsetAsync(sync, 0, ints * sizeof(int), c.st)) != cudaSuccess) return (int)e;
  }
  int rc = km ? tile_launch<T, true, true, false>(P, P, (int)n, nt, (int)n, W, c, base, sync, nt, mt)
              : tile_launch<T, false, false, false>(P, P, (int)n, nt, (int)n, W, c, base, sync, nt, mt);
  // keep_sync: the caller gates a concurrent kernel on the done flags
  // (done(i, j) at sync + SYNC_HDR + i * nt + j; abort at sync + 1; the task
  // counter at sync[0] is nonzero once a CTA has started) and frees the array
  // once that kernel is ordered after it.  *keep_sync non-null on entry: the
  // caller allocated and zeroed the array (potrf_sync_ints) on a stream both
  // kernels are ordered after.
  if (keep_sync) *keep_sync = sync;
  else cudaFreeAsync(sync, c.st);
  return rc;
}

// The whole SRPA factorization in one dataflow launch: region 0 = the tall
// panel P = [T1; S] (n x n1, T1 lower), region 1 = the lower view V of T2^T
// (n2 x n2, n = n1 + n2).  Every tile of the global lower triangle is a task
// of the one DAG, so potrf(T1), the S solve, T2 -= S S^H and potrf(T2) are a
// single chain of diagonal tiles with all other work overlapping it
// (rfp.py:70-89 in one kernel).  Real only; W needs ceil(n1/64) +
// ceil(n2/64) slabs.  -100: unsupported strides.
template <typename T> int potrf_rfp_tiles(Ctx c, View<T> P, View<T> V, int base, T* W) {
  if constexpr (is_cplx<T>::value) {
    return -100;
  } else {
    const i64 n1 = P.n, n2 = V.m, n = n1 + n2;
    if (n2 == 0) return potrf_panel_tiles(c, P, n1, base, W);
    if (!W || P.m != n || V.n != n2 || n1 == 0) return -100;
    const bool k0 = !(P.rs == 1), k1 = !(V.rs == 1);
    if ((k0 && P.cs != 1) || (k1 && V.cs != 1)) return -100;
    const int nt1 = (int)((n1 + TP - 1) / TP), nt = nt1 + (int)((n2 + TP - 1) / TP);
    const size_t ints = potrf_sync_ints(nt, nt);
    int* sync = nullptr;
    cudaError_t e = cudaMallocAsync((void**)&sync, ints * sizeof(int), c.st);
    if (e != cudaSuccess) return (int)e;
    if ((e = cudaMemsetAsync(sync, 0, ints * sizeof(int), c.st)) != cudaSuccess) return (int)e;
    const int a = (int)n1, b = (int)n;
    int rc = -100;
    if (k0 && !k1) rc = tile_launch<T, true, false, true>(P, V, a, nt1, b, W, c, base, sync, nt, nt);
    else if (!k0 && k1) rc = tile_launch<T, false, true, true>(P, V, a, nt1, b, W, c, base, sync, nt, nt);
    else if (!k0 && !k1) rc = tile_launch<T, false, false, true>(P, V, a, nt1, b, W, c, base, sync, nt, nt);
    // (both row-major: no RFP layout produces it)
    cudaFreeAsync(sync, c.st);
    return rc;
  }
}

template <typename T> int potrf_tiles(Ctx c, View<T> A, int base, T* W) {
  return potrf_panel_tiles(c, A, A.m, base, W);
}

// Library side streams for the overlapped steps, per host thread and device
// (thread_local): two callers on their own streams never share a fork/join
// event or a side stream, so a join can never silently lose a dependency.
OverlapStreams& overlap_streams() {
  static thread_local OverlapStreams per_dev[MAX_DEVICES];
  OverlapStreams& S = per_dev[cur_device() & (MAX_DEVICES - 1)];
  if (!S.ok) {
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    cudaStreamCreateWithPriority(&S.hi, cudaStreamNonBlocking, greatest);
    cudaStreamCreateWithPriority(&S.lo, cudaStreamNonBlocking, least);
    for (auto& e : S.ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    S.ok = true;
  }
  return S;
}

OverlapStreams::~OverlapStreams() {
  if (!ok) return;
  cudaStreamDestroy(hi);
  cudaStreamDestroy(lo);
  for (auto e : ev) cudaEventDestroy(e);
}

namespace {
// Device-wide order of the spin-coupled potrf || trsm pairs: the solve's
// waiting CTAs need the potrf's CTAs to become resident beside them, which
// one pair at a time guarantees (at most num_sms() waiting CTAs, see aguard)
// but several pairs from different host threads could not -- enough waiting
// CTAs of several solves could fill every slot.  Each pair's fork therefore
// waits (stream-ordered, never spinning) for the previous pair's join on the
// same device.
struct PairChain {
  std::mutex mu;
  cudaEvent_t last = nullptr;
};
PairChain& pair_chain() {
  static PairChain chains[MAX_DEVICES];
  return chains[cur_device() & (MAX_DEVICES - 1)];
}
}  // namespace

// potrf('L', A) and the solve conj?(A) X = B that consumes its factor, as
// two CONCURRENT dataflow launches: the tile potrf on a high-priority stream
// (two CTAs per SM at these orders, so every SM keeps a third slot), the tile
// trsm on a low-priority stream, each trsm task first waiting for the
// potrf's diagonal flag of its row block (done(i, i): row block i of L and
// W_i published).  The solve's first row blocks then run beside the
// factorization's chain instead of after it.  Deadlock-free: the potrf never
// waits on the solve and its CTAs are normally dispatched first (launched
// first, higher priority); should the solve's CTAs still reach the SMs first,
// every one beyond the first num_sms() exits at once while the potrf's task
// counter reads zero (TrsmArgs::aguard), so at most one SM's worth of waiting
// solve CTAs can be resident before the potrf runs.  A failing potrf raises
// its abort flag, on which every waiting trsm task exits.  The potrf's flag
// array is zeroed on the caller's stream before the fork (pool memory may
// hold an earlier run's flags).
template <typename T>
int potrf_trsm_overlap(Ctx c, View<T> A, T* W, bool conj, View<T> B, const int* pgate,
                       const int* bgate, int bgate_mode) {
  if constexpr (is_cplx<T>::value) {
    return -100;
  } else {
    if (!tune(TK_OVERLAP) || A.m <= TP || B.empty() || !W) return -100;
    // row-major B only: the column-major-B trsm variants take ~250 registers
    // and do not fit beside two potrf CTAs on an SM (UPLO='U' at n = 12000:
    // 11.18 ms overlapped vs 10.9 in sequence)
    if (A.rs != 1 || B.cs != 1 || B.rs == 1) return -100;
    // not under graph capture: captured kernel nodes lose the stream
    // priorities the dispatch order relies on
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(c.st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone)
      return -100;
    OverlapStreams& S = overlap_streams();
    // the potrf's flag array, zeroed on the caller's stream BEFORE the fork:
    // the trsm reads it from its first task on
    const int nt = (int)((A.m + TP - 1) / TP);
    const size_t ints = potrf_sync_ints(nt, nt);
    int* psync = nullptr;
    cudaError_t e = cudaMallocAsync((void**)&psync, ints * sizeof(int), c.st);
    if (e == cudaSuccess) e = cudaMemsetAsync(psync, 0, ints * sizeof(int), c.st);
    if (e != cudaSuccess) {
      if (psync) cudaFreeAsync(psync, c.st);
      return (int)e;
    }
    PairChain& pc = pair_chain();
    std::lock_guard<std::mutex> lk(pc.mu);
    e = cudaEventRecord(S.ev[0], c.st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(S.hi, S.ev[0], 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(S.lo, S.ev[0], 0);
    if (e == cudaSuccess && pc.last) e = cudaStreamWaitEvent(S.hi, pc.last, 0);
    if (e == cudaSuccess && pc.last) e = cudaStreamWaitEvent(S.lo, pc.last, 0);
    if (e != cudaSuccess) {
      cudaFreeAsync(psync, c.st);
      return (int)e;
    }
    // (pgate / bgate: host-streamed input, see InputGate -- the potrf reads
    // A's column chunks, the trsm B's chunks as the copy engine flags them)
    int rc;
    {
      InputGate g(pgate, 0);
      rc = potrf_panel_tiles(Ctx{S.hi, c.info}, A, A.m, 0, W, &psync);
    }
    if (!rc) {
      InputGate g(bgate, bgate_mode);
      rc = trsm_tiles(Ctx{S.lo, c.info}, true, conj, A, B, (const T*)W, false,
                      psync + SYNC_HDR, nt + 1, psync + 1);
    }
    // join both streams back into the caller's (also on the error paths)
    cudaEventRecord(S.ev[1], S.hi);
    cudaEventRecord(S.ev[2], S.lo);
    cudaStreamWaitEvent(c.st, S.ev[1], 0);
    cudaStreamWaitEvent(c.st, S.ev[2], 0);
    // this pair's join becomes the next pair's fork dependency
    cudaEvent_t joined = nullptr;
    if (cudaEventCreateWithFlags(&joined, cudaEventDisableTiming) == cudaSuccess) {
      cudaEventRecord(joined, c.st);
      if (pc.last) cudaEventDestroy(pc.last);  // pending waits keep their snapshot
      pc.last = joined;
    }
    cudaFreeAsync(psync, c.st);
    return rc;
  }
}
template int potrf_trsm_overlap<double>(Ctx, View<double>, double*, bool, View<double>,
                                        const int*, const int*, int);
template int potrf_trsm_overlap<Z>(Ctx, View<Z>, Z*, bool, View<Z>, const int*, const int*, int);

template int potrf_panel_tiles<double>(Ctx, View<double>, i64, int, double*, int**);
template int potrf_panel_tiles<Z>(Ctx, View<Z>, i64, int, Z*, int**);
template int potrf_tiles<double>(Ctx, View<double>, int, double*);
template int potrf_rfp_tiles<double>(Ctx, View<double>, View<double>, int, double*);
template int potrf_tiles<Z>(Ctx, View<Z>, int, Z*);

}  // namespace rfpk

#ifdef RFPK_CHAIN_TRACE
extern "C" int rfpk_chain_trace_read(unsigned long long* host, int count) {
  return (int)cudaMemcpyFromSymbol(host, rfpk::g_chain_trace,
                                   sizeof(unsigned long long) * (size_t)count);
}
extern "C" int rfpk_task_trace_read(unsigned long long* host, int count) {
  return (int)cudaMemcpyFromSymbol(host, rfpk::g_task_trace,
                                   sizeof(unsigned long long) * (size_t)count);
}
extern "C" int rfpk_chain_trace_clear() {
  static unsigned long long zero[rfpk::CT_MAX * rfpk::CT_EV] = {};
  return (int)cudaMemcpyToSymbol(rfpk::g_chain_trace, zero, sizeof(zero));
}
#endif
