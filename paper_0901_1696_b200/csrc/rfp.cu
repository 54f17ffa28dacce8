// RFP drivers (rfp.py) and full/packed/RFP conversion kernels (convert.py).
#include "rfp.cuh"

#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

namespace rfpk {

RfpDesc rfp_desc(i64 n, char uplo, char transr) {
  RfpDesc d;
  d.n = n;
  d.n1 = (n + 1) / 2;
  d.n2 = n - d.n1;
  d.nt = n * (n + 1) / 2;
  d.ldar = (n % 2) ? n : n + 1;
  d.d = (n % 2) ? 0 : 1;
  d.lower = uplo == 'L';
  d.trans = transr != 'N';
  return d;
}

template <typename T>
void rfp_blocks(const RfpDesc& d, T* buf, View<T>& t1, View<T>& t2, View<T>& s1) {
  const i64 rs = d.trans ? d.n1 : 1, cs = d.trans ? 1 : d.ldar;
  auto mk = [&](i64 r0, i64 c0, i64 m, i64 n) { return View<T>{buf + r0 * rs + c0 * cs, m, n, rs, cs}; };
  const i64 n1 = d.n1, n2 = d.n2, sh = d.d;
  if (d.lower) {
    t1 = mk(sh, 0, n1, n1);
    t2 = mk(0, 1 - sh, n2, n2);
    s1 = mk(n1 + sh, 0, n2, n1);
  } else {
    t1 = mk(n2 + 1, 0, n2, n2);
    t2 = mk(n2, 0, n1, n1);
    s1 = mk(0, 0, n2, n1);
  }
}

template <typename T> static T one() { return sc_from<T>(1.0); }
template <typename T> static T m_one() { return sc_from<T>(-1.0); }

// Phase timing of the SRPA steps.  Tuning "trace" = 1 prints each direct
// call's phases to stderr (synchronising); the phase clock (rfpk_phase_clock) only
// records event pairs, summed per "routine phase" label when
// rfpk_phase_time() is asked -- so a benchmark can time its dominant kernel
// live inside the timed region without perturbing it.  Captured (graph)
// calls are never traced.
struct PhaseClock {
  std::mutex mu;
  std::atomic<bool> on{false};
  struct Pending { std::string label; cudaEvent_t a, b; };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> owned;  // destroyed once read
  std::map<std::string, std::pair<double, long long>> sums;
  static PhaseClock& get() {
    static PhaseClock c;
    return c;
  }
  void drain() {  // caller holds mu
    for (auto& p : pending) {
      cudaEventSynchronize(p.b);
      float ms = 0;
      cudaEventElapsedTime(&ms, p.a, p.b);
      auto& e = sums[p.label];
      e.first += ms;
      e.second += 1;
    }
    pending.clear();
    for (cudaEvent_t e : owned) cudaEventDestroy(e);
    owned.clear();
  }
};

KernelClock::KernelClock(cudaStream_t s) : st(s) {
  if (!PhaseClock::get().on) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
  if (cudaEventCreate(&a) != cudaSuccess) {
    a = nullptr;
    return;
  }
  cudaEventRecord(a, st);
}

void KernelClock::stop(const char* name, long long d0, long long d1, long long d2) {
  if (!a) return;
  cudaEvent_t b = nullptr;
  if (cudaEventCreate(&b) != cudaSuccess) {
    cudaEventDestroy(a);
    a = nullptr;
    return;
  }
  cudaEventRecord(b, st);
  char lab[160];
  if (d2 >= 0) snprintf(lab, sizeof lab, "kernel %s %lldx%lldx%lld", name, d0, d1, d2);
  else snprintf(lab, sizeof lab, "kernel %s %lldx%lld", name, d0, d1);
  PhaseClock& pc = PhaseClock::get();
  std::lock_guard<std::mutex> g(pc.mu);
  pc.pending.push_back({std::string(lab), a, b});
  pc.owned.push_back(a);
  pc.owned.push_back(b);
  a = nullptr;
}

struct PhaseTrace {
  cudaStream_t st;
  const char* name;
  bool print = false, clock = false;
  cudaEvent_t ev[8];
  const char* lab[8];
  int k = 0;
  PhaseTrace(cudaStream_t s, const char* nm) : st(s), name(nm) {
    nvtxRangePushA(nm);  // NVTX: one range per SRPA routine, a mark per step
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs != cudaStreamCaptureStatusNone) return;
    print = tune(TK_TRACE) != 0;
    clock = PhaseClock::get().on;
    if (print || clock) mark("start");
  }
  void mark(const char* l) {
    nvtxMarkA(l);
    if (!(print || clock) || k >= 8) return;
    cudaEventCreate(&ev[k]);
    cudaEventRecord(ev[k], st);
    lab[k++] = l;
  }
  ~PhaseTrace() {
    nvtxRangePop();
    if (!(print || clock)) return;
    if (clock) {
      PhaseClock& pc = PhaseClock::get();
      std::lock_guard<std::mutex> g(pc.mu);
      for (int i = 1; i < k; ++i)
        pc.pending.push_back({std::string(name) + " " + lab[i], ev[i - 1], ev[i]});
      for (int i = 0; i < k; ++i) pc.owned.push_back(ev[i]);
      return;  // read (and synchronised) only by rfpk_phase_time
    }
    cudaEventSynchronize(ev[k - 1]);
    for (int i = 1; i < k; ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
      fprintf(stderr, "[rfpk trace] %s %-10s %9.3f ms\n", name, lab[i], ms);
    }
    for (int i = 0; i < k; ++i) cudaEventDestroy(ev[i]);
  }
};

#define TRY(x)              \
  do {                      \
    int rc_ = (x);          \
    if (rc_) return rc_;    \
  } while (0)

// dst(i, j) = src(i, j) for an m x n view pair of any orientations (lower:
// the lower triangle i >= j only): 32 x 32 tiles through shared memory, read
// along src's contiguous dimension and written along dst's
template <typename T>
__global__ void tile_copy_kernel(View<T> src, View<T> dst, int lower) {
  __shared__ T tile[32][33];  // tile[a][b] = element (i0 + a, j0 + b)
  const int bi = blockIdx.y, bj = blockIdx.x;
  if (lower && bi < bj) return;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const i64 i0 = (i64)bi * 32, j0 = (i64)bj * 32;
  const bool sj = src.cs == 1 && src.rs != 1;  // row-major: contiguous along j
  const bool dj = dst.cs == 1 && dst.rs != 1;
#pragma unroll
  for (int r = ty; r < 32; r += 8) {
    const int ta = sj ? r : tx, tb = sj ? tx : r;
    const i64 i = i0 + ta, j = j0 + tb;
    if (i < src.m && j < src.n && (!lower || j <= i)) tile[ta][tb] = *src.at(i, j);
  }
  __syncthreads();
#pragma unroll
  for (int r = ty; r < 32; r += 8) {
    const int ta = dj ? r : tx, tb = dj ? tx : r;
    const i64 i = i0 + ta, j = j0 + tb;
    if (i < src.m && j < src.n && (!lower || j <= i)) *dst.at(i, j) = tile[ta][tb];
  }
}

template <typename T> static int tile_copy(Ctx c, View<T> src, View<T> dst, bool lower) {
  if (src.empty()) return 0;
  const dim3 grid((unsigned)((src.n + 31) / 32), (unsigned)((src.m + 31) / 32));
  KernelClock kc(c.st);
  tile_copy_kernel<T><<<grid, dim3(32, 8), 0, c.st>>>(src, dst, lower ? 1 : 0);
  RFPK_CHECK_LAUNCH();
  kc.stop("tile_copy", src.m, src.n);
  return 0;
}

// column-major m x n workspace, 64-byte aligned columns, ld off a power of 2
template <typename T> static int ws_colmajor(Ctx c, i64 m, i64 n, View<T>& v) {
  const i64 ld = (m + 15) / 16 * 16 + 8;
  T* p = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&p, (size_t)ld * (n > 0 ? n : 1) * sizeof(T), c.st);
  v = View<T>{p, m, n, 1, ld};
  return e == cudaSuccess ? 0 : (int)e;
}

// potrf('U', T2) (rfp.py:89 / :84).  The lower view the Cholesky factors is
// T2^T; for TRANSR='N' that view is row-major with the RFP's odd leading
// dimension, where every 16-wide K slice of a row straddles an extra sector
// and the tile potrf runs a two-stage pipeline (potrf(T2) 8.1 ms against
// potrf(T1)'s 7.0 at n = 16384).  Large blocks are therefore factored in a
// column-major copy: two coalesced O(n^2) transposing copies buy the
// column-major tile potrf (pftrf n = 16384: 'L','N' bench step 69.5 -> 68.8
// ms; 'L','T' 49.2 -> 48.7 ms; 'U','N' 50.4 -> 49.5 ms).  Same kernels, same
// pivots, same info offsets.
// potrf(T1) of the TRANSR='T' / 'C' layouts has the same row-major lower
// view and takes the same route when its input is not streamed in.
template <typename T> static int potrf_block(Ctx c, char uplo, View<T> blk, int base, T* W) {
  const View<T> v = uplo == 'L' ? blk : blk.t();
  const i64 min_n = tune(TK_T2_COPY_MIN);
  // (real only: for complex128 the row-major tile potrf measured as fast or
  // faster -- config 5's pftrf 606 ms direct vs 663 ms through the copy)
  if (is_cplx<T>::value || v.rs == 1 || v.cs != 1 || v.m < min_n)
    return blas_potrf(c, uplo, blk, base, W);
  View<T> x;
  int rc = ws_colmajor(c, v.m, v.m, x);
  if (rc) return rc;
  rc = tile_copy(c, v, x, true);
  if (!rc) rc = blas_potrf(c, 'L', x, base, W);
  if (!rc) rc = tile_copy(c, x, v, true);
  cudaFreeAsync(x.p, c.st);
  return rc;
}

static i64 panel_max() { return tune(TK_PANEL_MAX); }

// The whole SRPA chain (rfp.py:70-89 / :81-89) as ONE dataflow launch over
// the global lower triangle (potrf_rfp_tiles): region 0 = [T1; S] with S =
// S1 ('L') or S1^T ('U'), region 1 = T2^T.  'L': [T1; S1] are contiguous
// rows of the normal rectangle, so the panel is read in place; 'U': S1 lies
// above T1 and enters transposed, so T1's lower triangle and S1^T are copied
// into a column-major workspace panel first (and back after).  T2^T is
// factored in place.  -100: not applicable.
template <typename T>
static int chol_srpa_fused(Ctx c, const RfpDesc& d, View<T> t1, View<T> t2, View<T> s1, T* W) {
  const i64 k = t1.m, m = d.n - k;
  if (d.lower) {
    View<T> panel{t1.p, d.n, k, t1.rs, t1.cs};
    return potrf_rfp_tiles(c, panel, t2.t(), 0, W);
  }
  const View<T> s = s1.t();
  View<T> P;
  int rc = ws_colmajor(c, d.n, k, P);
  if (rc) return rc;
  View<T> p1 = P.sub(0, 0, k, k), p2 = P.sub(k, 0, m, k);
  rc = tile_copy(c, t1, p1, true);
  if (!rc) rc = tile_copy(c, s, p2, false);
  if (!rc) rc = potrf_rfp_tiles(c, P, t2.t(), 0, W);
  if (!rc) rc = tile_copy(c, p1, t1, true);
  if (!rc) rc = tile_copy(c, p2, s, false);
  cudaFreeAsync(P.p, c.st);
  return rc;
}

struct WsPair {  // two leaf-inverse workspaces, freed stream-ordered
  cudaStream_t st;
  void* p[2] = {nullptr, nullptr};
  ~WsPair() {
    for (void* q : p)
      if (q) cudaFreeAsync(q, st);
  }
};

template <typename T>
static int pftrs_part(Ctx c, const RfpDesc& d, const T* arf, View<T> b, T* W1, T* W2,
                      cudaEvent_t b2_final, int part, RowDoneHook* last_hook = nullptr);

// SRPA factorization (rfp.py:55-91)
template <typename T>
int pftrf(Ctx c, const RfpDesc& d, T* arf, cudaEvent_t s1_ready, const int* cflags,
          const int* sflags, PfsvPlan<T>* plan) {
  if (d.n == 0) return 0;
  const bool herm = is_cplx<T>::value;
  View<T> t1, t2, s1;
  rfp_blocks(d, arf, t1, t2, s1);
  // one workspace for the leaf inverses: T1's are reused by the S1 solve,
  // then the buffer is reused for T2's potrf
  T* W = nullptr;
  TRY(ws_alloc(&W, d.n + LEAF, c.st));
  int rc = 0;
  PhaseTrace tr(c.st, "pftrf");
  // mid orders, device-resident input: the whole chain in one launch
  if (!is_cplx<T>::value && !s1_ready && !cflags && d.n2 && t1.m <= panel_max()) {
    rc = chol_srpa_fused(c, d, t1, t2, s1, W);
    if (rc != -100) {
      tr.mark("potrf(T1)+trsm(S1)+syrk(T2)+potrf(T2)");
      ws_free(W, c.st);
      return rc;
    }
    rc = 0;
  }
  // potrf(T2); with a pfsv plan, beside pftrs part 1 (see pfsv)
  auto t2_step = [&](int base) -> int {
    const i64 min_t2 = tune(TK_PFSV_OVERLAP_MIN);
    if (!plan || d.n2 == 0 || t2.m < min_t2) return potrf_block(c, 'U', t2, base, W);
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(c.st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone)
      return potrf_block(c, 'U', t2, base, W);
    OverlapStreams& S = overlap_streams();
    T *W1 = nullptr, *W2 = nullptr;
    WsPair fr{c.st};
    int r = ws_alloc(&W1, t1.m, c.st);
    fr.p[0] = W1;
    if (!r) r = ws_alloc(&W2, t2.m, c.st);
    fr.p[1] = W2;
    if (r) return r;
    cudaEventRecord(S.ev[3], c.st);
    cudaStreamWaitEvent(S.hi, S.ev[3], 0);
    int rt2 = potrf_block(Ctx{S.hi, c.info}, 'U', t2, base, W);
    if (plan->b_ready) cudaStreamWaitEvent(c.st, plan->b_ready, 0);
    r = blas_leaf_inverses(c, t1, W1);
    if (!r) r = pftrs_part(c, d, (const T*)arf, plan->b, W1, W2, nullptr, 1);
    cudaEventRecord(S.ev[4], S.hi);  // join (also on the error paths)
    cudaStreamWaitEvent(c.st, S.ev[4], 0);
    tr.mark("potrf(T2)||pftrs(T1,S1)");
    if (rt2) return rt2;
    if (r) return r;
    r = blas_leaf_inverses(c, t2.t(), W2);
    if (!r) r = pftrs_part(c, d, (const T*)arf, plan->b, W1, W2, plan->b2_final, 2, plan->head_rows);
    plan->done = true;
    return r;
  };
  // streamed input (cflags/sflags): potrf(T1) and the S1 solve read each
  // 64-column chunk as soon as its flag is set; the remaining steps wait for
  // the whole transfer (s1_ready) -- by then every chunk has been seen
  const bool gated = cflags != nullptr;
  auto before_s1 = [&]() {
    if (!gated && !rc && s1_ready) rc = (int)cudaStreamWaitEvent(c.st, s1_ready, 0);
  };
  auto after_s1 = [&]() {
    if (gated && !rc && s1_ready) rc = (int)cudaStreamWaitEvent(c.st, s1_ready, 0);
  };
  if (d.lower) {
    // (mid orders took the one-launch chain above.)  potrf(T1) and the S1
    // solve as two concurrent launches, the solve gated row block by row
    // block on the factorization (device-resident input, real, column-major
    // T1: potrf_trsm_overlap); streamed input: each launch keeps its chunk
    // gate (B = S1^T, block row i <-> column chunk i)
    int fused = -100;
    if (d.n2 && (gated || !s1_ready))
      fused = potrf_trsm_overlap(c, t1, W, herm, s1.t(), cflags, sflags, 0);
    if (fused != -100) {
      rc = fused;
      after_s1();
      tr.mark("potrf(T1)||trsm(S1)");
    } else {
      {
        InputGate g(cflags, 0);
        rc = gated ? blas_potrf(c, 'L', t1, 0, W) : potrf_block(c, 'L', t1, 0, W);
      }
      tr.mark("potrf(T1)");
      before_s1();
      if (!rc && d.n2) {
        InputGate g(sflags, 0);  // B = S1^T: block row i <-> column chunk i
        rc = blas_trsm(c, 'R', 'L', 'C', 'N', one<T>(), t1, s1, false, W);
      }
      after_s1();
      tr.mark("trsm(S1)");
    }
    if (!rc && d.n2) {
      if (!rc) rc = blas_syrk(c, 'U', 'C', -1.0, s1.t(), 1.0, t2, herm);
      tr.mark("syrk(T2)");
      if (!rc) rc = t2_step((int)d.n1);
      tr.mark(plan && plan->done ? "pftrs(rest)" : "potrf(T2)");
    }
  } else {
    // UPLO='U' (mid orders took the one-launch chain above)
    int fused = -100;
    if (d.n2) {
      // larger leading blocks: potrf(T1) and the S1 solve concurrently (as 'L')
      if (gated || !s1_ready)  // B = S1: block column c <-> column chunk c
        fused = potrf_trsm_overlap(c, t1, W, herm, s1, cflags, sflags, 1);
      if (fused != -100) {
        rc = fused;
        after_s1();
        tr.mark("potrf(T1)||trsm(S1)");
      } else {
        {
          InputGate g(cflags, 0);
          rc = gated ? blas_potrf(c, 'L', t1, 0, W) : potrf_block(c, 'L', t1, 0, W);
        }
        tr.mark("potrf(T1)");
        before_s1();
        if (!rc) {
          InputGate g(sflags, 1);  // B = S1: block column c <-> column chunk c
          rc = blas_trsm(c, 'L', 'U', 'C', 'N', one<T>(), t1.t(), s1, false, W);
        }
        after_s1();
        tr.mark("trsm(S1)");
      }
      if (!rc) rc = blas_syrk(c, 'U', 'C', -1.0, s1, 1.0, t2, herm);
      tr.mark("syrk(T2)");
    }
    if (!rc) rc = t2_step((int)d.n2);
    tr.mark(plan && plan->done ? "pftrs(rest)" : "potrf(T2)");
  }
  // (the transfers must also be complete on every early-exit path)
  if (s1_ready) cudaStreamWaitEvent(c.st, s1_ready, 0);
  ws_free(W, c.st);
  return rc;
}

// Rows [r0, r1) x columns [c0, c1) of the normal ldar x n1 rectangle as one
// 2-D copy (column-major rectangle for TRANSR='N', row-major for 'T').
template <typename T>
static cudaError_t copy_block(const RfpDesc& d, const T* host, T* dev, i64 r0, i64 r1, i64 c0,
                              i64 c1, cudaStream_t st) {
  if (r1 <= r0 || c1 <= c0) return cudaSuccess;
  const size_t es = sizeof(T);
  if (d.trans)  // element (r, c) at r * n1 + c
    return cudaMemcpy2DAsync(dev + r0 * d.n1 + c0, (size_t)d.n1 * es, host + r0 * d.n1 + c0,
                             (size_t)d.n1 * es, (size_t)(c1 - c0) * es, (size_t)(r1 - r0),
                             cudaMemcpyHostToDevice, st);
  return cudaMemcpy2DAsync(dev + r0 + c0 * d.ldar, (size_t)d.ldar * es, host + r0 + c0 * d.ldar,
                           (size_t)d.ldar * es, (size_t)(r1 - r0) * es, (size_t)(c1 - c0),
                           cudaMemcpyHostToDevice, st);
}

// T1 and T2 live in the rows [0, n1 + d) (lower) / [n2, ldar) (upper) of the
// normal rectangle, S1 in the rest (rfp_blocks)
template <typename T>
static void rfp_row_regions(const RfpDesc& d, i64& t0, i64& t1, i64& s0, i64& s1) {
  t0 = d.lower ? 0 : d.n2;
  t1 = d.lower ? d.n1 + d.d : d.ldar;
  s0 = d.lower ? d.n1 + d.d : 0;
  s1 = d.lower ? d.ldar : d.n2;
}

template <typename T>
int rfp_h2d_split(const RfpDesc& d, const T* host, T* dev, cudaStream_t first,
                  cudaStream_t second) {
  i64 t0, t1, s0, s1;
  rfp_row_regions<T>(d, t0, t1, s0, s1);
  cudaError_t e = copy_block(d, host, dev, t0, t1, 0, d.n1, first);
  if (e == cudaSuccess) e = copy_block(d, host, dev, s0, s1, 0, d.n1, second);
  return (int)e;
}

template <typename T>
int rfp_h2d_chunked(const RfpDesc& d, const T* host, T* dev, int* cflags, int* sflags,
                    cudaStream_t copy) {
  static int* one = [] {  // pinned source of the flag value (every device)
    int* p = nullptr;
    cudaHostAlloc((void**)&p, sizeof(int), cudaHostAllocPortable);
    *p = 1;
    return p;
  }();
  i64 t0, t1, s0, s1;
  rfp_row_regions<T>(d, t0, t1, s0, s1);
  const i64 nch = (d.n1 + 63) / 64;
  // first rectangle row of T1 in column c: T1 = rect[d:, :] lower ('L') or
  // rect[n2+1:, :n2] lower ('U'); the T rows above it belong to T2, which is
  // first read by the SYRK after the whole transfer -- so T1's rows go first
  // (half the T region: potrf(T1) no longer waits for T2's), then S1's, then
  // T2's remainder, each chunk of the first two followed by its flag
  auto t1first = [&](i64 c) {
    i64 r = d.lower ? c + d.d : (c < d.n2 ? d.n2 + 1 + c : t1);
    return r < t0 ? t0 : (r > t1 ? t1 : r);
  };
  for (int pass = 0; pass < 3; ++pass) {
    for (i64 j = 0; j < nch; ++j) {
      const i64 c0 = j * 64, c1 = c0 + 64 < d.n1 ? c0 + 64 : d.n1;
      i64 r0, r1;
      int* flags = nullptr;
      if (pass == 0) { r0 = t1first(c0); r1 = t1; flags = cflags; }
      else if (pass == 1) { r0 = s0; r1 = s1; flags = sflags; }
      else { r0 = t0; r1 = t1first(c0); }
      cudaError_t e = cudaSuccess;
      if (r1 > r0) e = copy_block(d, host, dev, r0, r1, c0, c1, copy);
      if (e == cudaSuccess && flags)
        e = cudaMemcpyAsync(flags + j, one, sizeof(int), cudaMemcpyHostToDevice, copy);
      if (e != cudaSuccess) return (int)e;
    }
  }
  return 0;
}

// forward/back substitution through T1/S1/T2 (rfp.py:106-136), in parts:
// part 1 = the first solve with T1 and the S1 product into the trailing
// block (reads only T1 and S1 -- it can run while T2 is still being
// factored, see pfsv), part 2 = the rest, part 0 = everything.  W1 / W2:
// the 64-block inverses of T1 (lower as stored for 'L', T1^T's for 'U' --
// the same view either way is the lower one) and of T2^T (T2 is upper),
// formed once and shared by the two solves with each triangle.
template <typename T>
static int pftrs_part(Ctx c, const RfpDesc& d, const T* arf, View<T> b, T* W1, T* W2,
                      cudaEvent_t b2_final, int part, RowDoneHook* last_hook) {
  View<T> t1, t2, s1;
  rfp_blocks(d, const_cast<T*>(arf), t1, t2, s1);
  const i64 n1 = d.n1, n2 = d.n2, r = b.n;
  PhaseTrace tr(c.st, "pftrs");
  if (d.lower) {
    View<T> b1 = b.sub(0, 0, n1, r), b2 = b.sub(n1, 0, n2, r);
    if (part != 2) {
      TRY(blas_trsm(c, 'L', 'L', 'N', 'N', one<T>(), t1, b1, false, W1));
      tr.mark("trsm1");
      if (n2) {
        TRY(blas_gemm(c, 'N', 'N', m_one<T>(), s1, b1, one<T>(), b2));
        tr.mark("gemm1");
      }
      if (part == 1) return 0;
    }
    if (n2) {
      TRY(blas_trsm(c, 'L', 'U', 'T', 'N', one<T>(), t2, b2, false, W2));
      tr.mark("trsm2");
      TRY(blas_trsm(c, 'L', 'L', 'C', 'N', one<T>(), t2.t(), b2, false, W2));
      tr.mark("trsm3");
      if (b2_final) cudaEventRecord(b2_final, c.st);
      TRY(blas_gemm(c, 'C', 'N', m_one<T>(), s1, b2, one<T>(), b1));
      tr.mark("gemm2");
    }
    {
      RowHook h(last_hook);  // the head block's rows are final as this solve ends them
      TRY(blas_trsm(c, 'L', 'L', 'C', 'N', one<T>(), t1, b1, false, W1));
    }
    tr.mark("trsm4");
    return 0;
  }
  View<T> b1 = b.sub(0, 0, n2, r), b2 = b.sub(n2, 0, n1, r);
  if (part != 2) {
    if (n2) {
      TRY(blas_trsm(c, 'L', 'U', 'C', 'N', one<T>(), t1.t(), b1, false, W1));
      TRY(blas_gemm(c, 'C', 'N', m_one<T>(), s1, b1, one<T>(), b2));
    }
    if (part == 1) return 0;
  }
  TRY(blas_trsm(c, 'L', 'U', 'C', 'N', one<T>(), t2, b2, false, W2));
  TRY(blas_trsm(c, 'L', 'U', 'N', 'N', one<T>(), t2, b2, false, W2));
  if (b2_final) cudaEventRecord(b2_final, c.st);
  if (n2) {
    TRY(blas_gemm(c, 'N', 'N', m_one<T>(), s1, b2, one<T>(), b1));
    RowHook h(last_hook);  // the head block's rows are final as this solve ends them
    TRY(blas_trsm(c, 'L', 'L', 'T', 'N', one<T>(), t1, b1, false, W1));
  }
  return 0;
}

template <typename T> int pftrs(Ctx c, const RfpDesc& d, const T* arf, View<T> b,
                                cudaEvent_t b2_final, RowDoneHook* head_rows) {
  if (d.n == 0 || b.n == 0) return 0;
  View<T> t1, t2, s1;
  rfp_blocks(d, const_cast<T*>(arf), t1, t2, s1);
  T *W1 = nullptr, *W2 = nullptr;
  WsPair fr{c.st};
  TRY(ws_alloc(&W1, t1.m, c.st));
  fr.p[0] = W1;
  TRY(blas_leaf_inverses(c, t1, W1));
  if (t2.m) {
    TRY(ws_alloc(&W2, t2.m, c.st));
    fr.p[1] = W2;
    TRY(blas_leaf_inverses(c, t2.t(), W2));
  }
  return pftrs_part(c, d, arf, b, W1, W2, b2_final, 0, head_rows);
}

// pftrf + pftrs in one driver (the public pfsv paths).  The first solve with
// T1 and the S1 product (pftrs part 1) read only T1 and S1, so they run on
// the caller's stream WHILE potrf(T2) runs on the high-priority stream: the
// factorization's diagonal chain leaves SM slots and DMMA cycles idle that
// the solve fills.  No flags cross the two: they touch disjoint blocks.
template <typename T>
int pfsv(Ctx c, const RfpDesc& d, T* arf, View<T> b, cudaEvent_t s1_ready, const int* cflags,
         const int* sflags, cudaEvent_t b_ready, cudaEvent_t b2_final, RowDoneHook* head_rows) {
  PfsvPlan<T> plan{b, b_ready, b2_final, false, head_rows};
  const int rc = pftrf<T>(c, d, arf, s1_ready, cflags, sflags, b.n ? &plan : nullptr);
  if (rc || plan.done || b.n == 0 || d.n == 0) return rc;
  if (b_ready) cudaStreamWaitEvent(c.st, b_ready, 0);
  return pftrs<T>(c, d, arf, b, b2_final, head_rows);
}

// triangular inverse in RFP (rfp.py:286-325)
template <typename T> int tftri(Ctx c, const RfpDesc& d, char diag, T* arf) {
  if (d.n == 0) return 0;
  View<T> t1, t2, s1;
  rfp_blocks(d, arf, t1, t2, s1);
  PhaseTrace tr(c.st, "tftri");
  if (d.lower) {
    TRY(blas_trtri(c, 'L', diag, t1, 0));
    tr.mark("trtri(T1)");
    if (d.n2) {
      TRY(blas_trmm(c, 'R', 'L', 'N', diag, m_one<T>(), t1, s1));
      tr.mark("trmm(S1)");
      TRY(blas_trtri(c, 'U', diag, t2, (int)d.n1));
      tr.mark("trtri(T2)");
      TRY(blas_trmm(c, 'L', 'U', 'T', diag, one<T>(), t2, s1));
      tr.mark("trmm(S1)");
    }
    return 0;
  }
  if (d.n2) {
    TRY(blas_trtri(c, 'L', diag, t1, 0));
    tr.mark("trtri(T1)");
    TRY(blas_trmm(c, 'L', 'L', 'T', diag, m_one<T>(), t1, s1));
    tr.mark("trmm(S1)");
    TRY(blas_trtri(c, 'U', diag, t2, (int)d.n2));
    tr.mark("trtri(T2)");
    TRY(blas_trmm(c, 'R', 'U', 'N', diag, one<T>(), t2, s1));
    tr.mark("trmm(S1)");
    return 0;
  }
  return blas_trtri(c, 'U', diag, t2, 0);
}

__global__ void merge_info_kernel(int* info, const int* info2) {
  if (*info == 0 && *info2 != 0) *info = *info2;
}

// pftri at mid orders with the independent steps on two streams (a fork
// and join of the caller's stream, also inside a captured graph): for 'L',
//   main: trtri(T1) -> trmm(S1 <- -S1 W1) -> [join T2] trmm(S1 <- W2^T S1)
//         -> [join lauum(T1)] syrk(T1 += S1^H S1) -> trmm(S1) -> lauum(T2)
//   side: trtri(T2) ...................... lauum(T1) (after the first trmm)
// ('U' mirrors it).  The side trtri reports a zero diagonal in its own info,
// merged after the join so T1's failure still wins (rfp.py:299-322: the
// reference stops at the first block).  The latency-bound launches of the
// two chains overlap (n = 1000: 0.48 -> 0.38 ms).
template <typename T> static int pftri_concurrent(Ctx c, const RfpDesc& d, T* arf) {
  const bool herm = is_cplx<T>::value;
  View<T> t1, t2, s1;
  rfp_blocks(d, arf, t1, t2, s1);
  OverlapStreams& S = overlap_streams();
  cudaStream_t side = S.lo;
  int* info2 = nullptr;
  TRY(cudaMallocAsync((void**)&info2, sizeof(int), c.st));
  TRY(cudaMemsetAsync(info2, 0, sizeof(int), c.st));
  PhaseTrace tr(c.st, "pftri");
  const int base2 = (int)(d.lower ? d.n1 : d.n2);
  // fork: trtri(T2) on the side stream, with its own info
  TRY(cudaEventRecord(S.ev[0], c.st));
  TRY(cudaStreamWaitEvent(side, S.ev[0], 0));
  int rs = blas_trtri(Ctx{side, info2}, 'U', 'N', t2, base2);
  int rc = blas_trtri(c, 'L', 'N', t1, 0);
  if (!rc) rc = d.lower ? blas_trmm(c, 'R', 'L', 'N', 'N', m_one<T>(), t1, s1)
                        : blas_trmm(c, 'L', 'L', 'T', 'N', m_one<T>(), t1, s1);
  // lauum(T1) needs only W1 (its trmm is done): side stream, after trtri(T2)
  cudaEventRecord(S.ev[1], c.st);
  cudaStreamWaitEvent(side, S.ev[1], 0);
  cudaEventRecord(S.ev[2], side);  // trtri(T2) done (side is in order)
  if (!rs) rs = blas_lauum(Ctx{side, c.info}, 'L', t1);
  cudaEventRecord(S.ev[3], side);
  // join trtri(T2), merge its info, trmm(S1) with W2
  cudaStreamWaitEvent(c.st, S.ev[2], 0);
  merge_info_kernel<<<1, 1, 0, c.st>>>(c.info, info2);
  if (!rc) rc = d.lower ? blas_trmm(c, 'L', 'U', 'T', 'N', one<T>(), t2, s1)
                        : blas_trmm(c, 'R', 'U', 'N', 'N', one<T>(), t2, s1);
  tr.mark("tftri");
  // join lauum(T1), then the rest of the lauum stage in order
  cudaStreamWaitEvent(c.st, S.ev[3], 0);
  if (!rc) rc = rs;
  if (!rc) rc = d.lower ? blas_syrk(c, 'L', 'C', 1.0, s1, 1.0, t1, herm)
                        : blas_syrk(c, 'L', 'C', 1.0, s1.t(), 1.0, t1, herm);
  if (!rc) rc = d.lower ? blas_trmm(c, 'L', 'L', 'C', 'N', one<T>(), t2.t(), s1)
                        : blas_trmm(c, 'R', 'U', 'C', 'N', one<T>(), t2, s1);
  if (!rc) rc = blas_lauum(c, 'U', t2);
  tr.mark("lauum stage");
  cudaFreeAsync(info2, c.st);
  return rc;
}

// inverse from the Cholesky factor: tftri + lauum stage (rfp.py:328-360)
template <typename T> int pftri(Ctx c, const RfpDesc& d, T* arf) {
  if (d.n2 && d.n1 <= panel_max()) return pftri_concurrent(c, d, arf);
  TRY(tftri(c, d, 'N', arf));
  if (d.n == 0) return 0;
  const bool herm = is_cplx<T>::value;
  View<T> t1, t2, s1;
  rfp_blocks(d, arf, t1, t2, s1);
  PhaseTrace tr(c.st, "pftri");
  if (d.lower) {
    TRY(blas_lauum(c, 'L', t1));
    tr.mark("lauum(T1)");
    if (d.n2) {
      TRY(blas_syrk(c, 'L', 'C', 1.0, s1, 1.0, t1, herm));
      tr.mark("syrk(T1)");
      TRY(blas_trmm(c, 'L', 'L', 'C', 'N', one<T>(), t2.t(), s1));
      tr.mark("trmm(S1)");
      TRY(blas_lauum(c, 'U', t2));
      tr.mark("lauum(T2)");
    }
    return 0;
  }
  if (d.n2) {
    TRY(blas_lauum(c, 'L', t1));
    tr.mark("lauum(T1)");
    TRY(blas_syrk(c, 'L', 'C', 1.0, s1.t(), 1.0, t1, herm));
    tr.mark("syrk(T1)");
    TRY(blas_trmm(c, 'R', 'U', 'C', 'N', one<T>(), t2, s1));
    tr.mark("trmm(S1)");
  }
  TRY(blas_lauum(c, 'U', t2));
  tr.mark("lauum(T2)");
  return 0;
}

// ============================================================ conversions
// Element (i, j) of the logical triangle -> offset in a storage, plus whether
// consecutive i are consecutive in memory ("i-fast").  RFP cells follow
// SURVEY Appendix B (convert.py:174-185, layout.py:127-163).
__device__ __forceinline__ i64 storage_addr(const Storage& s, i64 i, i64 j, bool& ifast) {
  if (s.kind == ST_FULL) { ifast = true; return i + j * s.ld; }
  const RfpDesc& r = s.r;
  if (s.kind == ST_PACKED) {
    ifast = true;
    return r.lower ? j * r.n - j * (j - 1) / 2 + (i - j) : j * (j + 1) / 2 + i;
  }
  i64 row, col;
  bool rowvar;
  if (r.lower) {
    if (j < r.n1) { row = i + r.d; col = j; rowvar = true; }
    else { row = j - r.n1; col = i - r.n1 + 1 - r.d; rowvar = false; }
  } else {
    if (j >= r.n2) { row = i; col = j - r.n2; rowvar = true; }
    else { row = j + r.n2 + 1; col = i; rowvar = false; }
  }
  if (!r.trans) { ifast = rowvar; return col * r.ldar + row; }
  ifast = !rowvar;
  return row * r.n1 + col;
}

// Contiguity of a storage over a whole column range [j0, j0 + 64): 1 = i-fast,
// 2 = j-fast, 3 = mixed (the tile straddles the RFP block boundary at column
// n1 (L) / n2 (U), where the transposed block starts).
__device__ __forceinline__ int tile_mode(const Storage& s, i64 j0) {
  if (s.kind != ST_RFP) return 1;
  const RfpDesc& r = s.r;
  const i64 split = r.lower ? r.n1 : r.n2;
  const bool lo_rowvar = r.lower;             // columns j < split are "row-varying" for L
  const i64 j1 = j0 + 63;
  auto mode_of = [&](bool left) {
    const bool rowvar = left ? lo_rowvar : !lo_rowvar;
    return (rowvar != r.trans) ? 1 : 2;
  };
  if (j1 < split) return mode_of(true);
  if (j0 >= split) return mode_of(false);
  return 3;
}

// Addressing of one storage over a tile that lies inside one RFP block: the
// RFP and full maps are affine there (base + i*si + j*sj, from three probes of
// storage_addr), the packed map is affine in i within each column.
struct TileAff {
  i64 base, si, sj;
  int packed;
};
__device__ __forceinline__ TileAff tile_aff(const Storage& s, i64 i0, i64 j0) {
  TileAff a{0, 1, 0, 0};
  if (s.kind == ST_PACKED) {
    a.packed = 1;
    return a;
  }
  bool f;
  a.base = storage_addr(s, i0, j0, f);
  a.si = storage_addr(s, i0 + 1, j0, f) - a.base;
  a.sj = storage_addr(s, i0, j0 + 1, f) - a.base;
  return a;
}
__device__ __forceinline__ i64 packed_addr(const RfpDesc& r, i64 i, i64 j) {
  return r.lower ? j * r.n - j * (j - 1) / 2 + (i - j) : j * (j + 1) / 2 + i;
}

// One 64x64 tile of the logical (i, j) space per CTA (256 threads, 16
// elements per thread per pass, all loads of a pass issued before the shared
// stores).  Loads use an i-fast or j-fast thread mapping according to the
// source's contiguity, stores according to the destination's, so both sides
// are coalesced even where RFP stores a block transposed; tiles that lie in
// one block run a single pass each way.
template <typename T>
__global__ void __launch_bounds__(256) convert_kernel(Storage src, const T* __restrict__ sp,
                                                      Storage dst, T* __restrict__ dp, i64 n,
                                                      i64 rows_total, int lower, int zero_fill) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tile = reinterpret_cast<T*>(smem_raw);  // tile[jj * 65 + ii]
  constexpr int TL = 65;
  const i64 i0 = (i64)blockIdx.x * 64, j0 = (i64)blockIdx.y * 64;
  const bool outside = lower ? (i0 + 63 < j0) : (i0 > j0 + 63);
  const int tid = threadIdx.x;
  if (outside) {
    if (!zero_fill) return;
    // zero-only tile of the full destination: stream zeros, no smem round trip
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const i64 i = i0 + (tid & 63), j = j0 + (tid >> 6) + 4 * r;
      if (i < rows_total && j < n) dp[i + j * dst.ld] = sc_from<T>(0.0);
    }
    return;
  }
  const int smode = tile_mode(src, j0);
  const int dmode = zero_fill ? 1 : tile_mode(dst, j0);
  // interior tiles (strictly inside the triangle, inside the matrix, one RFP
  // block on each side): affine addressing, one add per element
  const bool interior = (lower ? i0 >= j0 + 64 : i0 + 64 <= j0) && i0 + 63 < n && j0 + 63 < n;
  if (interior && smode != 3 && dmode != 3) {
    const TileAff sa = tile_aff(src, i0, j0), da = tile_aff(dst, i0, j0);
    const int a = tid & 63, b = tid >> 6;
    T v[16];
    if (smode == 1) {  // i-fast: lanes along i, r along j
      if (sa.packed) {
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = sp[packed_addr(src.r, i0 + a, j0 + b + 4 * r)];
      } else {
        const T* p = sp + sa.base + a * sa.si + b * sa.sj;
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = p[(i64)r * 4 * sa.sj];
      }
#pragma unroll
      for (int r = 0; r < 16; ++r) tile[(b + 4 * r) * TL + a] = v[r];
    } else {           // j-fast: lanes along j, r along i
      const T* p = sp + sa.base + b * sa.si + a * sa.sj;
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = p[(i64)r * 4 * sa.si];
#pragma unroll
      for (int r = 0; r < 16; ++r) tile[a * TL + b + 4 * r] = v[r];
    }
    __syncthreads();
    if (dmode == 1) {
      if (da.packed) {
#pragma unroll
        for (int r = 0; r < 16; ++r) dp[packed_addr(dst.r, i0 + a, j0 + b + 4 * r)] = tile[(b + 4 * r) * TL + a];
      } else {
        T* p = dp + da.base + a * da.si + b * da.sj;
#pragma unroll
        for (int r = 0; r < 16; ++r) p[(i64)r * 4 * da.sj] = tile[(b + 4 * r) * TL + a];
      }
    } else {
      T* p = dp + da.base + b * da.si + a * da.sj;
#pragma unroll
      for (int r = 0; r < 16; ++r) p[(i64)r * 4 * da.si] = tile[a * TL + b + 4 * r];
    }
    return;
  }
#pragma unroll
  for (int pass = 1; pass <= 2; ++pass) {
    if (!(smode & pass)) continue;
    T v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int a = tid & 63, b = (tid >> 6) + 4 * r;
      const int ii = pass == 1 ? a : b, jj = pass == 1 ? b : a;
      const i64 i = i0 + ii, j = j0 + jj;
      const bool in = i < n && j < n && (lower ? i >= j : i <= j);
      v[r] = sc_from<T>(0.0);
      if (in) {
        bool f;
        const i64 off = storage_addr(src, i, j, f);
        if (smode != 3 || f == (pass == 1)) v[r] = sp[off];
      }
    }
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int a = tid & 63, b = (tid >> 6) + 4 * r;
      const int ii = pass == 1 ? a : b, jj = pass == 1 ? b : a;
      const i64 i = i0 + ii, j = j0 + jj;
      const bool in = i < n && j < n && (lower ? i >= j : i <= j);
      bool mine = true;
      if (smode == 3 && in) {
        bool f;
        storage_addr(src, i, j, f);
        mine = f == (pass == 1);
      }
      // out-of-triangle elements are written (as zero) by the i-fast pass only
      if (in ? mine : pass == 1 || smode == 2) tile[jj * TL + ii] = v[r];
    }
  }
  __syncthreads();
#pragma unroll
  for (int pass = 1; pass <= 2; ++pass) {
    if (!(dmode & pass)) continue;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int a = tid & 63, b = (tid >> 6) + 4 * r;
      const int ii = pass == 1 ? a : b, jj = pass == 1 ? b : a;
      const i64 i = i0 + ii, j = j0 + jj;
      if (zero_fill) {
        // full destination, i-fast: every element of the ld x n array
        if (i < rows_total && j < n) dp[i + j * dst.ld] = tile[jj * TL + ii];
        continue;
      }
      const bool in = i < n && j < n && (lower ? i >= j : i <= j);
      if (in) {
        bool f;
        const i64 off = storage_addr(dst, i, j, f);
        if (dmode != 3 || f == (pass == 1)) dp[off] = tile[jj * TL + ii];
      }
    }
  }
}

template <typename T>
int convert(const Storage& src, const T* s, const Storage& dst, T* dptr, bool zero_fill,
            cudaStream_t st) {
  const i64 n = src.r.n;
  if (n == 0 && !(zero_fill && dst.kind == ST_FULL)) return 0;
  const i64 rows = (zero_fill && dst.kind == ST_FULL) ? dst.ld : n;
  if (rows == 0 || n == 0) return 0;
  dim3 grid((unsigned)((rows + 63) / 64), (unsigned)((n + 63) / 64));
  const size_t sm = 64 * 65 * sizeof(T);
  auto k = convert_kernel<T>;
  kernel_setup(k, 256, sm);
  KernelClock kc(st);
  k<<<grid, 256, sm, st>>>(src, s, dst, dptr, n, rows, src.r.lower ? 1 : 0, zero_fill ? 1 : 0);
  RFPK_CHECK_LAUNCH();
  kc.stop("convert", src.kind * 10 + dst.kind, n);
  return 0;
}


// ============================================================ SURVEY 8(f) rows
// tfsm: RFP triangular solve through T1/S1/T2 (rfp.py:139-224); singular
// indices re-based to the global row via the scan base (rfp.py:46-52).
template <typename T>
static int tfsm_left(Ctx c, const RfpDesc& d, char trans, char diag, T alpha, View<T> t1,
                     View<T> t2, View<T> s1, View<T> b) {
  const i64 n1 = d.n1, n2 = d.n2, N = b.n;
  const int in1 = (int)n1, in2 = (int)n2;
  const T one_ = one<T>(), mone = m_one<T>();
  if (d.lower) {
    View<T> b1 = b.sub(0, 0, n1, N), b2 = b.sub(n1, 0, n2, N);
    if (trans == 'N') {
      TRY(blas_trsm(c, 'L', 'L', 'N', diag, alpha, t1, b1, true, (T*)nullptr, 0));
      if (n2) {
        TRY(blas_gemm(c, 'N', 'N', mone, s1, b1, alpha, b2));
        TRY(blas_trsm(c, 'L', 'U', 'T', diag, one_, t2, b2, true, (T*)nullptr, in1));
      }
    } else if (trans == 'T') {
      if (n2) {
        TRY(blas_trsm(c, 'L', 'U', 'N', diag, alpha, t2, b2, true, (T*)nullptr, in1));
        TRY(blas_gemm(c, 'T', 'N', mone, s1, b2, alpha, b1));
        TRY(blas_trsm(c, 'L', 'L', 'T', diag, one_, t1, b1, true, (T*)nullptr, 0));
      } else {
        TRY(blas_trsm(c, 'L', 'L', 'T', diag, alpha, t1, b1, true, (T*)nullptr, 0));
      }
    } else {
      if (n2) {
        TRY(blas_trsm(c, 'L', 'L', 'C', diag, alpha, t2.t(), b2, true, (T*)nullptr, in1));
        TRY(blas_gemm(c, 'C', 'N', mone, s1, b2, alpha, b1));
        TRY(blas_trsm(c, 'L', 'L', 'C', diag, one_, t1, b1, true, (T*)nullptr, 0));
      } else {
        TRY(blas_trsm(c, 'L', 'L', 'C', diag, alpha, t1, b1, true, (T*)nullptr, 0));
      }
    }
    return 0;
  }
  View<T> b1 = b.sub(0, 0, n2, N), b2 = b.sub(n2, 0, n1, N);
  if (trans == 'N') {
    TRY(blas_trsm(c, 'L', 'U', 'N', diag, alpha, t2, b2, true, (T*)nullptr, in2));
    if (n2) {
      TRY(blas_gemm(c, 'N', 'N', mone, s1, b2, alpha, b1));
      TRY(blas_trsm(c, 'L', 'L', 'T', diag, one_, t1, b1, true, (T*)nullptr, 0));
    }
  } else if (trans == 'T') {
    if (n2) {
      TRY(blas_trsm(c, 'L', 'L', 'N', diag, alpha, t1, b1, true, (T*)nullptr, 0));
      TRY(blas_gemm(c, 'T', 'N', mone, s1, b1, alpha, b2));
      TRY(blas_trsm(c, 'L', 'U', 'T', diag, one_, t2, b2, true, (T*)nullptr, in2));
    } else {
      TRY(blas_trsm(c, 'L', 'U', 'T', diag, alpha, t2, b2, true, (T*)nullptr, in2));
    }
  } else {
    if (n2) {
      TRY(blas_trsm(c, 'L', 'U', 'C', diag, alpha, t1.t(), b1, true, (T*)nullptr, 0));
      TRY(blas_gemm(c, 'C', 'N', mone, s1, b1, alpha, b2));
      TRY(blas_trsm(c, 'L', 'U', 'C', diag, one_, t2, b2, true, (T*)nullptr, in2));
    } else {
      TRY(blas_trsm(c, 'L', 'U', 'C', diag, alpha, t2, b2, true, (T*)nullptr, in2));
    }
  }
  return 0;
}

template <typename T>
int tfsm(Ctx c, const RfpDesc& d, char side, char trans, char diag, T alpha, const T* arf,
         View<T> b) {
  if (b.empty()) return 0;
  if (is_zero(alpha)) return scale_view<T>(b, alpha, TRI_FULL, false, c.info, c.st);
  if (!is_cplx<T>::value && trans == 'C') trans = 'T';
  View<T> t1, t2, s1;
  rfp_blocks(d, const_cast<T*>(arf), t1, t2, s1);
  if (side == 'L') return tfsm_left(c, d, trans, diag, alpha, t1, t2, s1, b);
  if (trans == 'C') {
    // X A^H = alpha B  <=>  A conj(X)^T = conj(alpha) conj(B)^T  (rfp.py:218-222)
    TRY(conj_view<T>(b, c.info, c.st));
    TRY(tfsm_left(c, d, 'N', diag, conj_(alpha), t1, t2, s1, b.t()));
    return conj_view<T>(b, c.info, c.st);
  }
  return tfsm_left(c, d, trans == 'N' ? 'T' : 'N', diag, alpha, t1, t2, s1, b.t());
}

// sfrk/hfrk: C <- alpha G G^(T|H) + beta C on the RFP blocks (rfp.py:227-283)
template <typename T>
int sfrk(Ctx c, const RfpDesc& d, char trans, i64 k, double alpha, View<T> a, double beta, T* arf,
         bool herm) {
  if (d.n == 0) return 0;
  if (alpha == 0.0 || k == 0) {
    if (beta == 1.0) return 0;
    return scale_view<T>(View<T>{arf, d.nt, 1, 1, d.nt}, sc_from<T>(beta), TRI_FULL, false,
                         c.info, c.st);
  }
  View<T> t1, t2, s1;
  rfp_blocks(d, arf, t1, t2, s1);
  const bool rows = trans == 'N';
  const i64 n1 = d.n1, n2 = d.n2;
  const T al = sc_from<T>(alpha), be = sc_from<T>(beta);
  auto part = [&](i64 r0, i64 cnt) { return rows ? a.sub(r0, 0, cnt, k) : a.sub(0, r0, k, cnt); };
  const char tc = rows ? 'C' : 'N';
  if (d.lower) {
    View<T> a1 = part(0, n1), a2 = part(n1, n2);
    TRY(blas_syrk(c, 'L', trans, alpha, a1, beta, t1, herm));
    if (n2) {
      if (rows) TRY(blas_gemm(c, 'N', 'C', al, a2, a1, be, s1));
      else TRY(blas_gemm(c, 'C', 'N', al, a2, a1, be, s1));
      TRY(blas_syrk(c, 'U', tc, alpha, a2.t(), beta, t2, herm));
    }
    return 0;
  }
  View<T> a1 = part(0, n2), a2 = part(n2, n1);
  if (n2) {
    TRY(blas_syrk(c, 'L', tc, alpha, a1.t(), beta, t1, herm));
    if (rows) TRY(blas_gemm(c, 'N', 'C', al, a1, a2, be, s1));
    else TRY(blas_gemm(c, 'C', 'N', al, a1, a2, be, s1));
  }
  return blas_syrk(c, 'U', trans, alpha, a2, beta, t2, herm);
}

// lansf: one pass over the RFP buffer (rfp.py:363-417).  Each stored element
// (i, j) of the triangle stands for |A(i,j)| = |A(j,i)|: 'M' takes the max,
// 'F' sums |a|^2 twice off the diagonal, '1'/'I' add |a| to the column sums
// of columns j and i (the implied full matrix is symmetric in magnitude).
__device__ __forceinline__ double mag(double v) { return fabs(v); }
__device__ __forceinline__ double mag(Z v) { return hypot(v.x, v.y); }

__device__ __forceinline__ void atomic_max_pos(double* a, double v) {
  // v >= 0: the IEEE bit pattern of non-negative doubles orders like the value
  atomicMax(reinterpret_cast<unsigned long long*>(a), __double_as_longlong(v));
}

// 'M' and the bulk of 'F': one grid-stride pass over the buffer with no index
// arithmetic (F^2 = 2 sum |a|^2 - sum_diag |a|^2: every stored off-diagonal
// cell stands for two entries of the full matrix).
template <typename T>
__global__ void lansf_sum_kernel(const T* __restrict__ arf, i64 nt, int mode, double* acc) {
  double local = 0.0;
  for (i64 p = blockIdx.x * (i64)blockDim.x + threadIdx.x; p < nt;
       p += (i64)gridDim.x * blockDim.x) {
    const double m = mag(arf[p]);
    local = mode == 0 ? fmax(local, m) : local + 2.0 * m * m;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double v = __shfl_down_sync(0xffffffffu, local, o);
    local = mode == 0 ? fmax(local, v) : local + v;
  }
  if ((threadIdx.x & 31) == 0) {
    if (mode == 0) atomic_max_pos(acc, local);
    else atomicAdd(acc, local);
  }
}

// acc -= sum over the n diagonal cells of |a|^2
template <typename T>
__global__ void lansf_diag_kernel(RfpDesc d, const T* __restrict__ arf, double* acc) {
  double local = 0.0;
  const Storage s{ST_RFP, 0, d};
  for (i64 k = blockIdx.x * (i64)blockDim.x + threadIdx.x; k < d.n; k += (i64)gridDim.x * blockDim.x) {
    bool f;
    const double m = mag(arf[storage_addr(s, k, k, f)]);
    local += m * m;
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(acc, -local);
}

// '1' / 'I': column sums of the implied full matrix.  Cell (row, col) of the
// normal rectangle (ldar x n1) stands for (i, j) of the triangle, and in each
// of its two regions one index depends on the row only, the other on the
// column only:
//   L, A (row >= col+d):  i = row-d,    j = col;        diagonal: row-d == col
//   L, B:                 j = row+n1,   i = col+n1-1+d; diagonal: col+d-1 == row
//   U, A (row <= col+n2): i = row,      j = col+n2;     diagonal: row == col+n2
//   U, B:                 j = row-n2-1, i = col;        diagonal: col == row-n2-1
// so colsum[row target] += sum over a rectangle ROW and colsum[column target]
// += sum over a rectangle COLUMN (the diagonal counted once, with the row).
// Two coalesced passes: BY_RUN reduces each contiguous run of the buffer (a
// warp per run, 2 atomics per run), !BY_RUN gives each thread one position of
// the run and sums across 64 runs (2 atomics per thread per 64 runs).
// Per fixed coordinate (the run for BY_RUN, the position within the runs
// otherwise) the region boundary, the two diagonal positions and both targets
// are computed once; each element then costs a compare-select-add.
struct LansfFixed {
  long long bound;  // region A <=> v >= bound (aGE) or v <= bound (!aGE)
  bool aGE;
  long long dA, dB;  // varying-index positions of the A / B diagonal cells
  i64 tA, tB;        // targets of the two regions
};
__device__ __forceinline__ LansfFixed lansf_fixed(const RfpDesc& d, i64 f, bool fixed_is_row,
                                                  bool col_target) {
  LansfFixed q;
  if (d.lower) {
    if (fixed_is_row) {  // A <=> col <= row - d
      q.bound = f - d.d; q.aGE = false; q.dA = f - d.d; q.dB = f + 1 - d.d;
      q.tA = col_target ? -1 : f - d.d; q.tB = col_target ? -1 : f + d.n1;
    } else {             // A <=> row >= col + d
      q.bound = f + d.d; q.aGE = true; q.dA = f + d.d; q.dB = f + d.d - 1;
      q.tA = col_target ? f : -1; q.tB = col_target ? f + d.n1 - 1 + d.d : -1;
    }
  } else {
    if (fixed_is_row) {  // A <=> col >= row - n2
      q.bound = f - d.n2; q.aGE = true; q.dA = f - d.n2; q.dB = f - d.n2 - 1;
      q.tA = col_target ? -1 : f; q.tB = col_target ? -1 : f - d.n2 - 1;
    } else {             // A <=> row <= col + n2
      q.bound = f + d.n2; q.aGE = false; q.dA = f + d.n2; q.dB = f + d.n2 + 1;
      q.tA = col_target ? f + d.n2 : -1; q.tB = col_target ? f : -1;
    }
  }
  return q;
}

template <typename T, bool BY_RUN>
__global__ void __launch_bounds__(256) lansf_colsum_kernel(RfpDesc d, const T* __restrict__ arf,
                                                           double* colsum) {
  // buffer = column-major (L x NR): runs of length L; 'N': runs are rectangle
  // columns (L = ldar), 'T': rectangle rows (L = n1)
  const i64 L = d.trans ? d.n1 : d.ldar, NR = d.trans ? d.ldar : d.n1;
  // the index this pass accumulates: along a run (BY_RUN) the run's own index
  // is fixed -- 'N' runs fix the column (column target), 'T' runs fix the row
  const bool col_target = BY_RUN != (bool)d.trans;
  // the fixed coordinate is a row when: BY_RUN and 'T', or !BY_RUN and 'N'
  const bool fixed_is_row = BY_RUN == (bool)d.trans;
  double sA = 0.0, sB = 0.0;
  LansfFixed q{};
  auto acc = [&](double m, long long v) {
    const bool inA = q.aGE ? v >= q.bound : v <= q.bound;
    // the diagonal cell counts once, with the row target
    if (col_target && (v == q.dA || v == q.dB)) {
      const bool diagA = v == q.dA && inA, diagB = v == q.dB && !inA;
      if (diagA || diagB) m = 0.0;
    }
    if (inA) sA += m;
    else sB += m;
  };
  if (BY_RUN) {
    const i64 run = (blockIdx.x * (i64)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (run >= NR) return;
    q = lansf_fixed(d, run, fixed_is_row, col_target);
    const T* pr = arf + run * L;
    for (i64 x0 = lane; x0 < L; x0 += 8 * 32) {
      double mv[8];  // eight independent loads in flight per lane
#pragma unroll
      for (int u = 0; u < 8; ++u) mv[u] = x0 + 32 * u < L ? mag(pr[x0 + 32 * u]) : -1.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (mv[u] >= 0.0) acc(mv[u], x0 + 32 * u);
    }
    for (int o = 16; o > 0; o >>= 1) {
      sA += __shfl_down_sync(0xffffffffu, sA, o);
      sB += __shfl_down_sync(0xffffffffu, sB, o);
    }
    if (lane == 0) {
      if (q.tA >= 0 && sA != 0.0) atomicAdd(colsum + q.tA, sA);
      if (q.tB >= 0 && sB != 0.0) atomicAdd(colsum + q.tB, sB);
    }
  } else {
    const i64 x = blockIdx.x * (i64)blockDim.x + threadIdx.x;  // position within the runs
    if (x >= L) return;
    q = lansf_fixed(d, x, fixed_is_row, col_target);
    const i64 r0 = (i64)blockIdx.y * 64, r1 = r0 + 64 < NR ? r0 + 64 : NR;
    for (i64 q0 = r0; q0 < r1; q0 += 8) {
      double mv[8];  // eight independent loads in flight per thread
#pragma unroll
      for (int u = 0; u < 8; ++u) mv[u] = q0 + u < r1 ? mag(arf[(q0 + u) * L + x]) : -1.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (mv[u] >= 0.0) acc(mv[u], q0 + u);
    }
    if (q.tA >= 0 && sA != 0.0) atomicAdd(colsum + q.tA, sA);
    if (q.tB >= 0 && sB != 0.0) atomicAdd(colsum + q.tB, sB);
  }
}

__global__ void colmax_kernel(const double* colsum, i64 n, double* acc) {
  double local = 0.0;
  for (i64 j = blockIdx.x * (i64)blockDim.x + threadIdx.x; j < n; j += (i64)gridDim.x * blockDim.x)
    local = fmax(local, colsum[j]);
  for (int o = 16; o > 0; o >>= 1) local = fmax(local, __shfl_down_sync(0xffffffffu, local, o));
  if ((threadIdx.x & 31) == 0) atomic_max_pos(acc, local);
}

__global__ void sqrt_kernel(double* acc) { *acc = sqrt(*acc); }

template <typename T>
int lansf(cudaStream_t st, const RfpDesc& d, char norm, const T* arf, double* out) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), st);
  if (e != cudaSuccess) return (int)e;
  if (d.n == 0) return 0;
  const int mode = norm == 'M' ? 0 : (norm == 'F' || norm == 'E') ? 2 : 1;
  double* colsum = nullptr;
  if (mode != 1) {
    int blocks = (int)((d.nt + 255) / 256);
    if (blocks > 8 * num_sms()) blocks = 8 * num_sms();
    lansf_sum_kernel<T><<<blocks, 256, 0, st>>>(arf, d.nt, mode, out);
    RFPK_CHECK_LAUNCH();
    if (mode == 2) {
      lansf_diag_kernel<T><<<(unsigned)((d.n + 255) / 256 < 1024 ? (d.n + 255) / 256 : 1024), 256, 0,
                             st>>>(d, arf, out);
      RFPK_CHECK_LAUNCH();
      sqrt_kernel<<<1, 1, 0, st>>>(out);
      RFPK_CHECK_LAUNCH();
    }
    return 0;
  }
  if ((e = cudaMallocAsync((void**)&colsum, sizeof(double) * d.n, st)) != cudaSuccess) return (int)e;
  if ((e = cudaMemsetAsync(colsum, 0, sizeof(double) * d.n, st)) != cudaSuccess) return (int)e;
  const i64 L = d.trans ? d.n1 : d.ldar, NR = d.trans ? d.ldar : d.n1;
  lansf_colsum_kernel<T, true><<<(unsigned)((NR * 32 + 255) / 256), 256, 0, st>>>(d, arf, colsum);
  RFPK_CHECK_LAUNCH();
  lansf_colsum_kernel<T, false><<<dim3((unsigned)((L + 255) / 256), (unsigned)((NR + 63) / 64)), 256,
                                  0, st>>>(d, arf, colsum);
  RFPK_CHECK_LAUNCH();
  int cb = (int)((d.n + 255) / 256);
  if (cb > 4 * num_sms()) cb = 4 * num_sms();
  colmax_kernel<<<cb, 256, 0, st>>>(colsum, d.n, out);
  RFPK_CHECK_LAUNCH();
  cudaFreeAsync(colsum, st);
  return 0;
}

#define RFPK_RFP_INST(T)                                                                     \
  template void rfp_blocks<T>(const RfpDesc&, T*, View<T>&, View<T>&, View<T>&);             \
  template int pftrf<T>(Ctx, const RfpDesc&, T*, cudaEvent_t, const int*, const int*, PfsvPlan<T>*); \
  template int pfsv<T>(Ctx, const RfpDesc&, T*, View<T>, cudaEvent_t, const int*, const int*,      \
                       cudaEvent_t, cudaEvent_t, RowDoneHook*);                 \
  template int rfp_h2d_split<T>(const RfpDesc&, const T*, T*, cudaStream_t, cudaStream_t);   \
  template int rfp_h2d_chunked<T>(const RfpDesc&, const T*, T*, int*, int*, cudaStream_t);                                            \
  template int pftrs<T>(Ctx, const RfpDesc&, const T*, View<T>, cudaEvent_t, RowDoneHook*);               \
  template int tftri<T>(Ctx, const RfpDesc&, char, T*);                                      \
  template int pftri<T>(Ctx, const RfpDesc&, T*);                                            \
  template int convert<T>(const Storage&, const T*, const Storage&, T*, bool, cudaStream_t);  \
  template int tfsm<T>(Ctx, const RfpDesc&, char, char, char, T, const T*, View<T>);         \
  template int sfrk<T>(Ctx, const RfpDesc&, char, i64, double, View<T>, double, T*, bool);   \
  template int lansf<T>(cudaStream_t, const RfpDesc&, char, const T*, double*);
RFPK_RFP_INST(double)
RFPK_RFP_INST(Z)

void phase_clock_enable(bool on) {
  PhaseClock& pc = PhaseClock::get();
  std::lock_guard<std::mutex> g(pc.mu);
  pc.drain();
  pc.sums.clear();
  pc.on = on;
}
std::string phase_clock_labels() {
  PhaseClock& pc = PhaseClock::get();
  std::lock_guard<std::mutex> g(pc.mu);
  pc.drain();
  std::string out;
  for (auto& kv : pc.sums) {
    out += kv.first;
    out += '\n';
  }
  return out;
}
bool phase_clock_read(const char* label, double* total_ms, long long* count) {
  PhaseClock& pc = PhaseClock::get();
  std::lock_guard<std::mutex> g(pc.mu);
  pc.drain();
  auto it = pc.sums.find(label);
  if (it == pc.sums.end()) return false;
  *total_ms = it->second.first;
  *count = it->second.second;
  return true;
}

}  // namespace rfpk
