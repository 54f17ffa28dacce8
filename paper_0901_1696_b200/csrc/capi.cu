// extern "C" boundary (include/rfpk_b200.h): argument checking, info reset,
// and dispatch into the templated drivers.  No allocations, no host syncs.
#include "../../include/rfpk_b200.h"
#include "graph_cache.cuh"
#include "rfp.cuh"

#include <cstring>
#include <map>
#include <mutex>

using namespace rfpk;

namespace {

char up(char c) { return (c >= 'a' && c <= 'z') ? (char)(c - 32) : c; }
bool one_of(char c, const char* set) {
  for (; *set; ++set)
    if (c == *set) return true;
  return false;
}
cudaStream_t S(rfpk_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }


int reset_info(int* info, cudaStream_t st) {
  if (!info) return 0;
  cudaError_t e = cudaMemsetAsync(info, 0, sizeof(int), st);
  return e == cudaSuccess ? 0 : (int)e;
}

template <typename T> View<T> V(const void* p, int64_t r, int64_t c, int64_t rs, int64_t cs) {
  return View<T>{reinterpret_cast<T*>(const_cast<void*>(p)), r, c, rs, cs};
}
bool unit_stride(int64_t r, int64_t c, int64_t rs, int64_t cs) {
  return rs == 1 || cs == 1 || r <= 1 || c <= 1;
}

// ---------------------------------------------------------------- conversions
template <typename T>
int trttf_t(char transr, char uplo, int64_t n, const void* a, int64_t lda, void* arf,
            cudaStream_t st) {
  transr = up(transr); uplo = up(uplo);
  if (!one_of(transr, "NTC")) return -1;
  if (!one_of(uplo, "LU")) return -2;
  if (n < 0) return -3;
  if (lda < (n > 1 ? n : 1)) return -5;
  Storage src{ST_FULL, lda, rfp_desc(n, uplo, transr)};
  Storage dst{ST_RFP, 0, rfp_desc(n, uplo, transr)};
  return convert<T>(src, (const T*)a, dst, (T*)arf, false, st);
}
template <typename T>
int tfttr_t(char transr, char uplo, int64_t n, const void* arf, void* a, int64_t lda,
            cudaStream_t st) {
  transr = up(transr); uplo = up(uplo);
  if (!one_of(transr, "NTC")) return -1;
  if (!one_of(uplo, "LU")) return -2;
  if (n < 0) return -3;
  if (lda < (n > 1 ? n : 1)) return -6;
  Storage src{ST_RFP, 0, rfp_desc(n, uplo, transr)};
  Storage dst{ST_FULL, lda, rfp_desc(n, uplo, transr)};
  return convert<T>(src, (const T*)arf, dst, (T*)a, true, st);
}
template <typename T>
int tpttf_t(char transr, char uplo, int64_t n, const void* ap, void* arf, cudaStream_t st) {
  transr = up(transr); uplo = up(uplo);
  if (!one_of(transr, "NTC")) return -1;
  if (!one_of(uplo, "LU")) return -2;
  if (n < 0) return -3;
  Storage src{ST_PACKED, 0, rfp_desc(n, uplo, transr)};
  Storage dst{ST_RFP, 0, rfp_desc(n, uplo, transr)};
  return convert<T>(src, (const T*)ap, dst, (T*)arf, false, st);
}
template <typename T>
int tfttp_t(char transr, char uplo, int64_t n, const void* arf, void* ap, cudaStream_t st) {
  transr = up(transr); uplo = up(uplo);
  if (!one_of(transr, "NTC")) return -1;
  if (!one_of(uplo, "LU")) return -2;
  if (n < 0) return -3;
  Storage src{ST_RFP, 0, rfp_desc(n, uplo, transr)};
  Storage dst{ST_PACKED, 0, rfp_desc(n, uplo, transr)};
  return convert<T>(src, (const T*)arf, dst, (T*)ap, false, st);
}
template <typename T>
int trttp_t(char uplo, int64_t n, const void* a, int64_t lda, void* ap, cudaStream_t st) {
  uplo = up(uplo);
  if (!one_of(uplo, "LU")) return -1;
  if (n < 0) return -2;
  if (lda < (n > 1 ? n : 1)) return -4;
  Storage src{ST_FULL, lda, rfp_desc(n, uplo, 'N')};
  Storage dst{ST_PACKED, 0, rfp_desc(n, uplo, 'N')};
  return convert<T>(src, (const T*)a, dst, (T*)ap, false, st);
}
template <typename T>
int tpttr_t(char uplo, int64_t n, const void* ap, void* a, int64_t lda, cudaStream_t st) {
  uplo = up(uplo);
  if (!one_of(uplo, "LU")) return -1;
  if (n < 0) return -2;
  if (lda < (n > 1 ? n : 1)) return -5;
  Storage src{ST_PACKED, 0, rfp_desc(n, uplo, 'N')};
  Storage dst{ST_FULL, lda, rfp_desc(n, uplo, 'N')};
  return convert<T>(src, (const T*)ap, dst, (T*)a, true, st);
}

// ---------------------------------------------------------------- RFP ops
template <typename T>
int pftrf_t(char transr, char uplo, int64_t n, void* arf, int* info, cudaStream_t st) {
  transr = up(transr); uplo = up(uplo);
  if (!one_of(transr, "NTC")) return -1;
  if (!one_of(uplo, "LU")) return -2;
  if (n < 0) return -3;
  if (!info) return -5;
  GraphKey key{1, is_cplx<T>::value ? 'z' : 'd', transr, uplo, 'N', n, 0, 0, 0, arf, nullptr, info,
               cur_device()};
  return GraphCache::get().run(key, st, [&](cudaStream_t s) {
    if (int rc = reset_info(info, s)) return rc;
    return pftrf<T>(Ctx{s, info}, rfp_desc(n, uplo, transr), (T*)arf);
  });
}
template <typename T>
int pftrs_t(char transr, char uplo, int64_t n, int64_t nrhs, const void* arf, void* b,
            int64_t rsb, int64_t csb, int* info, cudaStream_t st) {
  transr = up(transr); uplo = up(uplo);
  if (!one_of(transr, "NTC")) return -1;
  if (!one_of(uplo, "LU")) return -2;
  if (n < 0) return -3;
  if (nrhs < 0) return -4;
  if (!unit_stride(n, nrhs, rsb, csb)) return -7;
  if (!info) return -8;
  GraphKey key{2, is_cplx<T>::value ? 'z' : 'd', transr, uplo, 'N', n, nrhs, rsb, csb, arf, b, info,
               cur_device()};
  return GraphCache::get().run(key, st, [&](cudaStream_t s) {
    if (int rc = reset_info(info, s)) return rc;
    return pftrs<T>(Ctx{s, info}, rfp_desc(n, uplo, transr), (const T*)arf,
                    V<T>(b, n, nrhs, rsb, csb));
  });
}
template <typename T>
int tftri_t(char transr, char uplo, char diag, int64_t n, void* arf, int* info, cudaStream_t st) {
  transr = up(transr); uplo = up(uplo); diag = up(diag);
  if (!one_of(transr, "NTC")) return -1;
  if (!one_of(uplo, "LU")) return -2;
  if (!one_of(diag, "NU")) return -3;
  if (n < 0) return -4;
  if (!info) return -6;
  GraphKey key{3, is_cplx<T>::value ? 'z' : 'd', transr, uplo, diag, n, 0, 0, 0, arf, nullptr, info,
               cur_device()};
  return GraphCache::get().run(key, st, [&](cudaStream_t s) {
    if (int rc = reset_info(info, s)) return rc;
    return tftri<T>(Ctx{s, info}, rfp_desc(n, uplo, transr), diag, (T*)arf);
  });
}
template <typename T>
int pftri_t(char transr, char uplo, int64_t n, void* arf, int* info, cudaStream_t st) {
  transr = up(transr); uplo = up(uplo);
  if (!one_of(transr, "NTC")) return -1;
  if (!one_of(uplo, "LU")) return -2;
  if (n < 0) return -3;
  if (!info) return -5;
  GraphKey key{4, is_cplx<T>::value ? 'z' : 'd', transr, uplo, 'N', n, 0, 0, 0, arf, nullptr, info,
               cur_device()};
  return GraphCache::get().run(key, st, [&](cudaStream_t s) {
    if (int rc = reset_info(info, s)) return rc;
    return pftri<T>(Ctx{s, info}, rfp_desc(n, uplo, transr), (T*)arf);
  });
}

Z zc(double re, double im) { return Z{re, im}; }

}  // namespace

namespace rfpk {
std::atomic<long long> g_launch_count{0};

namespace {
struct TuneTable {
  const char* name;
  long long dflt;
};
constexpr TuneTable kTune[TK_COUNT] = {
    {"oop_max", 4096},       {"t2_copy_min", 2048}, {"panel_max", 4096},
    {"pfsv_overlap_min", 512}, {"overlap", 1},      {"graphs", 1},
    {"graph_max_n", 8192},   {"gemm_wide", 0},      {"batched_generic", 0},
    {"trace", 0},            {"trsm_split", 1},
    {"zpotrf_split_min", 9000}};
std::atomic<long long> g_tune[TK_COUNT] = {
    {kTune[0].dflt}, {kTune[1].dflt}, {kTune[2].dflt}, {kTune[3].dflt}, {kTune[4].dflt},
    {kTune[5].dflt}, {kTune[6].dflt}, {kTune[7].dflt}, {kTune[8].dflt}, {kTune[9].dflt},
    {kTune[10].dflt}, {kTune[11].dflt}};
int tune_index(const char* name) {
  if (!name) return -1;
  for (int i = 0; i < TK_COUNT; ++i)
    if (std::strcmp(name, kTune[i].name) == 0) return i;
  return -1;
}

std::mutex g_setup_mu;
std::map<std::pair<const void*, int>, int> g_setup;
}  // namespace

long long tune(TuneKey k) { return g_tune[k].load(std::memory_order_relaxed); }

int kernel_setup(const void* kern, int threads, size_t smem) {
  const int dev = cur_device();
  std::lock_guard<std::mutex> lk(g_setup_mu);
  auto it = g_setup.find({kern, dev});
  if (it != g_setup.end()) return it->second;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem);
  cudaGetLastError();
  if (nb < 1) nb = 1;
  g_setup.emplace(std::make_pair(kern, dev), nb);
  return nb;
}
}  // namespace rfpk

// ---------------------------------------------------------------- host streaming
// Start the host->device transfer of an RFP buffer on `copy` (forked from
// `st`).  Real data at orders where pftrf's potrf(T1) and S1 solve run on
// the dataflow tile kernels: 64-column chunks with per-chunk flags, so those
// two steps consume the buffer while it arrives (*cflags / *sflags set,
// `in_done` marks the end).  Otherwise two region copies, the S1 rows on the
// copy stream (`in_done` = the S1 rows landed) and T1/T2's on `st`.
template <typename T>
static int h2d_rfp_begin(const RfpDesc& d, const void* h, void* dv, cudaStream_t st,
                         cudaStream_t copy, cudaEvent_t fork, cudaEvent_t in_done, int** cflags,
                         int** sflags) {
  *cflags = *sflags = nullptr;
  const bool chunked = !is_cplx<T>::value && d.n1 >= 512;
  const i64 nch = (d.n1 + 63) / 64;
  cudaError_t e = cudaSuccess;
  if (chunked) {
    int* f = nullptr;
    if ((e = cudaMallocAsync((void**)&f, (size_t)2 * nch * sizeof(int), st)) != cudaSuccess)
      return (int)e;
    if ((e = cudaMemsetAsync(f, 0, (size_t)2 * nch * sizeof(int), st)) != cudaSuccess) return (int)e;
    *cflags = f;
    *sflags = f + nch;
  }
  if ((e = cudaEventRecord(fork, st)) != cudaSuccess) return (int)e;
  if ((e = cudaStreamWaitEvent(copy, fork, 0)) != cudaSuccess) return (int)e;
  int rc = chunked ? rfp_h2d_chunked<T>(d, (const T*)h, (T*)dv, *cflags, *sflags, copy)
                   : rfp_h2d_split<T>(d, (const T*)h, (T*)dv, st, copy);
  if (rc) return rc;
  return (int)cudaEventRecord(in_done, copy);
}

// cuStreamWaitValue32 (GEQ) through the runtime's driver entry point (no
// link-time dependency on libcuda); null if the driver does not offer it
using WaitValueFn = int (*)(cudaStream_t, const int*, unsigned);
namespace {
typedef int (*cu_wait_value32_t)(void* stream, unsigned long long addr, unsigned value,
                                 unsigned flags);
cu_wait_value32_t g_cu_wait = nullptr;
int wait_value_geq(cudaStream_t s, const int* addr, unsigned value) {
  return g_cu_wait((void*)s, (unsigned long long)(uintptr_t)addr, value, 0x0 /* GEQ */);
}
}  // namespace
static WaitValueFn stream_wait_value_fn() {
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_cu_wait = reinterpret_cast<cu_wait_value32_t>(fn);
    else
      cudaGetLastError();
  });
  return g_cu_wait ? wait_value_geq : nullptr;
}

// Side stream and events of the host-buffer drivers, per host thread and
// DEVICE (streams and events belong to the device current at creation; a
// thread may serve streams of several devices, see StreamDevice)
struct HostPathRes {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, s1_done = nullptr, b_done = nullptr, b2_final = nullptr,
              launched = nullptr, last_join = nullptr;
  int* rowcnt = nullptr;  // row-block counters (plain cudaMalloc: stream memory
  int rowcnt_len = 0;     // operations reject stream-ordered pool allocations)
};
static HostPathRes& host_path_res() {
  static thread_local HostPathRes per_dev[MAX_DEVICES];
  HostPathRes& r = per_dev[cur_device() & (MAX_DEVICES - 1)];
  if (!r.side) {
    cudaStreamCreateWithFlags(&r.side, cudaStreamNonBlocking);
    for (cudaEvent_t* e : {&r.fork, &r.s1_done, &r.b_done, &r.b2_final, &r.launched, &r.last_join})
      cudaEventCreateWithFlags(e, cudaEventDisableTiming);
    cudaEventRecord(r.last_join, r.side);
  }
  return r;
}

// ---------------------------------------------------------------- pftrf from host
// The factorization of a pinned HOST RFP buffer with the transfer streamed:
// the rows holding T1/T2 are copied on `st` and potrf(T1) starts as soon as
// they land, while the S1 rows come over on a side stream; the S1 solve
// waits for them.  The PCIe/C2C copy of S1 (about half the buffer) thus
// hides under potrf(T1).  Result and info as rfpk_?pftrf, in d_arf.
template <typename T>
int pftrf_host_t(char transr, char uplo, int64_t n, const void* h_arf, void* d_arf, int* info,
                 cudaStream_t st) {
  transr = up(transr); uplo = up(uplo);
  if (!one_of(transr, "NTC")) return -1;
  if (!one_of(uplo, "LU")) return -2;
  if (n < 0) return -3;
  if (!info) return -6;
  if (int rc = reset_info(info, st)) return rc;
  if (n == 0) return 0;
  const RfpDesc d = rfp_desc(n, uplo, transr);
  HostPathRes& R = host_path_res();
  cudaStream_t side = R.side;
  cudaEvent_t fork = R.fork, s1_done = R.s1_done;
  int* cflags;
  int* sflags;
  if (int rc = h2d_rfp_begin<T>(d, h_arf, d_arf, st, side, fork, s1_done, &cflags, &sflags))
    return rc;
  int rc = pftrf<T>(Ctx{st, info}, d, (T*)d_arf, s1_done, cflags, sflags);
  if (cflags) cudaFreeAsync(cflags, st);
  return rc;
}

// pftrf + pftrs of a pinned HOST problem with every transfer overlapped:
// T1/T2 rows first (stream), S1 rows then the right-hand side on a side
// stream (hidden under potrf(T1) and the S1 solve), and the solution's
// trailing block copied back while the last two solve steps still run.
template <typename T>
int pfsv_host_t(char transr, char uplo, int64_t n, int64_t nrhs, const void* h_arf, void* d_arf,
                const void* h_b, void* d_b, void* h_x, int64_t ldb, int* info, cudaStream_t st) {
  transr = up(transr); uplo = up(uplo);
  if (!one_of(transr, "NTC")) return -1;
  if (!one_of(uplo, "LU")) return -2;
  if (n < 0) return -3;
  if (nrhs < 0) return -4;
  if (ldb < (n > 1 ? n : 1)) return -10;
  if (!info) return -11;
  if (int rc = reset_info(info, st)) return rc;
  if (n == 0) return 0;
  const RfpDesc d = rfp_desc(n, uplo, transr);
  HostPathRes& R = host_path_res();
  cudaStream_t side = R.side;
  cudaEvent_t fork = R.fork, s1_done = R.s1_done, b_done = R.b_done, b2_final = R.b2_final;
  // the previous call's row-block waits (side stream) read the same counter
  // buffer: order this call after them, whatever stream it is on
  cudaStreamWaitEvent(st, R.last_join, 0);
  int* cflags;
  int* sflags;
  if (int rc = h2d_rfp_begin<T>(d, h_arf, d_arf, st, side, fork, s1_done, &cflags, &sflags))
    return rc;
  cudaError_t e;
  const size_t col = (size_t)n * sizeof(T), pitch = (size_t)ldb * sizeof(T);
  if (nrhs) {
    e = cudaMemcpy2DAsync(d_b, pitch, h_b, pitch, col, (size_t)nrhs, cudaMemcpyHostToDevice, side);
    if (e != cudaSuccess) return (int)e;
  }
  cudaEventRecord(b_done, side);
  // pftrf + pftrs as one driver (pfsv: the first T1 solve and the S1 product
  // run beside potrf(T2)); after a failed factorization every solve kernel
  // skips on *info
  const i64 split = d.lower ? d.n1 : d.n2;  // first row of the trailing block
  const bool trail = nrhs > 0 && n - split > 0 && !(d.lower && d.n2 == 0);
  // the head block [0, split) is final only as the last solve ends each of its
  // 64-row blocks: with the row-completion hook every block is copied back as
  // soon as its column tasks are done (a stream-ordered wait on the solve's
  // per-row counter), so only the last block's copy follows the solve
  RowDoneHook hook;
  hook.launched = R.launched;
  const int nbh = (int)((split + 63) / 64);
  int* rowcnt = nullptr;
  if (trail && stream_wait_value_fn()) {
    if (R.rowcnt_len < nbh) {
      cudaStreamSynchronize(side);  // (a previous call's waits may still read the old buffer)
      if (R.rowcnt) cudaFree(R.rowcnt);
      R.rowcnt = nullptr;
      R.rowcnt_len = 0;
      if (cudaMalloc((void**)&R.rowcnt, (size_t)nbh * sizeof(int)) == cudaSuccess)
        R.rowcnt_len = nbh;
      else
        cudaGetLastError();
    }
    if (R.rowcnt_len >= nbh) rowcnt = R.rowcnt;
    hook.rowcnt = rowcnt;
  }
  int rcf = pfsv<T>(Ctx{st, info}, d, (T*)d_arf, V<T>(d_b, n, nrhs, 1, ldb), s1_done, cflags,
                    sflags, b_done, trail ? b2_final : nullptr, rowcnt ? &hook : nullptr);
  if (cflags) cudaFreeAsync(cflags, st);
  if (rcf) return rcf;
  if (nrhs == 0) return 0;
  if (trail) {
    cudaStreamWaitEvent(side, b2_final, 0);
    e = cudaMemcpy2DAsync((T*)h_x + split, pitch, (const T*)d_b + split, pitch,
                          (size_t)(n - split) * sizeof(T), (size_t)nrhs, cudaMemcpyDeviceToHost,
                          side);
    if (e != cudaSuccess) return (int)e;
  }
  bool rows_copied = false;
  if (hook.used && hook.nb == nbh) {
    cudaStreamWaitEvent(side, hook.launched, 0);
    auto wait32 = stream_wait_value_fn();
    for (int k = 0; k < nbh; ++k) {
      const int i = hook.forward ? k : nbh - 1 - k;
      const i64 r0 = (i64)i * 64, rows = split - r0 < 64 ? split - r0 : 64;
      const int we = wait32(side, rowcnt + i, (unsigned)hook.nc);
      if (we != 0) {
        if (k == 0) {  // not offered for this memory / device: copy after the solve
          static bool once = [&] {
            fprintf(stderr, "rfpk: cuStreamWaitValue32 unavailable (CUresult %d): the "
                            "solution is copied back after the last solve\n", we);
            return true;
          }();
          (void)once;
          break;
        }
        return (int)cudaErrorUnknown;
      }
      e = cudaMemcpy2DAsync((T*)h_x + r0, pitch, (const T*)d_b + r0, pitch, (size_t)rows * sizeof(T),
                            (size_t)nrhs, cudaMemcpyDeviceToHost, side);
      if (e != cudaSuccess) return (int)e;
      rows_copied = true;
    }
  }
  if (!rows_copied) {
    e = cudaMemcpy2DAsync(h_x, pitch, d_b, pitch, (size_t)(trail ? split : n) * sizeof(T),
                          (size_t)nrhs, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return (int)e;
  }
  cudaEventRecord(fork, side);  // join the side stream back into `st`
  cudaStreamWaitEvent(st, fork, 0);
  cudaEventRecord(R.last_join, side);
  return 0;
}

// pftrf + pftrs of a device-resident problem in one call (the pfsv driver:
// the first solve with T1 and the S1 product overlap potrf(T2))
template <typename T>
int pfsv_t(char transr, char uplo, int64_t n, int64_t nrhs, void* arf, void* b, int64_t ldb,
           int* info, cudaStream_t st) {
  transr = up(transr); uplo = up(uplo);
  if (!one_of(transr, "NTC")) return -1;
  if (!one_of(uplo, "LU")) return -2;
  if (n < 0) return -3;
  if (nrhs < 0) return -4;
  if (ldb < (n > 1 ? n : 1)) return -7;
  if (!info) return -8;
  if (int rc = reset_info(info, st)) return rc;
  if (n == 0) return 0;
  return pfsv<T>(Ctx{st, info}, rfp_desc(n, uplo, transr), (T*)arf, V<T>(b, n, nrhs, 1, ldb));
}

// ---------------------------------------------------------------- packed Cholesky
// the reference's Level-2 packed comparator
// (packed.py:70-146 pptrf_ref / pptrs_ref).  B200 design: the column-packed
// triangle is converted to RFP (TRANSR='N', the tiled copy kernel) in a
// stream-ordered workspace, factored / solved there with the RFP drivers,
// and (pptrf) converted back -- the conversions move 2*nt elements each,
// negligible next to the n^3/3 factorization.  info = first non-positive
// leading minor, as pptrf_ref.
template <typename T>
int pptrf_t(char uplo, int64_t n, void* ap, int* info, cudaStream_t st) {
  uplo = up(uplo);
  if (!one_of(uplo, "LU")) return -1;
  if (n < 0) return -2;
  if (!info) return -4;
  if (int rc = reset_info(info, st)) return rc;
  if (n == 0) return 0;
  const RfpDesc d = rfp_desc(n, uplo, 'N');
  T* w = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&w, (size_t)d.nt * sizeof(T), st);
  if (e != cudaSuccess) return (int)e;
  const Storage pk{ST_PACKED, 0, d}, rf{ST_RFP, 0, d};
  int rc = convert<T>(pk, (const T*)ap, rf, w, false, st);
  if (!rc) rc = pftrf<T>(Ctx{st, info}, d, w);
  if (!rc) rc = convert<T>(rf, w, pk, (T*)ap, false, st);
  cudaFreeAsync(w, st);
  return rc;
}
template <typename T>
int pptrs_t(char uplo, int64_t n, int64_t nrhs, const void* ap, void* b, int64_t rsb,
            int64_t csb, int* info, cudaStream_t st) {
  uplo = up(uplo);
  if (!one_of(uplo, "LU")) return -1;
  if (n < 0) return -2;
  if (nrhs < 0) return -3;
  if (!unit_stride(n, nrhs, rsb, csb)) return -6;
  if (!info) return -8;
  if (int rc = reset_info(info, st)) return rc;
  if (n == 0 || nrhs == 0) return 0;
  const RfpDesc d = rfp_desc(n, uplo, 'N');
  T* w = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&w, (size_t)d.nt * sizeof(T), st);
  if (e != cudaSuccess) return (int)e;
  const Storage pk{ST_PACKED, 0, d}, rf{ST_RFP, 0, d};
  int rc = convert<T>(pk, (const T*)ap, rf, w, false, st);
  if (!rc) rc = pftrs<T>(Ctx{st, info}, d, w, V<T>(b, n, nrhs, rsb, csb));
  cudaFreeAsync(w, st);
  return rc;
}

extern "C" {

const char* rfpk_version(void) { return "rfpk_b200 0.1 (sm_100a, FP64 DMMA)"; }

long long rfpk_launch_count(void) { return g_launch_count.load(); }

int rfpk_graph_cache_clear(void) {
  GraphCache::get().clear();
  return 0;
}

int rfpk_set_tuning(const char* name, long long value) {
  const int i = tune_index(name);
  if (i < 0) return -1;
  g_tune[i].store(value);
  GraphCache::get().clear();  // no replay of a path chosen under the old value
  return 0;
}

int rfpk_get_tuning(const char* name, long long* value) {
  const int i = tune_index(name);
  if (i < 0 || !value) return -1;
  *value = g_tune[i].load();
  return 0;
}

int rfpk_reset_tuning(void) {
  for (int i = 0; i < TK_COUNT; ++i) g_tune[i].store(kTune[i].dflt);
  GraphCache::get().clear();
  return 0;
}

int rfpk_device_sms(void) {
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return -(int)e;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return e == cudaSuccess ? sms : -(int)e;
}

int rfpk_dtrttf(char t, char u, int64_t n, const double* a, int64_t lda, double* arf, rfpk_stream_t s) { StreamDevice dg_(s); return trttf_t<double>(t, u, n, a, lda, arf, S(s)); }
int rfpk_ztrttf(char t, char u, int64_t n, const void* a, int64_t lda, void* arf, rfpk_stream_t s) { StreamDevice dg_(s); return trttf_t<Z>(t, u, n, a, lda, arf, S(s)); }
int rfpk_dtfttr(char t, char u, int64_t n, const double* arf, double* a, int64_t lda, rfpk_stream_t s) { StreamDevice dg_(s); return tfttr_t<double>(t, u, n, arf, a, lda, S(s)); }
int rfpk_ztfttr(char t, char u, int64_t n, const void* arf, void* a, int64_t lda, rfpk_stream_t s) { StreamDevice dg_(s); return tfttr_t<Z>(t, u, n, arf, a, lda, S(s)); }
int rfpk_dtpttf(char t, char u, int64_t n, const double* ap, double* arf, rfpk_stream_t s) { StreamDevice dg_(s); return tpttf_t<double>(t, u, n, ap, arf, S(s)); }
int rfpk_ztpttf(char t, char u, int64_t n, const void* ap, void* arf, rfpk_stream_t s) { StreamDevice dg_(s); return tpttf_t<Z>(t, u, n, ap, arf, S(s)); }
int rfpk_dtfttp(char t, char u, int64_t n, const double* arf, double* ap, rfpk_stream_t s) { StreamDevice dg_(s); return tfttp_t<double>(t, u, n, arf, ap, S(s)); }
int rfpk_ztfttp(char t, char u, int64_t n, const void* arf, void* ap, rfpk_stream_t s) { StreamDevice dg_(s); return tfttp_t<Z>(t, u, n, arf, ap, S(s)); }
int rfpk_dtrttp(char u, int64_t n, const double* a, int64_t lda, double* ap, rfpk_stream_t s) { StreamDevice dg_(s); return trttp_t<double>(u, n, a, lda, ap, S(s)); }
int rfpk_ztrttp(char u, int64_t n, const void* a, int64_t lda, void* ap, rfpk_stream_t s) { StreamDevice dg_(s); return trttp_t<Z>(u, n, a, lda, ap, S(s)); }
int rfpk_dtpttr(char u, int64_t n, const double* ap, double* a, int64_t lda, rfpk_stream_t s) { StreamDevice dg_(s); return tpttr_t<double>(u, n, ap, a, lda, S(s)); }
int rfpk_ztpttr(char u, int64_t n, const void* ap, void* a, int64_t lda, rfpk_stream_t s) { StreamDevice dg_(s); return tpttr_t<Z>(u, n, ap, a, lda, S(s)); }

int rfpk_dpftrf(char t, char u, int64_t n, double* arf, int* info, rfpk_stream_t s) { StreamDevice dg_(s); return pftrf_t<double>(t, u, n, arf, info, S(s)); }
int rfpk_zpftrf(char t, char u, int64_t n, void* arf, int* info, rfpk_stream_t s) { StreamDevice dg_(s); return pftrf_t<Z>(t, u, n, arf, info, S(s)); }
int rfpk_dpftrs(char t, char u, int64_t n, int64_t nrhs, const double* arf, double* b, int64_t ldb, int* info, rfpk_stream_t s) { StreamDevice dg_(s);
  if (ldb < (n > 1 ? n : 1)) return -7;
  return pftrs_t<double>(t, u, n, nrhs, arf, b, 1, ldb, info, S(s));
}
int rfpk_zpftrs(char t, char u, int64_t n, int64_t nrhs, const void* arf, void* b, int64_t ldb, int* info, rfpk_stream_t s) { StreamDevice dg_(s);
  if (ldb < (n > 1 ? n : 1)) return -7;
  return pftrs_t<Z>(t, u, n, nrhs, arf, b, 1, ldb, info, S(s));
}
int rfpk_dpftrs_ex(char t, char u, int64_t n, int64_t nrhs, const double* arf, double* b, int64_t rsb, int64_t csb, int* info, rfpk_stream_t s) { StreamDevice dg_(s); return pftrs_t<double>(t, u, n, nrhs, arf, b, rsb, csb, info, S(s)); }
int rfpk_zpftrs_ex(char t, char u, int64_t n, int64_t nrhs, const void* arf, void* b, int64_t rsb, int64_t csb, int* info, rfpk_stream_t s) { StreamDevice dg_(s); return pftrs_t<Z>(t, u, n, nrhs, arf, b, rsb, csb, info, S(s)); }
int rfpk_dtftri(char t, char u, char d, int64_t n, double* arf, int* info, rfpk_stream_t s) { StreamDevice dg_(s); return tftri_t<double>(t, u, d, n, arf, info, S(s)); }
int rfpk_ztftri(char t, char u, char d, int64_t n, void* arf, int* info, rfpk_stream_t s) { StreamDevice dg_(s); return tftri_t<Z>(t, u, d, n, arf, info, S(s)); }
int rfpk_dpftri(char t, char u, int64_t n, double* arf, int* info, rfpk_stream_t s) { StreamDevice dg_(s); return pftri_t<double>(t, u, n, arf, info, S(s)); }
int rfpk_zpftri(char t, char u, int64_t n, void* arf, int* info, rfpk_stream_t s) { StreamDevice dg_(s); return pftri_t<Z>(t, u, n, arf, info, S(s)); }

int rfpk_dpftrf_host(char t, char u, int64_t n, const double* h, double* d, int* info, rfpk_stream_t s) { StreamDevice dg_(s); return pftrf_host_t<double>(t, u, n, h, d, info, S(s)); }
int rfpk_zpftrf_host(char t, char u, int64_t n, const void* h, void* d, int* info, rfpk_stream_t s) { StreamDevice dg_(s); return pftrf_host_t<Z>(t, u, n, h, d, info, S(s)); }
int rfpk_phase_clock(int enable) {
  phase_clock_enable(enable != 0);
  return 0;
}
int64_t rfpk_phase_labels(char* out, int64_t cap) {
  const std::string l = phase_clock_labels();
  if (out && cap > 0) {
    const size_t k = l.size() < (size_t)cap - 1 ? l.size() : (size_t)cap - 1;
    std::memcpy(out, l.data(), k);
    out[k] = '\0';
  }
  return (int64_t)l.size() + 1;
}
int rfpk_phase_time(const char* label, double* total_ms, int64_t* count) {
  if (!label || !total_ms || !count) return -1;
  long long c = 0;
  double t = 0;
  if (!phase_clock_read(label, &t, &c)) { *total_ms = 0; *count = 0; return 1; }
  *total_ms = t;
  *count = c;
  return 0;
}
int rfpk_dpfsv(char t, char u, int64_t n, int64_t nrhs, double* arf, double* b, int64_t ldb, int* info, rfpk_stream_t s) { StreamDevice dg_(s); return pfsv_t<double>(t, u, n, nrhs, arf, b, ldb, info, S(s)); }
int rfpk_zpfsv(char t, char u, int64_t n, int64_t nrhs, void* arf, void* b, int64_t ldb, int* info, rfpk_stream_t s) { StreamDevice dg_(s); return pfsv_t<Z>(t, u, n, nrhs, arf, b, ldb, info, S(s)); }
int rfpk_dpfsv_host(char t, char u, int64_t n, int64_t nrhs, const double* h_arf, double* d_arf, const double* h_b, double* d_b, double* h_x, int64_t ldb, int* info, rfpk_stream_t s) { StreamDevice dg_(s); return pfsv_host_t<double>(t, u, n, nrhs, h_arf, d_arf, h_b, d_b, h_x, ldb, info, S(s)); }
int rfpk_zpfsv_host(char t, char u, int64_t n, int64_t nrhs, const void* h_arf, void* d_arf, const void* h_b, void* d_b, void* h_x, int64_t ldb, int* info, rfpk_stream_t s) { StreamDevice dg_(s); return pfsv_host_t<Z>(t, u, n, nrhs, h_arf, d_arf, h_b, d_b, h_x, ldb, info, S(s)); }
int rfpk_dpptrf(char u, int64_t n, double* ap, int* info, rfpk_stream_t s) { StreamDevice dg_(s); return pptrf_t<double>(u, n, ap, info, S(s)); }
int rfpk_zpptrf(char u, int64_t n, void* ap, int* info, rfpk_stream_t s) { StreamDevice dg_(s); return pptrf_t<Z>(u, n, ap, info, S(s)); }
int rfpk_dpptrs(char u, int64_t n, int64_t nrhs, const double* ap, double* b, int64_t rsb, int64_t csb, int* info, rfpk_stream_t s) { StreamDevice dg_(s); return pptrs_t<double>(u, n, nrhs, ap, b, rsb, csb, info, S(s)); }
int rfpk_zpptrs(char u, int64_t n, int64_t nrhs, const void* ap, void* b, int64_t rsb, int64_t csb, int* info, rfpk_stream_t s) { StreamDevice dg_(s); return pptrs_t<Z>(u, n, nrhs, ap, b, rsb, csb, info, S(s)); }

// ---------------------------------------------------------------- SURVEY 8(f) rows
static int tfsm_check(char& transr, char& side, char& uplo, char& trans, char& diag, int64_t m,
                      int64_t n, int64_t rsb, int64_t csb, int* info) {
  transr = up(transr); side = up(side); uplo = up(uplo); trans = up(trans); diag = up(diag);
  if (!one_of(transr, "NTC")) return -1;
  if (!one_of(side, "LR")) return -2;
  if (!one_of(uplo, "LU")) return -3;
  if (!one_of(trans, "NTC")) return -4;
  if (!one_of(diag, "NU")) return -5;
  if (m < 0) return -6;
  if (n < 0) return -7;
  if (!unit_stride(m, n, rsb, csb)) return -10;
  if (!info) return -13;
  return 0;
}
int rfpk_dtfsm(char transr, char side, char uplo, char trans, char diag, int64_t m, int64_t n, double alpha,
               const double* arf, double* b, int64_t rsb, int64_t csb, int* info, rfpk_stream_t s) { StreamDevice dg_(s);
  if (int rc = tfsm_check(transr, side, uplo, trans, diag, m, n, rsb, csb, info)) return rc;
  if (int rc = reset_info(info, S(s))) return rc;
  const int64_t order = side == 'L' ? m : n;
  return tfsm<double>(Ctx{S(s), info}, rfp_desc(order, uplo, transr), side, trans, diag, alpha, arf,
                      V<double>(b, m, n, rsb, csb));
}
int rfpk_ztfsm(char transr, char side, char uplo, char trans, char diag, int64_t m, int64_t n, double are,
               double aim, const void* arf, void* b, int64_t rsb, int64_t csb, int* info, rfpk_stream_t s) { StreamDevice dg_(s);
  if (int rc = tfsm_check(transr, side, uplo, trans, diag, m, n, rsb, csb, info)) return rc;
  if (int rc = reset_info(info, S(s))) return rc;
  const int64_t order = side == 'L' ? m : n;
  return tfsm<Z>(Ctx{S(s), info}, rfp_desc(order, uplo, transr), side, trans, diag, zc(are, aim),
                 (const Z*)arf, V<Z>(b, m, n, rsb, csb));
}
static int sfrk_check(char& transr, char& uplo, char& trans, int64_t n, int64_t k, int64_t rsa, int64_t csa) {
  transr = up(transr); uplo = up(uplo); trans = up(trans);
  if (!one_of(transr, "NTC")) return -1;
  if (!one_of(uplo, "LU")) return -2;
  if (!one_of(trans, "NTC")) return -3;
  if (n < 0) return -4;
  if (k < 0) return -5;
  const int64_t r = trans == 'N' ? n : k, c = trans == 'N' ? k : n;
  if (!unit_stride(r, c, rsa, csa)) return -8;
  return 0;
}
int rfpk_dsfrk(char transr, char uplo, char trans, int64_t n, int64_t k, double alpha, const double* a,
               int64_t rsa, int64_t csa, double beta, double* arf, rfpk_stream_t s) { StreamDevice dg_(s);
  if (int rc = sfrk_check(transr, uplo, trans, n, k, rsa, csa)) return rc;
  const int64_t r = trans == 'N' ? n : k, c = trans == 'N' ? k : n;
  return sfrk<double>(Ctx{S(s), nullptr}, rfp_desc(n, uplo, transr), trans, k, alpha,
                      V<double>(a, r, c, rsa, csa), beta, arf, false);
}
int rfpk_zhfrk(char transr, char uplo, char trans, int64_t n, int64_t k, double alpha, const void* a,
               int64_t rsa, int64_t csa, double beta, void* arf, int hermitian, rfpk_stream_t s) { StreamDevice dg_(s);
  if (int rc = sfrk_check(transr, uplo, trans, n, k, rsa, csa)) return rc;
  const int64_t r = trans == 'N' ? n : k, c = trans == 'N' ? k : n;
  return sfrk<Z>(Ctx{S(s), nullptr}, rfp_desc(n, uplo, transr), trans, k, alpha,
                 V<Z>(a, r, c, rsa, csa), beta, (Z*)arf, hermitian != 0);
}
static int lansf_check(char& norm, char& transr, char& uplo, int64_t n, const double* out) {
  norm = up(norm); transr = up(transr); uplo = up(uplo);
  if (norm == 'O') norm = '1';
  if (norm == 'E') norm = 'F';
  if (!one_of(norm, "M1IF")) return -1;
  if (!one_of(transr, "NTC")) return -2;
  if (!one_of(uplo, "LU")) return -3;
  if (n < 0) return -4;
  if (!out) return -6;
  return 0;
}
int rfpk_dlansf(char norm, char transr, char uplo, int64_t n, const double* arf, double* out, rfpk_stream_t s) { StreamDevice dg_(s);
  if (int rc = lansf_check(norm, transr, uplo, n, out)) return rc;
  return lansf<double>(S(s), rfp_desc(n, uplo, transr), norm, arf, out);
}
int rfpk_zlansf(char norm, char transr, char uplo, int64_t n, const void* arf, double* out, rfpk_stream_t s) { StreamDevice dg_(s);
  if (int rc = lansf_check(norm, transr, uplo, n, out)) return rc;
  return lansf<Z>(S(s), rfp_desc(n, uplo, transr), norm, (const Z*)arf, out);
}

// ---------------------------------------------------------------- dense kernels
int rfpk_dgemm(char ta, char tb, double alpha, const double* a, int64_t ar, int64_t ac, int64_t ars, int64_t acs,
               const double* b, int64_t br, int64_t bc, int64_t brs, int64_t bcs, double beta,
               double* c, int64_t cr, int64_t cc, int64_t crs, int64_t ccs, rfpk_stream_t s) { StreamDevice dg_(s);
  ta = up(ta); tb = up(tb);
  if (!one_of(ta, "NTC")) return -1;
  if (!one_of(tb, "NTC")) return -2;
  if (!unit_stride(ar, ac, ars, acs)) return -4;
  if (!unit_stride(br, bc, brs, bcs)) return -9;
  if (!unit_stride(cr, cc, crs, ccs)) return -15;
  View<double> A = V<double>(a, ar, ac, ars, acs), B = V<double>(b, br, bc, brs, bcs),
               C = V<double>(c, cr, cc, crs, ccs);
  int64_t m = ta == 'N' ? ar : ac, k = ta == 'N' ? ac : ar;
  int64_t kb = tb == 'N' ? br : bc, nn = tb == 'N' ? bc : br;
  if (alpha != 0 && (m != cr || nn != cc || k != kb)) return -4;
  return blas_gemm<double>(Ctx{S(s), nullptr}, ta, tb, alpha, A, B, beta, C);
}
int rfpk_zgemm(char ta, char tb, double are, double aim, const void* a, int64_t ar, int64_t ac, int64_t ars, int64_t acs,
               const void* b, int64_t br, int64_t bc, int64_t brs, int64_t bcs, double bre, double bim,
               void* c, int64_t cr, int64_t cc, int64_t crs, int64_t ccs, rfpk_stream_t s) { StreamDevice dg_(s);
  ta = up(ta); tb = up(tb);
  if (!one_of(ta, "NTC")) return -1;
  if (!one_of(tb, "NTC")) return -2;
  if (!unit_stride(ar, ac, ars, acs)) return -5;
  if (!unit_stride(br, bc, brs, bcs)) return -10;
  if (!unit_stride(cr, cc, crs, ccs)) return -17;
  View<Z> A = V<Z>(a, ar, ac, ars, acs), B = V<Z>(b, br, bc, brs, bcs), C = V<Z>(c, cr, cc, crs, ccs);
  int64_t m = ta == 'N' ? ar : ac, k = ta == 'N' ? ac : ar;
  int64_t kb = tb == 'N' ? br : bc, nn = tb == 'N' ? bc : br;
  if (!(are == 0 && aim == 0) && (m != cr || nn != cc || k != kb)) return -5;
  return blas_gemm<Z>(Ctx{S(s), nullptr}, ta, tb, zc(are, aim), A, B, zc(bre, bim), C);
}

#define TRI_ARGS_CHECK()                          \
  side = up(side); uplo = up(uplo); trans = up(trans); diag = up(diag); \
  if (!one_of(side, "LR")) return -1;             \
  if (!one_of(uplo, "LU")) return -2;             \
  if (!one_of(trans, "NTC")) return -3;           \
  if (!one_of(diag, "NU")) return -4;             \
  if (!unit_stride(an, an, ars, acs)) return -6;  \
  if (!unit_stride(br, bc, brs, bcs)) return -10; \
  if ((side == 'L' ? br : bc) != an) return -7;

int rfpk_dtrsm(char side, char uplo, char trans, char diag, double alpha, const double* a, int64_t an, int64_t ars, int64_t acs,
               double* b, int64_t br, int64_t bc, int64_t brs, int64_t bcs, int* info, rfpk_stream_t s) { StreamDevice dg_(s);
  TRI_ARGS_CHECK();
  if (int rc = reset_info(info, S(s))) return rc;
  return blas_trsm<double>(Ctx{S(s), info}, side, uplo, trans, diag, alpha, V<double>(a, an, an, ars, acs),
                           V<double>(b, br, bc, brs, bcs), info != nullptr);
}
int rfpk_ztrsm(char side, char uplo, char trans, char diag, double are, double aim, const void* a, int64_t an, int64_t ars, int64_t acs,
               void* b, int64_t br, int64_t bc, int64_t brs, int64_t bcs, int* info, rfpk_stream_t s) { StreamDevice dg_(s);
  TRI_ARGS_CHECK();
  if (int rc = reset_info(info, S(s))) return rc;
  return blas_trsm<Z>(Ctx{S(s), info}, side, uplo, trans, diag, zc(are, aim), V<Z>(a, an, an, ars, acs),
                      V<Z>(b, br, bc, brs, bcs), info != nullptr);
}
int rfpk_dtrmm(char side, char uplo, char trans, char diag, double alpha, const double* a, int64_t an, int64_t ars, int64_t acs,
               double* b, int64_t br, int64_t bc, int64_t brs, int64_t bcs, rfpk_stream_t s) { StreamDevice dg_(s);
  TRI_ARGS_CHECK();
  return blas_trmm<double>(Ctx{S(s), nullptr}, side, uplo, trans, diag, alpha, V<double>(a, an, an, ars, acs),
                           V<double>(b, br, bc, brs, bcs));
}
int rfpk_ztrmm(char side, char uplo, char trans, char diag, double are, double aim, const void* a, int64_t an, int64_t ars, int64_t acs,
               void* b, int64_t br, int64_t bc, int64_t brs, int64_t bcs, rfpk_stream_t s) { StreamDevice dg_(s);
  TRI_ARGS_CHECK();
  return blas_trmm<Z>(Ctx{S(s), nullptr}, side, uplo, trans, diag, zc(are, aim), V<Z>(a, an, an, ars, acs),
                      V<Z>(b, br, bc, brs, bcs));
}
int rfpk_dsyrk(char uplo, char trans, double alpha, const double* a, int64_t ar, int64_t ac, int64_t ars, int64_t acs,
               double beta, double* c, int64_t cn, int64_t crs, int64_t ccs, rfpk_stream_t s) { StreamDevice dg_(s);
  uplo = up(uplo); trans = up(trans);
  if (!one_of(uplo, "LU")) return -1;
  if (!one_of(trans, "NTC")) return -2;
  if (!unit_stride(ar, ac, ars, acs)) return -4;
  if (!unit_stride(cn, cn, crs, ccs)) return -10;
  if (alpha != 0 && (trans == 'N' ? ar : ac) != cn) return -4;
  return blas_syrk<double>(Ctx{S(s), nullptr}, uplo, trans, alpha, V<double>(a, ar, ac, ars, acs), beta,
                           V<double>(c, cn, cn, crs, ccs), false);
}
int rfpk_zsyrk(char uplo, char trans, double alpha, const void* a, int64_t ar, int64_t ac, int64_t ars, int64_t acs,
               double beta, void* c, int64_t cn, int64_t crs, int64_t ccs, int hermitian, rfpk_stream_t s) { StreamDevice dg_(s);
  uplo = up(uplo); trans = up(trans);
  if (!one_of(uplo, "LU")) return -1;
  if (!one_of(trans, "NTC")) return -2;
  if (!unit_stride(ar, ac, ars, acs)) return -4;
  if (!unit_stride(cn, cn, crs, ccs)) return -10;
  if (alpha != 0 && (trans == 'N' ? ar : ac) != cn) return -4;
  return blas_syrk<Z>(Ctx{S(s), nullptr}, uplo, trans, alpha, V<Z>(a, ar, ac, ars, acs), beta,
                      V<Z>(c, cn, cn, crs, ccs), hermitian != 0);
}
int rfpk_dpotrf(char uplo, double* a, int64_t n, int64_t rs, int64_t cs, int* info, rfpk_stream_t s) { StreamDevice dg_(s);
  uplo = up(uplo);
  if (!one_of(uplo, "LU")) return -1;
  if (!unit_stride(n, n, rs, cs)) return -4;
  if (!info) return -6;
  if (int rc = reset_info(info, S(s))) return rc;
  return blas_potrf<double>(Ctx{S(s), info}, uplo, V<double>(a, n, n, rs, cs), 0);
}
int rfpk_zpotrf(char uplo, void* a, int64_t n, int64_t rs, int64_t cs, int* info, rfpk_stream_t s) { StreamDevice dg_(s);
  uplo = up(uplo);
  if (!one_of(uplo, "LU")) return -1;
  if (!unit_stride(n, n, rs, cs)) return -4;
  if (!info) return -6;
  if (int rc = reset_info(info, S(s))) return rc;
  return blas_potrf<Z>(Ctx{S(s), info}, uplo, V<Z>(a, n, n, rs, cs), 0);
}
int rfpk_dtrtri(char uplo, char diag, double* a, int64_t n, int64_t rs, int64_t cs, int* info, rfpk_stream_t s) { StreamDevice dg_(s);
  uplo = up(uplo); diag = up(diag);
  if (!one_of(uplo, "LU")) return -1;
  if (!one_of(diag, "NU")) return -2;
  if (!unit_stride(n, n, rs, cs)) return -5;
  if (!info) return -7;
  if (int rc = reset_info(info, S(s))) return rc;
  return blas_trtri<double>(Ctx{S(s), info}, uplo, diag, V<double>(a, n, n, rs, cs), 0);
}
int rfpk_ztrtri(char uplo, char diag, void* a, int64_t n, int64_t rs, int64_t cs, int* info, rfpk_stream_t s) { StreamDevice dg_(s);
  uplo = up(uplo); diag = up(diag);
  if (!one_of(uplo, "LU")) return -1;
  if (!one_of(diag, "NU")) return -2;
  if (!unit_stride(n, n, rs, cs)) return -5;
  if (!info) return -7;
  if (int rc = reset_info(info, S(s))) return rc;
  return blas_trtri<Z>(Ctx{S(s), info}, uplo, diag, V<Z>(a, n, n, rs, cs), 0);
}
int rfpk_dlauum(char uplo, double* a, int64_t n, int64_t rs, int64_t cs, rfpk_stream_t s) { StreamDevice dg_(s);
  uplo = up(uplo);
  if (!one_of(uplo, "LU")) return -1;
  if (!unit_stride(n, n, rs, cs)) return -4;
  return blas_lauum<double>(Ctx{S(s), nullptr}, uplo, V<double>(a, n, n, rs, cs));
}
int rfpk_zlauum(char uplo, void* a, int64_t n, int64_t rs, int64_t cs, rfpk_stream_t s) { StreamDevice dg_(s);
  uplo = up(uplo);
  if (!one_of(uplo, "LU")) return -1;
  if (!unit_stride(n, n, rs, cs)) return -4;
  return blas_lauum<Z>(Ctx{S(s), nullptr}, uplo, V<Z>(a, n, n, rs, cs));
}

}  // extern "C"
