// Common device/host definitions for the B200 RFPF library.
//
// Every matrix operand is a strided *view* into a caller-owned device
// buffer: element (i, j) of an m x n view lives at p[i*rs + j*cs].  RFP
// blocks T1/T2/S1 are such views of the flat RFP buffer (normal layout:
// rs = 1, cs = ldar; transposed layout: rs = n1, cs = 1), which is how the
// reference addresses them too (convert.py:76-87, 142-153).  All kernels
// require one of the two strides to be 1 (column- or row-major view).
#pragma once

#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdio>

namespace rfpk {

using i64 = long long;

// ---------------------------------------------------------------- scalars
struct Z {  // complex128, interleaved (re, im) -- numpy/torch complex128 layout
  double x, y;
};

template <typename T> struct is_cplx { static constexpr bool value = false; };
template <> struct is_cplx<Z> { static constexpr bool value = true; };

__host__ __device__ __forceinline__ double sc_re(double a) { return a; }
__host__ __device__ __forceinline__ double sc_re(Z a) { return a.x; }
__host__ __device__ __forceinline__ double conj_(double a) { return a; }
__host__ __device__ __forceinline__ Z conj_(Z a) { return Z{a.x, -a.y}; }
__host__ __device__ __forceinline__ double cj(double a, bool c) { return a; }
__host__ __device__ __forceinline__ Z cj(Z a, bool c) { return c ? Z{a.x, -a.y} : a; }
__host__ __device__ __forceinline__ Z operator+(Z a, Z b) { return Z{a.x + b.x, a.y + b.y}; }
__host__ __device__ __forceinline__ Z operator-(Z a, Z b) { return Z{a.x - b.x, a.y - b.y}; }
__host__ __device__ __forceinline__ Z operator-(Z a) { return Z{-a.x, -a.y}; }
__host__ __device__ __forceinline__ Z operator*(Z a, Z b) {
  return Z{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
__host__ __device__ __forceinline__ Z operator*(double s, Z b) { return Z{s * b.x, s * b.y}; }
__host__ __device__ __forceinline__ Z operator/(Z a, Z b) {
  // numpy-compatible complex division (Smith's algorithm is what numpy uses)
  double ar = fabs(b.x), ai = fabs(b.y);
  if (ar >= ai) {
    if (ar == 0 && ai == 0) return Z{a.x / ar, a.y / ai};
    double r = b.y / b.x, den = b.x + b.y * r;
    return Z{(a.x + a.y * r) / den, (a.y - a.x * r) / den};
  }
  double r = b.x / b.y, den = b.y + b.x * r;
  return Z{(a.x * r + a.y) / den, (a.y * r - a.x) / den};
}
__host__ __device__ __forceinline__ Z operator/(Z a, double s) { return Z{a.x / s, a.y / s}; }
__host__ __device__ __forceinline__ bool is_zero(double a) { return a == 0.0; }
__host__ __device__ __forceinline__ bool is_zero(Z a) { return a.x == 0.0 && a.y == 0.0; }
template <typename T> __host__ __device__ __forceinline__ T sc_from(double v);
template <> __host__ __device__ __forceinline__ double sc_from<double>(double v) { return v; }
template <> __host__ __device__ __forceinline__ Z sc_from<Z>(double v) { return Z{v, 0.0}; }
// a*b + c  with a, b, c scalars (complex: 4 real FMAs)
__device__ __forceinline__ double fmac(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ Z fmac(Z a, Z b, Z c) {
  return Z{fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y))};
}
// c - a*b
__device__ __forceinline__ double fnmac(double a, double b, double c) { return fma(-a, b, c); }
__device__ __forceinline__ Z fnmac(Z a, Z b, Z c) {
  return Z{fma(-a.x, b.x, fma(a.y, b.y, c.x)), fma(-a.x, b.y, fma(-a.y, b.x, c.y))};
}

// 1/sqrt(x) for a Cholesky pivot x > 0 (normal): the MUFU seed
// (rsqrt.approx.f64) and one cubic Newton step, y (1 + e/2 + 3e^2/8) with
// e = 1 - x y^2 -- the seed's error cubed, below double rounding.  No range
// checks: a pivot that is not > 0 is reported before its rsqrt is used (the
// library's rsqrt() spends ~12 instructions on those checks, on the serial
// chain of every pivot).
__device__ __forceinline__ double rsqrt_pivot(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  // (four dependent FP64 operations after the seed: y^2 | e | {3e/8 + 1/2,
  // y e} | the sum -- this value heads the serial chain of every pivot)
  const double e = fma(-x, y * y, 1.0);
  return fma(y * e, fma(0.375, e, 0.5), y);
}

// CTA barrier for code where single threads run the flag protocol (spins,
// atomics, releases) or record failures: __syncthreads() is bar.sync, an
// .aligned barrier that a warp must reach CONVERGED, and under independent
// thread scheduling the compiler does not always reconverge a warp after a
// thread-0-only block (measured: one thread-0 store ahead of a task's first
// barrier let the warp's other lanes run a barrier ahead of lane 0 and read
// a tile before lane 0 had acquired its flag).  Reconverge first.
__device__ __forceinline__ void cta_sync() {
  __syncwarp();
  __syncthreads();
}

// ---------------------------------------------------------------- views
template <typename T> struct View {
  T* p;
  i64 m, n, rs, cs;
  __host__ __device__ T* at(i64 i, i64 j) const { return p + i * rs + j * cs; }
  __host__ __device__ View t() const { return View{p, n, m, cs, rs}; }
  __host__ __device__ View sub(i64 i0, i64 j0, i64 mm, i64 nn) const {
    return View{p + i0 * rs + j0 * cs, mm, nn, rs, cs};
  }
  __host__ __device__ bool empty() const { return m <= 0 || n <= 0; }
  // column-major if rs == 1 (or degenerate), row-major if cs == 1
  __host__ bool colmajor() const { return rs == 1 || (m == 1 && cs != 1); }
};

// ---------------------------------------------------------------- errors
// Every kernel launch site ends with RFPK_CHECK_LAUNCH, which also counts the
// launch (exported as rfpk_launch_count() so benchmarks can report how many
// of the library's kernels ran).
extern std::atomic<long long> g_launch_count;
#define RFPK_CHECK_LAUNCH()                                                   \
  do {                                                                        \
    g_launch_count.fetch_add(1, std::memory_order_relaxed);                   \
    cudaError_t e_ = cudaGetLastError();                                      \
    if (e_ != cudaSuccess) {                                                  \
      fprintf(stderr, "rfpk: launch failed %s at %s:%d\n",                    \
              cudaGetErrorString(e_), __FILE__, __LINE__);                    \
      return (int)e_;                                                         \
    }                                                                         \
  } while (0)

// status codes returned by the internal drivers (>0: CUDA error codes)
enum { RFPK_OK = 0 };

// ---------------------------------------------------------------- enums
enum Uplo : int { LOWER = 0, UPPER = 1 };
enum TriMode : int { TRI_FULL = 0, TRI_LOWER = 1, TRI_UPPER = 2 };

inline int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

constexpr int MAX_DEVICES = 64;

// SM count of the CURRENT device (cached per device)
inline int num_sms() {
  static std::atomic<int> sms[MAX_DEVICES];
  const int dev = cur_device() & (MAX_DEVICES - 1);
  int v = sms[dev].load(std::memory_order_relaxed);
  if (!v) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
    sms[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

// One-time per-(kernel, device) configuration: opts the kernel into `smem`
// bytes of dynamic shared memory ON THE CURRENT DEVICE (function attributes
// are per device context) and returns its resident CTAs per SM at
// `threads` threads (>= 1).  Defined in capi.cu.
int kernel_setup(const void* kern, int threads, size_t smem);
template <typename K> int kernel_setup(K* kern, int threads, size_t smem) {
  return kernel_setup(reinterpret_cast<const void*>(kern), threads, smem);
}

// Every entry point runs on the device that owns the caller's stream: the
// drivers query the current device (SM count, library streams, kernel
// attributes, graph keys), so a stream of device k is served with device k
// current for the duration of the call, and the caller's current device is
// restored on return.  The default streams (0 / legacy / per-thread) belong
// to the current device already.
struct StreamDevice {
  int prev = -1;
  explicit StreamDevice(void* s) {
    cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
    if (st == nullptr || st == cudaStreamLegacy || st == cudaStreamPerThread) return;
    int dev = -1, cur = -1;
    if (cudaStreamGetDevice(st, &dev) != cudaSuccess) {
      cudaGetLastError();  // leave the error to the launch that uses the stream
      return;
    }
    if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess)
      prev = cur;
  }
  ~StreamDevice() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// ---------------------------------------------------------------- kernel clock
// With the phase clock on (rfpk_phase_clock(1)), a launch site bracketed by
// a KernelClock records a CUDA event pair ON THE STREAM IT LAUNCHES ON and
// files the pair under `label` ("kernel <name> <shape>"); rfpk_phase_time
// sums them.  Nothing is recorded under graph capture or with the clock off.
// Defined in rfp.cu.
struct KernelClock {
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  explicit KernelClock(cudaStream_t s);
  void stop(const char* name, long long d0, long long d1, long long d2 = -1);
};

// ---------------------------------------------------------------- tuning
// Path thresholds, set only through the explicit C-ABI call
// rfpk_set_tuning(name, value) (include/rfpk_b200.h) -- there are no
// environment knobs.  The defaults are the measured crossovers (DESIGN.md
// section 4); tests use the setter to force the alternative paths at small
// orders.  Changing a value drops every cached CUDA graph, so a replay can
// never run a path chosen under the old setting.
enum TuneKey : int {
  TK_OOP_MAX = 0,          // one-launch trmm / lauum / trtri up to this order (4096)
  TK_T2_COPY_MIN,          // column-major workspace potrf of row-major blocks from (2048)
  TK_PANEL_MAX,            // one-launch [T1; S1] panel Cholesky up to n1 (4096)
  TK_PFSV_OVERLAP_MIN,     // pfsv: pftrs part 1 beside potrf(T2) from order (512)
  TK_OVERLAP,              // potrf(T1) || S1 solve as two concurrent launches (1)
  TK_GRAPHS,               // CUDA-graph replay of repeated calls (1)
  TK_GRAPH_MAX_N,          // ... below this order (8192)
  TK_GEMM_WIDE,            // force the 64 x 128 GEMM tile for every product (0)
  TK_BATCHED_GENERIC,      // force the generic batched kernel at n = 64 (0)
  TK_TRACE,                // print per-phase SRPA times to stderr (0)
  TK_TRSM_SPLIT,           // tile trsm: split tasks: 0 off, 1 automatic, > 1 kept chunks (1)
  TK_ZPOTRF_SPLIT_MIN,     // complex potrf: one GEMM-level split from this order (9000)
  TK_COUNT
};
long long tune(TuneKey k);  // defined in capi.cu

}  // namespace rfpk
