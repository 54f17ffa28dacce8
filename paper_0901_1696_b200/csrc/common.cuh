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

inline int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

}  // namespace rfpk
