// clock64 timing of the 64x64x64 shared-memory DMMA product used on the
// tile-Cholesky critical path (smem_mm_yh pattern), one CTA of 128 threads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//      -I../paper_0901_1696_b200/csrc -o mmbench mmbench.cu
#include <cstdio>
#include "dmma.cuh"
#include "leaf.cuh"
using namespace rfpk;

template <int LDX>
__device__ __forceinline__ void mm_yh(const double* X, const double* Y, double (&acc)[2][4][4]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp & 1, wn = warp >> 1, g = lane >> 2, t = lane & 3;
#pragma unroll 4
  for (int k = 0; k < 64; k += 4) {
    double a[2][2], b[4];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      a[mi][0] = X[(wm * 32 + mi * 16 + g) + (k + t) * LDX];
      a[mi][1] = X[(wm * 32 + mi * 16 + g + 8) + (k + t) * LDX];
    }
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = Y[(wn * 32 + ni * 8 + g) + (k + t) * LDX];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma16x8x4(acc[mi][ni], a[mi][0], a[mi][1], b[ni]);
  }
}

template <int LDX>
__global__ void bench(double* out, long long* tick) {
  __shared__ double X[64 * LDX];
  double* Y = X;
  for (int e = threadIdx.x; e < 64 * LDX; e += 128) X[e] = e * 1e-3;
  __syncthreads();
  double acc[2][4][4] = {};
  long long t0 = clock64();
  for (int rep = 0; rep < 10; ++rep) mm_yh<LDX>(X, Y, acc);
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int mi = 0; mi < 2; ++mi) for (int ni = 0; ni < 4; ++ni) for (int r = 0; r < 4; ++r) s += acc[mi][ni][r];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) tick[0] = (t1 - t0) / 10;
}
int main() {
  double* o; long long* t; cudaMallocManaged(&o, 128 * 8); cudaMallocManaged(&t, 8);
  bench<65><<<1, 128>>>(o, t); cudaDeviceSynchronize();
  bench<65><<<1, 128>>>(o, t); cudaDeviceSynchronize(); printf("LD 65: %lld cycles per 64^3\n", t[0]);
  bench<68><<<1, 128>>>(o, t); cudaDeviceSynchronize();
  bench<68><<<1, 128>>>(o, t); cudaDeviceSynchronize(); printf("LD 68: %lld cycles per 64^3\n", t[0]);
  bench<72><<<1, 128>>>(o, t); cudaDeviceSynchronize();
  bench<72><<<1, 128>>>(o, t); cudaDeviceSynchronize(); printf("LD 72: %lld cycles per 64^3\n", t[0]);
}
