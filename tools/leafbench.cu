// Phase-timed 64-leaf (clock64) to see where the leaf latency goes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//        -I../paper_0901_1696_b200/csrc -shared -Xcompiler -fPIC -o leafbench.so leafbench.cu
#include "leaf.cuh"

using namespace rfpk;

template <typename T>
__global__ void __launch_bounds__(128) leaf_phases(T* A, long long* tick) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* S = reinterpret_cast<T*>(smem_raw);
  T* Ws = S + 64 * LD64;
  T* scr = Ws + 64 * LD64;
  const int warp = threadIdx.x >> 5;
  View<T> v{A, 64, 64, 1, 64};
  long long t0 = clock64();
  leaf_load_lower(S, v, 64);
  __syncthreads();
  long long t1 = clock64();
  if (warp == 0) chol32_warp(S, 0, scr);
  __syncthreads();
  long long t2 = clock64();
  if (warp == 0) inv32_warp(S, 0, Ws, 0, false, scr);
  __syncthreads();
  long long t3 = clock64();
  Frag32<T> f;
  mm32_mma<T, true, true>(S, 32, 0, Ws, 0, 0, f);
  __syncthreads();
  frag32_each(f, [&](int i, int j, T v) { S[(32 + i) + j * LD64] = v; });
  __syncthreads();
  long long t4 = clock64();
  mm32_mma<T, true, true>(S, 32, 0, S, 32, 0, f);
  frag32_each(f, [&](int i, int j, T v) {
    if (j <= i) S[(32 + i) + (32 + j) * LD64] = S[(32 + i) + (32 + j) * LD64] - v;
  });
  __syncthreads();
  long long t5 = clock64();
  if (warp == 0) chol32_warp(S, 32, scr);
  __syncthreads();
  long long t6 = clock64();
  if (warp == 1) inv32_warp(S, 32, Ws, 32, false, scr + 32);
  __syncthreads();
  long long t7 = clock64();
  inv64_block(S, Ws, false, true, scr);
  __syncthreads();
  long long t8 = clock64();
  leaf_store_lower(S, v, 64, false);
  __syncthreads();
  long long t9 = clock64();
  if (threadIdx.x == 0) {
    long long t[] = {t0, t1, t2, t3, t4, t5, t6, t7, t8, t9};
    for (int k = 0; k < 10; ++k) tick[k] = t[k] - t0;
  }
}

extern "C" int run_leaf_phases(int cplx, void* A, long long* tick) {
  size_t sm = (2 * 64 * 65 + 128) * (cplx ? 16 : 8);
  if (cplx) {
    cudaFuncSetAttribute(leaf_phases<Z>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    leaf_phases<Z><<<1, 128, sm>>>((Z*)A, tick);
  } else {
    cudaFuncSetAttribute(leaf_phases<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    leaf_phases<double><<<1, 128, sm>>>((double*)A, tick);
  }
  return (int)cudaDeviceSynchronize();
}

// whole leaf (leaf_factor_inv64) timed, and its result written back for checking
template <typename T>
__global__ void __launch_bounds__(128) leaf_full(T* A, T* Wout, long long* tick) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* S = reinterpret_cast<T*>(smem_raw);
  T* Ws = S + 64 * LD64;
  T* scr = Ws + 64 * LD64;
  __shared__ int fail;
  View<T> v{A, 64, 64, 1, 64};
  leaf_load_lower(S, v, 64);
  __syncthreads();
  long long t0 = clock64();
  int f = leaf_factor_inv64(S, Ws, scr, &fail);
  __syncthreads();
  long long t1 = clock64();
  leaf_store_lower(S, v, 64, false);
  for (int e = threadIdx.x; e < 4096; e += 128) Wout[e] = Ws[(e & 63) + (e >> 6) * LD64];
  if (threadIdx.x == 0) { tick[0] = t1 - t0; tick[1] = f; }
}

extern "C" int run_leaf_full(int cplx, void* A, void* W, long long* tick) {
  size_t sm = (2 * 64 * 65 + 128) * (cplx ? 16 : 8);
  if (cplx) {
    cudaFuncSetAttribute(leaf_full<Z>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    leaf_full<Z><<<1, 128, sm>>>((Z*)A, (Z*)W, tick);
  } else {
    cudaFuncSetAttribute(leaf_full<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    leaf_full<double><<<1, 128, sm>>>((double*)A, (double*)W, tick);
  }
  return (int)cudaDeviceSynchronize();
}

