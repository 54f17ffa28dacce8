// Dependent-chain latency probes on the B200 (cycles per op, one warp).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_probe lat_probe.cu
#include <cstdio>
__global__ void probe(double* out, long long* t, double x0) {
  __shared__ double sh[64];
  double x = x0 + threadIdx.x * 1e-9;
  long long c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) x = fma(x, 0.999999, 1e-7);
  long long c1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) x = rsqrt(x) + 0.5;
  long long c2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) x = __shfl_sync(0xffffffffu, x, (i + 1) & 31) * 1.0000001;
  long long c3 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
    sh[threadIdx.x] = x;
    __syncwarp();
    x = sh[(threadIdx.x + 1) & 31] * 1.0000001;
    __syncwarp();
  }
  long long c4 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) x = x * 0.999999;
  long long c5 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) x = 1.0 / x;
  long long c6 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { t[0] = c1 - c0; t[1] = c2 - c1; t[2] = c3 - c2; t[3] = c4 - c3; t[4] = c5 - c4; t[5] = c6 - c5; }
}
int main() {
  double* o; long long* t; cudaMallocManaged(&o, 64 * 8); cudaMallocManaged(&t, 64 * 8);
  for (int r = 0; r < 2; ++r) { probe<<<1, 32>>>(o, t, 1.5); cudaDeviceSynchronize(); }
  const char* nm[] = {"dfma", "rsqrt+dadd", "shfl+dmul", "sts/syncwarp/lds+dmul", "dmul", "1/x"};
  for (int i = 0; i < 6; ++i) printf("%-24s %.1f cyc/iter\n", nm[i], t[i] / 256.0);
}
