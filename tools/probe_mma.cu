// Probe: verify the assumed register-fragment layouts of the FP64 mma.sync
// shapes on sm_100a (m8n8k4, m16n8k4, m16n8k8, m16n8k16).  One warp; A is
// M x K row-major, B is K x N row-major, D is M x N row-major.
#include <cuda_runtime.h>

extern "C" __global__ void probe_m8n8k4(const double* A, const double* B, double* D) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a = A[g * 4 + t];
  double b = B[t * 8 + g];
  double c0 = 0, c1 = 0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  D[g * 8 + 2 * t] = c0;
  D[g * 8 + 2 * t + 1] = c1;
}

extern "C" __global__ void probe_m16n8k4(const double* A, const double* B, double* D) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a0 = A[g * 4 + t], a1 = A[(g + 8) * 4 + t];
  double b = B[t * 8 + g];
  double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3) : "d"(a0), "d"(a1), "d"(b));
  D[g * 8 + 2 * t] = c0; D[g * 8 + 2 * t + 1] = c1;
  D[(g + 8) * 8 + 2 * t] = c2; D[(g + 8) * 8 + 2 * t + 1] = c3;
}

extern "C" __global__ void probe_m16n8k8(const double* A, const double* B, double* D) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a0 = A[g * 8 + t], a1 = A[(g + 8) * 8 + t], a2 = A[g * 8 + t + 4], a3 = A[(g + 8) * 8 + t + 4];
  double b0 = B[t * 8 + g], b1 = B[(t + 4) * 8 + g];
  double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3) : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  D[g * 8 + 2 * t] = c0; D[g * 8 + 2 * t + 1] = c1;
  D[(g + 8) * 8 + 2 * t] = c2; D[(g + 8) * 8 + 2 * t + 1] = c3;
}

extern "C" __global__ void probe_m16n8k16(const double* A, const double* B, double* D) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = A[(g + 8 * (i & 1)) * 16 + t + 4 * (i >> 1)];
  for (int i = 0; i < 4; ++i) b[i] = B[(t + 4 * i) * 8 + g];
  double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
               : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3)
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  D[g * 8 + 2 * t] = c0; D[g * 8 + 2 * t + 1] = c1;
  D[(g + 8) * 8 + 2 * t] = c2; D[(g + 8) * 8 + 2 * t + 1] = c3;
}

// Throughput probe: each warp runs `iters` iterations of 16 independent m16n8k4 mmas.
extern "C" __global__ void probe_dmma_rate(double* out, int iters) {
  double acc[16][4];
  for (int i = 0; i < 16; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) for (int j = 0; j < 4; ++j) s += acc[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// DFMA throughput probe: 16 independent FMA chains per thread.
extern "C" __global__ void probe_dfma_rate(double* out, int iters) {
  double acc[16];
  double x = threadIdx.x * 1e-3, y = 0.999999;
  for (int i = 0; i < 16; ++i) acc[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], y, x);
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

extern "C" int launch_probe(int which, const double* A, const double* B, double* D) {
  switch (which) {
    case 0: probe_m8n8k4<<<1, 32>>>(A, B, D); break;
    case 1: probe_m16n8k4<<<1, 32>>>(A, B, D); break;
    case 2: probe_m16n8k8<<<1, 32>>>(A, B, D); break;
    case 3: probe_m16n8k16<<<1, 32>>>(A, B, D); break;
  }
  return (int)cudaDeviceSynchronize();
}

extern "C" int launch_rate(int which, double* out, int blocks, int threads, int iters) {
  if (which == 0) probe_dmma_rate<<<blocks, threads>>>(out, iters);
  else probe_dfma_rate<<<blocks, threads>>>(out, iters);
  return (int)cudaGetLastError();
}
