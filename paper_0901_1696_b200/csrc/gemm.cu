// FP64 / complex128 DMMA GEMM for sm_100a (see gemm.cuh for the contract).
#include "gemm.cuh"
#include "dmma.cuh"

#include <cstdlib>

namespace rfpk {

__device__ __forceinline__ void tri_tile(int mode, long long b, int& tm, int& tn) {
  // b enumerates the tiles (ti >= tj) of a lower-triangular tile grid
  int ti = (int)((sqrt(8.0 * (double)b + 1.0) - 1.0) * 0.5);
  while ((long long)(ti + 1) * (ti + 2) / 2 <= b) ++ti;
  while ((long long)ti * (ti + 1) / 2 > b) --ti;
  int tj = (int)(b - (long long)ti * (ti + 1) / 2);
  if (mode == TRI_LOWER) { tm = ti; tn = tj; } else { tm = tj; tn = ti; }
}

// Banded order of the same lower-triangular tile grid: bands of H tile rows,
// each band walked column by column (the H tiles of a column, then the next
// column; the band's own triangle last).  The tiles resident at one time
// then share ~H row panels and ~(resident / H) column panels instead of a
// few rows and every column panel up to them, so the operand panels they
// stream stay in L2 (SYRK T2 -= S1 S1^T at n = 16384, ncu: DRAM reads per
// launch 20.6 GB row by row -> 7.05 GB at H = 24, 17.12 -> 16.73 ms; H = 16
// and 32 measured the same time).  RFPK_TRI_BAND = H (0: row by row).
__device__ __forceinline__ void tri_tile_banded(int mode, long long b, int tiles, int H, int& tm,
                                                int& tn) {
  int r0 = 0;
  for (;;) {  // band starting at tile row r0: h full columns of r0 tiles + its triangle
    const int h = tiles - r0 < H ? tiles - r0 : H;
    const long long cnt = (long long)r0 * h + (long long)h * (h + 1) / 2;
    if (b < cnt) {
      int ti, tj;
      if (b < (long long)r0 * h) {
        tj = (int)(b / h);
        ti = r0 + (int)(b % h);
      } else {
        long long o = b - (long long)r0 * h;
        tj = r0;
        while (o >= r0 + h - tj) {
          o -= r0 + h - tj;
          ++tj;
        }
        ti = tj + (int)o;
      }
      if (mode == TRI_LOWER) { tm = ti; tn = tj; } else { tm = tj; tn = ti; }
      return;
    }
    b -= cnt;
    r0 += h;
  }
}

// the same for BM x BN tiles with BN a multiple of BM (64 x 128): column tile
// tn spans rows tiles from (TRI_LOWER) BN/BM*tn, or up to (TRI_UPPER)
// BN/BM*(tn+1)-1; scanned column by column (<= tiles_n steps per CTA)
template <int BM, int BN>
__host__ __device__ inline long long tri_rect_count(int mode, int tn, int tiles_m) {
  constexpr int R = BN / BM;
  if (mode == TRI_LOWER) return tiles_m > R * tn ? tiles_m - R * tn : 0;
  return R * (tn + 1) < tiles_m ? R * (tn + 1) : tiles_m;
}
template <int BM, int BN>
__device__ __forceinline__ void tri_tile_rect(int mode, long long b, int tiles_m, int& tm, int& tn) {
  constexpr int R = BN / BM;
  tn = 0;
  for (;;) {
    const long long c = tri_rect_count<BM, BN>(mode, tn, tiles_m);
    if (b < c) break;
    b -= c;
    ++tn;
  }
  tm = (mode == TRI_LOWER ? R * tn : 0) + (int)b;
}

__device__ __forceinline__ bool tri_keep(int mode, int row, int col) {
  return mode == TRI_FULL || (mode == TRI_LOWER ? row >= col : row <= col);
}

// ------------------------------------------------------------ kernel
// One CTA computes a BM x BN tile of C with (BM/WM) x (BN/WN) warps; each warp
// a WM x WN sub-tile of m16n8k4 DMMA fragments.  Real: one DMMA per fragment
// pair.  Complex: 4 real DMMAs (Re += Ar Br - Ai Bi, Im += Ar Bi + Ai Br),
// conjugation by sign flips.  Padded smem rows (P = BM + 4 real / + 2 complex)
// make the fragment loads bank-conflict free.
template <typename T, int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BKM, int MODE>
__device__ __forceinline__ void gemm_tile(const GemmArgs<T>& g, int tm, int tn, T* As, T* Bs) {
  constexpr bool CPLX = is_cplx<T>::value;
  constexpr int WARPS_M = BM / WM;
  constexpr int NT = WARPS_M * (BN / WN) * 32;
  using LA = SmemLayout<T, BM, BK, AK>;
  using LB = SmemLayout<T, BN, BK, BKM>;
  constexpr int MI = WM / 16, NI = WN / 8;
  constexpr int NACC = CPLX ? 2 : 1;
  const int m0 = tm * BM, n0 = tn * BN;
  const int M = g.M, N = g.N, K = g.K;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % WARPS_M, wn = warp / WARPS_M;
  const int gq = lane >> 2, tq = lane & 3;

  TileLoader<T, BM, BK, NT, AK> la;
  TileLoader<T, BN, BK, NT, BKM> lb;
  la.init(g.A, g.lda, m0, M, tid);
  lb.init(g.B, g.ldb, n0, N, tid);
  const bool masked = (g.a_tri != A_FULL && g.a_tri != A_UBAND) ||
                      (g.b_tri != A_FULL && g.b_tri != A_UBAND);
  // a triangular operand is zero outside a band of K for this tile: lower
  // (k <= row) ends the K loop at the tile's last row, upper (k >= row)
  // starts it at the tile's first -- half the flops of a masked trmm GEMM
  int kbeg = 0, kend = g.K;
  if (g.a_tri == A_LOWER || g.a_tri == A_SLOWER) kend = min(kend, m0 + BM);
  if (g.a_tri == A_UPPER || g.a_tri == A_SUPPER || g.a_tri == A_UBAND) kbeg = max(kbeg, m0);
  if (g.b_tri == A_LOWER || g.b_tri == A_SLOWER) kend = min(kend, n0 + BN);
  if (g.b_tri == A_UPPER || g.b_tri == A_SUPPER || g.b_tri == A_UBAND) kbeg = max(kbeg, n0);
  const int kt0 = kbeg / BK;
  la.skip(kt0);
  lb.skip(kt0);

  double acc[NACC][MI][NI][4];
#pragma unroll
  for (int c = 0; c < NACC; ++c)
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[c][i][j][r] = 0.0;

  const int KT = kend > kbeg ? (kend + BK - 1) / BK - kt0 : 0;  // stages of this tile
  auto load_stage = [&](int stage, int kt) {  // kt counts from kt0
    T* as = As + stage * LA::SIZE;
    T* bs = Bs + stage * LB::SIZE;
    const int k0 = (kt + kt0) * BK;
    if (!masked && k0 + BK <= K) {  // uniform
      la.load(as);
      lb.load(bs);
    } else {
      la.load_pred(as, k0, K, m0, g.a_tri);
      lb.load_pred(bs, k0, K, n0, g.b_tri);
    }
    la.advance();
    lb.advance();
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_async_commit();
  }
  const double sa = (CPLX && g.conjA) ? -1.0 : 1.0, sb = (CPLX && g.conjB) ? -1.0 : 1.0;
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nk = kt + STAGES - 1;
    if (nk < KT) load_stage(nk % STAGES, nk);
    cp_async_commit();
    const T* as = As + (kt % STAGES) * LA::SIZE + (wm * WM + gq) * LA::RS + tq * LA::KS;
    const T* bs = Bs + (kt % STAGES) * LB::SIZE + (wn * WN + gq) * LB::RS + tq * LB::KS;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      if constexpr (!CPLX) {
        double af[MI][2], bf[NI];
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          af[i][0] = as[kk * LA::KS + (i * 16) * LA::RS];
          af[i][1] = as[kk * LA::KS + (i * 16 + 8) * LA::RS];
        }
#pragma unroll
        for (int j = 0; j < NI; ++j) bf[j] = bs[kk * LB::KS + (j * 8) * LB::RS];
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NI; ++j) dmma16x8x4(acc[0][i][j], af[i][0], af[i][1], bf[j]);
      } else {
        double ar[MI][2], ai[MI][2], nai[MI][2], br[NI], bi[NI];
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const Z v0 = as[kk * LA::KS + (i * 16) * LA::RS];
          const Z v1 = as[kk * LA::KS + (i * 16 + 8) * LA::RS];
          ar[i][0] = v0.x; ai[i][0] = sa * v0.y;
          ar[i][1] = v1.x; ai[i][1] = sa * v1.y;
          nai[i][0] = -ai[i][0]; nai[i][1] = -ai[i][1];
        }
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          const Z w = bs[kk * LB::KS + (j * 8) * LB::RS];
          br[j] = w.x; bi[j] = sb * w.y;
        }
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NI; ++j) {
            dmma16x8x4(acc[0][i][j], ar[i][0], ar[i][1], br[j]);
            dmma16x8x4(acc[0][i][j], nai[i][0], nai[i][1], bi[j]);
            dmma16x8x4(acc[1][i][j], ar[i][0], ar[i][1], bi[j]);
            dmma16x8x4(acc[1][i][j], ai[i][0], ai[i][1], br[j]);
          }
      }
    }
  }
  cp_async_wait<0>();

  const T alpha = g.alpha, beta = g.beta;
  const bool use_beta = !is_zero(beta);
  // Epilogue, one MI row-block at a time: all C loads of the block are issued
  // before any store (so their latencies overlap), then alpha/beta are
  // applied and the triangle-masked stores issued.
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    T cv[NI][4];
#pragma unroll
    for (int j = 0; j < NI; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int row = m0 + wm * WM + i * 16 + gq + ((r & 2) ? 8 : 0);
        const int col = n0 + wn * WN + j * 8 + 2 * tq + (r & 1);
        cv[j][r] = (use_beta && row < M && col < N && tri_keep(MODE, row, col))
                       ? g.C[row + (i64)col * g.ldc]
                       : sc_from<T>(0.0);
      }
#pragma unroll
    for (int j = 0; j < NI; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int row = m0 + wm * WM + i * 16 + gq + ((r & 2) ? 8 : 0);
        const int col = n0 + wn * WN + j * 8 + 2 * tq + (r & 1);
        if (row < M && col < N && tri_keep(MODE, row, col)) {
          T* c = g.C + row + (i64)col * g.ldc;
          if constexpr (!CPLX) {
            double v = alpha * acc[0][i][j][r];
            if (use_beta) v = fma(beta, cv[j][r], v);
            *c = v;
          } else {
            Z v = alpha * Z{acc[0][i][j][r], acc[1][i][j][r]};
            if (use_beta) v = v + beta * cv[j][r];
            if (MODE != TRI_FULL && g.herm_diag && row == col) v.y = 0.0;
            *c = v;
          }
        }
      }
  }
}

template <typename T, int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BKM, int MODE>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32,
                                  (BM * BN <= 64 * 64) ? (is_cplx<T>::value ? 2 : (STAGES <= 3 ? 4 : 3)) : 1)
    gemm_kernel(GemmArgs<T> g) {
  using LA = SmemLayout<T, BM, BK, AK>;
  extern __shared__ __align__(16) double smem_d[];
  T* As = reinterpret_cast<T*>(smem_d);
  T* Bs = As + STAGES * LA::SIZE;
  if (g.skip && *g.skip) return;
  for (long long t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
    int tm, tn;
    if (MODE == TRI_FULL) {
      if (g.band > 0) {  // bands of g.band tile rows, column by column inside a band
        const int tiles_n = (g.N + BN - 1) / BN;
        const long long per = (long long)g.band * tiles_n;
        const int b = (int)(t / per), r0 = b * g.band;
        const int h = g.tiles_m - r0 < g.band ? g.tiles_m - r0 : g.band;
        const long long o = t - (long long)b * per;
        tn = (int)(o / h);
        tm = r0 + (int)(o % h);
      } else {
        tm = (int)(t % g.tiles_m);
        tn = (int)(t / g.tiles_m);
      }
    }
    else if constexpr (BM == BN) {
      if (g.band > 0) tri_tile_banded(MODE, t, g.tiles_m, g.band, tm, tn);
      else tri_tile(MODE, t, tm, tn);
    }
    else tri_tile_rect<BM, BN>(MODE, t, g.tiles_m, tm, tn);
    gemm_tile<T, BM, BN, BK, WM, WN, STAGES, AK, BKM, MODE>(g, tm, tn, As, Bs);
    if (t + gridDim.x < g.ntiles) __syncthreads();  // smem stages are reused
  }
}

// ------------------------------------------------------------ split-K
// Few output tiles and a long K (pftrs' C = B2 -= S1 B1 at nrhs = 64: 32
// tiles, K = 2000): split K into S slices, one CTA per (tile, slice) writes
// its partial product to a workspace, and a second kernel sums the slices in
// a fixed order -- deterministic, unlike atomics.
template <typename T, int BM, int BN, int BK, int WM, int WN, int STAGES, bool AK, bool BKM>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * 32, 4)
    gemm_splitk_kernel(GemmArgs<T> g, T* ws, int kchunk) {
  using LA = SmemLayout<T, BM, BK, AK>;
  extern __shared__ __align__(16) double smem_d[];
  T* As = reinterpret_cast<T*>(smem_d);
  T* Bs = As + STAGES * LA::SIZE;
  if (g.skip && *g.skip) return;
  const int s = blockIdx.y;
  const int k0 = s * kchunk;
  GemmArgs<T> p = g;
  p.K = g.K - k0 < kchunk ? g.K - k0 : kchunk;
  p.A = g.A + (AK ? (i64)k0 : (i64)k0 * g.lda);
  p.B = g.B + (BKM ? (i64)k0 : (i64)k0 * g.ldb);
  p.C = ws + (i64)s * g.M * g.N;
  p.ldc = g.M;
  p.alpha = sc_from<T>(1.0);
  p.beta = sc_from<T>(0.0);
  const int tm = (int)(blockIdx.x % g.tiles_m), tn = (int)(blockIdx.x / g.tiles_m);
  gemm_tile<T, BM, BN, BK, WM, WN, STAGES, AK, BKM, TRI_FULL>(p, tm, tn, As, Bs);
}

template <typename T>
__global__ void splitk_reduce_kernel(GemmArgs<T> g, const T* ws, int S) {
  if (g.skip && *g.skip) return;
  const i64 total = (i64)g.M * g.N;
  const bool use_beta = !is_zero(g.beta);
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total;
       e += (i64)gridDim.x * blockDim.x) {
    T acc = ws[e];
    for (int s = 1; s < S; ++s) acc = acc + ws[(i64)s * total + e];
    const i64 i = e % g.M, j = e / g.M;
    T* c = g.C + i + j * g.ldc;
    T v = g.alpha * acc;
    if (use_beta) v = v + g.beta * (*c);
    *c = v;
  }
}

// ------------------------------------------------------------ scale kernel
template <typename T>
__global__ void scale_kernel(View<T> C, T beta, int mode, int herm_diag, const int* skip) {
  if (skip && *skip) return;
  i64 total = C.m * C.n;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total;
       e += (i64)gridDim.x * blockDim.x) {
    i64 i = e % C.m, j = e / C.m;
    if (!tri_keep(mode, (int)i, (int)j)) continue;
    T* c = C.at(i, j);
    T v = is_zero(beta) ? sc_from<T>(0.0) : beta * (*c);
    if constexpr (is_cplx<T>::value) {
      if (herm_diag && i == j) v.y = 0.0;
    }
    *c = v;
  }
}

template <typename T>
int scale_view(View<T> C, T beta, int tri_mode, bool herm_diag, const int* skip, cudaStream_t st) {
  if (C.empty()) return 0;
  i64 total = C.m * C.n;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 4 * num_sms()) blocks = 4 * num_sms();
  scale_kernel<T><<<blocks, 256, 0, st>>>(C, beta, tri_mode, herm_diag ? 1 : 0, skip);
  RFPK_CHECK_LAUNCH();
  return 0;
}

// elementwise conjugation of a complex view (no-op launch for real)
template <typename T> __global__ void conj_kernel(View<T> C, const int* skip) {
  if (skip && *skip) return;
  const i64 total = C.m * C.n;
  for (i64 e = blockIdx.x * (i64)blockDim.x + threadIdx.x; e < total;
       e += (i64)gridDim.x * blockDim.x) {
    T* c = C.at(e % C.m, e / C.m);
    *c = conj_(*c);
  }
}

template <typename T> int conj_view(View<T> C, const int* skip, cudaStream_t st) {
  if (!is_cplx<T>::value || C.empty()) return 0;
  i64 total = C.m * C.n;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 4 * num_sms()) blocks = 4 * num_sms();
  conj_kernel<T><<<blocks, 256, 0, st>>>(C, skip);
  RFPK_CHECK_LAUNCH();
  return 0;
}

// ------------------------------------------------------------ dispatch
namespace {

struct OperandLayout {
  bool kmajor;  // contiguous along K
  i64 ld;
  bool ok;
};

// A is an M x K view (or B a K x N view, passed transposed as N x K): report
// whether it is contiguous along its first dim (MN-major) or its second (K).
template <typename T> OperandLayout classify(const View<T>& v) {
  if (v.rs == 1 || v.m == 1) {
    i64 ld = (v.n == 1) ? (v.m > 0 ? v.m : 1) : v.cs;
    return {false, ld, true};
  }
  if (v.cs == 1 || v.n == 1) {
    i64 ld = (v.m == 1) ? (v.n > 0 ? v.n : 1) : v.rs;
    return {true, ld, true};
  }
  return {false, 0, false};
}

template <typename T, int BM, int BN, int BK, int WM, int WN, int ST, bool AK, bool BKM, int MODE>
int launch_one(const GemmArgs<T>& a, cudaStream_t st) {
  constexpr int NT = (BM / WM) * (BN / WN) * 32;
  constexpr size_t smem = (size_t)ST *
                          (SmemLayout<T, BM, BK, AK>::SIZE + SmemLayout<T, BN, BK, BKM>::SIZE) *
                          sizeof(T);
  auto kern = gemm_kernel<T, BM, BN, BK, WM, WN, ST, AK, BKM, MODE>;
  kernel_setup(kern, NT, smem);
  const int tm = (a.M + BM - 1) / BM, tn = (a.N + BN - 1) / BN;
  GemmArgs<T> g = a;
  g.tiles_m = tm;
  constexpr int band = 24, full_band = 24;  // tile rows per band (see GemmArgs::band)
  // full products: banded only when C is narrow (few column tiles, e.g.
  // pftrs's 8192 x 1024 gemms: 32.0 -> 33.0 TFLOP/s, A streamed from DRAM once
  // instead of once per resident column group); square products keep the
  // column-major order (8192^3: 33.9 vs 33.5 TFLOP/s banded)
  g.band = MODE == TRI_FULL ? (tn <= 32 ? full_band : 0) : band;
  if (MODE == TRI_FULL) {
    g.ntiles = (long long)tm * tn;
  } else if (BM == BN) {
    g.ntiles = (long long)tm * (tm + 1) / 2;
  } else {
    g.ntiles = 0;
    for (int j = 0; j < tn; ++j) g.ntiles += tri_rect_count<BM, BN>(MODE, j, tm);
  }
  const long long grid = g.ntiles;
  KernelClock kc(st);
  kern<<<(unsigned)grid, NT, smem, st>>>(g);
  RFPK_CHECK_LAUNCH();
  kc.stop(MODE == TRI_FULL ? "gemm" : "syrk", a.M, a.N, a.K);
  return 0;
}

template <typename T, int BM, int BN, int BK, int WM, int WN, int ST, int MODE>
int launch_major(const GemmArgs<T>& a, bool ak, bool bk, cudaStream_t st) {
  if (ak) {
    return bk ? launch_one<T, BM, BN, BK, WM, WN, ST, true, true, MODE>(a, st)
              : launch_one<T, BM, BN, BK, WM, WN, ST, true, false, MODE>(a, st);
  }
  return bk ? launch_one<T, BM, BN, BK, WM, WN, ST, false, true, MODE>(a, st)
            : launch_one<T, BM, BN, BK, WM, WN, ST, false, false, MODE>(a, st);
}

template <typename T, int BM, int BN, int BK, int WM, int WN, int ST>
int launch_mode(const GemmArgs<T>& a, int mode, bool ak, bool bk, cudaStream_t st) {
  switch (mode) {
    case TRI_LOWER: return launch_major<T, BM, BN, BK, WM, WN, ST, TRI_LOWER>(a, ak, bk, st);
    case TRI_UPPER: return launch_major<T, BM, BN, BK, WM, WN, ST, TRI_UPPER>(a, ak, bk, st);
    default: return launch_major<T, BM, BN, BK, WM, WN, ST, TRI_FULL>(a, ak, bk, st);
  }
}

template <typename T, bool AK, bool BKM>
int splitk_launch(const GemmArgs<T>& a, int S, int kchunk, cudaStream_t st) {
  constexpr int BM = 64, BN = 64, BK = is_cplx<T>::value ? 8 : 16, WM = 32, WN = 32, ST = 3;
  constexpr size_t smem = (size_t)ST *
                          (SmemLayout<T, BM, BK, AK>::SIZE + SmemLayout<T, BN, BK, BKM>::SIZE) *
                          sizeof(T);
  auto kern = gemm_splitk_kernel<T, BM, BN, BK, WM, WN, ST, AK, BKM>;
  kernel_setup(kern, (BM / WM) * (BN / WN) * 32, smem);
  GemmArgs<T> g = a;
  g.tiles_m = (g.M + BM - 1) / BM;
  const int tiles = g.tiles_m * ((g.N + BN - 1) / BN);
  T* ws = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&ws, (size_t)S * g.M * g.N * sizeof(T), st);
  if (e != cudaSuccess) return (int)e;
  KernelClock kc(st);
  kern<<<dim3((unsigned)tiles, (unsigned)S), (BM / WM) * (BN / WN) * 32, smem, st>>>(g, ws, kchunk);
  RFPK_CHECK_LAUNCH();
  kc.stop("gemm_splitk", g.M, g.N, g.K);
  const i64 total = (i64)g.M * g.N;
  int blocks = (int)((total + 255) / 256);
  if (blocks > 4 * num_sms()) blocks = 4 * num_sms();
  splitk_reduce_kernel<T><<<blocks, 256, 0, st>>>(g, ws, S);
  RFPK_CHECK_LAUNCH();
  cudaFreeAsync(ws, st);
  return 0;
}

// -100: not worth splitting (enough tiles, or a short K)
template <typename T> int gemm_splitk(const GemmArgs<T>& g, bool ak, bool bk, cudaStream_t st) {
  constexpr int min_k = 256;
  const long long tiles = (long long)((g.M + 63) / 64) * ((g.N + 63) / 64);
  if (g.K < min_k || tiles * 2 > num_sms()) return -100;
  // about two CTAs per SM in total, slices of at least 128 (a multiple of 16)
  int S = (int)((2 * num_sms() + tiles - 1) / tiles);
  const int smax = g.K / 128;
  if (S > smax) S = smax;
  if (S < 2) return -100;
  const int kchunk = ((g.K + S - 1) / S + 15) / 16 * 16;
  S = (g.K + kchunk - 1) / kchunk;
  if (ak) return bk ? splitk_launch<T, true, true>(g, S, kchunk, st)
                    : splitk_launch<T, true, false>(g, S, kchunk, st);
  return bk ? splitk_launch<T, false, true>(g, S, kchunk, st)
            : splitk_launch<T, false, false>(g, S, kchunk, st);
}

}  // namespace



template <typename T>
int gemm(int tri_mode, T alpha, View<T> A, bool conjA, View<T> B, bool conjB, T beta,
         View<T> C, bool herm_diag, const int* skip, cudaStream_t st, int a_tri,
         bool inplace_leaf) {
  if (C.empty()) return 0;
  if (A.n == 0 || is_zero(alpha)) {
    bool unit_beta;
    if constexpr (is_cplx<T>::value) unit_beta = beta.x == 1.0 && beta.y == 0.0;
    else unit_beta = beta == 1.0;
    if (unit_beta && !herm_diag) return 0;
    return scale_view(C, beta, tri_mode, herm_diag, skip, st);
  }
  // in-place leaf: the leaf dimension (M) must fit one 64-wide tile; after the
  // optional transpose below it becomes N, and the 64x64 config covers it
  // either way, so each CTA reads its whole slab of B before overwriting it.
  if (inplace_leaf && C.m > 64) return -101;
  bool transposed = false;
  if (!(C.rs == 1 || C.m == 1)) {
    // C not column-major: solve C^T = op(B)^T op(A)^T (column-major)
    View<T> At = B.t(), Bt = A.t();
    A = At; B = Bt;
    bool c = conjA; conjA = conjB; conjB = c;
    transposed = true;
    C = C.t();
    if (tri_mode == TRI_LOWER) tri_mode = TRI_UPPER;
    else if (tri_mode == TRI_UPPER) tri_mode = TRI_LOWER;
  }
  OperandLayout la = classify(A);
  OperandLayout lb = classify(B.t());  // B^T is N x K
  if (!la.ok || !lb.ok || !(C.rs == 1 || C.m == 1)) return -100;
  GemmArgs<T> g;
  g.M = (int)C.m; g.N = (int)C.n; g.K = (int)A.n;
  g.A = A.p; g.lda = la.ld;
  g.B = B.p; g.ldb = lb.ld;
  g.C = C.p; g.ldc = (C.n == 1) ? (C.m > 0 ? C.m : 1) : C.cs;
  g.alpha = alpha; g.beta = beta;
  g.conjA = conjA; g.conjB = conjB;
  g.herm_diag = herm_diag ? 1 : 0;
  g.skip = skip;
  g.tiles_m = 0;
  g.ntiles = 0;  // set by launch_one
  g.a_tri = transposed ? A_FULL : a_tri;
  g.b_tri = transposed ? a_tri : A_FULL;
  // operand "K-major": A contiguous along K  <=> la.kmajor; for B, B^T (N x K)
  // contiguous along K <=> lb.kmajor.
  const bool ak = la.kmajor, bk = lb.kmajor;
  if (inplace_leaf) {
    return launch_mode<T, 64, 64, 16 / (is_cplx<T>::value ? 2 : 1), 32, 32, 3>(g, tri_mode, ak,
                                                                               bk, st);
  }
  if (tri_mode == TRI_FULL && a_tri == A_FULL) {
    const int rc = gemm_splitk(g, ak, bk, st);
    if (rc != -100) return rc;
  }
  if constexpr (is_cplx<T>::value) {
    long long tiles = (long long)((g.M + 63) / 64) * ((g.N + 63) / 64);
    if (tiles >= num_sms())
      // (four stages of 8 k: config 5's pftrf 578.6 -> 574.9 ms against three)
      return launch_mode<T, 64, 64, 8, 32, 32, 4>(g, tri_mode, ak, bk, st);
    return launch_mode<T, 32, 32, 8, 16, 16, 3>(g, tri_mode, ak, bk, st);
  } else {
    // 64 x 64 tiles, 4 warps of 32 x 32, FOUR stages of EIGHT k, three CTAs
    // per SM at 150 registers: the measured best FP64 config.  Against the
    // former three stages of 16 k at four CTAs per SM (128 registers, 52 KB of
    // shared memory per CTA instead of 35): config 3's SYRK 16.73 -> 16.45 ms
    // by itself (tools/dom_syrk.py; 16 k x 4 stages 16.80, 8 k x 3 / 5 / 6
    // stages 17.07 / 17.28 / 18.23, 32 k x 2 17.80, 4 k x 8 19.33) and 16.42
    // -> 16.20 ms inside the bench step; capped at 128 registers for four
    // CTAs per SM it is 16.40 ms alone but 16.45 in the step (bench 65.00 vs
    // 64.50 ms).  (33 TFLOP/s at 8192^3 vs 31 for a 1-CTA/SM 128 x 128 tile:
    // more resident CTAs hide the per-stage barrier.)
    const bool force_wide = tune(TK_GEMM_WIDE) != 0;
    // 64 x 128 tiles (4 warps of 32 x 64: 12 fragment loads per 16 DMMAs
    // instead of 8 per 8) for full products with >= 4 waves of them at 2
    // CTAs/SM: DGEMM 8192^3 32.4-33.5 -> 34.2-34.4 TFLOP/s; at 8192 x 1024 the
    // tile count is too small (29.8 vs 32.5).  SYRK/HERK keep 64 x 64: on the
    // odd-ld RFP operands of pftrf the wide tiles measured slower (T2 -= S1
    // S1^T at n = 16384: 17.46 vs 17.02 ms); tuning "gemm_wide" forces them.
    const long long t128 = (long long)((g.M + 63) / 64) * ((g.N + 127) / 128);
    if (force_wide || (tri_mode == TRI_FULL && t128 >= 8LL * num_sms()))
      return launch_mode<T, 64, 128, 16, 32, 64, 3>(g, tri_mode, ak, bk, st);
    return launch_mode<T, 64, 64, 8, 32, 32, 4>(g, tri_mode, ak, bk, st);
  }
}

template int gemm<double>(int, double, View<double>, bool, View<double>, bool, double,
                          View<double>, bool, const int*, cudaStream_t, int, bool);
template int gemm<Z>(int, Z, View<Z>, bool, View<Z>, bool, Z, View<Z>, bool, const int*,
                     cudaStream_t, int, bool);
template int conj_view<double>(View<double>, const int*, cudaStream_t);
template int conj_view<Z>(View<Z>, const int*, cudaStream_t);
template int scale_view<double>(View<double>, double, int, bool, const int*, cudaStream_t);
template int scale_view<Z>(View<Z>, Z, int, bool, const int*, cudaStream_t);

}  // namespace rfpk
