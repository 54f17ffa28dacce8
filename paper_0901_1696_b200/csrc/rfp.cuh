// RFP-level drivers: the SRPA compositions of pftrf / pftrs / tftri / pftri
// over the T1 / T2 / S1 views of one flat RFP buffer, and the full / packed /
// RFP conversion kernels.
#pragma once
#include "blas.cuh"

#include <string>

namespace rfpk {

struct RfpDesc {
  i64 n, n1, n2, nt, ldar;
  int d;       // 1 for even n (layout.py:75-78)
  bool lower;  // uplo 'L'
  bool trans;  // transr 'T' (or 'C', its verbatim alias)
};

RfpDesc rfp_desc(i64 n, char uplo, char transr);

// T1, T2, S1 as views of the normal ldar x n1 rectangle (convert.py:142-153)
template <typename T> void rfp_blocks(const RfpDesc& d, T* buf, View<T>& t1, View<T>& t2,
                                      View<T>& s1);

// pfsv plan: pftrf runs the whole pftrs of b at its end (part of it beside
// potrf(T2)) and sets done; b_ready: b's transfer, b2_final as for pftrs
template <typename T> struct PfsvPlan {
  View<T> b;
  cudaEvent_t b_ready;
  cudaEvent_t b2_final;
  bool done;
  RowDoneHook* head_rows = nullptr;  // hook for the last solve (the head block's rows)
};
template <typename T>
int pftrf(Ctx c, const RfpDesc& d, T* arf, cudaEvent_t s1_ready = nullptr,
          const int* cflags = nullptr, const int* sflags = nullptr,
          PfsvPlan<T>* plan = nullptr);
// pftrf + pftrs(b) with the independent parts overlapped (see rfp.cu)
template <typename T>
int pfsv(Ctx c, const RfpDesc& d, T* arf, View<T> b, cudaEvent_t s1_ready = nullptr,
         const int* cflags = nullptr, const int* sflags = nullptr,
         cudaEvent_t b_ready = nullptr, cudaEvent_t b2_final = nullptr,
         RowDoneHook* head_rows = nullptr);
// (s1_ready: the S1 rows' transfer; with cflags / sflags the input is being
//  streamed in 64-column chunks of the normal rectangle, chunk j of the T1/T2
//  rows flagged in cflags[j] and of the S1 rows in sflags[j], and s1_ready
//  marks the end of the whole transfer; see rfp_h2d_chunked)
// host -> device streaming helper for pftrf: the rows of the normal rectangle
// holding T1 and T2 (first needed) and those holding S1 (needed from the S1
// solve on) as two copies; see rfpk_?pftrf_host
template <typename T>
int rfp_h2d_split(const RfpDesc& d, const T* host, T* dev, cudaStream_t first, cudaStream_t second);
// the same two row regions, each in 64-column chunks of the normal
// rectangle, on ONE copy stream, setting cflags[j] / sflags[j] (device ints,
// zeroed by the caller) after chunk j of the T1/T2 rows / of the S1 rows
template <typename T>
int rfp_h2d_chunked(const RfpDesc& d, const T* host, T* dev, int* cflags, int* sflags,
                    cudaStream_t copy);
template <typename T> int pftrs(Ctx c, const RfpDesc& d, const T* arf, View<T> b,
                                cudaEvent_t b2_final = nullptr, RowDoneHook* head_rows = nullptr);
// (head_rows: see RowHook -- the last solve, which finalizes the head block
//  rows [0, n1) for 'L' / [0, n2) for 'U', reports its row blocks as done)
// (b2_final: recorded once the trailing block of b -- rows [n1, n) for 'L',
//  [n2, n) for 'U' -- holds its final values, before the last two steps)
template <typename T> int tftri(Ctx c, const RfpDesc& d, char diag, T* arf);
template <typename T> int pftri(Ctx c, const RfpDesc& d, T* arf);

// SURVEY 8(f) rows
template <typename T>
int tfsm(Ctx c, const RfpDesc& d, char side, char trans, char diag, T alpha, const T* arf,
         View<T> b);
template <typename T>
int sfrk(Ctx c, const RfpDesc& d, char trans, i64 k, double alpha, View<T> a, double beta, T* arf,
         bool herm);
// norm of the implied full matrix into *out (device double): 'M', '1', 'I', 'F'
template <typename T> int lansf(cudaStream_t st, const RfpDesc& d, char norm, const T* arf,
                                double* out);

// phase clock (see PhaseTrace in rfp.cu)
void phase_clock_enable(bool on);
bool phase_clock_read(const char* label, double* total_ms, long long* count);
std::string phase_clock_labels();  // every label seen, one per line

// Storage descriptors for the conversion kernel.
enum StorageKind : int { ST_FULL = 0, ST_PACKED = 1, ST_RFP = 2 };
struct Storage {
  int kind;
  i64 ld;  // full: leading dimension
  RfpDesc r;
};

// Copy the triangle between two storages (verbatim).  When dst is ST_FULL and
// zero_fill is set, every other element of the ld x n destination is +0.0
// (convert.py:200, packed.py:62).
template <typename T>
int convert(const Storage& src, const T* s, const Storage& dst, T* dptr, bool zero_fill,
            cudaStream_t st);

}  // namespace rfpk
