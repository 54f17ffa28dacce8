/*
 * rfpk_b200.h -- C ABI of the B200-native RFPF Cholesky library
 * (librfpk_b200.so, built from paper_0901_1696_b200/csrc).
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/pkg/src/rfpk).  Argument order follows the LAPACK RFPF
 * calling sequences the paper describes (PAPER.md:1313-1333:
 * PFTRF(TRANSR,UPLO,N,A,INFO), PFTRS(TRANSR,UPLO,N,NR,A,B,LDB,INFO), ...),
 * which is what a ctypes/cffi binding of the reference's Python entry points
 * (convert.py / rfp.py / packed.py) lowers to.
 *
 * Conventions
 *  - All array arguments are DEVICE pointers (CUDA global memory) owned by
 *    the caller.  Complex arrays are complex128 interleaved (re, im), i.e.
 *    numpy / torch complex128 layout, passed as void*.
 *  - Every call is asynchronous and stream-ordered on `stream` (a
 *    cudaStream_t; NULL = legacy default stream).
 *  - Return value: 0 = launched; -k = illegal value of argument k (LAPACK
 *    convention, nothing launched); > 0 = CUDA runtime error code.
 *  - `info` is a DEVICE int.  It is reset to 0 on the stream at the start of
 *    the call and receives, stream-ordered, the LAPACK/reference info:
 *    pftrf: 1-based order of the first non-positive (or NaN) leading minor
 *    (rfp.py:71-79, 88-89); tftri/pftri: 1-based index of a zero diagonal
 *    (rfp.py:299-322, kernels.py:526-529).  After a failure the remaining
 *    kernels of the call are skipped and the buffer contents are unspecified
 *    (the reference also leaves a partially overwritten buffer).
 *  - transr: 'N', 'T' or 'C'.  'C' is an alias of 'T' (the verbatim
 *    transposed rectangle of the reference, layout.py:31; convert.py:83-87):
 *    values are never conjugated by the storage format.
 *  - uplo: 'L' or 'U'; diag: 'N' or 'U'; trans: 'N', 'T', 'C'; side 'L'/'R'.
 *    Lower-case letters are accepted.
 */
#ifndef RFPK_B200_H
#define RFPK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* rfpk_stream_t; /* == cudaStream_t */

/* library identification ------------------------------------------------ */
const char* rfpk_version(void);
/* number of SMs of the current device, or a negative CUDA error */
int rfpk_device_sms(void);
/* total kernels this library has launched in the process (monotonic;
   kernels replayed from a cached CUDA graph are counted per replay) */
long long rfpk_launch_count(void);
/* pftrf/pftrs/tftri/pftri calls are captured into CUDA graphs keyed by their
   full argument tuple (pointers included) and replayed on repeat calls
   (tuning "graphs" = 0 disables).  This drops every cached graph. */
int rfpk_graph_cache_clear(void);
/* Path thresholds (process-wide; there are no environment knobs).  Names and
   defaults: "oop_max" 4096, "t2_copy_min" 2048, "panel_max" 4096,
   "pfsv_overlap_min" 512, "overlap" 1, "graphs" 1, "graph_max_n" 8192,
   "gemm_wide" 0, "batched_generic" 0, "trace" 0, "trsm_split" 1, "zpotrf_split_min" 9000 (see
   DESIGN.md section 4).
   Setting a value drops every cached graph.  Returns 0, or -1 for an
   unknown name.  Not meant to be changed while other threads are inside
   the library. */
int rfpk_set_tuning(const char* name, long long value);
int rfpk_get_tuning(const char* name, long long* value);
int rfpk_reset_tuning(void);

/* conversions: verbatim copies, bit-exact (convert.py:156-275) ----------- */
/* replaces convert.trttf(a, uplo, transr)   convert.py:156-186 */
int rfpk_dtrttf(char transr, char uplo, int64_t n, const double* a, int64_t lda, double* arf,
                rfpk_stream_t stream);
int rfpk_ztrttf(char transr, char uplo, int64_t n, const void* a, int64_t lda, void* arf,
                rfpk_stream_t stream);
/* replaces convert.tfttr(r, ld)   convert.py:189-217; writes all lda x n
   entries (triangle + zeros), as the reference's zero-filled result */
int rfpk_dtfttr(char transr, char uplo, int64_t n, const double* arf, double* a, int64_t lda,
                rfpk_stream_t stream);
int rfpk_ztfttr(char transr, char uplo, int64_t n, const void* arf, void* a, int64_t lda,
                rfpk_stream_t stream);
/* replaces convert.tpttf(p, transr)   convert.py:220-246 */
int rfpk_dtpttf(char transr, char uplo, int64_t n, const double* ap, double* arf,
                rfpk_stream_t stream);
int rfpk_ztpttf(char transr, char uplo, int64_t n, const void* ap, void* arf,
                rfpk_stream_t stream);
/* replaces convert.tfttp(r)   convert.py:249-275 */
int rfpk_dtfttp(char transr, char uplo, int64_t n, const double* arf, double* ap,
                rfpk_stream_t stream);
int rfpk_ztfttp(char transr, char uplo, int64_t n, const void* arf, void* ap,
                rfpk_stream_t stream);
/* replaces packed.pack(a, uplo)   packed.py:41-51 */
int rfpk_dtrttp(char uplo, int64_t n, const double* a, int64_t lda, double* ap,
                rfpk_stream_t stream);
int rfpk_ztrttp(char uplo, int64_t n, const void* a, int64_t lda, void* ap,
                rfpk_stream_t stream);
/* replaces packed.unpack(p, ld)   packed.py:54-67 (zero-filled lda x n) */
int rfpk_dtpttr(char uplo, int64_t n, const double* ap, double* a, int64_t lda,
                rfpk_stream_t stream);
int rfpk_ztpttr(char uplo, int64_t n, const void* ap, void* a, int64_t lda,
                rfpk_stream_t stream);

/* factorization / solve / inversion (rfp.py) ------------------------------ */
/* replaces rfp.pftrf(r)   rfp.py:55-91 */
int rfpk_dpftrf(char transr, char uplo, int64_t n, double* arf, int* info,
                rfpk_stream_t stream);
int rfpk_zpftrf(char transr, char uplo, int64_t n, void* arf, int* info, rfpk_stream_t stream);
/* replaces rfp.pftrs(r, b)   rfp.py:106-136; B column-major n x nrhs, ldb >= n */
int rfpk_dpftrs(char transr, char uplo, int64_t n, int64_t nrhs, const double* arf, double* b,
                int64_t ldb, int* info, rfpk_stream_t stream);
int rfpk_zpftrs(char transr, char uplo, int64_t n, int64_t nrhs, const void* arf, void* b,
                int64_t ldb, int* info, rfpk_stream_t stream);
/* same, B element (i, j) at b[i*rsb + j*csb] with rsb == 1 or csb == 1
   (the reference accepts any strided b; rfp.py:94-103) */
int rfpk_dpftrs_ex(char transr, char uplo, int64_t n, int64_t nrhs, const double* arf, double* b,
                   int64_t rsb, int64_t csb, int* info, rfpk_stream_t stream);
int rfpk_zpftrs_ex(char transr, char uplo, int64_t n, int64_t nrhs, const void* arf, void* b,
                   int64_t rsb, int64_t csb, int* info, rfpk_stream_t stream);
/* rfp.pftrf(r) on a buffer that still sits in pinned HOST memory h_arf:
   the host->device copy into d_arf is streamed (T1/T2 rows first on `stream`,
   S1 rows on an internal side stream) and overlapped with potrf(T1);
   factor and info as rfpk_?pftrf.  rfp.py:55-91 + the caller's H2D copy. */
int rfpk_dpftrf_host(char transr, char uplo, int64_t n, const double* h_arf, double* d_arf,
                     int* info, rfpk_stream_t stream);
int rfpk_zpftrf_host(char transr, char uplo, int64_t n, const void* h_arf, void* d_arf, int* info,
                     rfpk_stream_t stream);
/* rfp.pftrf(r) then rfp.pftrs(r, b) on a device-resident problem in one
   call (B column-major n x nrhs, ld ldb): the first solve with T1 and the S1
   product run concurrently with potrf(T2).  info as rfpk_?pftrf (after a
   failure b is unspecified).  rfp.py:55-136 (the pair of calls). */
int rfpk_dpfsv(char transr, char uplo, int64_t n, int64_t nrhs, double* arf, double* b,
               int64_t ldb, int* info, rfpk_stream_t stream);
int rfpk_zpfsv(char transr, char uplo, int64_t n, int64_t nrhs, void* arf, void* b, int64_t ldb,
               int* info, rfpk_stream_t stream);
/* rfp.pftrf(r) then rfp.pftrs(r, b) on a problem that sits in pinned HOST
   memory (h_arf: the RFP buffer; h_b: n x nrhs column-major, ld ldb), with
   every transfer overlapped with the computation; the solution lands in
   h_x (may equal h_b), the factor in d_arf, the device copy of B in d_b
   (n x nrhs, ld ldb).  info as rfpk_?pftrf; on failure h_x is unspecified.
   rfp.py:55-136 + the caller's copies. */
int rfpk_dpfsv_host(char transr, char uplo, int64_t n, int64_t nrhs, const double* h_arf,
                    double* d_arf, const double* h_b, double* d_b, double* h_x, int64_t ldb,
                    int* info, rfpk_stream_t stream);
int rfpk_zpfsv_host(char transr, char uplo, int64_t n, int64_t nrhs, const void* h_arf,
                    void* d_arf, const void* h_b, void* d_b, void* h_x, int64_t ldb, int* info,
                    rfpk_stream_t stream);
/* replaces rfp.tftri(r, diag)   rfp.py:286-325 */
int rfpk_dtftri(char transr, char uplo, char diag, int64_t n, double* arf, int* info,
                rfpk_stream_t stream);
int rfpk_ztftri(char transr, char uplo, char diag, int64_t n, void* arf, int* info,
                rfpk_stream_t stream);
/* replaces rfp.pftri(r)   rfp.py:328-360 */
int rfpk_dpftri(char transr, char uplo, int64_t n, double* arf, int* info, rfpk_stream_t stream);
int rfpk_zpftri(char transr, char uplo, int64_t n, void* arf, int* info, rfpk_stream_t stream);

/* Phase clock (measurement only, no reference counterpart): when enabled,
   every direct (non-graph) pftrf / pftrs call records CUDA events around its
   SRPA steps on its own stream without synchronising; rfpk_phase_time()
   waits for them and returns the summed milliseconds and the count for one
   label, e.g. "pftrf trsm(S1)".  Enabling resets the sums.  Returns 1 if
   the label was never seen. */
int rfpk_phase_clock(int enable);
int rfpk_phase_time(const char* label, double* total_ms, int64_t* count);
/* every label the clock has seen since it was enabled, newline-separated, into
   out[cap] (truncated, NUL-terminated); returns the length needed incl. NUL.
   Kernel launches appear as "kernel <name> <dims>" (see KernelClock) */
int64_t rfpk_phase_labels(char* out, int64_t cap);

/* packed Cholesky ------------------------------------ */
/* replaces packed.pptrf_ref(p)   packed.py:70-108 -- in place on the
   column-packed triangle ap (n(n+1)/2 elements, LAPACK 'L'/'U' packing);
   info (device) = 0 or the 1-based order of the first non-positive leading
   minor.  Computed through RFP (tpttf -> pftrf -> tfttp) in a workspace. */
int rfpk_dpptrf(char uplo, int64_t n, double* ap, int* info, rfpk_stream_t stream);
int rfpk_zpptrf(char uplo, int64_t n, void* ap, int* info, rfpk_stream_t stream);
/* replaces packed.pptrs_ref(p, b)   packed.py:111-146 -- solve A X = B in
   place from a packed factor; b is n x nrhs with element (i, j) at
   b[i*rsb + j*csb] (one of the strides 1) */
int rfpk_dpptrs(char uplo, int64_t n, int64_t nrhs, const double* ap, double* b, int64_t rsb,
                int64_t csb, int* info, rfpk_stream_t stream);
int rfpk_zpptrs(char uplo, int64_t n, int64_t nrhs, const void* ap, void* b, int64_t rsb,
                int64_t csb, int* info, rfpk_stream_t stream);

/* SURVEY 8(f) rows ------------------------------------------------------- */
/* replaces rfp.tfsm(transr, side, uplo, trans, diag, m, n, alpha, a, b)
   rfp.py:181-224; a holds the order-m (side L) / order-n (side R) triangle;
   b is m x n with element (i, j) at b[i*rsb + j*csb]; info (device) receives
   the 1-based global index of a zero diagonal (SingularMatrixError) */
int rfpk_dtfsm(char transr, char side, char uplo, char trans, char diag, int64_t m, int64_t n,
               double alpha, const double* arf, double* b, int64_t rsb, int64_t csb, int* info,
               rfpk_stream_t stream);
int rfpk_ztfsm(char transr, char side, char uplo, char trans, char diag, int64_t m, int64_t n,
               double alpha_re, double alpha_im, const void* arf, void* b, int64_t rsb,
               int64_t csb, int* info, rfpk_stream_t stream);
/* replaces rfp.sfrk_hfrk(transr, uplo, trans, n, k, alpha, a, beta, c)
   rfp.py:227-283: C <- alpha G G^(T|H) + beta C; a is n x k (trans 'N') or
   k x n, element (i, j) at a[i*rsa + j*csa] */
int rfpk_dsfrk(char transr, char uplo, char trans, int64_t n, int64_t k, double alpha,
               const double* a, int64_t rsa, int64_t csa, double beta, double* arf,
               rfpk_stream_t stream);
int rfpk_zhfrk(char transr, char uplo, char trans, int64_t n, int64_t k, double alpha,
               const void* a, int64_t rsa, int64_t csa, double beta, void* arf, int hermitian,
               rfpk_stream_t stream);
/* replaces rfp.lansf(norm, r)   rfp.py:363-417: 'M', '1'/'O', 'I', 'F'/'E' norm
   of the implied full matrix, written to the device double *result */
int rfpk_dlansf(char norm, char transr, char uplo, int64_t n, const double* arf, double* result,
                rfpk_stream_t stream);
int rfpk_zlansf(char norm, char transr, char uplo, int64_t n, const void* arf, double* result,
                rfpk_stream_t stream);

/* batched small-n (BASELINE config 4; no reference counterpart beyond a loop
   over rfp.pftrf / rfp.pftrs per matrix) --------------------------------- */
/* batch independent RFP buffers at arf + k*stride_arf; info[k] per matrix */
int rfpk_dpftrf_batched(char transr, char uplo, int64_t n, double* arf, int64_t stride_arf,
                        int64_t batch, int* info, rfpk_stream_t stream);
/* B_k column-major n x nrhs at b + k*stride_b with leading dimension ldb */
int rfpk_dpftrs_batched(char transr, char uplo, int64_t n, int64_t nrhs, const double* arf,
                        int64_t stride_arf, double* b, int64_t ldb, int64_t stride_b,
                        int64_t batch, int* info, rfpk_stream_t stream);
/* fused pftrf + pftrs, one pass over HBM per matrix */
int rfpk_dpftrf_pftrs_batched(char transr, char uplo, int64_t n, int64_t nrhs, double* arf,
                              int64_t stride_arf, double* b, int64_t ldb, int64_t stride_b,
                              int64_t batch, int* info, rfpk_stream_t stream);

/* full-format kernels on strided device views (kernels.py) ----------------
   A matrix argument is (ptr, rows, cols, rs, cs): element (i, j) at
   ptr[i*rs + j*cs], with rs == 1 or cs == 1.  Complex alpha/beta are passed
   as (re, im).  info (device) receives a 1-based singular index (trsm,
   trtri) or failing pivot (potrf). */
int rfpk_dgemm(char transa, char transb, double alpha, const double* a, int64_t ar, int64_t ac,
               int64_t ars, int64_t acs, const double* b, int64_t br, int64_t bc, int64_t brs,
               int64_t bcs, double beta, double* c, int64_t cr, int64_t cc, int64_t crs,
               int64_t ccs, rfpk_stream_t stream);
int rfpk_zgemm(char transa, char transb, double alpha_re, double alpha_im, const void* a,
               int64_t ar, int64_t ac, int64_t ars, int64_t acs, const void* b, int64_t br,
               int64_t bc, int64_t brs, int64_t bcs, double beta_re, double beta_im, void* c,
               int64_t cr, int64_t cc, int64_t crs, int64_t ccs, rfpk_stream_t stream);
int rfpk_dtrsm(char side, char uplo, char trans, char diag, double alpha, const double* a,
               int64_t an, int64_t ars, int64_t acs, double* b, int64_t br, int64_t bc,
               int64_t brs, int64_t bcs, int* info, rfpk_stream_t stream);
int rfpk_ztrsm(char side, char uplo, char trans, char diag, double alpha_re, double alpha_im,
               const void* a, int64_t an, int64_t ars, int64_t acs, void* b, int64_t br,
               int64_t bc, int64_t brs, int64_t bcs, int* info, rfpk_stream_t stream);
int rfpk_dtrmm(char side, char uplo, char trans, char diag, double alpha, const double* a,
               int64_t an, int64_t ars, int64_t acs, double* b, int64_t br, int64_t bc,
               int64_t brs, int64_t bcs, rfpk_stream_t stream);
int rfpk_ztrmm(char side, char uplo, char trans, char diag, double alpha_re, double alpha_im,
               const void* a, int64_t an, int64_t ars, int64_t acs, void* b, int64_t br,
               int64_t bc, int64_t brs, int64_t bcs, rfpk_stream_t stream);
int rfpk_dsyrk(char uplo, char trans, double alpha, const double* a, int64_t ar, int64_t ac,
               int64_t ars, int64_t acs, double beta, double* c, int64_t cn, int64_t crs,
               int64_t ccs, rfpk_stream_t stream);
/* hermitian != 0: C <- alpha G G^H + beta C (diag imag forced 0); else G G^T */
int rfpk_zsyrk(char uplo, char trans, double alpha, const void* a, int64_t ar, int64_t ac,
               int64_t ars, int64_t acs, double beta, void* c, int64_t cn, int64_t crs,
               int64_t ccs, int hermitian, rfpk_stream_t stream);
int rfpk_dpotrf(char uplo, double* a, int64_t n, int64_t rs, int64_t cs, int* info,
                rfpk_stream_t stream);
int rfpk_zpotrf(char uplo, void* a, int64_t n, int64_t rs, int64_t cs, int* info,
                rfpk_stream_t stream);
int rfpk_dtrtri(char uplo, char diag, double* a, int64_t n, int64_t rs, int64_t cs, int* info,
                rfpk_stream_t stream);
int rfpk_ztrtri(char uplo, char diag, void* a, int64_t n, int64_t rs, int64_t cs, int* info,
                rfpk_stream_t stream);
int rfpk_dlauum(char uplo, double* a, int64_t n, int64_t rs, int64_t cs, rfpk_stream_t stream);
int rfpk_zlauum(char uplo, void* a, int64_t n, int64_t rs, int64_t cs, rfpk_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* RFPK_B200_H */
