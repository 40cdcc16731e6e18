/*
 * wf4dvar_testing.h -- kernel-level hooks of libwf4dvar.so for unit tests and
 * micro-benchmarks.  NOT part of the method's ABI (include/wf4dvar.h); they expose
 * the two FP64 tensor-core building blocks of the hot path on caller-owned DEVICE
 * buffers, enqueued on `stream` (cudaStream_t, NULL = default), asynchronous.
 *
 *   wf4dvar_test_gemm : Y = alpha * A X + beta * Z, all row-major
 *                       (A: M x K, lda; X: K x N, ldx; Y, Z: M x N, ldy / ldz;
 *                        Z may be NULL (then beta is ignored) and may alias Y).
 *                       The covariance products of P:L637-639, L651, L663.
 *   wf4dvar_test_trsm : Y = G^{-1} X (upper == 0, G lower triangular) or
 *                       Y = U^{-1} X (upper == 1, U upper triangular), n x n
 *                       row-major factor (ld = n), X / Y n x ncols row-major
 *                       (ld = ncols), X may alias Y; blk > 0 declares the factor
 *                       block diagonal with blocks of blk rows.  The Cholesky-factor
 *                       solves of D_hat^{-1} / R_hat^{-1}.
 * Both return 0 on success, WF4DVAR_EINVAL on bad arguments, WF4DVAR_ECUDA on a
 * launch failure.
 */
#ifndef WF4DVAR_TESTING_H
#define WF4DVAR_TESTING_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
int wf4dvar_test_gemm(int M, int N, int K, double alpha, const double *A, int64_t lda,
                      const double *X, int64_t ldx, double beta, const double *Z, int64_t ldz,
                      double *Y, int64_t ldy, void *stream);
int wf4dvar_test_trsm(int n, int ncols, int upper, int blk, const double *G, const double *X,
                      double *Y, void *stream);
#ifdef __cplusplus
}
#endif
#endif
