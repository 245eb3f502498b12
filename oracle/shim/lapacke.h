/* Minimal LAPACKE shim so the reference's linalg_lapack.cpp compiles against
 * scipy's bundled OpenBLAS 0.3.30 (LP64, exports prefixed with "scipy_").
 * Test infrastructure only: used by oracle/Makefile to build oracle/_ref.
 * Only the three calls the reference makes are declared
 * (proj/src/linalg_lapack.cpp:18-19, 36-37, 55-58). */
#pragma once

typedef int lapack_int;
#define LAPACK_ROW_MAJOR 101
#define LAPACK_COL_MAJOR 102

#ifdef __cplusplus
extern "C" {
#endif
lapack_int scipy_LAPACKE_dsyev(int layout, char jobz, char uplo, lapack_int n, double* a,
                               lapack_int lda, double* w);
lapack_int scipy_LAPACKE_dposv(int layout, char uplo, lapack_int n, lapack_int nrhs, double* a,
                               lapack_int lda, double* b, lapack_int ldb);
lapack_int scipy_LAPACKE_dgesvd(int layout, char jobu, char jobvt, lapack_int m, lapack_int n,
                                double* a, lapack_int lda, double* s, double* u, lapack_int ldu,
                                double* vt, lapack_int ldvt, double* superb);
#ifdef __cplusplus
}
#endif

#define LAPACKE_dsyev scipy_LAPACKE_dsyev
#define LAPACKE_dposv scipy_LAPACKE_dposv
#define LAPACKE_dgesvd scipy_LAPACKE_dgesvd
