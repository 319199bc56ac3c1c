// Hand-written LAPACKE prototypes (standard ABI, lapack_int = int) for the
// reference CPU oracle build. Test infrastructure only.
#pragma once
#ifdef __cplusplus
extern "C" {
#endif
typedef int lapack_int;
#define LAPACK_ROW_MAJOR 101
#define LAPACK_COL_MAJOR 102
lapack_int LAPACKE_dgesdd(int matrix_layout, char jobz, lapack_int m, lapack_int n, double *a, lapack_int lda,
                          double *s, double *u, lapack_int ldu, double *vt, lapack_int ldvt);
lapack_int LAPACKE_dgesvd(int matrix_layout, char jobu, char jobvt, lapack_int m, lapack_int n, double *a,
                          lapack_int lda, double *s, double *u, lapack_int ldu, double *vt, lapack_int ldvt,
                          double *superb);
#ifdef __cplusplus
}
#endif
