// Hand-written CBLAS prototypes (standard ABI) so the reference CPU oracle
// compiles against the OpenBLAS shared object bundled in this image.
// Test infrastructure only.
#pragma once
#ifdef __cplusplus
extern "C" {
#endif
enum CBLAS_ORDER { CblasRowMajor = 101, CblasColMajor = 102 };
enum CBLAS_TRANSPOSE { CblasNoTrans = 111, CblasTrans = 112, CblasConjTrans = 113 };
void cblas_dgemm(enum CBLAS_ORDER, enum CBLAS_TRANSPOSE, enum CBLAS_TRANSPOSE, int m, int n, int k, double alpha,
                 const double *a, int lda, const double *b, int ldb, double beta, double *c, int ldc);
void cblas_dgemv(enum CBLAS_ORDER, enum CBLAS_TRANSPOSE, int m, int n, double alpha, const double *a, int lda,
                 const double *x, int incx, double beta, double *y, int incy);
void openblas_set_num_threads(int n);
#ifdef __cplusplus
}
#endif
