/* Minimal CBLAS declarations (test infrastructure for the oracle build only).
 * The reference's matmul.cpp (proj/src/matmul.cpp:1-27) includes <cblas.h>; the
 * image has no OpenBLAS dev package, so the oracle links the OpenBLAS 0.3.15
 * shipped inside the opencv wheel, whose exported symbols match these. */
#ifndef ORACLE_SHIM_CBLAS_H
#define ORACLE_SHIM_CBLAS_H
#ifdef __cplusplus
extern "C" {
#endif
enum CBLAS_ORDER { CblasRowMajor = 101, CblasColMajor = 102 };
enum CBLAS_TRANSPOSE { CblasNoTrans = 111, CblasTrans = 112, CblasConjTrans = 113 };
void cblas_sgemm(enum CBLAS_ORDER order, enum CBLAS_TRANSPOSE ta, enum CBLAS_TRANSPOSE tb,
                 int m, int n, int k, float alpha, const float* a, int lda, const float* b,
                 int ldb, float beta, float* c, int ldc);
void openblas_set_num_threads(int n);
#ifdef __cplusplus
}
#endif
#endif
