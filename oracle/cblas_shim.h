/* Minimal cblas.h for building the reference's tensor.cpp against the OpenBLAS
 * 0.3.15 that ships inside the image (opencv_python_headless.libs). Only the
 * symbols the reference uses (tensor.cpp:3,15,138-175,483-539) are declared.
 * Test infrastructure only (oracle/), never linked into the product. */
#ifndef P2R_ORACLE_CBLAS_SHIM_H
#define P2R_ORACLE_CBLAS_SHIM_H
#ifdef __cplusplus
extern "C" {
#endif
enum CBLAS_ORDER { CblasRowMajor = 101, CblasColMajor = 102 };
enum CBLAS_TRANSPOSE { CblasNoTrans = 111, CblasTrans = 112, CblasConjTrans = 113 };
void cblas_sgemm(enum CBLAS_ORDER order, enum CBLAS_TRANSPOSE ta, enum CBLAS_TRANSPOSE tb, int m,
                 int n, int k, float alpha, const float* a, int lda, const float* b, int ldb,
                 float beta, float* c, int ldc);
void openblas_set_num_threads(int n);
#ifdef __cplusplus
}
#endif
#endif
