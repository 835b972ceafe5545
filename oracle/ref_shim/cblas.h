/* Minimal CBLAS declarations so the reference's gemm_kernel.cpp (which does
 * `#include <cblas.h>`, /root/reference/proj/src/gemm_kernel.cpp:5-7) compiles
 * against the OpenBLAS shipped in the image (opencv_python_headless.libs).
 * TEST INFRASTRUCTURE ONLY: used by oracle/Makefile to build oracle/_ref. */
#ifndef FPMM_REF_SHIM_CBLAS_H
#define FPMM_REF_SHIM_CBLAS_H
#ifdef __cplusplus
extern "C" {
#endif
enum CBLAS_ORDER { CblasRowMajor = 101, CblasColMajor = 102 };
enum CBLAS_TRANSPOSE { CblasNoTrans = 111, CblasTrans = 112, CblasConjTrans = 113 };
void cblas_dgemm(enum CBLAS_ORDER, enum CBLAS_TRANSPOSE, enum CBLAS_TRANSPOSE, int, int, int,
                 double, const double*, int, const double*, int, double, double*, int);
void cblas_sgemm(enum CBLAS_ORDER, enum CBLAS_TRANSPOSE, enum CBLAS_TRANSPOSE, int, int, int,
                 float, const float*, int, const float*, int, float, float*, int);
void openblas_set_num_threads(int);
int openblas_get_num_threads(void);
#ifdef __cplusplus
}
#endif
#endif
