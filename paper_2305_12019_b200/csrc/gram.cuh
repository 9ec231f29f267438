#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gdwd {

cudaError_t gemm_f64(const double* a, int64_t sam, int64_t sak, const double* b, int64_t sbn, int64_t sbk,
                     int64_t M, int64_t N, int64_t K, double alpha, double beta, double* C, int64_t ldc,
                     cudaStream_t st);
int gram_slices(int64_t M, int64_t K);
int64_t gram_workspace_doubles(int64_t M, int64_t K);
cudaError_t gram_syrk(const double* Zs, int64_t R, int64_t Lc, int64_t ldz, bool sum_over_rows, double div,
                      double shift, double* C, int64_t ldc, double* W, cudaStream_t st, bool accumulate = false);
cudaError_t chol_inverse(double* A, double* Li, double* T, int64_t ld, int64_t m, int* info, cudaStream_t st);

}  // namespace gdwd
