#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gdwd {

// tri: structural zeros of triangular operands the tiles may skip (the
// skipped products are exact zeros, so results are unchanged):
//   GEMM_B_KLE_N  B(n,k) = 0 for k > n     GEMM_B_KGE_N  B(n,k) = 0 for k < n
//   GEMM_A_KLE_M  A(m,k) = 0 for k > m     GEMM_A_KGE_M  A(m,k) = 0 for k < m
//   GEMM_C_LOWER  only C's tiles on or below the diagonal are needed
enum : int { GEMM_B_KLE_N = 1, GEMM_B_KGE_N = 2, GEMM_A_KLE_M = 4, GEMM_A_KGE_M = 8, GEMM_C_LOWER = 16 };
cudaError_t gemm_f64(const double* a, int64_t sam, int64_t sak, const double* b, int64_t sbn, int64_t sbk,
                     int64_t M, int64_t N, int64_t K, double alpha, double beta, double* C, int64_t ldc,
                     cudaStream_t st, int tri = 0);
int gram_slices(int64_t M, int64_t K);
int64_t gram_workspace_doubles(int64_t M, int64_t K);
cudaError_t gram_syrk(const double* Zs, int64_t R, int64_t Lc, int64_t ldz, bool sum_over_rows, double div,
                      double shift, double* C, int64_t ldc, double* W, cudaStream_t st, bool accumulate = false);
cudaError_t chol_inverse(double* A, double* Li, double* T, int64_t ld, int64_t m, int* info, cudaStream_t st);

}  // namespace gdwd
