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
// row-block (bordered) forms used while the samples are still being uploaded
int64_t gram_rowblock_workspace(int64_t n, int64_t d, int64_t mb);
cudaError_t gram_rowblock(const double* Zs, int64_t ldz, int64_t d, int64_t r0, int64_t r1, double* K, int64_t ldk,
                          double* G, int64_t ldg, double mu2, double* W, cudaStream_t st);
cudaError_t bordered_chol_step(double* G, double* Wi, double* T, double* Ginv, int64_t ld, int64_t r0, int64_t r1,
                               int* info, cudaStream_t chain, cudaStream_t side, cudaStream_t acc, double* ws,
                               int64_t wcap);
// split-K workspace (doubles) of the bordered chain for blocks of mb rows of an n x n matrix
inline int64_t bordered_workspace(int64_t n, int64_t mb) { return 2 * 8 * mb * n; }
cudaError_t mirror_lower(double* A, int64_t ld, int64_t m, cudaStream_t st);

}  // namespace gdwd
