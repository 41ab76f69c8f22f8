// cublasLt vs cublasDgemm for the plane-GS DST shape (M=K=nx, N=ny*planes): which
// DMMA kernels exist and how fast each runs.  nvcc -o lt_probe lt_probe.cu -lcublasLt -lcublas
#include <cublasLt.h>
#include <cublas_v2.h>
#include <cstdio>
#include <vector>
int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 128, N = argc > 2 ? atoi(argv[2]) : 8192, K = M;
  double *A, *B, *C;
  cudaMalloc(&A, sizeof(double) * M * K);
  cudaMalloc(&B, sizeof(double) * K * N);
  cudaMalloc(&C, sizeof(double) * M * N);
  cudaMemset(A, 0, sizeof(double) * M * K);
  cudaMemset(B, 0, sizeof(double) * K * N);
  const double one = 1, zero = 0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cublasHandle_t h;
  cublasCreate(&h);
  for (int w = 0; w < 5; ++w) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, M, N, K, &one, A, M, B, K, &zero, C, M);
  cudaEventRecord(e0);
  for (int r = 0; r < 50; ++r) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, M, N, K, &one, A, M, B, K, &zero, C, M);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("cublasDgemm M=%d N=%d K=%d: %.2f us  %.1f TF/s\n", M, N, K, ms * 20, 2.0 * M * N * K / (ms / 50 * 1e-3) / 1e12);
  cublasLtHandle_t lt;
  cublasLtCreate(&lt);
  cublasLtMatmulDesc_t op;
  cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_64F, CUDA_R_64F);
  cublasLtMatrixLayout_t la, lb, lc;
  cublasLtMatrixLayoutCreate(&la, CUDA_R_64F, M, K, M);
  cublasLtMatrixLayoutCreate(&lb, CUDA_R_64F, K, N, K);
  cublasLtMatrixLayoutCreate(&lc, CUDA_R_64F, M, N, M);
  cublasLtMatmulPreference_t pref;
  cublasLtMatmulPreferenceCreate(&pref);
  size_t ws = 32 << 20;
  void* wsp;
  cudaMalloc(&wsp, ws);
  cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws, sizeof ws);
  cublasLtMatmulHeuristicResult_t res[16];
  int n = 0;
  cublasLtMatmulAlgoGetHeuristic(lt, op, la, lb, lc, lc, pref, 16, res, &n);
  printf("heuristic algos: %d\n", n);
  for (int i = 0; i < n; ++i) {
    for (int w = 0; w < 3; ++w)
      cublasLtMatmul(lt, op, &one, A, la, B, lb, &zero, C, lc, C, lc, &res[i].algo, wsp, ws, 0);
    cudaEventRecord(e0);
    for (int r = 0; r < 50; ++r)
      cublasLtMatmul(lt, op, &one, A, la, B, lb, &zero, C, lc, C, lc, &res[i].algo, wsp, ws, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("  algo %d: %.2f us  %.1f TF/s (ws %zu)\n", i, ms * 20, 2.0 * M * N * K / (ms / 50 * 1e-3) / 1e12,
           res[i].workspaceSize);
  }
  return 0;
}
