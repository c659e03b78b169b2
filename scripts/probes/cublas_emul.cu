// Probe: which cuBLAS configurations run FP32 GEMMs with BF16x9 emulation here.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
int main() {
  int ver = 0;
  cublasHandle_t h;
  cublasCreate(&h);
  cublasGetVersion(h, &ver);
  printf("cublas version %d\n", ver);
  const int M = 262144, N = 128, K = 256;
  float *A, *B, *C;
  cudaMalloc(&A, sizeof(float) * M * K);
  cudaMalloc(&B, sizeof(float) * K * N);
  cudaMalloc(&C, sizeof(float) * M * N);
  cudaMemset(A, 0, sizeof(float) * M * K);
  cudaMemset(B, 0, sizeof(float) * K * N);
  float alpha = 1, beta = 0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto fn) {
    cublasStatus_t s = fn();
    if (s != CUBLAS_STATUS_SUCCESS) { printf("%-55s status %d (%s)\n", name, (int)s, cublasGetStatusString(s)); return; }
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
    printf("%-55s %.3f ms  %.1f TFLOP/s\n", name, ms, 2.0 * M * N * K / ms / 1e9);
  };
  for (int strat = 0; strat < 3; ++strat) {
    cublasSetEmulationStrategy(h, (cublasEmulationStrategy_t)strat);
    printf("-- emulation strategy %d\n", strat);
    cublasSetMathMode(h, CUBLAS_DEFAULT_MATH);
    timeit("GemmEx NN COMPUTE_32F_EMULATED_16BFX9", [&] {
      return cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, N, M, K, &alpha, B, CUDA_R_32F, N, A, CUDA_R_32F, K, &beta, C, CUDA_R_32F, N, CUBLAS_COMPUTE_32F_EMULATED_16BFX9, CUBLAS_GEMM_DEFAULT); });
    timeit("GemmEx TN COMPUTE_32F_EMULATED_16BFX9", [&] {
      return cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, N, M, K, &alpha, B, CUDA_R_32F, K, A, CUDA_R_32F, K, &beta, C, CUDA_R_32F, N, CUBLAS_COMPUTE_32F_EMULATED_16BFX9, CUBLAS_GEMM_DEFAULT); });
    cublasSetMathMode(h, CUBLAS_FP32_EMULATED_BF16X9_MATH);
    timeit("Sgemm NN mathmode BF16X9", [&] {
      return cublasSgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, N, M, K, &alpha, B, N, A, K, &beta, C, N); });
    timeit("GemmEx NN COMPUTE_32F + mathmode BF16X9", [&] {
      return cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, N, M, K, &alpha, B, CUDA_R_32F, N, A, CUDA_R_32F, K, &beta, C, CUDA_R_32F, N, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT); });
    cublasSetMathMode(h, CUBLAS_DEFAULT_MATH);
  }
  timeit("GemmEx NN COMPUTE_32F_PEDANTIC", [&] {
    return cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, N, M, K, &alpha, B, CUDA_R_32F, N, A, CUDA_R_32F, K, &beta, C, CUDA_R_32F, N, CUBLAS_COMPUTE_32F_PEDANTIC, CUBLAS_GEMM_DEFAULT); });
  timeit("GemmEx NN COMPUTE_32F_FAST_TF32 (not accurate, ref)", [&] {
    return cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, N, M, K, &alpha, B, CUDA_R_32F, N, A, CUDA_R_32F, K, &beta, C, CUDA_R_32F, N, CUBLAS_COMPUTE_32F_FAST_TF32, CUBLAS_GEMM_DEFAULT); });
  return 0;
}
