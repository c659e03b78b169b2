// FP32 CUDA-core FMA throughput microbenchmark (roofline denominator for the
// SIMT circuit kernels; MEASURED_PEAKS.json only carries HBM and bf16 GEMM).
// Not part of the QPINN ABI: built into libqpinn_tools.so for bench.py.
#include <cuda_runtime.h>
#include <stdint.h>

template <int CHAINS, bool IMM>
__global__ void __launch_bounds__(256) fma_kernel(float* out, int iters, float b, float c) {
  float a[CHAINS];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) a[k] = threadIdx.x * 1e-3f + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) {
      if (IMM) a[k] = fmaf(a[k], 0.9999f, 1e-4f);
      else a[k] = fmaf(a[k], b, c);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += a[k];
  if (s == 1234.5f) out[threadIdx.x] = s;  // keep the work alive
}

extern "C" int qpinn_tool_fp32_peak(double* tflops_imm, double* tflops_reg, int* sms) {
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  *sms = nsm;
  float* out = nullptr;
  if (cudaMalloc(&out, 1024 * sizeof(float)) != cudaSuccess) return 1;
  const int blocks = nsm * 8, threads = 256, iters = 4096;
  const double flops = 2.0 * 16 * (double)iters * blocks * threads;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int variant = 0; variant < 2; ++variant) {
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      if (variant == 0) fma_kernel<16, true><<<blocks, threads>>>(out, iters, 0.9999f, 1e-4f);
      else fma_kernel<16, false><<<blocks, threads>>>(out, iters, 0.9999f, 1e-4f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    const double t = flops / (best * 1e-3) / 1e12;
    if (variant == 0) *tflops_imm = t; else *tflops_reg = t;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
