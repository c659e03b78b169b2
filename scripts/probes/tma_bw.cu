// Probe: HBM read bandwidth of TMA tile loads as the 3xTF32 GEMM issues them
// (tc_gemm.cu: one thread per CTA, fp32 boxes of 32 columns x ROWS rows, 128-byte
// swizzle, S stages in flight), against 1-D bulk copies of contiguous memory.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2506_23246_b200/csrc \
//        scripts/probes/tma_bw.cu -o scripts/probes/tma_bw -lcuda
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "tc_gemm.cuh"

using namespace qpinn::tc;

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// mode 0: 2-D TMA boxes (32 cols x rows), walking (row tile, k-block) like the GEMM;
// mode 1: 1-D bulk copies of `box_bytes` contiguous bytes
__global__ void __launch_bounds__(32, 1) tma_bw(const __grid_constant__ CUtensorMap map,
                                                const float* base, int mode, int rows, int K,
                                                int64_t M, int S, int box_bytes) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[16];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s) mbar_init(full + s, 1);
  mbar_init_fence();
  const int nk = K / 32;
  const int64_t n_tiles = M / rows;
  int64_t j = 0;
  if (mode == 0) {
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x)
      for (int kb = 0; kb < nk; ++kb, ++j) {
        const int s = (int)(j % S);
        if (j >= S) mbar_wait(full + s, (uint32_t)(((j / S) - 1) & 1));
        mbar_expect_tx(full + s, rows * 128);
        tma_load_2d(smem + s * box_bytes, &map, full + s, kb * 32, (int)(t * rows));
      }
  } else {
    const int64_t total = M * K * 4, n_chunks = total / box_bytes;
    for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x, ++j) {
      const int s = (int)(j % S);
      if (j >= S) mbar_wait(full + s, (uint32_t)(((j / S) - 1) & 1));
      mbar_expect_tx(full + s, box_bytes);
      bulk_load(smem + s * box_bytes, (const unsigned char*)base + c * box_bytes, box_bytes,
                full + s);
    }
  }
  for (int64_t i = (j > S ? j - S : 0); i < j; ++i) mbar_wait(full + (int)(i % S), (uint32_t)((i / S) & 1));
}

int main() {
  const int64_t M = 262144;
  const int K = 256;
  float* A;
  cudaMalloc(&A, M * K * 4);
  cudaMemset(A, 0, M * K * 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  cudaFuncSetAttribute(tma_bw, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, int mode, int rows, int S, int box, int grid) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
    cuuint64_t strides[1] = {(cuuint64_t)K * 4};
    cuuint32_t bx[2] = {32, (cuuint32_t)(rows > 256 ? 256 : rows)};
    cuuint32_t es[2] = {1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, A, dims, strides, bx, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int bb = mode == 0 ? rows * 128 : box;
    tma_bw<<<grid, 32, 200 * 1024>>>(map, A, mode, rows, K, M, S, bb);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) tma_bw<<<grid, 32, 200 * 1024>>>(map, A, mode, rows, K, M, S, bb);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-34s S=%2d grid=%3d: %6.1f us  %6.0f GB/s  %s\n", name, S, grid, ms / 5 * 1e3,
           M * K * 4.0 / (ms / 5 * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
  };
  for (int S : {3, 6, 12}) run("2-D box 32 cols x 128 rows", 0, 128, S, 0, sms);
  run("2-D box 32 cols x 256 rows", 0, 256, 6, 0, sms);
  run("2-D box 32 cols x 64 rows", 0, 64, 12, 0, sms);
  run("2-D box 32 x 128, 2 CTAs/SM", 0, 128, 6, 0, 2 * sms);
  for (int S : {3, 6, 12}) run("1-D bulk 16 KB", 1, 0, S, 16384, sms);
  run("1-D bulk 32 KB", 1, 0, 6, 32768, sms);
  return 0;
}
