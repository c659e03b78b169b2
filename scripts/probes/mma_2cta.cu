// Probe: tcgen05.mma.cta_group::2 kind::tf32 with A in TMEM (the 3xTF32 GEMM's
// "ts" operand pattern on a CTA pair).  Checks the operand semantics on known
// integer data and measures the issue rate.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2506_23246_b200/csrc \
//        scripts/probes/mma_2cta.cu -o scripts/probes/mma_2cta
//
// Layout under test: M = 256 rows, CTA r holds rows 128 r .. in its TMEM lanes
// (A operand, K along columns) and its accumulator D; B (N x K, K-major, 128-byte
// swizzle) is split by rows between the CTAs' shared memory at the same offset:
// CTA r holds B rows (N/2) r ...
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_gemm.cuh"

using namespace qpinn::tc;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

constexpr int N = 128;

// A[m][k] = (m % 7) - 3 + k,  B[n][k] = (n % 5) - 2 + (k & 1)   (small integers, exact)
__host__ __device__ inline float Aval(int m, int k) { return float((m % 7) - 3 + k); }
__host__ __device__ inline float Bval(int n, int k) { return float((n % 5) - 2 + (k & 1)); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma2(int iters, float* out, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  // B half: rows n_local = 0..63 of this CTA = global rows 64 rank + n_local; K = 8 used
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) ((float*)smem)[i] = 0.f;
  __syncthreads();
  for (int i = threadIdx.x; i < (N / 2) * 8; i += blockDim.x) {
    const int nl = i / 8, k = i % 8, n = (N / 2) * rank + nl;
    const int chunk = k / 4, within = k % 4;
    const int off = (nl / 8) * 1024 + (nl % 8) * 128 + ((chunk ^ (nl % 8)) << 4) + within * 4;
    *(float*)(smem + off) = Bval(n, k);
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init_fence();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tslot)),
                 "r"(256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tslot;
  // A in TMEM columns 128..135: lane = local row, global row m = 128 rank + lane
  {
    float v[32];
    const int m = 128 * rank + warp * 32 + lane;
    for (int k = 0; k < 32; ++k) v[k] = k < 8 ? Aval(m, k) : 0.f;
    tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + 128, v);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  constexpr uint32_t idesc = idesc_tf32(256, N);
  if (rank == 0 && threadIdx.x == 0) {
    mma2_ts(tmem, tmem + 128, desc_k_sw128(smem_u32(smem)), idesc, 0);
    commit2(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  {  // D rows of this CTA: N columns
    float v[32];
    const int m = 128 * rank + warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 32) {
      tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
      for (int i = 0; i < 32; ++i) out[(size_t)m * N + c0 + i] = v[i];
    }
  }
  // rate: chains of 48 MMAs per commit
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  uint32_t ph = 1;
  if (rank == 0 && threadIdx.x == 0) {
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int c = 0; c < 48; ++c) mma2_ts(tmem, tmem + 128, desc_k_sw128(smem_u32(smem)), idesc, 1);
      commit2(&bar);
      mbar_wait(&bar, ph);
      ph ^= 1;
    }
    cyc[blockIdx.x / 2] = (unsigned long long)(clock64() - t0);
  } else if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&bar, ph);
      ph ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256)
                 : "memory");
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int pairs = sms / 2;
  float* d_out;
  unsigned long long* d_cyc;
  cudaMalloc(&d_out, (size_t)pairs * 0 + 256 * N * sizeof(float));
  cudaMalloc(&d_cyc, pairs * sizeof(unsigned long long));
  cudaFuncSetAttribute(mma2, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  const int iters = 2000;
  mma2<<<2, 128, 40 * 1024>>>(10, d_out, d_cyc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("launch: %s\n", cudaGetErrorString(e));
    return 1;
  }
  static float h[256 * N];
  cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  int bad_split = 0, bad_alt = 0;
  for (int m = 0; m < 256; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < 8; ++k) ref += (double)Aval(m, k) * Bval(n, k);
      if (h[m * N + n] != (float)ref) ++bad_split;
    }
  printf("cta_group::2 ts M=256 N=%d K=8: %d / %d mismatches (B rows split in halves by CTA)\n", N,
         bad_split, 256 * N);
  if (bad_split) {
    printf("sample D[0][0..7]:");
    for (int i = 0; i < 8; ++i) printf(" %g", h[i]);
    printf("\nsample D[128][0..7]:");
    for (int i = 0; i < 8; ++i) printf(" %g", h[128 * N + i]);
    printf("\nsample D[0][64..71]:");
    for (int i = 64; i < 72; ++i) printf(" %g", h[i]);
    printf("\n");
    (void)bad_alt;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma2<<<2 * pairs, 128, 40 * 1024>>>(iters, d_out, d_cyc);
  cudaEventRecord(e1);
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("rate launch: %s\n", cudaGetErrorString(e));
    return 1;
  }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  static unsigned long long hc[256];
  cudaMemcpy(hc, d_cyc, pairs * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < pairs; ++i) cyc += hc[i];
  cyc /= pairs;
  const double per = cyc / (iters * 48.0);
  printf("cta_group::2 ts M256 N%d chain 48: %.1f cyc/MMA  %.0f MAC/cyc/SM  %.1f TFLOP/s tf32\n", N,
         per, 256.0 * N * 8 / per / 2, 2.0 * 256 * N * 8 * iters * 48.0 * pairs / (ms * 1e-3) / 1e12);
  return 0;
}
