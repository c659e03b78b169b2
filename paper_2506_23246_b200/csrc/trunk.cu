// Classical trunk with forward-mode x/y/t tangents: forward and reverse pass.
//
// Reference: network.py:133-147 (periodic map, frozen RFF), :284-298 (tanh
// layers + tanh adapter on BatchedDuals, tangents riding as one stacked GEMM,
// ops.py:282-298) and the tape's reverse pass through them.
//
// Activations are channel-major [4, R, width] (value, d/dx, d/dy, d/dt), so
// every dense layer is ONE GEMM [4R, in] x [in, out].  float32: the forward
// layers and the input-gradient GEMMs run on our tcgen05 3xTF32 kernels
// (tc_gemm.cu, FP32-class accuracy) with the dual tanh fused into the
// epilogue, the weight gradients as a deterministic split-K; the adapter's
// 7-wide GEMMs in the backward use cuBLAS FP32.  float64 uses cuBLAS DGEMM throughout.  Around the GEMMs:
// the feature map + RFF with tangents, the dual tanh (y = tanh(u0 + b),
// dy_k = (1 - y^2) du_k) and its reverse written on the stored outputs
// (g_u0 = g_y s - 2 y sum_k g_dy_k dy_k, g_du_k = g_dy_k s, s = 1 - y^2),
// deterministic bias column sums, and the tau gradient through the learned
// time period.
#include <cublas_v2.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "gates.cuh"
#include "tc_gemm.h"

namespace qpinn {

// ---- cuBLAS handle per device ---------------------------------------------------------
struct BlasSlot {
  cublasHandle_t h = nullptr;
  void* ws = nullptr;
};
static BlasSlot g_blas[64];
static std::mutex g_blas_mu;
constexpr size_t kBlasWorkspace = 64ull << 20;

static int blas_handle(cudaStream_t st, cublasHandle_t* out) {
  int dev = 0;
  QPINN_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_blas_mu);
  BlasSlot& b = g_blas[dev & 63];
  if (!b.h) {
    if (cublasCreate(&b.h) != CUBLAS_STATUS_SUCCESS) return fail(QPINN_ERR_CUDA, "cublasCreate");
    QPINN_CUDA_CHECK(cudaMalloc(&b.ws, kBlasWorkspace));
    cublasSetWorkspace(b.h, b.ws, kBlasWorkspace);
    cublasSetAtomicsMode(b.h, CUBLAS_ATOMICS_NOT_ALLOWED);  // deterministic reductions
  }
  if (cublasSetStream(b.h, st) != CUBLAS_STATUS_SUCCESS) return fail(QPINN_ERR_CUDA, "cublasSetStream");
  *out = b.h;
  return QPINN_OK;
}

// row-major C[M,N] = op(A) op(B) (+ beta C); op(A) is [M,K], op(B) is [K,N]
template <typename T>
static int gemm_rm(cublasHandle_t h, bool ta, bool tb, int64_t M, int64_t N, int64_t K, const T* A,
                   int64_t lda, const T* B, int64_t ldb, T* C, int64_t ldc, T beta) {
  const T alpha = T(1);
  const cudaDataType dt = sizeof(T) == 8 ? CUDA_R_64F : CUDA_R_32F;
  const cublasComputeType_t ct =
      sizeof(T) == 8 ? CUBLAS_COMPUTE_64F : CUBLAS_COMPUTE_32F_EMULATED_16BFX9;
  // column-major view: C^T[N,M] = op(B)^T op(A)^T
  auto call = [&](cublasComputeType_t c) {
    return cublasGemmEx(h, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N, (int)N,
                        (int)M, (int)K, &alpha, B, dt, (int)ldb, A, dt, (int)lda, &beta, C, dt,
                        (int)ldc, c, CUBLAS_GEMM_DEFAULT);
  };
  cublasStatus_t s = call(ct);
  if (s == CUBLAS_STATUS_NOT_SUPPORTED && sizeof(T) == 4) {
    // shapes the BF16x9 emulation does not cover run as plain FP32 (same accuracy class)
    static int logged = 0;
    if (getenv("QPINN_VERBOSE") && logged++ < 16)
      fprintf(stderr, "[qpinn] BF16x9 emulation unsupported for M=%ld N=%ld K=%ld ta=%d tb=%d: FP32\n",
              (long)M, (long)N, (long)K, (int)ta, (int)tb);
    s = call(CUBLAS_COMPUTE_32F_PEDANTIC);
  }
  if (s != CUBLAS_STATUS_SUCCESS)
    return fail(QPINN_ERR_CUDA, std::string("cublasGemmEx: ") + cublasGetStatusString(s));
  return QPINN_OK;
}

__device__ __forceinline__ void sincos_t(float x, float* s, float* c) { sincosf(x, s, c); }
__device__ __forceinline__ void sincos_t(double x, double* s, double* c) { sincos(x, s, c); }
__device__ __forceinline__ void sincospi_t(float x, float* s, float* c) { sincospif(x, s, c); }
__device__ __forceinline__ void sincospi_t(double x, double* s, double* c) { sincospi(x, s, c); }

template <typename T>
__device__ __forceinline__ T tau_of(const T* params, int64_t off_tau, T t_dom) {
  const T raw = params[off_tau];
  const T sp = raw > T(20) ? raw : log1p(exp(raw));  // softplus (network.py:292-293)
  return (T(1) + sp) * t_dom;
}

// periodic map (network.py:133-141) + RFF (network.py:144-147) with tangents.
// The per-point trig (x, y, t) is computed once per point into shared memory
// (kFeatPB points per block iteration); the (point, feature) items then stream.
constexpr int kFeatPB = 32;
template <typename T>
__global__ void __launch_bounds__(256) features_fwd(int64_t R, int F, const T* __restrict__ x,
                                                    const T* __restrict__ y, const T* __restrict__ t,
                                                    const T* __restrict__ omega,
                                                    const T* __restrict__ params, int64_t off_tau,
                                                    T t_dom, T* __restrict__ H0, int nch) {
  __shared__ T trig[kFeatPB][6];
  const T tau = tau_of(params, off_tau, t_dom);
  const T w = T(2.0 * kPi) / tau;
  const int64_t W = 2 * (int64_t)F;
  for (int64_t p0 = (int64_t)blockIdx.x * kFeatPB; p0 < R; p0 += (int64_t)gridDim.x * kFeatPB) {
    if (threadIdx.x < kFeatPB && p0 + threadIdx.x < R) {
      const int64_t p = p0 + threadIdx.x;
      T* tr = trig[threadIdx.x];
      sincospi_t(x[p], &tr[0], &tr[1]);  // x * 2 pi / lx, lx = 2
      sincospi_t(y[p], &tr[2], &tr[3]);
      const T at = (t[p] * T(2.0 * kPi)) / tau;
      sincos_t(at, &tr[4], &tr[5]);
    }
    __syncthreads();
    const int np = R - p0 < kFeatPB ? (int)(R - p0) : kFeatPB;
    for (int i = threadIdx.x; i < np * F; i += blockDim.x) {
      const int pl = i / F, f = i % F;
      const int64_t p = p0 + pl;
      const T* tr = trig[pl];
      const T sx = tr[0], cx = tr[1], sy = tr[2], cy = tr[3], st = tr[4], ct = tr[5];
      const T* om = omega + 6 * f;
      const T proj = sx * om[0] + cx * om[1] + sy * om[2] + cy * om[3] + st * om[4] + ct * om[5];
      T sp, cp;
      sincos_t(proj, &sp, &cp);
      H0[p * W + f] = cp;
      H0[p * W + F + f] = sp;
      if (nch == 1) continue;  // value only (inference)
      const T dps[3] = {T(kPi) * cx * om[0] - T(kPi) * sx * om[1],
                        T(kPi) * cy * om[2] - T(kPi) * sy * om[3], w * ct * om[4] - w * st * om[5]};
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        T* Hk = H0 + (int64_t)(k + 1) * R * W + p * W;
        Hk[f] = -sp * dps[k];
        Hk[F + f] = cp * dps[k];
      }
    }
    __syncthreads();
  }
}

// dual tanh epilogue: H[0] = tanh(U[0] + b), H[k] = (1 - H[0]^2) U[k]
template <typename T>
__global__ void tanh_fwd(int64_t R, int N, const T* __restrict__ U, const T* __restrict__ b,
                         T* __restrict__ H, int nch) {
  const int64_t n = R * N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(i % N);
    const T yv = tanh(U[i] + b[j]);
    const T s = T(1) - yv * yv;
    H[i] = yv;
    if (nch == 1) continue;
    H[n + i] = s * U[n + i];
    H[2 * n + i] = s * U[2 * n + i];
    H[3 * n + i] = s * U[3 * n + i];
  }
}

// reverse of the dual tanh on its outputs H (dy_k = s du_k):
// g_u0 = g_y s - 2 y sum_k g_dy_k dy_k, g_du_k = g_dy_k s
template <typename T>
__global__ void tanh_bwd(int64_t R, int N, const T* __restrict__ GY, const T* __restrict__ Y,
                         T* __restrict__ GU) {
  const int64_t n = R * N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T yv = Y[i];
    const T s = T(1) - yv * yv;
    const T g1 = GY[n + i], g2 = GY[2 * n + i], g3 = GY[3 * n + i];
    GU[i] = GY[i] * s + (g1 * Y[n + i] + g2 * Y[2 * n + i] + g3 * Y[3 * n + i]) * (T(-2) * yv);
    GU[n + i] = g1 * s;
    GU[2 * n + i] = g2 * s;
    GU[3 * n + i] = g3 * s;
  }
}

// tanh_bwd fused with the bias gradient: block b owns rows [b*rows_per, ...),
// thread t column t % N; the value-channel dL/du column sums of the block go
// to partial[b][N] (reduced in block order by colsum_reduce: deterministic)
template <typename T>
__global__ void tanh_bwd_bias(int64_t R, int N, int64_t rows_per, const T* __restrict__ GY,
                              const T* __restrict__ Y, T* __restrict__ GU,
                              double* __restrict__ partial) {
  extern __shared__ double red[];
  const int per = blockDim.x / N;  // rows processed together
  const int j = threadIdx.x % N, r_off = threadIdx.x / N;
  const int64_t n = R * N;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per;
  const int64_t r1 = r0 + rows_per < R ? r0 + rows_per : R;
  double acc = 0.0;
  if (r_off < per) {
    for (int64_t r = r0 + r_off; r < r1; r += per) {
      const int64_t i = r * N + j;
      const T yv = Y[i];
      const T s = T(1) - yv * yv;
      const T g1 = GY[n + i], g2 = GY[2 * n + i], g3 = GY[3 * n + i];
      const T gu = GY[i] * s + (g1 * Y[n + i] + g2 * Y[2 * n + i] + g3 * Y[3 * n + i]) * (T(-2) * yv);
      GU[i] = gu;
      GU[n + i] = g1 * s;
      GU[2 * n + i] = g2 * s;
      GU[3 * n + i] = g3 * s;
      acc += (double)gu;
    }
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < N) {
    double v = 0.0;
    for (int k = 0; k < per; ++k) v += red[k * N + threadIdx.x];
    partial[(int64_t)blockIdx.x * N + threadIdx.x] = v;
  }
}

// fp32, N % 4 == 0, N <= 256: tanh_bwd_bias with a float4 of columns per thread
// (N / 4 threads per row, 256 / (N / 4) rows per block iteration): a quarter of the
// memory instructions for the same 12 N floats per point (HBM-bound pass)
__global__ void __launch_bounds__(256) tanh_bwd_bias_v4(int64_t R, int N, int64_t rows_per,
                                                        const float* __restrict__ GY,
                                                        const float* __restrict__ Y,
                                                        float* __restrict__ GU,
                                                        double* __restrict__ partial) {
  __shared__ double red[256 * 4];
  const int tpr = N / 4;              // threads per row
  const int per = blockDim.x / tpr;   // rows per iteration
  const int c4 = threadIdx.x % tpr, r_off = threadIdx.x / tpr;
  const int64_t n = R * N;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per;
  const int64_t r1 = r0 + rows_per < R ? r0 + rows_per : R;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (r_off < per) {
#pragma unroll 2
    for (int64_t r = r0 + r_off; r < r1; r += per) {
      const int64_t i = r * N + 4 * c4;
      const float4 y0 = __ldg(reinterpret_cast<const float4*>(Y + i));
      const float4 y1 = __ldg(reinterpret_cast<const float4*>(Y + n + i));
      const float4 y2 = __ldg(reinterpret_cast<const float4*>(Y + 2 * n + i));
      const float4 y3 = __ldg(reinterpret_cast<const float4*>(Y + 3 * n + i));
      const float4 g0 = __ldg(reinterpret_cast<const float4*>(GY + i));
      const float4 g1 = __ldg(reinterpret_cast<const float4*>(GY + n + i));
      const float4 g2 = __ldg(reinterpret_cast<const float4*>(GY + 2 * n + i));
      const float4 g3 = __ldg(reinterpret_cast<const float4*>(GY + 3 * n + i));
      const float yv[4] = {y0.x, y0.y, y0.z, y0.w}, a1[4] = {y1.x, y1.y, y1.z, y1.w},
                  a2[4] = {y2.x, y2.y, y2.z, y2.w}, a3[4] = {y3.x, y3.y, y3.z, y3.w};
      const float h0[4] = {g0.x, g0.y, g0.z, g0.w}, h1[4] = {g1.x, g1.y, g1.z, g1.w},
                  h2[4] = {g2.x, g2.y, g2.z, g2.w}, h3[4] = {g3.x, g3.y, g3.z, g3.w};
      float u0[4], u1[4], u2[4], u3[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {  // the order of tanh_bwd_bias
        const float s = 1.f - yv[e] * yv[e];
        u0[e] = h0[e] * s + (h1[e] * a1[e] + h2[e] * a2[e] + h3[e] * a3[e]) * (-2.f * yv[e]);
        u1[e] = h1[e] * s;
        u2[e] = h2[e] * s;
        u3[e] = h3[e] * s;
        acc[e] += (double)u0[e];
      }
      *reinterpret_cast<float4*>(GU + i) = make_float4(u0[0], u0[1], u0[2], u0[3]);
      *reinterpret_cast<float4*>(GU + n + i) = make_float4(u1[0], u1[1], u1[2], u1[3]);
      *reinterpret_cast<float4*>(GU + 2 * n + i) = make_float4(u2[0], u2[1], u2[2], u2[3]);
      *reinterpret_cast<float4*>(GU + 3 * n + i) = make_float4(u3[0], u3[1], u3[2], u3[3]);
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) red[threadIdx.x * 4 + e] = acc[e];
  __syncthreads();
  for (int j = threadIdx.x; j < N; j += blockDim.x) {  // column j: thread (row group k, j / 4)
    double v = 0.0;
    for (int k = 0; k < per; ++k) v += red[(k * tpr + j / 4) * 4 + (j & 3)];
    partial[(int64_t)blockIdx.x * N + j] = v;
  }
}

// Adapter backward fused with the last hidden layer's reverse dual tanh:
//   GUa = reverse dual tanh of the adapter (g_act, act)           [4, R, n]
//   G_H = GUa Wa^T (n-term dot products)                          [4, R, Hd]
//   GU  = reverse dual tanh of the last hidden layer (G_H, Hl)    [4, R, Hd]
// plus block partials of dWa = Hl^T GUa, dba = sum GUa_0, db = sum GU_0 (all
// four channels of a point meet in one block; reduced later in block order).
// Replaces two library GEMMs and two elementwise passes; G_H never hits HBM.
constexpr int kAdMaxN = 16;

// NV contiguous values from 16-byte aligned shared memory with vector loads
template <typename T, int NV>
__device__ __forceinline__ void lds_vec(const T* src, T (&dst)[NV]) {
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int i = 0; i < NV / 4; ++i) {
      const float4 v = reinterpret_cast<const float4*>(src)[i];
      dst[4 * i] = v.x;
      dst[4 * i + 1] = v.y;
      dst[4 * i + 2] = v.z;
      dst[4 * i + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < NV / 2; ++i) {
      const double2 v = reinterpret_cast<const double2*>(src)[i];
      dst[2 * i] = v.x;
      dst[2 * i + 1] = v.y;
    }
  }
}
#ifndef QPINN_ADB_MINB
#define QPINN_ADB_MINB 5  // 102 registers, 5 blocks per SM: 69 -> 60 us (4 and 6-8 measured worse)
#endif
#ifndef QPINN_ADB_PB
#define QPINN_ADB_PB 8
#endif
template <typename T, int NA>
__global__ void __launch_bounds__(128, QPINN_ADB_MINB) adapter_bwd(int64_t R, int Hd, int64_t rows_per, const T* __restrict__ g_act,
                            const T* __restrict__ act, const T* __restrict__ Hl,
                            const T* __restrict__ Wa, T* __restrict__ GU,
                            double* __restrict__ part) {
  // partials: one row per block, [db (Hd) | dWa (Hd x n) | dba (n)] -- the order of
  // h_last.b, adapter.W, adapter.b in the flat parameter vector (network.py layout)
  constexpr int n = NA;
  constexpr int NAP = (NA + 3) / 4 * 4;  // padded rows: vector shared-memory loads
  __shared__ __align__(16) T gua[32][4][NAP];
  const int tid = threadIdx.x;
  const int j = tid;  // column of the hidden layer
  const bool col = j < Hd;
  const int64_t nA = R * n, nH = R * Hd;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per;
  const int64_t r1 = r0 + rows_per < R ? r0 + rows_per : R;
  T wrow[NA];
#pragma unroll
  for (int k = 0; k < NA; ++k) wrow[k] = col ? Wa[(int64_t)j * n + k] : T(0);
  T acc_w[NA];  // per-thread partials over the block's points (fixed order)
#pragma unroll
  for (int k = 0; k < NA; ++k) acc_w[k] = T(0);
  double acc_b = 0.0, acc_ba = 0.0;
  for (int64_t p0 = r0; p0 < r1; p0 += 32) {
    const int np = (int)(r1 - p0 < 32 ? r1 - p0 : 32);
    for (int idx = tid; idx < 32 * n; idx += blockDim.x) {
      const int pt = idx / n, k = idx % n;
      T g[4] = {T(0), T(0), T(0), T(0)};
      if (pt < np) {
        const int64_t i = (p0 + pt) * n + k;
        const T y0 = act[i], s = T(1) - y0 * y0;
        const T a1 = g_act[nA + i], a2 = g_act[2 * nA + i], a3 = g_act[3 * nA + i];
        g[0] = g_act[i] * s + (a1 * act[nA + i] + a2 * act[2 * nA + i] + a3 * act[3 * nA + i]) *
                                  (T(-2) * y0);
        g[1] = a1 * s;
        g[2] = a2 * s;
        g[3] = a3 * s;
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) gua[pt][c][k] = g[c];
    }
    __syncthreads();
    if (tid < n)
      for (int pt = 0; pt < np; ++pt) acc_ba += (double)gua[pt][0][tid];
    if (col) {
      // PB points at a time with their 4 PB loads issued up front (latency bound otherwise)
      constexpr int PB = QPINN_ADB_PB;
      for (int pb = 0; pb < np; pb += PB) {
        T hb[PB][4];
#pragma unroll
        for (int u = 0; u < PB; ++u)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            hb[u][c] = pb + u < np ? Hl[c * nH + (p0 + pb + u) * Hd + j] : T(0);
#pragma unroll
      for (int u = 0; u < PB; ++u) {
        const int pt = pb + u;
        if (pt >= np) break;
        const int64_t i = (p0 + pt) * Hd + j;
        T gv[4][NAP];  // the point's adapter gradients, 16-byte shared loads (broadcast)
#pragma unroll
        for (int c = 0; c < 4; ++c) lds_vec<T, NAP>(&gua[pt][c][0], gv[c]);
        T h[4], gh[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          h[c] = hb[u][c];
          T v = T(0);
#pragma unroll
          for (int k = 0; k < NA; ++k) v += gv[c][k] * wrow[k];
          gh[c] = v;
        }
        const T s = T(1) - h[0] * h[0];
        const T gu0 = gh[0] * s + (gh[1] * h[1] + gh[2] * h[2] + gh[3] * h[3]) * (T(-2) * h[0]);
        GU[i] = gu0;
        GU[nH + i] = gh[1] * s;
        GU[2 * nH + i] = gh[2] * s;
        GU[3 * nH + i] = gh[3] * s;
        acc_b += (double)gu0;
#pragma unroll
        for (int k = 0; k < NA; ++k)
          acc_w[k] += h[0] * gv[0][k] + h[1] * gv[1][k] + h[2] * gv[2][k] + h[3] * gv[3][k];
      }
      }
    }
    __syncthreads();
  }
  double* row = part + (int64_t)blockIdx.x * (Hd + Hd * n + n);
  if (col) {
    row[j] = acc_b;
#pragma unroll
    for (int k = 0; k < NA; ++k) row[Hd + (int64_t)j * n + k] = (double)acc_w[k];
  }
  if (tid < n) row[Hd + Hd * n + tid] = acc_ba;
}

// deterministic column sums of X [R, N]: block b sums rows [b*rows_per, ...)
template <typename T>
__global__ void colsum_partial(int64_t R, int N, int64_t rows_per, const T* __restrict__ X,
                               double* __restrict__ partial) {
  const int64_t r0 = (int64_t)blockIdx.x * rows_per;
  const int64_t r1 = r0 + rows_per < R ? r0 + rows_per : R;
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    double acc = 0.0;
    for (int64_t r = r0; r < r1; ++r) acc += (double)X[r * N + j];
    partial[(int64_t)blockIdx.x * N + j] = acc;
  }
}

// out[j] = sum_b partial[b][j]: a CTA owns kCsCols columns and splits the partial rows
// into blockDim / kCsCols interleaved groups (group g sums rows g, g + G, ...); the
// group sums are combined in fixed order (deterministic).  8 columns x 128 groups:
// ~5 rows per thread, all loads in flight at once, and N / 8 CTAs (with 32 columns x
// 32 groups the 592-row partials took ~8.7 us per launch, a chain of dependent loads
// on N / 32 CTAs)
constexpr int kCsCols = 8;
template <typename T>
__global__ void __launch_bounds__(1024) colsum_reduce(int nb, int N, const double* __restrict__ partial,
                                                      T* __restrict__ out, int64_t ld = 0) {
  __shared__ double red[1024 / kCsCols][kCsCols + 1];
  const int c = threadIdx.x % kCsCols, grp = threadIdx.x / kCsCols, G = blockDim.x / kCsCols;
  const int j = blockIdx.x * kCsCols + c;
  const int64_t rs = ld ? ld : N;  // partial rows ld apart (0: N)
  double acc = 0.0;
  if (j < N) {
#pragma unroll 8
    for (int b = grp; b < nb; b += G) acc += __ldg(partial + (int64_t)b * rs + j);
  }
  red[grp][c] = acc;
  __syncthreads();
  if (grp == 0 && j < N) {
    double v = 0.0;
    for (int g = 0; g < G; ++g) v += red[g][c];
    out[j] = T(v);
  }
}
constexpr int colsum_grid(int N) { return (N + kCsCols - 1) / kCsCols; }

// dL/dtau_raw through at = 2 pi t / tau and the t-tangent features (one warp per point;
// the per-point trig of a block's kFeatBPB points is computed once into shared memory)
// (cos, sin of the projections are read back from the forward's H0 value channel)
#ifndef QPINN_FEATB_RECOMP
#define QPINN_FEATB_RECOMP 1  // 81 vs 88 us: the pass is latency-bound, the trig is cheaper than the loads
#endif
constexpr int kFeatBPB = 64;
#ifndef QPINN_FEATB_UNROLL
#define QPINN_FEATB_UNROLL 2  // with the 4-deep feature loop: 89 vs 95 us (measured)
#endif
constexpr int kFeatBUnroll = QPINN_FEATB_UNROLL;
template <typename T>
__global__ void __launch_bounds__(256) features_bwd(int64_t R, int F, const T* __restrict__ x,
                                                    const T* __restrict__ y, const T* __restrict__ t,
                                                    const T* __restrict__ omega,
                                                    const T* __restrict__ params, int64_t off_tau,
                                                    T t_dom, const T* __restrict__ H0,
                                                    const T* __restrict__ G0,
                                                    double* __restrict__ partial) {
  __shared__ T trig[kFeatBPB][7];
  const T tau = tau_of(params, off_tau, t_dom);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
  const int64_t W = 2 * (int64_t)F;
  const T w = T(2.0 * kPi) / tau;
  double acc = 0.0;
  for (int64_t p0 = (int64_t)blockIdx.x * kFeatBPB; p0 < R; p0 += (int64_t)gridDim.x * kFeatBPB) {
    if (threadIdx.x < kFeatBPB && p0 + threadIdx.x < R) {
      const int64_t p = p0 + threadIdx.x;
      T* tr = trig[threadIdx.x];
      sincospi_t(x[p], &tr[0], &tr[1]);
      sincospi_t(y[p], &tr[2], &tr[3]);
      const T at = (t[p] * T(2.0 * kPi)) / tau;
      sincos_t(at, &tr[4], &tr[5]);
      tr[6] = at;
    }
    __syncthreads();
#pragma unroll kFeatBUnroll
    for (int pl = warp; pl < kFeatBPB && p0 + pl < R; pl += warps) {
      const int64_t p = p0 + pl;
      const T* tr = trig[pl];
      const T sx = tr[0], cx = tr[1], sy = tr[2], cy = tr[3], st = tr[4], ct = tr[5], at = tr[6];
      T G4 = 0, G5 = 0, D4 = 0, D5 = 0;
#pragma unroll 4
      for (int f = lane; f < F; f += 32) {
        const T* om = omega + 6 * f;
        const T dps[3] = {T(kPi) * cx * om[0] - T(kPi) * sx * om[1],
                          T(kPi) * cy * om[2] - T(kPi) * sy * om[3], w * ct * om[4] - w * st * om[5]};
#if QPINN_FEATB_RECOMP
        // cos/sin of the projection recomputed (as features_fwd) instead of read back
        const T proj = sx * om[0] + cx * om[1] + sy * om[2] + cy * om[3] + st * om[4] + ct * om[5];
        T sp, cp;
        sincos_t(proj, &sp, &cp);
#else
        const T cp = H0[p * W + f], sp = H0[p * W + F + f];
#endif
        const T gc = G0[p * W + f], gs = G0[p * W + F + f];
        T gproj = -sp * gc + cp * gs, gdp2 = 0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const T* Gk = G0 + (int64_t)(k + 1) * R * W + p * W;
          const T gdc = Gk[f], gds = Gk[F + f];
          gproj += -cp * dps[k] * gdc - sp * dps[k] * gds;
          if (k == 2) gdp2 = -sp * gdc + cp * gds;
        }
        G4 += gproj * om[4];
        G5 += gproj * om[5];
        D4 += gdp2 * om[4];
        D5 += gdp2 * om[5];
      }
      // gt is linear in the feature sums, so each lane folds its partial sums with
      // the point's coefficients and the warp reduces once, after the last point
      const T dat = -at / tau;
      const T w2 = T(2.0 * kPi) / (tau * tau);
      const T gt = G4 * ct * dat + G5 * (-st) * dat + D4 * (-w2 * ct + w2 * at * st) +
                   D5 * (w2 * st + w2 * at * ct);
      acc += (double)gt;
    }
    __syncthreads();
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
  __shared__ double red[32];
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w3 = 0; w3 < warps; ++w3) v += red[w3];
    partial[blockIdx.x] = v;
  }
}

// fp32, F = 128 NC: the same two passes with a warp per point and a lane per 4
// consecutive features of each 128-feature chunk, so every H0 / G0 row moves as 16-byte
// vectors (HBM-bound passes; the scalar versions above issue 4x the memory instructions).
// The lane's omega rows stay in registers across points.
template <int NC>
__global__ void __launch_bounds__(256) features_fwd_v4(int64_t R, int F, const float* __restrict__ x,
                                                       const float* __restrict__ y,
                                                       const float* __restrict__ t,
                                                       const float* __restrict__ omega,
                                                       const float* __restrict__ params,
                                                       int64_t off_tau, float t_dom,
                                                       float* __restrict__ H0, int nch) {
  __shared__ float trig[kFeatPB][6];
  const float tau = tau_of(params, off_tau, t_dom);
  const float w = float(2.0 * kPi) / tau;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t W = 2 * (int64_t)F;
  float om[NC][4][6];
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
      for (int j = 0; j < 6; ++j) om[c][e][j] = __ldg(omega + 6 * (128 * c + 4 * lane + e) + j);
  for (int64_t p0 = (int64_t)blockIdx.x * kFeatPB; p0 < R; p0 += (int64_t)gridDim.x * kFeatPB) {
    if (threadIdx.x < kFeatPB && p0 + threadIdx.x < R) {
      const int64_t p = p0 + threadIdx.x;
      float* tr = trig[threadIdx.x];
      sincospif(x[p], &tr[0], &tr[1]);
      sincospif(y[p], &tr[2], &tr[3]);
      sincosf((t[p] * float(2.0 * kPi)) / tau, &tr[4], &tr[5]);
    }
    __syncthreads();
    for (int pl = warp; pl < kFeatPB && p0 + pl < R; pl += 8) {
      const int64_t p = p0 + pl;
      const float* tr = trig[pl];
      const float sx = tr[0], cx = tr[1], sy = tr[2], cy = tr[3], st = tr[4], ct = tr[5];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        float cp[4], sp[4], dps[3][4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float* o = om[c][e];
          const float proj = sx * o[0] + cx * o[1] + sy * o[2] + cy * o[3] + st * o[4] + ct * o[5];
          sincosf(proj, &sp[e], &cp[e]);
          dps[0][e] = float(kPi) * cx * o[0] - float(kPi) * sx * o[1];
          dps[1][e] = float(kPi) * cy * o[2] - float(kPi) * sy * o[3];
          dps[2][e] = w * ct * o[4] - w * st * o[5];
        }
        const int64_t f0 = 128 * c + 4 * lane;
        float* row = H0 + p * W;
        *reinterpret_cast<float4*>(row + f0) = make_float4(cp[0], cp[1], cp[2], cp[3]);
        *reinterpret_cast<float4*>(row + F + f0) = make_float4(sp[0], sp[1], sp[2], sp[3]);
        if (nch == 1) continue;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          float* rk = H0 + (int64_t)(k + 1) * R * W + p * W;
          *reinterpret_cast<float4*>(rk + f0) =
              make_float4(-sp[0] * dps[k][0], -sp[1] * dps[k][1], -sp[2] * dps[k][2], -sp[3] * dps[k][3]);
          *reinterpret_cast<float4*>(rk + F + f0) =
              make_float4(cp[0] * dps[k][0], cp[1] * dps[k][1], cp[2] * dps[k][2], cp[3] * dps[k][3]);
        }
      }
    }
    __syncthreads();
  }
}

#ifndef QPINN_FB4_MINB
#define QPINN_FB4_MINB 3  // 85 registers: 65 -> 62 us (4: 66 us)
#endif
template <int NC>
__global__ void __launch_bounds__(256, QPINN_FB4_MINB) features_bwd_v4(int64_t R, int F, const float* __restrict__ x,
                                                       const float* __restrict__ y,
                                                       const float* __restrict__ t,
                                                       const float* __restrict__ omega,
                                                       const float* __restrict__ params,
                                                       int64_t off_tau, float t_dom,
                                                       const float* __restrict__ G0,
                                                       double* __restrict__ partial) {
  __shared__ float trig[kFeatBPB][7];
  const float tau = tau_of(params, off_tau, t_dom);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t W = 2 * (int64_t)F;
  const float w = float(2.0 * kPi) / tau;
  float om[NC][4][6];
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
      for (int j = 0; j < 6; ++j) om[c][e][j] = __ldg(omega + 6 * (128 * c + 4 * lane + e) + j);
  double acc = 0.0;
  for (int64_t p0 = (int64_t)blockIdx.x * kFeatBPB; p0 < R; p0 += (int64_t)gridDim.x * kFeatBPB) {
    if (threadIdx.x < kFeatBPB && p0 + threadIdx.x < R) {
      const int64_t p = p0 + threadIdx.x;
      float* tr = trig[threadIdx.x];
      sincospif(x[p], &tr[0], &tr[1]);
      sincospif(y[p], &tr[2], &tr[3]);
      const float at = (t[p] * float(2.0 * kPi)) / tau;
      sincosf(at, &tr[4], &tr[5]);
      tr[6] = at;
    }
    __syncthreads();
#pragma unroll 2
    for (int pl = warp; pl < kFeatBPB && p0 + pl < R; pl += 8) {
      const int64_t p = p0 + pl;
      const float* tr = trig[pl];
      const float sx = tr[0], cx = tr[1], sy = tr[2], cy = tr[3], st = tr[4], ct = tr[5], at = tr[6];
      float G4 = 0.f, G5 = 0.f, D4 = 0.f, D5 = 0.f;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int64_t f0 = 128 * c + 4 * lane;
        float4 gv[4][2];  // [channel][cos half, sin half]
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float* rk = G0 + (int64_t)k * R * W + p * W;
          gv[k][0] = __ldg(reinterpret_cast<const float4*>(rk + f0));
          gv[k][1] = __ldg(reinterpret_cast<const float4*>(rk + F + f0));
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float* o = om[c][e];
          const float dps[3] = {float(kPi) * cx * o[0] - float(kPi) * sx * o[1],
                                float(kPi) * cy * o[2] - float(kPi) * sy * o[3],
                                w * ct * o[4] - w * st * o[5]};
          const float proj = sx * o[0] + cx * o[1] + sy * o[2] + cy * o[3] + st * o[4] + ct * o[5];
          float sp, cp;
          sincosf(proj, &sp, &cp);
          const float* g0c = &gv[0][0].x;
          const float* g0s = &gv[0][1].x;
          float gproj = -sp * g0c[e] + cp * g0s[e], gdp2 = 0.f;
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const float gdc = (&gv[k + 1][0].x)[e], gds = (&gv[k + 1][1].x)[e];
            gproj += -cp * dps[k] * gdc - sp * dps[k] * gds;
            if (k == 2) gdp2 = -sp * gdc + cp * gds;
          }
          G4 += gproj * o[4];
          G5 += gproj * o[5];
          D4 += gdp2 * o[4];
          D5 += gdp2 * o[5];
        }
      }
      const float dat = -at / tau;
      const float w2 = float(2.0 * kPi) / (tau * tau);
      const float gt = G4 * ct * dat + G5 * (-st) * dat + D4 * (-w2 * ct + w2 * at * st) +
                       D5 * (w2 * st + w2 * at * ct);
      acc += (double)gt;
    }
    __syncthreads();
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
  __shared__ double red[8];
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w3 = 0; w3 < 8; ++w3) v += red[w3];
    partial[blockIdx.x] = v;
  }
}

// one block: strided per-thread sums, then a fixed-order tree (deterministic)
template <typename T>
__global__ void tau_grad_reduce(int nb, const double* __restrict__ partial, const T* __restrict__ params,
                                int64_t off_tau, T t_dom, T* __restrict__ grad) {
  __shared__ double red[256];
  double v = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) v += partial[b];
  red[threadIdx.x] = v;
  __syncthreads();
  for (int m = blockDim.x / 2; m > 0; m >>= 1) {
    if (threadIdx.x < m) red[threadIdx.x] += red[threadIdx.x + m];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double raw = (double)params[off_tau];
    const double sig = 0.5 * (1.0 + tanh(0.5 * raw));  // d softplus / d raw
    grad[off_tau] = T(red[0] * (double)t_dom * sig);
  }
}

// ---- workspace plan ----------------------------------------------------------------------------
struct TrunkWS {
  size_t h0, u, h[8], g0, g1, part, apart, tau_part, wcache, wsplit, total;
};

// float32: every dense layer's weights split into tf32 hi / lo once per forward (one
// split_weights launch), in the two layouts the GEMMs take: forward B = W^T [H, K_in]
// and input-gradient B = W [K_in, H]; the backward reuses the forward's splits (it
// already requires the forward's activations in the same workspace)
struct WCache {
  tc::Wsplit fwd[8], bwd[8], ad;
};

static size_t wcache_bytes(const qpinn_trunk_desc* d) {
  size_t b = 0;
  const int H = d->hidden;
  for (int i = 0; i < d->n_hidden; ++i) {
    const int K = i == 0 ? 2 * d->rff : H;
    b += 2 * ((size_t)H * tc::split_ldk(K) + (size_t)K * tc::split_ldk(H)) * 4;
  }
  const int Kl = d->n_hidden ? H : 2 * d->rff;
  b += 2 * (size_t)d->n_out * tc::split_ldk(Kl) * 4;
  return b + 256;
}

// carve the cache and, when jobs is given, list the splits that fill it
static WCache wcache_of(const qpinn_trunk_desc* d, unsigned char* base, const float* params,
                        tc::SplitJob* jobs, int* njobs) {
  WCache c{};
  float* o = (float*)(((uintptr_t)base + 255) & ~(uintptr_t)255);
  const int H = d->hidden;
  int nj = 0;
  auto take = [&](int N, int K, const float* src, int transpose, int64_t ld) {
    const int ldk = tc::split_ldk(K);
    float* hi = o;
    float* lo = o + (size_t)N * ldk;
    o = lo + (size_t)N * ldk;
    if (jobs) jobs[nj++] = tc::SplitJob{src, N, K, transpose, ldk, ld, hi, lo};
    return tc::Wsplit{hi, lo, ldk};
  };
  for (int i = 0; i < d->n_hidden; ++i) {
    const int K = i == 0 ? 2 * d->rff : H;
    const float* W = params + d->off_w[i];  // [K, H] row-major
    c.fwd[i] = take(H, K, W, 1, H);
    c.bwd[i] = take(K, H, W, 0, H);
  }
  const int Kl = d->n_hidden ? H : 2 * d->rff;
  c.ad = take(d->n_out, Kl, params + d->off_adapter_w, 1, d->n_out);
  if (njobs) *njobs = nj;
  return c;
}

constexpr int kColBlocks = 256;
constexpr int kTanhBlocks = 592;  // 4 per SM for the fused reverse dual tanh
constexpr int kAdBlocks = 592;    // fused adapter backward (4 per SM)
constexpr int kTauBlocks = 1184;  // 8 per SM: the tau pass is latency bound

static TrunkWS trunk_ws(const qpinn_trunk_desc* d, size_t es, int64_t R) {
  TrunkWS w{};
  size_t o = 0;
  auto take = [&](size_t n) {
    size_t at = o;
    o += (n * es + 255) / 256 * 256;
    return at;
  };
  const size_t F2 = 2 * (size_t)d->rff, H = d->hidden;
  w.h0 = take(4 * R * F2);
  // GEMM output before the dual tanh (cuBLAS layers: float64, unaligned float32 widths)
  w.u = take(4 * R * (H > (size_t)d->n_out ? H : d->n_out));
  for (int i = 0; i < d->n_hidden; ++i) w.h[i] = take(4 * R * H);
  const size_t gmax = 4 * R * (F2 > H ? F2 : H);
  w.g0 = take(gmax);
  w.g1 = take(gmax);
  w.part = o;
  o += ((size_t)(kColBlocks > kTanhBlocks ? kColBlocks : kTanhBlocks) *
            (H > (size_t)d->n_out ? H : d->n_out) * 8 + 255) / 256 * 256;
  w.apart = o;  // adapter backward partials: [blocks][Hd * n + Hd + n] doubles
  o += ((size_t)kAdBlocks * (H * d->n_out + H + d->n_out) * 8 + 255) / 256 * 256;
  w.tau_part = o;
  o += (kTauBlocks * 8 + 255) / 256 * 256;
  w.wcache = o;
  if (es == 4) o += (wcache_bytes(d) + 255) / 256 * 256;
  // float32 tensor-core scratch, used by one GEMM at a time: the tf32 hi/lo
  // split of a weight matrix, or the split-K partials of a weight gradient
  w.wsplit = o;
  if (es == 4) {
    const int KM = (int)(F2 > H ? F2 : H);
    size_t b = tc::gemm3_workspace_bytes(KM, KM);
    const size_t b1 = tc::wgrad_workspace_bytes(4 * R, (int)F2, (int)H);
    const size_t b2 = tc::wgrad_workspace_bytes(4 * R, (int)H, (int)H);
    b = b > b1 ? b : b1;
    o += (b > b2 ? b : b2);
  }
  w.total = o;
  return w;
}

static int grid_1d(int64_t n) {
  int64_t g = (n + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  return (int)(g < 1 ? 1 : g > cap ? cap : g);
}

template <typename T>
static int bias_grad(int64_t R, int N, const T* GU0, double* part, T* out, cudaStream_t st);

// QPINN_TANH_V4=0: the scalar reverse dual tanh (A/B experiments)
static bool tanh_v4_off() {
  static const bool off = [] {
    const char* e = getenv("QPINN_TANH_V4");
    return e && atoi(e) == 0;
  }();
  return off;
}

// GU = reverse dual tanh (GY, Y) and out = column sums of GU's value channel
template <typename T>
static int tanh_bwd_and_bias(int64_t R, int N, const T* GY, const T* Y, T* GU, double* part,
                             T* out, cudaStream_t st) {
  const int threads = N <= 256 ? (256 / N) * N : 0;
  if (threads == 0) {  // wide layers: separate kernels
    tanh_bwd<T><<<grid_1d(R * N), 256, 0, st>>>(R, N, GY, Y, GU);
    QPINN_CUDA_CHECK(cudaGetLastError());
    return bias_grad<T>(R, N, GU, part, out, st);
  }
  const int64_t rows_per = (R + kTanhBlocks - 1) / kTanhBlocks;
  const int nb = (int)((R + rows_per - 1) / rows_per);
  if (sizeof(T) == 4 && N % 4 == 0 && !tanh_v4_off()) {
    tanh_bwd_bias_v4<<<nb, 256, 0, st>>>(R, N, rows_per, (const float*)GY, (const float*)Y,
                                         (float*)GU, part);
  } else {
    tanh_bwd_bias<T><<<nb, threads, threads * sizeof(double), st>>>(R, N, rows_per, GY, Y, GU,
                                                                    part);
  }
  colsum_reduce<T><<<colsum_grid(N), 1024, 0, st>>>(nb, N, part, out);
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

template <typename T>
static int bias_grad(int64_t R, int N, const T* GU0, double* part, T* out, cudaStream_t st) {
  const int64_t rows_per = (R + kColBlocks - 1) / kColBlocks;
  const int nb = (int)((R + rows_per - 1) / rows_per);
  colsum_partial<T><<<nb, N < 128 ? 32 * ((N + 31) / 32) : 128, 0, st>>>(R, N, rows_per, GU0, part);
  colsum_reduce<T><<<colsum_grid(N), 1024, 0, st>>>(nb, N, part, out);
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

// QPINN_FEAT_V4=0: the scalar feature passes (A/B experiments)
static bool feat_v4_off() {
  static const bool off = [] {
    const char* e = getenv("QPINN_FEAT_V4");
    return e && atoi(e) == 0;
  }();
  return off;
}

// QPINN_FUSE_ADAPTER=0: the adapter as its own tensor-core layer (A/B experiments)
static bool adapter_fusion_off() {
  static const bool off = [] {
    const char* e = getenv("QPINN_FUSE_ADAPTER");
    return e && atoi(e) == 0;
  }();
  return off;
}

template <typename T>
static int forward_impl(const qpinn_trunk_desc* d, int64_t R, const T* x, const T* y, const T* t,
                        const T* params, T* act, unsigned char* ws, cudaStream_t st,
                        int nch = 4) {
  const TrunkWS w = trunk_ws(d, sizeof(T), R);
  const int F = d->rff, H = d->hidden, n = d->n_out;
  T* H0 = (T*)(ws + w.h0);
  const int fb = (int)((R + kFeatPB - 1) / kFeatPB < num_sms() * 8 ? (R + kFeatPB - 1) / kFeatPB
                                                                   : num_sms() * 8);
  if (sizeof(T) == 4 && (F == 128 || F == 256) && !feat_v4_off()) {
    auto kern = F == 128 ? features_fwd_v4<1> : features_fwd_v4<2>;
    kern<<<fb > 0 ? fb : 1, 256, 0, st>>>(R, F, (const float*)x, (const float*)y, (const float*)t,
                                          (const float*)d->omega, (const float*)params,
                                          d->off_tau_raw, (float)d->t_domain, (float*)H0, nch);
  } else {
    features_fwd<T><<<fb > 0 ? fb : 1, 256, 0, st>>>(R, F, x, y, t, (const T*)d->omega, params,
                                                    d->off_tau_raw, (T)d->t_domain, H0, nch);
  }
  QPINN_CUDA_CHECK(cudaGetLastError());
  const T* in = H0;
  int K = 2 * F;
  cublasHandle_t h;
  if (int rc = blas_handle(st, &h)) return rc;
  T* U = (T*)(ws + w.u);
  WCache wc{};
  if constexpr (sizeof(T) == 4) {  // this forward's weight splits, one launch
    tc::SplitJob jobs[tc::kMaxSplitJobs];
    int nj = 0;
    wc = wcache_of(d, ws + w.wcache, (const float*)params, jobs, &nj);
    if (int rc = tc::split_weights(jobs, nj, st)) return rc;
  }
  // one dense layer + dual tanh: tensor cores (float32, 16-byte aligned rows) or cuBLAS
  auto dense = [&](int Kin, int N, const T* X, int64_t off_w, int64_t off_b, T* out,
                   const tc::Wsplit* pre) -> int {
    if constexpr (sizeof(T) == 4) {
      if (Kin % 4 == 0)
        return nch == 4 ? tc::dense_tanh(R, N, Kin, X, params + off_w, params + off_b, out,
                                         ws + w.wsplit, w.total - w.wsplit, st, pre)
                        : tc::dense_tanh1(R, N, Kin, X, params + off_w, params + off_b, out,
                                          ws + w.wsplit, w.total - w.wsplit, st, pre);
    }
    if (int rc = gemm_rm<T>(h, false, false, nch * R, N, Kin, X, Kin, params + off_w, N, U, N,
                            T(0)))
      return rc;
    tanh_fwd<T><<<grid_1d(R * N), 256, 0, st>>>(R, N, U, params + off_b, out, nch);
    QPINN_CUDA_CHECK(cudaGetLastError());
    return QPINN_OK;
  };
  // the tanh adapter (128 -> n) rides in the last hidden layer's epilogue when
  // that layer runs on the tensor cores with a single N-tile
  bool fuse_adapter = false;
  if constexpr (sizeof(T) == 4)
    fuse_adapter = nch == 4 && d->n_hidden > 0 && H <= 128 && H % 4 == 0 && n <= 8 &&
                   !adapter_fusion_off();
  for (int i = 0; i < d->n_hidden; ++i) {
    T* Hn = (T*)(ws + w.h[i]);
    if constexpr (sizeof(T) == 4) {
      if (fuse_adapter && i == d->n_hidden - 1 && K % 4 == 0)
        return tc::dense_tanh_adapter(R, H, K, (const float*)in, params + d->off_w[i],
                                      params + d->off_b[i], Hn, params + d->off_adapter_w,
                                      params + d->off_adapter_b, n, act, ws + w.wsplit,
                                      w.total - w.wsplit, st, &wc.fwd[i]);
    }
    if (int rc = dense(K, H, in, d->off_w[i], d->off_b[i], Hn, &wc.fwd[i])) return rc;
    in = Hn;
    K = H;
  }
  return dense(K, n, in, d->off_adapter_w, d->off_adapter_b, act, &wc.ad);
}

template <typename T>
static int backward_impl(const qpinn_trunk_desc* d, int64_t R, const T* x, const T* y, const T* t,
                         const T* params, const T* act, const T* g_act, T* grad, unsigned char* ws,
                         cudaStream_t st) {
  const TrunkWS w = trunk_ws(d, sizeof(T), R);
  cublasHandle_t h;
  if (int rc = blas_handle(st, &h)) return rc;
  const int F = d->rff, H = d->hidden, n = d->n_out;
  double* part = (double*)(ws + w.part);
  T* g0 = (T*)(ws + w.g0);
  T* g1 = (T*)(ws + w.g1);
  // adapter: GU = tanh_bwd(g_act); dWa = H_last^T GU; dba = colsum(GU0); G_H = GU Wa^T
  const T* Hl = (const T*)(ws + (d->n_hidden ? w.h[d->n_hidden - 1] : w.h0));
  const int Kl = d->n_hidden ? H : 2 * F;
  const bool fused = d->n_hidden > 0 && n <= kAdMaxN && H <= 128;
  if (fused) {  // adapter + last hidden layer's reverse dual tanh in one pass (g1 = its dL/dU)
    double* pa = (double*)(ws + w.apart);  // [blocks][H + H n + n]
    const int W = H + H * n + n;
    const int64_t rows_per = (R + kAdBlocks - 1) / kAdBlocks;
    const int nb = (int)((R + rows_per - 1) / rows_per);
    const int thr = (H + 31) / 32 * 32;
    const T* Wa = params + d->off_adapter_w;
    switch (n) {
#define QPINN_AD(NN)                                                                        \
  case NN:                                                                                  \
    adapter_bwd<T, NN><<<nb, thr, 0, st>>>(R, H, rows_per, g_act, act, Hl, Wa, g1, pa); \
    break;
      QPINN_AD(1) QPINN_AD(2) QPINN_AD(3) QPINN_AD(4) QPINN_AD(5) QPINN_AD(6) QPINN_AD(7)
      QPINN_AD(8) QPINN_AD(9) QPINN_AD(10) QPINN_AD(11) QPINN_AD(12) QPINN_AD(13)
      QPINN_AD(14) QPINN_AD(15) QPINN_AD(16)
#undef QPINN_AD
    }
    const int ob = d->off_b[d->n_hidden - 1];
    if (d->off_adapter_w == ob + H && d->off_adapter_b == ob + H + H * n) {  // contiguous
      colsum_reduce<T><<<colsum_grid(W), 1024, 0, st>>>(nb, W, pa, grad + ob);
    } else {
      colsum_reduce<T><<<colsum_grid(H), 1024, 0, st>>>(nb, H, pa, grad + ob, W);
      colsum_reduce<T><<<colsum_grid(H * n), 1024, 0, st>>>(nb, H * n, pa + H,
                                                          grad + d->off_adapter_w, W);
      colsum_reduce<T><<<colsum_grid(n), 1024, 0, st>>>(nb, n, pa + H + H * n,
                                                      grad + d->off_adapter_b, W);
    }
    QPINN_CUDA_CHECK(cudaGetLastError());
  } else {
    if (int rc = tanh_bwd_and_bias<T>(R, n, g_act, act, g1, part, grad + d->off_adapter_b, st))
      return rc;
    if (int rc = gemm_rm<T>(h, true, false, Kl, n, 4 * R, Hl, Kl, g1, n, grad + d->off_adapter_w,
                            n, T(0)))
      return rc;
    if (int rc = gemm_rm<T>(h, false, true, 4 * R, Kl, n, g1, n, params + d->off_adapter_w, n, g0,
                            Kl, T(0)))
      return rc;
  }
  // hidden layers, last to first; g0 holds dL/dH_{i+1} (g1 already dL/dU_i when fused)
  for (int i = d->n_hidden - 1; i >= 0; --i) {
    const int K = i == 0 ? 2 * F : H;
    const T* Hin = (const T*)(ws + (i == 0 ? w.h0 : w.h[i - 1]));
    if (!(fused && i == d->n_hidden - 1)) {
      if (int rc = tanh_bwd_and_bias<T>(R, H, g0, (const T*)(ws + w.h[i]), g1, part,
                                        grad + d->off_b[i], st))
        return rc;
    }
    if (sizeof(T) == 4 && K % 4 == 0 && H % 4 == 0) {  // dW = H_in^T GU on the tensor cores
      if (int rc = tc::wgrad(4 * R, K, H, (const float*)Hin, K, (const float*)g1, H,
                             (float*)(grad + d->off_w[i]), ws + w.wsplit, w.total - w.wsplit, st))
        return rc;
    } else if (int rc = gemm_rm<T>(h, true, false, K, H, 4 * R, Hin, K, g1, H, grad + d->off_w[i],
                                   H, T(0))) {
      return rc;
    }
    if (sizeof(T) == 4 && H % 4 == 0) {  // dL/dH_in = GU W^T on the tensor cores
      const WCache wc = wcache_of(d, ws + w.wcache, (const float*)params, nullptr, nullptr);
      if (int rc = tc::gemm3(4 * R, K, H, (const float*)g1, H, (const float*)(params + d->off_w[i]),
                             H, (float*)g0, K, ws + w.wsplit, w.total - w.wsplit, st, &wc.bwd[i]))
        return rc;
    } else if (int rc = gemm_rm<T>(h, false, true, 4 * R, K, H, g1, H, params + d->off_w[i], H, g0,
                                   K, T(0))) {
      return rc;
    }
  }
  // tau_raw through the time features
  double* tp = (double*)(ws + w.tau_part);
  if (sizeof(T) == 4 && (F == 128 || F == 256) && !feat_v4_off()) {
    auto kern = F == 128 ? features_bwd_v4<1> : features_bwd_v4<2>;
    kern<<<kTauBlocks, 256, 0, st>>>(R, F, (const float*)x, (const float*)y, (const float*)t,
                                     (const float*)d->omega, (const float*)params,
                                     d->off_tau_raw, (float)d->t_domain, (const float*)g0, tp);
  } else {
    features_bwd<T><<<kTauBlocks, 256, 0, st>>>(R, F, x, y, t, (const T*)d->omega, params,
                                                 d->off_tau_raw, (T)d->t_domain,
                                                 (const T*)(ws + w.h0), g0, tp);
  }
  tau_grad_reduce<T><<<1, 256, 0, st>>>(kTauBlocks, tp, params, d->off_tau_raw, (T)d->t_domain, grad);
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

static int check_desc(const qpinn_trunk_desc* d, int dtype) {
  if (!d) return fail(QPINN_ERR_CONFIG, "null trunk descriptor");
  if (dtype != QPINN_F32 && dtype != QPINN_F64) return fail(QPINN_ERR_CONFIG, "bad dtype");
  if (d->n_hidden < 0 || d->n_hidden > 8 || d->rff < 1 || d->hidden < 1 || d->n_out < 1 || !d->omega)
    return fail(QPINN_ERR_CONFIG, "bad trunk descriptor");
  return QPINN_OK;
}

}  // namespace qpinn

using namespace qpinn;

extern "C" {

size_t qpinn_trunk_workspace_bytes(const qpinn_trunk_desc* d, int dtype, int64_t rows) {
  if (!d || rows < 0) return 0;
  return trunk_ws(d, dtype == QPINN_F64 ? 8 : 4, rows).total;
}

int qpinn_trunk_forward(const qpinn_trunk_desc* d, int dtype, int64_t rows, const void* x,
                        const void* y, const void* t, const void* params, void* act,
                        void* workspace, size_t workspace_bytes, void* stream) {
  if (int rc = check_desc(d, dtype)) return rc;
  if (workspace_bytes < qpinn_trunk_workspace_bytes(d, dtype, rows))
    return fail(QPINN_ERR_CONFIG, "trunk workspace too small");
  if (rows <= 0) return QPINN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == QPINN_F32)
    return forward_impl<float>(d, rows, (const float*)x, (const float*)y, (const float*)t,
                               (const float*)params, (float*)act, (unsigned char*)workspace, st);
  return forward_impl<double>(d, rows, (const double*)x, (const double*)y, (const double*)t,
                              (const double*)params, (double*)act, (unsigned char*)workspace, st);
}

int qpinn_trunk_forward_value(const qpinn_trunk_desc* d, int dtype, int64_t rows, const void* x,
                              const void* y, const void* t, const void* params, void* act,
                              void* workspace, size_t workspace_bytes, void* stream) {
  if (int rc = check_desc(d, dtype)) return rc;
  if (workspace_bytes < qpinn_trunk_workspace_bytes(d, dtype, rows))
    return fail(QPINN_ERR_CONFIG, "trunk workspace too small");
  if (rows <= 0) return QPINN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == QPINN_F32)
    return forward_impl<float>(d, rows, (const float*)x, (const float*)y, (const float*)t,
                               (const float*)params, (float*)act, (unsigned char*)workspace, st, 1);
  return forward_impl<double>(d, rows, (const double*)x, (const double*)y, (const double*)t,
                              (const double*)params, (double*)act, (unsigned char*)workspace, st,
                              1);
}

int qpinn_trunk_backward(const qpinn_trunk_desc* d, int dtype, int64_t rows, const void* x,
                         const void* y, const void* t, const void* params, const void* act,
                         const void* g_act, void* grad, void* workspace, size_t workspace_bytes,
                         void* stream) {
  if (int rc = check_desc(d, dtype)) return rc;
  if (workspace_bytes < qpinn_trunk_workspace_bytes(d, dtype, rows))
    return fail(QPINN_ERR_CONFIG, "trunk workspace too small");
  if (rows <= 0) return QPINN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == QPINN_F32)
    return backward_impl<float>(d, rows, (const float*)x, (const float*)y, (const float*)t,
                                (const float*)params, (const float*)act, (const float*)g_act,
                                (float*)grad, (unsigned char*)workspace, st);
  return backward_impl<double>(d, rows, (const double*)x, (const double*)y, (const double*)t,
                               (const double*)params, (const double*)act, (const double*)g_act,
                               (double*)grad, (unsigned char*)workspace, st);
}

}  // extern "C"
