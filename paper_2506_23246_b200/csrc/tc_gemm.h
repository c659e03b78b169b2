// Host entry points of the tensor-core trunk GEMMs (tc_gemm.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace qpinn {
namespace tc {
// a weight operand already split into tf32 hi / lo parts, [N, ldk] each (ldk = K rounded
// up to 4, zero padded): passed as `pre`, the GEMM skips its own split kernel
struct Wsplit {
  const float* hi;
  const float* lo;
  int ldk;
};
// one split of a batched split_weights launch: B = src [N, K] (ld) or, with transpose,
// B = src^T for src [K, N] row-major (ld = N); writes hi / lo [N, ldk]
struct SplitJob {
  const float* src;
  int N, K, transpose, ldk;
  int64_t ld;
  float* hi;
  float* lo;
};
constexpr int kMaxSplitJobs = 20;
inline int split_ldk(int K) { return (K + 3) & ~3; }
int split_weights(const SplitJob* jobs, int njobs, cudaStream_t st);
size_t gemm3_workspace_bytes(int N, int K);
// C[M,N] = A[M,K] B[N,K]^T (fp32, 3xTF32 tensor cores)
int gemm3(int64_t M, int N, int K, const float* A, int64_t lda, const float* B, int64_t ldb,
          float* C, int64_t ldc, void* ws, size_t ws_bytes, cudaStream_t st,
          const Wsplit* pre = nullptr);
// Psi [4R, 256] = Phi [4R, 128] Wt[256, 128]^T with the fused n = 7 Pauli-Z readout
// z [R, 7], dz [3, R, 7] (transfer-matrix PQC forward with tangents)
int gemm3_readout(int64_t R, const float* Phi, const float* Wt, float* Psi, float* z, float* dz,
                  void* ws, size_t ws_bytes, cudaStream_t st, const Wsplit* pre = nullptr);
size_t wgrad_workspace_bytes(int64_t rows, int Kin, int Nout);
// dW [Kin,Nout] = X [rows,Kin]^T G [rows,Nout] (split-K over rows, deterministic)
int wgrad(int64_t rows, int Kin, int Nout, const float* X, int64_t ldx, const float* G,
          int64_t ldg, float* dW, void* ws, size_t ws_bytes, cudaStream_t st);
// H [R,N] = tanh(X [R,K] W [K,N] + b) (value only)
int dense_tanh1(int64_t R, int N, int K, const float* X, const float* W, const float* bias,
                float* H, void* ws, size_t ws_bytes, cudaStream_t st,
                const Wsplit* pre = nullptr);
// H [4R,N] = dual tanh of X [4R,K] W [K,N] + b (value / tangent channel blocks)
int dense_tanh(int64_t R, int N, int K, const float* X, const float* W, const float* bias,
               float* H, void* ws, size_t ws_bytes, cudaStream_t st,
               const Wsplit* pre = nullptr);
// dense_tanh with the tanh adapter fused into the epilogue: also
// act [4R, n_ad] = dual tanh(H Wa + ba)  (N <= 128, n_ad <= 8)
int dense_tanh_adapter(int64_t R, int N, int K, const float* X, const float* W, const float* bias,
                       float* H, const float* Wa, const float* ba, int n_ad, float* act, void* ws,
                       size_t ws_bytes, cudaStream_t st, const Wsplit* pre = nullptr);
}  // namespace tc
}  // namespace qpinn
