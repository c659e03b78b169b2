// Adam with bias correction (training.py:87-111), in place on the flat
// parameter vector.  The reference raises RunAborted on a non-finite gradient
// before touching any state (training.py:104-105): a first pass ORs a device
// flag, the update pass is skipped when the flag is set.  An optional veto
// (the step's reduced domain flag) skips it the same way: the reference
// raises DomainError in the forward, before any update (ansatz.py:51-58).
#include "common.cuh"

namespace qpinn {

template <typename T>
__global__ void adam_check(int64_t n, const T* __restrict__ g, const double* __restrict__ loss,
                           const double* __restrict__ veto, int* __restrict__ flag) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (loss && blockIdx.x == 0 && threadIdx.x == 0 && !isfinite(*loss)) atomicOr(flag, 2);
  if (veto && blockIdx.x == 0 && threadIdx.x == 0 && *veto != 0.0) atomicOr(flag, 4);
  int bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    bad |= !isfinite(g[i]);
  bad = __any_sync(0xffffffffu, bad);
  if (bad && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

template <typename T>
__global__ void adam_update(int64_t n, T* __restrict__ p, const T* __restrict__ g, T* __restrict__ m,
                            T* __restrict__ v, T b1, T b2, T bc1, T bc2, T lr, T eps,
                            const int* __restrict__ flag) {
  if (*flag) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const T gi = g[i];
    const T mi = b1 * m[i] + (T(1) - b1) * gi;
    const T vi = b2 * v[i] + (T(1) - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    const T mhat = mi / bc1, vhat = vi / bc2;
    p[i] -= lr * mhat / (sqrt(vhat) + eps);
  }
}

}  // namespace qpinn

using namespace qpinn;

extern "C" int qpinn_adam_step(int dtype, int64_t n, void* params, const void* grad, void* m, void* v,
                               int64_t t, double lr, double b1, double b2, double eps,
                               const double* loss, const double* veto, int32_t* flag,
                               void* stream) {
  if (dtype != QPINN_F32 && dtype != QPINN_F64) return fail(QPINN_ERR_CONFIG, "bad dtype");
  if (t < 1) return fail(QPINN_ERR_CONFIG, "adam step t must be >= 1");
  if (!flag) return fail(QPINN_ERR_CONFIG, "adam needs a device flag");
  cudaStream_t st = (cudaStream_t)stream;
  QPINN_CUDA_CHECK(cudaMemsetAsync(flag, 0, sizeof(int32_t), st));
  if (n <= 0) return QPINN_OK;
  const double bc1 = 1.0 - pow(b1, (double)t), bc2 = 1.0 - pow(b2, (double)t);
  int64_t need = (n + 255) / 256;
  const int grid = (int)(need < (int64_t)num_sms() * 4 ? need : (int64_t)num_sms() * 4);
  if (dtype == QPINN_F32) {
    adam_check<float><<<grid, 256, 0, st>>>(n, (const float*)grad, loss, veto, flag);
    adam_update<float><<<grid, 256, 0, st>>>(n, (float*)params, (const float*)grad, (float*)m,
                                             (float*)v, (float)b1, (float)b2, (float)bc1,
                                             (float)bc2, (float)lr, (float)eps, flag);
  } else {
    adam_check<double><<<grid, 256, 0, st>>>(n, (const double*)grad, loss, veto, flag);
    adam_update<double><<<grid, 256, 0, st>>>(n, (double*)params, (const double*)grad, (double*)m,
                                              (double*)v, b1, b2, bc1, bc2, lr, eps, flag);
  }
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}
