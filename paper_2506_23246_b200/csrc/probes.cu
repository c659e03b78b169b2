// Value-only inference head and the diagnostic probes' reductions
// (SURVEY 8f row 3): network.py:302 (linear head), training.py:187-217
// (energy probe, L2 against the FDTD reference), fdtd.py:194-197 (energy).
// One block per time slice with a fixed-order tree: deterministic.
#include "common.cuh"

namespace qpinn {

template <typename T>
__global__ void head_forward(int64_t R, int n, const T* __restrict__ z, const T* __restrict__ W,
                             const T* __restrict__ b, T* __restrict__ out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < R;
       p += (int64_t)gridDim.x * blockDim.x) {
    T o0 = b[0], o1 = b[1], o2 = b[2];
    for (int k = 0; k < n; ++k) {
      const T v = z[p * n + k];
      o0 += v * W[k * 3 + 0];
      o1 += v * W[k * 3 + 1];
      o2 += v * W[k * 3 + 2];
    }
    out[p * 3 + 0] = o0;
    out[p * 3 + 1] = o1;
    out[p * 3 + 2] = o2;
  }
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int m = blockDim.x / 2; m > 0; m >>= 1) {
    if (threadIdx.x < m) red[threadIdx.x] += red[threadIdx.x + m];
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

// u[t] = dxdy * sum_p 0.5 (eps_p Ez^2 + Hx^2 + Hy^2) over slice t's P points
template <typename T>
__global__ void probe_energy(int64_t P, const T* __restrict__ f, const double* __restrict__ eps,
                             double dxdy, double* __restrict__ u) {
  __shared__ double red[256];
  const T* s = f + (int64_t)blockIdx.x * P * 3;
  double acc = 0.0;
  for (int64_t p = threadIdx.x; p < P; p += blockDim.x) {
    const double ez = s[3 * p], hx = s[3 * p + 1], hy = s[3 * p + 2];
    acc += 0.5 * (eps[p] * ez * ez + hx * hx + hy * hy);
  }
  const double tot = block_sum(acc, red);
  if (threadIdx.x == 0) u[blockIdx.x] = tot * dxdy;
}

// out[2t] = sum (Ez - ref)^2, out[2t+1] = sum ref^2 over slice t
template <typename T>
__global__ void probe_l2(int64_t P, const T* __restrict__ f, const double* __restrict__ ref,
                         double* __restrict__ out) {
  __shared__ double red[256];
  const T* s = f + (int64_t)blockIdx.x * P * 3;
  const double* r = ref + (int64_t)blockIdx.x * P;
  double num = 0.0, den = 0.0;
  for (int64_t p = threadIdx.x; p < P; p += blockDim.x) {
    const double d = (double)s[3 * p] - r[p];
    num += d * d;
    den += r[p] * r[p];
  }
  const double a = block_sum(num, red);
  const double b2 = block_sum(den, red);
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = a;
    out[2 * blockIdx.x + 1] = b2;
  }
}

}  // namespace qpinn

using namespace qpinn;

extern "C" {

int qpinn_head_forward(int dtype, int64_t rows, int n, const void* z, const void* w_out,
                       const void* b_out, void* fields, void* stream) {
  if (rows < 0 || n < 1) return fail(QPINN_ERR_CONFIG, "head: bad shape");
  if (rows == 0) return QPINN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int blocks = (int)((rows + 255) / 256 < 4096 ? (rows + 255) / 256 : 4096);
  if (dtype == QPINN_F32)
    head_forward<float><<<blocks, 256, 0, st>>>(rows, n, (const float*)z, (const float*)w_out,
                                                (const float*)b_out, (float*)fields);
  else if (dtype == QPINN_F64)
    head_forward<double><<<blocks, 256, 0, st>>>(rows, n, (const double*)z,
                                                 (const double*)w_out, (const double*)b_out,
                                                 (double*)fields);
  else
    return fail(QPINN_ERR_CONFIG, "bad dtype");
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

int qpinn_probe_energy(int dtype, int n_slices, int64_t points, const void* fields,
                       const double* eps, double dxdy, double* u, void* stream) {
  if (n_slices < 0 || points < 1) return fail(QPINN_ERR_CONFIG, "probe_energy: bad shape");
  if (n_slices == 0) return QPINN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == QPINN_F32)
    probe_energy<float><<<n_slices, 256, 0, st>>>(points, (const float*)fields, eps, dxdy, u);
  else
    probe_energy<double><<<n_slices, 256, 0, st>>>(points, (const double*)fields, eps, dxdy, u);
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

int qpinn_probe_l2(int dtype, int n_slices, int64_t points, const void* fields, const double* ref,
                   double* sums, void* stream) {
  if (n_slices < 0 || points < 1) return fail(QPINN_ERR_CONFIG, "probe_l2: bad shape");
  if (n_slices == 0) return QPINN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == QPINN_F32)
    probe_l2<float><<<n_slices, 256, 0, st>>>(points, (const float*)fields, ref, sums);
  else
    probe_l2<double><<<n_slices, 256, 0, st>>>(points, (const double*)fields, ref, sums);
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

}  // extern "C"
