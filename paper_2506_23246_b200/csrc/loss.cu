// K4: fused Maxwell residual / loss block-reduce and its closed-form gradient.
//
// Reference: physics.LossEvaluator.evaluate (physics.py:334-428) computes,
// per chunk of whole time slices, the TEz residuals (physics.py:123-128), the
// per-bin residual sums, the Poynting energy residual (physics.py:157-164),
// the mirror-parity terms through exact grid permutations (physics.py:397-404)
// and the t = 0 initial-condition term (physics.py:406-411), then
// back-propagates the weighted chunk scalar through its tape.  Every term is a
// sum of squares of pointwise quantities with static coefficients, so the
// gradient w.r.t. (fields, jacobians) is closed-form per point; the mirror
// terms need the partner point's field only.  One thread per point; sums are
// reduced warp -> block (fixed order, float64) -> grid (fixed order).
#include "common.cuh"

namespace qpinn {

constexpr int kLossThreads = 128;
constexpr int kNS = QPINN_LOSS_NSUMS;

struct LossDev {
  int nx, ny, S, nloc;
  const int* bin;
  const int* is_ic;
  const double* eps;
  const double* ic_target;
  int balanced, energy, n_sym;
  int sym_field[6], sym_axis[6];
  double sym_sign[6];
  double coef[5][4];  // per-point coefficient of the squared residual sums
  double c_energy, c_sym, c_ic;
};

template <typename T>
__global__ void __launch_bounds__(kLossThreads)
loss_kernel(LossDev L, int64_t R, const T* __restrict__ out, const T* __restrict__ dout,
            const double* __restrict__ weights, T* __restrict__ g_out, T* __restrict__ g_dout,
            double* __restrict__ partial) {
  double acc[kNS];
#pragma unroll
  for (int i = 0; i < kNS; ++i) acc[i] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < R; i += stride) {
    const int ls = (int)(i / L.S), p = (int)(i % L.S);
    const int m = L.bin[ls];
    const T eps = (T)L.eps[p];
    const T ez = out[i * 3], hx = out[i * 3 + 1], hy = out[i * 3 + 2];
    const T* d0 = dout + i * 3;            // d/dx
    const T* d1 = dout + (R + i) * 3;      // d/dy
    const T* d2 = dout + (2 * R + i) * 3;  // d/dt
    const T ezx = d0[0], hyx = d0[2];
    const T ezy = d1[0], hxy = d1[1];
    const T ezt = d2[0], hxt = d2[1], hyt = d2[2];
    // TEz residuals (physics.py:123-128)
    const T res1 = ezt - (hyx - hxy) / eps;
    const T res2 = hxt + ezy;
    const T res3 = hyt - ezx;
    const int k1 = (L.balanced && L.eps[p] != 1.0) ? 1 : 0;
    const double wm = weights ? weights[m] : 1.0;
    const T c1 = (T)(wm * L.coef[m][k1]), c2 = (T)(wm * L.coef[m][2]), c3 = (T)(wm * L.coef[m][3]);
#pragma unroll
    for (int mm = 0; mm < 5; ++mm) {
      if (mm != m) continue;
      acc[4 * mm + k1] += (double)(res1 * res1);
      acc[4 * mm + 2] += (double)(res2 * res2);
      acc[4 * mm + 3] += (double)(res3 * res3);
    }
    T g[3] = {T(0), T(0), T(0)};
    T gd[3][3] = {{T(0), T(0), T(0)}, {T(0), T(0), T(0)}, {T(0), T(0), T(0)}};  // [k][field]
    gd[2][0] += T(2) * c1 * res1;
    gd[0][2] += T(-2) * c1 * res1 / eps;
    gd[1][1] += T(2) * c1 * res1 / eps;
    gd[2][1] += T(2) * c2 * res2;
    gd[1][0] += T(2) * c2 * res2;
    gd[2][2] += T(2) * c3 * res3;
    gd[0][0] += T(-2) * c3 * res3;
    if (L.energy) {  // Poynting residual (physics.py:157-164)
      const T rE = (eps * ez * ezt + hx * hxt + hy * hyt) - (ezx * hy + ez * hyx) +
                   (ezy * hx + ez * hxy);
      acc[20] += (double)(rE * rE);
      const T gE = T(2) * (T)L.c_energy * rE;
      g[0] += gE * (eps * ezt - hyx + hxy);
      g[1] += gE * (hxt + ezy);
      g[2] += gE * (hyt - ezx);
      gd[2][0] += gE * eps * ez;
      gd[2][1] += gE * hx;
      gd[2][2] += gE * hy;
      gd[0][0] -= gE * hy;
      gd[0][2] -= gE * ez;
      gd[1][0] += gE * hx;
      gd[1][1] += gE * ez;
    }
    if (L.n_sym) {  // parity terms through mirror partners (physics.py:397-404)
      const int ix = p % L.nx, iy = p / L.nx;
      const int64_t base = (int64_t)ls * L.S;
      const int64_t imx = base + iy * L.nx + (L.nx - ix) % L.nx;
      const int64_t imy = base + (int64_t)((L.ny - iy) % L.ny) * L.nx + ix;
      for (int t = 0; t < L.n_sym; ++t) {
        const int f = L.sym_field[t];
        const T fv = out[i * 3 + f];
        const T fm = out[(L.sym_axis[t] ? imy : imx) * 3 + f];
        const T d = fv - (T)L.sym_sign[t] * fm;
        acc[21] += (double)(d * d);
        // d/df_i of sum_j (f_j - s f_m(j))^2 with an involutive mirror = 4 (f_i - s f_m(i))
        g[f] += T(4) * (T)L.c_sym * d;
      }
    }
    if (L.is_ic[ls]) {  // initial condition on the t = 0 slice (physics.py:406-411)
      const T dzv = ez - (T)L.ic_target[p];
      acc[22] += (double)(dzv * dzv + hx * hx + hy * hy);
      const T ci = T(2) * (T)L.c_ic;
      g[0] += ci * dzv;
      g[1] += ci * hx;
      g[2] += ci * hy;
    }
#pragma unroll
    for (int f = 0; f < 3; ++f) g_out[i * 3 + f] = g[f];
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int f = 0; f < 3; ++f) g_dout[((int64_t)k * R + i) * 3 + f] = gd[k][f];
  }
  // warp reduce (fixed butterfly) -> per-warp smem -> block partial
  __shared__ double red[kLossThreads / 32][kNS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int v = 0; v < kNS; ++v) {
    double x = acc[v];
#pragma unroll
    for (int mk = 16; mk >= 1; mk >>= 1) x += __shfl_xor_sync(0xffffffffu, x, mk);
    if (lane == 0) red[warp][v] = x;
  }
  __syncthreads();
  if (threadIdx.x < kNS) {
    double x = 0.0;
    for (int w = 0; w < kLossThreads / 32; ++w) x += red[w][threadIdx.x];
    partial[(size_t)blockIdx.x * kNS + threadIdx.x] = x;
  }
}

__global__ void loss_reduce(const double* __restrict__ partial, int blocks, double* __restrict__ sums) {
  const int v = threadIdx.x;
  if (v >= kNS) return;
  double x = 0.0;
  for (int b = 0; b < blocks; ++b) x += partial[(size_t)b * kNS + v];
  sums[v] = x;
}

struct FinDev {
  double inv_count_bin[5][4];
  double inv_count_all[4];
  double n_total, slice_size;
  int energy;
};

// breakdown (physics.py:416-426) and next time-bin weights (physics.py:172-180)
__global__ void loss_finalize_kernel(FinDev F, const double* __restrict__ sums,
                                     const double* __restrict__ weights, int weighted,
                                     double kappa, double* __restrict__ bd,
                                     double* __restrict__ wnext) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double bin_phys[5];
  for (int m = 0; m < 5; ++m) {
    double b = 0.0;
    for (int k = 0; k < 4; ++k) b += sums[4 * m + k] * F.inv_count_bin[m][k];
    bin_phys[m] = b;
  }
  double phys = 0.0;
  if (weighted) {
    for (int m = 0; m < 5; ++m) phys += weights[m] * bin_phys[m];
    phys /= 5.0;
  } else {
    for (int k = 0; k < 4; ++k) {
      double tot = 0.0;
      for (int m = 0; m < 5; ++m) tot += sums[4 * m + k];
      phys += tot * F.inv_count_all[k];
    }
  }
  const double ic = sums[22] / F.slice_size;
  const double sym = sums[21] / F.n_total;
  const double energy = F.energy ? sums[20] / F.n_total : 0.0;
  double total = phys + 10.0 * ic + 10.0 * sym;
  if (F.energy) total += 10.0 * energy;
  bd[0] = phys; bd[1] = ic; bd[2] = sym; bd[3] = energy; bd[4] = total;
  for (int m = 0; m < 5; ++m) bd[5 + m] = bin_phys[m];
  if (wnext) {
    double cum = 0.0;
    wnext[0] = 1.0;
    for (int m = 1; m < 5; ++m) {
      cum += bin_phys[m - 1];
      const double e = exp(-kappa * cum);
      wnext[m] = e < 1.0 ? e : 1.0;
    }
  }
}

static int loss_grid(int64_t R) {
  int64_t need = (R + kLossThreads - 1) / kLossThreads;
  int64_t cap = (int64_t)num_sms() * 8;
  int64_t g = need < cap ? need : cap;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace qpinn

using namespace qpinn;

extern "C" {

size_t qpinn_loss_workspace_bytes(const qpinn_loss_spec*, int, int64_t) {
  return sizeof(double) * kNS * (size_t)num_sms() * 8 + 256;
}

int qpinn_loss_forward_backward(const qpinn_loss_spec* s, int dtype, int64_t R, const void* out,
                                const void* dout, const double* weights_dev, void* g_out,
                                void* g_dout, double* sums_dev, void* workspace,
                                size_t workspace_bytes, void* stream) {
  if (!s) return fail(QPINN_ERR_CONFIG, "null loss spec");
  if (dtype != QPINN_F32 && dtype != QPINN_F64) return fail(QPINN_ERR_CONFIG, "bad dtype");
  const int64_t S = (int64_t)s->nx * s->ny;
  if (S <= 0 || R != S * s->n_local_slices)
    return fail(QPINN_ERR_INVALID_BATCH, "rows must equal n_local_slices * nx * ny");
  if (s->n_sym < 0 || s->n_sym > 6) return fail(QPINN_ERR_CONFIG, "bad symmetry term count");
  if (workspace_bytes < qpinn_loss_workspace_bytes(s, dtype, R))
    return fail(QPINN_ERR_CONFIG, "workspace too small");
  LossDev L;
  L.nx = s->nx; L.ny = s->ny; L.S = (int)S; L.nloc = s->n_local_slices;
  L.bin = s->slice_bin; L.is_ic = s->slice_is_ic; L.eps = s->eps; L.ic_target = s->ic_target;
  L.balanced = s->balanced; L.energy = s->energy; L.n_sym = s->n_sym;
  for (int t = 0; t < 6; ++t) {
    L.sym_field[t] = s->sym_field[t];
    L.sym_axis[t] = s->sym_axis[t];
    L.sym_sign[t] = s->sym_sign[t];
  }
  // weighted: w_m / (5 count(key, bin m)); pooled: 1 / count(key, all slices)
  for (int m = 0; m < 5; ++m)
    for (int k = 0; k < 4; ++k)
      L.coef[m][k] = weights_dev ? s->inv_count_bin[m][k] / 5.0 : s->inv_count_all[k];
  L.c_energy = 10.0 / s->n_total;
  L.c_sym = 10.0 / s->n_total;
  L.c_ic = 10.0 / s->slice_size;
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = loss_grid(R);
  double* partial = (double*)workspace;
  if (R == 0) {
    QPINN_CUDA_CHECK(cudaMemsetAsync(sums_dev, 0, sizeof(double) * kNS, st));
    return QPINN_OK;
  }
  if (dtype == QPINN_F32)
    loss_kernel<float><<<grid, kLossThreads, 0, st>>>(L, R, (const float*)out, (const float*)dout,
                                                      weights_dev, (float*)g_out, (float*)g_dout,
                                                      partial);
  else
    loss_kernel<double><<<grid, kLossThreads, 0, st>>>(L, R, (const double*)out,
                                                       (const double*)dout, weights_dev,
                                                       (double*)g_out, (double*)g_dout, partial);
  QPINN_CUDA_CHECK(cudaGetLastError());
  loss_reduce<<<1, 32, 0, st>>>(partial, grid, sums_dev);
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

int qpinn_loss_finalize(const qpinn_loss_spec* s, const double* sums_dev, const double* weights_dev,
                        int weighted, double kappa, double* breakdown_dev, double* weights_next_dev,
                        void* stream) {
  if (!s) return fail(QPINN_ERR_CONFIG, "null loss spec");
  if (weighted && !weights_dev) return fail(QPINN_ERR_CONFIG, "weighted finalize needs weights");
  FinDev F;
  for (int m = 0; m < 5; ++m)
    for (int k = 0; k < 4; ++k) F.inv_count_bin[m][k] = s->inv_count_bin[m][k];
  for (int k = 0; k < 4; ++k) F.inv_count_all[k] = s->inv_count_all[k];
  F.n_total = s->n_total;
  F.slice_size = s->slice_size;
  F.energy = s->energy;
  loss_finalize_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(F, sums_dev, weights_dev, weighted, kappa,
                                                           breakdown_dev, weights_next_dev);
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

}  // extern "C"
