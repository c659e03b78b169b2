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

// Per-point residuals, loss sums and closed-form loss gradient w.r.t. the
// fields (g[f]) and their jacobians (gd[k][f]).  field_at(row, f) returns the
// value of field f at another row of the same slice (mirror partners).
template <typename T, typename FieldAt>
__device__ __forceinline__ void point_loss(const LossDev& L, const double* __restrict__ weights,
                                           int64_t i, const T (&fv)[3], const T (&dv)[3][3],
                                           FieldAt field_at, double (&acc)[kNS], T (&g)[3],
                                           T (&gd)[3][3]) {
  const int ls = (int)(i / L.S), p = (int)(i % L.S);
  const int m = L.bin[ls];
  const T eps = (T)L.eps[p];
  const T ez = fv[0], hx = fv[1], hy = fv[2];
  const T ezx = dv[0][0], hyx = dv[0][2];
  const T ezy = dv[1][0], hxy = dv[1][1];
  const T ezt = dv[2][0], hxt = dv[2][1], hyt = dv[2][2];
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
    // static indices only (a runtime one would put acc in local memory)
    const double r1 = (double)(res1 * res1);
    if (k1) acc[4 * mm + 1] += r1;
    else acc[4 * mm] += r1;
    acc[4 * mm + 2] += (double)(res2 * res2);
    acc[4 * mm + 3] += (double)(res3 * res3);
  }
#pragma unroll
  for (int f = 0; f < 3; ++f) {
    g[f] = T(0);
#pragma unroll
    for (int k = 0; k < 3; ++k) gd[k][f] = T(0);
  }
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
      const T fm = field_at(L.sym_axis[t] ? imy : imx, f);
      const T d = fv[f] - (T)L.sym_sign[t] * fm;
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
}

// fixed-order block reduction of NV per-thread values -> partial[block][NV]
template <int NV>
__device__ __forceinline__ void block_reduce_store(double (&v)[NV], double* __restrict__ partial) {
  __shared__ double red[kLossThreads / 32][NV];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    double x = v[j];
#pragma unroll
    for (int mk = 16; mk >= 1; mk >>= 1) x += __shfl_xor_sync(0xffffffffu, x, mk);
    if (lane == 0) red[warp][j] = x;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < NV; j += blockDim.x) {
    double x = 0.0;
    for (int w = 0; w < kLossThreads / 32; ++w) x += red[w][j];
    partial[(size_t)blockIdx.x * NV + j] = x;
  }
}

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
    T fv[3], dv[3][3], g[3], gd[3][3];
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      fv[f] = out[i * 3 + f];
#pragma unroll
      for (int k = 0; k < 3; ++k) dv[k][f] = dout[((int64_t)k * R + i) * 3 + f];
    }
    point_loss<T>(L, weights, i, fv, dv, [&](int64_t j, int f) { return out[j * 3 + f]; }, acc, g, gd);
#pragma unroll
    for (int f = 0; f < 3; ++f) g_out[i * 3 + f] = g[f];
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int f = 0; f < 3; ++f) g_dout[((int64_t)k * R + i) * 3 + f] = gd[k][f];
  }
  block_reduce_store<kNS>(acc, partial);
}

// Head fused in: out = z Wo + bo, dout_k = dz_k Wo (network.py:302) from
// z [4, R, W]; writes dL/dz [4, R, W] and accumulates dL/dWo, dL/dbo.
template <typename T, int W>
__global__ void __launch_bounds__(kLossThreads)
loss_head_kernel(LossDev L, int64_t R, const T* __restrict__ Z, const T* __restrict__ Wo,
                 const T* __restrict__ bo, const double* __restrict__ weights,
                 T* __restrict__ GZ, double* __restrict__ partial) {
  constexpr int NV = kNS + 3 * W + 3;
  __shared__ T sw[3 * W + 3];
  for (int j = threadIdx.x; j < 3 * W; j += blockDim.x) sw[j] = Wo[j];
  if (threadIdx.x < 3) sw[3 * W + threadIdx.x] = bo[threadIdx.x];
  __syncthreads();
  double acc[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) acc[j] = 0.0;
  const int64_t n = R * W;
  auto field_at = [&](int64_t j, int f) {
    T v = sw[3 * W + f];
#pragma unroll
    for (int w = 0; w < W; ++w) v += Z[j * W + w] * sw[w * 3 + f];
    return v;
  };
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < R; i += stride) {
    T z[4][W];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int w = 0; w < W; ++w) z[c][w] = Z[c * n + i * W + w];
    T fv[3], dv[3][3];
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      T v = sw[3 * W + f];
#pragma unroll
      for (int w = 0; w < W; ++w) v += z[0][w] * sw[w * 3 + f];
      fv[f] = v;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        T d = T(0);
#pragma unroll
        for (int w = 0; w < W; ++w) d += z[1 + k][w] * sw[w * 3 + f];
        dv[k][f] = d;
      }
    }
    T g[3], gd[3][3];
    point_loss<T>(L, weights, i, fv, dv, field_at, *reinterpret_cast<double(*)[kNS]>(&acc[0]), g, gd);
    // dL/dz = g Wo^T, dL/d(dz_k) = gd_k Wo^T; dWo += z^T g + sum_k dz_k^T gd_k; dbo += g
#pragma unroll
    for (int w = 0; w < W; ++w) {
      GZ[i * W + w] = g[0] * sw[w * 3] + g[1] * sw[w * 3 + 1] + g[2] * sw[w * 3 + 2];
#pragma unroll
      for (int k = 0; k < 3; ++k)
        GZ[(1 + k) * n + i * W + w] =
            gd[k][0] * sw[w * 3] + gd[k][1] * sw[w * 3 + 1] + gd[k][2] * sw[w * 3 + 2];
#pragma unroll
      for (int f = 0; f < 3; ++f)
        acc[kNS + w * 3 + f] += (double)(z[0][w] * g[f] + z[1][w] * gd[0][f] +
                                         z[2][w] * gd[1][f] + z[3][w] * gd[2][f]);
    }
#pragma unroll
    for (int f = 0; f < 3; ++f) acc[kNS + 3 * W + f] += (double)g[f];
  }
  block_reduce_store<NV>(acc, partial);
}

// fixed-order grid reduction: sums[0..23) (double) and the head gradient (dtype);
// 32 values x 32 interleaved block groups per CTA, groups combined in order
template <typename T>
__global__ void __launch_bounds__(1024) loss_head_reduce(const double* __restrict__ partial, int blocks, int nv,
                                 double* __restrict__ sums, T* __restrict__ g_wo,
                                 T* __restrict__ g_bo) {
  __shared__ double red[32][33];  // 32 row groups (blockDim 1024), added in order
  const int c = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int v = blockIdx.x * 32 + c;
  double x = 0.0;
  if (v < nv) {
#pragma unroll 4
    for (int b = grp; b < blocks; b += 32) x += __ldg(partial + (size_t)b * nv + v);
  }
  red[grp][c] = x;
  __syncthreads();
  if (grp == 0 && v < nv) {
    double t = 0.0;
    for (int g2 = 0; g2 < 32; ++g2) t += red[g2][c];
    if (v < kNS) sums[v] = t;
    else if (v < nv - 3) g_wo[v - kNS] = T(t);
    else g_bo[v - (nv - 3)] = T(t);
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

LossDev make_loss_dev(const qpinn_loss_spec* s, bool weighted);

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
  return sizeof(double) * (kNS + 3 * 16 + 3) * (size_t)num_sms() * 8 + 256;
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
  LossDev L = make_loss_dev(s, weights_dev != nullptr);
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

}  // extern "C"

namespace qpinn {
LossDev make_loss_dev(const qpinn_loss_spec* s, bool weighted) {
  LossDev L;
  const int64_t S = (int64_t)s->nx * s->ny;
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
      L.coef[m][k] = weighted ? s->inv_count_bin[m][k] / 5.0 : s->inv_count_all[k];
  L.c_energy = 10.0 / s->n_total;
  L.c_sym = 10.0 / s->n_total;
  L.c_ic = 10.0 / s->slice_size;
  return L;
}

template <typename T, int W>
static int launch_head(const LossDev& L, int64_t R, const T* z, const T* wo, const T* bo,
                       const double* weights, T* gz, T* g_wo, T* g_bo, double* sums,
                       double* partial, cudaStream_t st) {
  const int grid = loss_grid(R);
  loss_head_kernel<T, W><<<grid, kLossThreads, 0, st>>>(L, R, z, wo, bo, weights, gz, partial);
  QPINN_CUDA_CHECK(cudaGetLastError());
  loss_head_reduce<T><<<(kNS + 3 * W + 3 + 31) / 32, 1024, 0, st>>>(partial, grid,
                                                                    kNS + 3 * W + 3, sums, g_wo,
                                                                    g_bo);
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

template <typename T>
static int head_dispatch(int W, const LossDev& L, int64_t R, const T* z, const T* wo, const T* bo,
                         const double* weights, T* gz, T* g_wo, T* g_bo, double* sums,
                         double* partial, cudaStream_t st) {
#define QPINN_HEAD_W(WW) \
  case WW: return launch_head<T, WW>(L, R, z, wo, bo, weights, gz, g_wo, g_bo, sums, partial, st);
  switch (W) {
    QPINN_HEAD_W(1) QPINN_HEAD_W(2) QPINN_HEAD_W(3) QPINN_HEAD_W(4) QPINN_HEAD_W(5)
    QPINN_HEAD_W(6) QPINN_HEAD_W(7) QPINN_HEAD_W(8) QPINN_HEAD_W(9) QPINN_HEAD_W(10)
    QPINN_HEAD_W(11) QPINN_HEAD_W(12) QPINN_HEAD_W(13) QPINN_HEAD_W(14) QPINN_HEAD_W(15)
    QPINN_HEAD_W(16)
    default: return fail(QPINN_ERR_CONFIG, "head width must be in [1, 16]");
  }
#undef QPINN_HEAD_W
}
}  // namespace qpinn

extern "C" {

int qpinn_loss_head_forward_backward(const qpinn_loss_spec* s, int dtype, int64_t R, int width,
                                     const void* z, const void* w_out, const void* b_out,
                                     const double* weights_dev, void* g_z, void* g_w_out,
                                     void* g_b_out, double* sums_dev, void* workspace,
                                     size_t workspace_bytes, void* stream) {
  if (!s) return fail(QPINN_ERR_CONFIG, "null loss spec");
  if (dtype != QPINN_F32 && dtype != QPINN_F64) return fail(QPINN_ERR_CONFIG, "bad dtype");
  const int64_t S = (int64_t)s->nx * s->ny;
  if (S <= 0 || R != S * s->n_local_slices)
    return fail(QPINN_ERR_INVALID_BATCH, "rows must equal n_local_slices * nx * ny");
  if (s->n_sym < 0 || s->n_sym > 6) return fail(QPINN_ERR_CONFIG, "bad symmetry term count");
  if (workspace_bytes < qpinn_loss_workspace_bytes(s, dtype, R))
    return fail(QPINN_ERR_CONFIG, "workspace too small");
  const LossDev L = make_loss_dev(s, weights_dev != nullptr);
  cudaStream_t st = (cudaStream_t)stream;
  if (R == 0) {
    QPINN_CUDA_CHECK(cudaMemsetAsync(sums_dev, 0, sizeof(double) * kNS, st));
    return QPINN_OK;
  }
  if (dtype == QPINN_F32)
    return head_dispatch<float>(width, L, R, (const float*)z, (const float*)w_out,
                                (const float*)b_out, weights_dev, (float*)g_z, (float*)g_w_out,
                                (float*)g_b_out, sums_dev, (double*)workspace, st);
  return head_dispatch<double>(width, L, R, (const double*)z, (const double*)w_out,
                               (const double*)b_out, weights_dev, (double*)g_z, (double*)g_w_out,
                               (double*)g_b_out, sums_dev, (double*)workspace, st);
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
