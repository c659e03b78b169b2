// K2 in the HBM regime (n = 15, 16): the adjoint beyond what a 16-CTA cluster
// can hold resident (x and the adjoint together need 64 D bytes per point at
// fp32 -- 4 MB at n = 16).
//
// Same algorithm as the layer kernels (pqc_layer.cu): the forward is re-run
// for a batch of B points with the four states (psi, d psi/dx,y,t) in global
// memory, storing the state at every layer boundary (after the layer's
// single-qubit gates); the reverse sweep then keeps only the adjoint live,
// takes every gate's post-gate state from the boundary checkpoint (gates of
// one layer commute), and propagates the adjoint through U^dagger.  Each gate
// is one bandwidth-bound pass over the batch's [B][4][D] array; the per-gate
// 2x2 outer products and the per-basis-state phase sums are reduced in a
// fixed order (deterministic), and the embedding gradient follows the oracle
// (qpinn_oracle.pqc_backward).  Reference: the taped backward of
// quantum_layer_forward via="gates" (ansatz.py:341-400, tape.py:118-148).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pqc_layer.h"

namespace qpinn {

namespace {

constexpr int kGbThreads = 256;

inline int gb_blocks(int64_t n) {
  const int64_t b = (n + kGbThreads - 1) / kGbThreads;
  const int64_t cap = (int64_t)num_sms() * 8;
  return (int)(b < 1 ? 1 : b > cap ? cap : b);
}

// u1 matrices [n_u1][4] and phase diagonals [n_phase][D], natural basis order
template <typename T>
__global__ void gb_tables(PlanDev p, const T* __restrict__ qp, cplx<T>* __restrict__ U,
                          cplx<T>* __restrict__ ph) {
  const int D = 1 << p.n;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int i = tid; i < p.n_u1; i += nt) {
    const int kind = p.u1[i * 4];
    double th[3] = {0, 0, 0};
    for (int j = 0; j < u1_nslots(kind); ++j) th[j] = (double)qp[p.u1[i * 4 + 1 + j]];
    double M[8];
    u1_matrix_d(kind, th, M);
    for (int e = 0; e < 4; ++e) U[i * 4 + e] = {T(M[2 * e]), T(M[2 * e + 1])};
  }
  for (int i = tid; i < p.n_phase * D; i += nt) {
    const int st = i / D, b = i % D;
    double phi = 0.0;
    for (int k = p.phase_off[st]; k < p.phase_off[st + 1]; ++k) {
      const int c = p.pairs[3 * k], t = p.pairs[3 * k + 1], s = p.pairs[3 * k + 2];
      const int on = (b >> (p.n - 1 - c)) & 1, tb = (b >> (p.n - 1 - t)) & 1;
      phi += on * (tb - 0.5) * (double)qp[s];  // qsim.py:212-225
    }
    double sp, cp;
    sincos(phi, &sp, &cp);
    ph[i] = {T(cp), T(sp)};
  }
}

// per point and qubit: cos, sin of theta/2, S', S'', dtheta_k (k = x, y, t)
template <typename T>
__global__ void gb_point(int n, int scale, int64_t R, int64_t p0, int B,
                         const T* __restrict__ act, const T* __restrict__ tan, T* __restrict__ PT) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B * n; i += gridDim.x * blockDim.x) {
    const int pb = i / n, q = i % n;
    const int64_t s = p0 + pb;
    T* o = PT + (int64_t)i * 8;
    if (s >= R) {
      for (int k = 0; k < 8; ++k) o[k] = T(0);
      continue;
    }
    T a = act[s * n + q];
    a = fmin(fmax(a, T(-1)), T(1));
    T c, sn, s1, s2;
    half_angle<T>(scale, a, c, sn, s1, s2);
    o[0] = c;
    o[1] = sn;
    o[2] = s1;
    o[3] = s2;
    for (int k = 0; k < 3; ++k) o[4 + k] = tan ? s1 * tan[((int64_t)k * R + s) * n + q] : T(0);
  }
}

// embedded state and its tangents (ansatz.py:233-243, :380-390); wire q is bit n-1-q
template <typename T>
__global__ void gb_embed(int n, int B, int nstates, const T* __restrict__ PT,
                         cplx<T>* __restrict__ X) {
  const int64_t D = (int64_t)1 << n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < B * D;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int pb = (int)(i / D);
    const int64_t b = i % D;
    const T* pt = PT + (int64_t)pb * n * 8;
    T pre[17];
    pre[0] = T(1);
    for (int q = 0; q < n; ++q) {
      const int bit = (b >> (n - 1 - q)) & 1;
      pre[q + 1] = pre[q] * (bit ? pt[q * 8 + 1] : pt[q * 8]);
    }
    T tk[3] = {T(0), T(0), T(0)}, suf = T(1);
    for (int q = n - 1; q >= 0; --q) {
      const int bit = (b >> (n - 1 - q)) & 1;
      const T df = bit ? T(0.5) * pt[q * 8] : T(-0.5) * pt[q * 8 + 1];
      const T rest = pre[q] * suf;
      for (int k = 0; k < 3; ++k) tk[k] += pt[q * 8 + 4 + k] * df * rest;
      suf *= bit ? pt[q * 8 + 1] : pt[q * 8];
    }
    const int ph = __popcll(b) & 3;  // (-i)^popcount
    auto put = [&](int s, T m) {
      X[((int64_t)pb * 4 + s) * D + b] = {ph == 0 ? m : ph == 2 ? -m : T(0),
                                           ph == 1 ? -m : ph == 3 ? m : T(0)};
    };
    put(0, pre[n]);
    if (nstates == 4)
      for (int k = 0; k < 3; ++k) put(k + 1, tk[k]);
  }
}

// one single-qubit step on every state of the batch (U or U^dagger)
template <typename T>
__global__ void gb_u1(int n, int64_t rows, cplx<T>* __restrict__ X, int q,
                      const cplx<T>* __restrict__ U, int dagger) {
  const int64_t half = (int64_t)1 << (n - 1), D = half * 2;
  const int pos = n - 1 - q;
  cplx<T> u00 = U[0], u01 = U[1], u10 = U[2], u11 = U[3];
  if (dagger) {
    const cplx<T> t01 = u01;
    u00 = {u00.re, -u00.im};
    u11 = {u11.re, -u11.im};
    u01 = {u10.re, -u10.im};
    u10 = {t01.re, -t01.im};
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows * half;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / half, k = i % half;
    const int64_t i0 = ((k >> pos) << (pos + 1)) | (k & (((int64_t)1 << pos) - 1));
    cplx<T>* x = X + row * D;
    const cplx<T> a = x[i0], b = x[i0 | ((int64_t)1 << pos)];
    x[i0] = cmul2(u00, a, u01, b);
    x[i0 | ((int64_t)1 << pos)] = cmul2(u10, a, u11, b);
  }
}

// out[row][b] = in[row][tab[b]] (a fused CNOT run or its inverse, qsim.py:198-209)
template <typename T>
__global__ void gb_perm(int n, int64_t rows, const cplx<T>* __restrict__ in,
                        cplx<T>* __restrict__ out, const uint16_t* __restrict__ tab) {
  const int64_t D = (int64_t)1 << n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows * D;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[(i / D) * D + tab[i % D]];
}

template <typename T>
__global__ void gb_phase(int n, int64_t rows, cplx<T>* __restrict__ X,
                         const cplx<T>* __restrict__ ph, int conj_) {
  const int64_t D = (int64_t)1 << n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows * D;
       i += (int64_t)gridDim.x * blockDim.x) {
    cplx<T> e = ph[i % D];
    if (conj_) e.im = -e.im;
    X[i] = cmul(X[i], e);
  }
}

// adjoint seeds: lambda = 2 w psi + 2 sum_k v_k dpsi_k, mu_k = 2 v_k psi
template <typename T>
__global__ void gb_seed(int n, int B, int64_t p0, int64_t R, const T* __restrict__ gz,
                        const T* __restrict__ gdz, const cplx<T>* __restrict__ X,
                        cplx<T>* __restrict__ A) {
  const int64_t D = (int64_t)1 << n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < B * D;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int pb = (int)(i / D);
    const int64_t b = i % D, s = p0 + pb;
    cplx<T>* a = A + (int64_t)pb * 4 * D + b;
    if (s >= R) {
      for (int k = 0; k < 4; ++k) a[k * D] = {T(0), T(0)};
      continue;
    }
    T w = T(0), v[3] = {T(0), T(0), T(0)};
    for (int q = 0; q < n; ++q) {
      const T sg = ((b >> (n - 1 - q)) & 1) ? T(-1) : T(1);
      w += sg * gz[s * n + q];
      for (int k = 0; k < 3; ++k) v[k] += sg * gdz[((int64_t)k * R + s) * n + q];
    }
    const cplx<T>* x = X + (int64_t)pb * 4 * D + b;
    const cplx<T> psi = x[0];
    cplx<T> l = {T(2) * w * psi.re, T(2) * w * psi.im};
    for (int k = 0; k < 3; ++k) {
      const cplx<T> d = x[(k + 1) * D];
      l.re += T(2) * v[k] * d.re;
      l.im += T(2) * v[k] * d.im;
      a[(k + 1) * D] = {T(2) * v[k] * psi.re, T(2) * v[k] * psi.im};
    }
    a[0] = l;
  }
}

// block partials of the post-gate outer product M'_ij = sum conj(a_i) x_j on wire q
template <typename T>
__global__ void gb_outer(int n, int64_t rows, const cplx<T>* __restrict__ X,
                         const cplx<T>* __restrict__ A, int q, double* __restrict__ part) {
  __shared__ double red[8][kGbThreads];
  const int64_t half = (int64_t)1 << (n - 1), D = half * 2;
  const int pos = n - 1 - q;
  T m[8] = {T(0), T(0), T(0), T(0), T(0), T(0), T(0), T(0)};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows * half;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / half, k = i % half;
    const int64_t i0 = row * D + (((k >> pos) << (pos + 1)) | (k & (((int64_t)1 << pos) - 1)));
    const int64_t i1 = i0 + ((int64_t)1 << pos);
    const cplx<T> x0 = X[i0], x1 = X[i1], a0 = A[i0], a1 = A[i1];
    cmac_c(m[0], m[1], a0, x0);
    cmac_c(m[2], m[3], a0, x1);
    cmac_c(m[4], m[5], a1, x0);
    cmac_c(m[6], m[7], a1, x1);
  }
  for (int k = 0; k < 8; ++k) red[k][threadIdx.x] = (double)m[k];
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int k = 0; k < 8; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x < 8) part[(size_t)blockIdx.x * 8 + threadIdx.x] = red[threadIdx.x][0];
}

// acc[0..8) += sum over blocks in order
__global__ void gb_sum8(int nblk, const double* __restrict__ part, double* __restrict__ acc) {
  if (threadIdx.x < 8) {
    double v = 0.0;
    for (int b = 0; b < nblk; ++b) v += part[(size_t)b * 8 + threadIdx.x];
    acc[threadIdx.x] += v;
  }
}

// phase step gradient per basis state: accP[b] += sum over the batch's rows of
// Im(conj(a_b) x'_b), x' = x ph (the post-entangler state)
template <typename T>
__global__ void gb_phase_grad(int n, int64_t rows, const cplx<T>* __restrict__ X,
                              const cplx<T>* __restrict__ A, const cplx<T>* __restrict__ ph,
                              double* __restrict__ accP) {
  const int64_t D = (int64_t)1 << n;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < D;
       b += (int64_t)gridDim.x * blockDim.x) {
    const cplx<T> e = ph[b];
    double v = 0.0;
    for (int64_t r = 0; r < rows; ++r) {
      const cplx<T> xp = cmul(X[r * D + b], e), a = A[r * D + b];
      v += (double)(a.im * xp.re - a.re * xp.im);
    }
    accP[b] += v;
  }
}

// embedding gradient partials (qpinn_oracle.pqc_backward):
//   eta = (i/2) phibar - 1/4 sum_k sum_q dth_kq X_q mu_k
//   g_th[q] = Re sum conj(eta) X_q phi, g_dth[k][q] = Re sum conj((i/2) mu_k) X_q phi
template <typename T>
__global__ void gb_embed_grad(int n, int chunks, const T* __restrict__ PT,
                              const cplx<T>* __restrict__ PHI, const cplx<T>* __restrict__ A,
                              double* __restrict__ egp) {
  extern __shared__ double eg_red[];  // [4 n][blockDim]
  const int64_t D = (int64_t)1 << n;
  const int pb = blockIdx.y;
  const T* pt = PT + (int64_t)pb * n * 8;
  const cplx<T>* phi = PHI + (int64_t)pb * 4 * D;  // state 0 of the re-embedded batch
  const cplx<T>* ab = A + (int64_t)pb * 4 * D;
  T acc[4 * 16];
  for (int j = 0; j < 4 * n; ++j) acc[j] = T(0);
  const int64_t per = (D + chunks - 1) / chunks;
  const int64_t b0 = blockIdx.x * per, b1 = b0 + per < D ? b0 + per : D;
  for (int64_t b = b0 + threadIdx.x; b < b1; b += blockDim.x) {
    const cplx<T> phib = ab[b];
    cplx<T> eta = {T(-0.5) * phib.im, T(0.5) * phib.re};  // (i/2) phibar
    for (int q = 0; q < n; ++q) {
      const int64_t f = b ^ ((int64_t)1 << (n - 1 - q));
      for (int k = 0; k < 3; ++k) {
        const cplx<T> m = ab[(k + 1) * D + f];
        const T w = T(0.25) * pt[q * 8 + 4 + k];
        eta.re -= w * m.re;
        eta.im -= w * m.im;
      }
    }
    for (int q = 0; q < n; ++q) {
      const cplx<T> y = phi[b ^ ((int64_t)1 << (n - 1 - q))];
      acc[q] += eta.re * y.re + eta.im * y.im;  // Re(conj(eta) y)
      for (int k = 0; k < 3; ++k) {
        const cplx<T> m = ab[(k + 1) * D + b];
        // (i/2) mu = (-mu.im/2, mu.re/2); Re(conj(that) y)
        acc[n + k * n + q] += T(-0.5) * m.im * y.re + T(0.5) * m.re * y.im;
      }
    }
  }
  for (int j = 0; j < 4 * n; ++j) eg_red[j * blockDim.x + threadIdx.x] = (double)acc[j];
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int j = 0; j < 4 * n; ++j)
        eg_red[j * blockDim.x + threadIdx.x] += eg_red[j * blockDim.x + threadIdx.x + s];
    __syncthreads();
  }
  for (int j = threadIdx.x; j < 4 * n; j += blockDim.x)
    egp[((int64_t)pb * chunks + blockIdx.x) * 4 * n + j] = eg_red[j * blockDim.x];
}

template <typename T>
__global__ void gb_embed_final(int n, int B, int chunks, int64_t p0, int64_t R,
                               const double* __restrict__ egp, const T* __restrict__ PT,
                               const T* __restrict__ tan, T* __restrict__ g_act,
                               T* __restrict__ g_tan) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B * n; i += gridDim.x * blockDim.x) {
    const int pb = i / n, q = i % n;
    const int64_t s = p0 + pb;
    if (s >= R) continue;
    double g[4] = {0, 0, 0, 0};
    for (int c = 0; c < chunks; ++c) {
      const double* e = egp + ((int64_t)pb * chunks + c) * 4 * n;
      for (int k = 0; k < 4; ++k) g[k] += e[k * n + q];
    }
    const T* pt = PT + ((int64_t)pb * n + q) * 8;
    const T s1 = pt[2], s2 = pt[3];
    T ga = T(g[0]) * s1;
    for (int k = 0; k < 3; ++k) {
      ga += T(g[1 + k]) * tan[((int64_t)k * R + s) * n + q] * s2;
      g_tan[((int64_t)k * R + s) * n + q] = T(g[1 + k]) * s1;
    }
    g_act[s * n + q] = ga;
  }
}

// readout partials (qsim.py:369-381, ansatz.py:395-399): per point
// z_q = sum_b |psi_b|^2 s_bq, dz_kq = sum_b 2 Re(conj(psi_b) dpsi_kb) s_bq
template <typename T>
__global__ void gb_readout(int n, int chunks, int nstates, const cplx<T>* __restrict__ X,
                           double* __restrict__ rp) {
  // per-thread partial sums, then a fixed warp-shuffle tree and a fixed
  // cross-warp order (deterministic); the dynamic shared memory is [warps][4 n]
  extern __shared__ double ro_red[];
  const int64_t D = (int64_t)1 << n;
  const int pb = blockIdx.y;
  const cplx<T>* x = X + (int64_t)pb * 4 * D;
  T acc[4 * 16];
#pragma unroll
  for (int j = 0; j < 4 * 16; ++j) acc[j] = T(0);
  const int64_t per = (D + chunks - 1) / chunks;
  const int64_t b0 = blockIdx.x * per, b1 = b0 + per < D ? b0 + per : D;
  for (int64_t b = b0 + threadIdx.x; b < b1; b += blockDim.x) {
    const cplx<T> psi = x[b];
    T v[4];
    v[0] = psi.re * psi.re + psi.im * psi.im;
#pragma unroll
    for (int k = 1; k < 4; ++k) {
      if (k < nstates) {
        const cplx<T> d = x[k * D + b];
        v[k] = T(2) * (psi.re * d.re + psi.im * d.im);
      } else {
        v[k] = T(0);
      }
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      if (q < n) {
        const bool neg = (b >> (n - 1 - q)) & 1;
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k * 16 + q] += neg ? -v[k] : v[k];
      }
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int j = 0; j < 4 * 16; ++j) {
    T v = acc[j];
    for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    acc[j] = v;
  }
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < 4; ++k)
      for (int q = 0; q < n; ++q) ro_red[w * 4 * n + k * n + q] = (double)acc[k * 16 + q];
  __syncthreads();
  for (int j = threadIdx.x; j < 4 * n; j += blockDim.x) {
    double t = 0.0;
    for (int i = 0; i < nw; ++i) t += ro_red[i * 4 * n + j];
    rp[((int64_t)pb * chunks + blockIdx.x) * 4 * n + j] = t;
  }
}

template <typename T>
__global__ void gb_readout_final(int n, int B, int chunks, int nstates, int64_t p0, int64_t R,
                                 const double* __restrict__ rp, T* __restrict__ z,
                                 T* __restrict__ dz) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < B * n; i += gridDim.x * blockDim.x) {
    const int pb = i / n, q = i % n;
    const int64_t s = p0 + pb;
    if (s >= R) continue;
    double g[4] = {0, 0, 0, 0};
    for (int c = 0; c < chunks; ++c)
      for (int k = 0; k < nstates; ++k) g[k] += rp[((int64_t)pb * chunks + c) * 4 * n + k * n + q];
    z[s * n + q] = T(g[0]);
    for (int k = 1; k < nstates; ++k) dz[((int64_t)(k - 1) * R + s) * n + q] = T(g[k]);
  }
}

template <typename T>
__global__ void gb_maxabs(int64_t count, const T* __restrict__ act,
                          unsigned long long* __restrict__ maxabs) {
  T m = T(0);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(act[i]));
  for (int s = 16; s >= 1; s >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, s));
  if ((threadIdx.x & 31) == 0) atomic_max_abs(maxabs, m);
}

constexpr int kGbChunks = 32;  // blocks per point for the embedding gradient / readout

struct GbLayout {
  int B;
  size_t acc, part, U, ph, PT, X, A, TMP, CK, EG, total;
};

template <typename T>
GbLayout gb_layout(const qpinn_circuit* c) {
  const size_t D = (size_t)1 << c->n, es = sizeof(cplx<T>);
  const size_t per_point = (3 + (size_t)c->L) * 4 * D * es;
  int B = (int)((size_t)(1u << 30) / per_point);  // ~1 GB of batch state
  B = B < 1 ? 1 : B > 16 ? 16 : B;
  GbLayout g{};
  g.B = B;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o += align_up(bytes, 256);
    return at;
  };
  g.acc = take(8 * (8 * (size_t)c->n_u1 + D * c->n_phase));
  g.part = take(8 * 8 * (size_t)num_sms() * 8);
  g.U = take(es * 4 * c->n_u1);
  g.ph = take(es * D * c->n_phase);
  g.PT = take(sizeof(T) * 8 * (size_t)B * c->n);
  g.X = take(4 * D * B * es);
  g.A = take(4 * D * B * es);
  g.TMP = take(4 * D * B * es);
  g.CK = take((size_t)c->L * 4 * D * B * es);
  g.EG = take(8 * (size_t)B * kGbChunks * 4 * c->n);
  g.total = o;
  return g;
}

// ---- several gates per HBM pass (forward with tangents, fp32, n >= 13) -------------
// The one-pass-per-gate forward above streams the [B][4][D] state through HBM once
// per gate.  Here the basis index is split as b = (s, l): the top h = n - kHbT bits
// s (wires 0 .. h-1) and the low kHbT bits l.  Two pass kinds each apply a run of
// gates in one read + write of the state:
//   SM pass: one CTA per (row, s) holds the 2^kHbT amplitudes of that slice in
//            shared memory -- gates on low wires, CNOTs whose target is a low wire
//            (a high control is fixed per slice), phase diagonals;
//   CS pass: one thread per (row, l) holds the 2^h amplitudes (s, l) in registers --
//            gates on high wires, CNOTs whose target is a high wire (a low control
//            is fixed per thread), phase diagonals.
// The CNOT runs are kept as individual CNOTs (qpinn_circuit::cnot_ct): a CNOT is
// local to the pass kind of its TARGET wire.  A host scheduler places every op of
// the fused plan (in gate order) into the earliest pass of its kind that follows
// every op it does not commute with, so a strongly-entangling layer costs one SM
// and one CS pass instead of n + 1 gate passes (plus one per CNOT run).
constexpr int kHbT = 12;  // low bits per SM tile: 2^12 complex = 32 KB of shared memory
enum { HB_U1 = 0, HB_CNOT = 1, HB_PHASE = 2 };
enum { HB_SM = 0, HB_CS = 1, HB_ANY = 2 };
struct HbOp {
  int type, a, b, idx;  // U1: a = bit, idx = u1 index; CNOT: a = control bit, b = target bit;
};                      // PHASE: idx = phase step
struct HbPass {
  int kind, op0, nops;
};
struct HbPlan {
  std::vector<HbOp> ops;
  std::vector<HbPass> passes;
  std::vector<int> luts;  // per CNOT run of an SM pass: [64 low | 64 high | 16 slice] index maps
};
constexpr int kHbLut = 64 + 64 + 16;

HbPlan hb_plan(const qpinn_circuit* c) {
  const int n = c->n, h = n - kHbT;
  struct Op {
    HbOp op;
    int kind;
    std::vector<int> wires;
  };
  std::vector<Op> seq;
  const int n_steps = (int)c->steps.size() / 3;
  for (int i = 0; i < n_steps; ++i) {
    const int type = c->steps[3 * i], wire = c->steps[3 * i + 1], idx = c->steps[3 * i + 2];
    if (type == STEP_U1) {
      seq.push_back({{HB_U1, n - 1 - wire, 0, idx}, wire < h ? HB_CS : HB_SM, {wire}});
    } else if (type == STEP_PERM) {
      for (int j = c->cnot_off[idx]; j < c->cnot_off[idx + 1]; ++j) {
        const int cw = c->cnot_ct[2 * j], tw = c->cnot_ct[2 * j + 1];
        seq.push_back({{HB_CNOT, n - 1 - cw, n - 1 - tw, 0}, tw < h ? HB_CS : HB_SM, {cw, tw}});
      }
    } else {
      std::vector<int> ws;
      for (int k = c->phase_off[idx]; k < c->phase_off[idx + 1]; ++k) {
        ws.push_back(c->pairs[3 * k]);
        ws.push_back(c->pairs[3 * k + 1]);
      }
      seq.push_back({{HB_PHASE, 0, 0, idx}, HB_ANY, ws});
    }
  }
  auto has = [](const std::vector<int>& v, int w) {
    for (int x : v)
      if (x == w) return true;
    return false;
  };
  auto commute = [&](const Op& x, const Op& y) {
    if (x.op.type == HB_PHASE && y.op.type == HB_PHASE) return true;
    if (x.op.type == HB_PHASE || y.op.type == HB_PHASE) {
      const Op& ph = x.op.type == HB_PHASE ? x : y;
      const Op& o = x.op.type == HB_PHASE ? y : x;
      if (o.op.type == HB_U1) return !has(ph.wires, o.wires[0]);
      return !has(ph.wires, o.wires[1]);  // a diagonal commutes with CNOT unless it reads the target
    }
    if (x.op.type == HB_U1 && y.op.type == HB_U1) return x.wires[0] != y.wires[0];
    if (x.op.type == HB_U1 || y.op.type == HB_U1) {
      const Op& u = x.op.type == HB_U1 ? x : y;
      const Op& cn = x.op.type == HB_U1 ? y : x;
      return !has(cn.wires, u.wires[0]);
    }
    return x.wires[1] != y.wires[0] && x.wires[0] != y.wires[1];  // CNOT, CNOT
  };
  std::vector<int> kinds;
  std::vector<std::vector<int>> members;  // op indices per pass, in gate order
  for (int i = 0; i < (int)seq.size(); ++i) {
    int kstar = -1;
    for (int k = 0; k < (int)members.size(); ++k)
      for (int j : members[k])
        if (!commute(seq[j], seq[i])) kstar = k;
    int k = kstar < 0 ? 0 : kstar;
    if (seq[i].kind == HB_ANY) {
      if (members.empty()) {
        kinds.push_back(HB_SM);
        members.emplace_back();
      }
    } else {
      while (k < (int)members.size() && kinds[k] != seq[i].kind) ++k;
      if (k == (int)members.size()) {
        kinds.push_back(seq[i].kind);
        members.emplace_back();
      }
    }
    members[k].push_back(i);
  }
  HbPlan plan;
  for (size_t k = 0; k < members.size(); ++k) {
    plan.passes.push_back({kinds[k], (int)plan.ops.size(), (int)members[k].size()});
    for (int j : members[k]) plan.ops.push_back(seq[j].op);
  }
  // A run of CNOTs in an SM pass is one GF(2)-linear index map on the 12 low bits
  // (plus the slice bits as fixed controls): new[i] = old[f(i, s)] with
  // f = g_first o ... o g_last, g(j) = j ^ (bit_c(j) << t).  f is tabulated as
  // f(i, s) = lo[i & 63] ^ hi[i >> 6] ^ sl[s]; the run head's idx is its table
  // offset and b its length (all of the run's CNOTs are then skipped).
  for (const HbPass& ps : plan.passes) {
    if (ps.kind != HB_SM) continue;
    int o = ps.op0;
    const int end = ps.op0 + ps.nops;
    while (o < end) {
      if (plan.ops[o].type != HB_CNOT) {
        ++o;
        continue;
      }
      int e = o + 1;
      while (e < end && plan.ops[e].type == HB_CNOT) ++e;
      auto f = [&](int i, int sl) {  // the run's map on a combined index
        int j = i;
        for (int q = e - 1; q >= o; --q) {
          const HbOp& c = plan.ops[q];
          const int on = c.a >= kHbT ? (sl >> (c.a - kHbT)) & 1 : (j >> c.a) & 1;
          j ^= on << c.b;
        }
        return j;
      };
      const int off = (int)plan.luts.size();
      plan.luts.resize(off + kHbLut, 0);
      int* lo = plan.luts.data() + off;
      int* hi = lo + 64;
      int* sl = hi + 64;
      for (int v = 0; v < 64; ++v) {
        lo[v] = f(v, 0);
        hi[v] = f(v << 6, 0);
      }
      for (int v = 0; v < 16; ++v) sl[v] = f(0, v);
      plan.ops[o].idx = off;
      plan.ops[o].b = plan.ops[o].b | ((e - o) << 8);  // run length rides in b's upper bits
      o = e;
    }
  }
  return plan;
}

__device__ __forceinline__ int hb_insert0(int k, int bit) {
  return ((k >> bit) << (bit + 1)) | (k & ((1 << bit) - 1));
}

// SM pass: CTA = (row, slice s); ops on the 2^kHbT low-bit amplitudes in shared memory.
// Runs of up to 3 single-qubit gates on distinct bits are applied together (8
// amplitudes per work item in registers, one barrier per run), and a run of CNOTs is
// one gather through the composed index map (one barrier per run).
template <int G>
__device__ __forceinline__ void hb_sm_u1_group(cplx<float>* t, const HbOp* op,
                                               const cplx<float>* __restrict__ U) {
  constexpr int TS = 1 << kHbT, M = 1 << G;
  int bits[G], sorted[G];
  cplx<float> u[G][4];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    bits[g] = op[g].a;
    sorted[g] = op[g].a;
#pragma unroll
    for (int e = 0; e < 4; ++e) u[g][e] = U[4 * op[g].idx + e];
  }
#pragma unroll
  for (int i = 0; i < G; ++i)
#pragma unroll
    for (int j = i + 1; j < G; ++j)
      if (sorted[j] < sorted[i]) {
        const int x = sorted[i];
        sorted[i] = sorted[j];
        sorted[j] = x;
      }
  for (int k = threadIdx.x; k < TS / M; k += blockDim.x) {
    int base = k;
#pragma unroll
    for (int g = 0; g < G; ++g) base = hb_insert0(base, sorted[g]);
    int idx[M];
    cplx<float> v[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      int i = base;
#pragma unroll
      for (int g = 0; g < G; ++g)
        if ((m >> g) & 1) i |= 1 << bits[g];
      idx[m] = i;
      v[m] = t[i];
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int m = 0; m < M; ++m) {
        if ((m >> g) & 1) continue;
        const int m1 = m | (1 << g);
        const cplx<float> a0 = v[m], a1 = v[m1];
        v[m] = cmul2(u[g][0], a0, u[g][1], a1);
        v[m1] = cmul2(u[g][2], a0, u[g][3], a1);
      }
    }
#pragma unroll
    for (int m = 0; m < M; ++m) t[idx[m]] = v[m];
  }
}

#ifndef QPINN_HB_MINB
#define QPINN_HB_MINB 4
#endif
#ifndef QPINN_HB_G
#define QPINN_HB_G 2
#endif
__global__ void __launch_bounds__(256, QPINN_HB_MINB) hb_sm_pass(int n, cplx<float>* __restrict__ X,
                                                  const HbOp* __restrict__ ops, int nops,
                                                  const int* __restrict__ luts,
                                                  const cplx<float>* __restrict__ U,
                                                  const cplx<float>* __restrict__ ph) {
  constexpr int TS = 1 << kHbT, PER = TS / 256;
  __shared__ cplx<float> t[TS];
  const int h = n - kHbT;
  const int64_t D = (int64_t)1 << n;
  const int64_t row = blockIdx.x >> h;
  const int s = blockIdx.x & ((1 << h) - 1);
  cplx<float>* x = X + row * D + ((int64_t)s << kHbT);
  {  // all of the thread's loads in flight before any shared-memory store
    cplx<float> r[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) r[j] = x[threadIdx.x + 256 * j];
#pragma unroll
    for (int j = 0; j < PER; ++j) t[threadIdx.x + 256 * j] = r[j];
  }
  __syncthreads();
  int o = 0;
  while (o < nops) {
    const HbOp op = ops[o];
    if (op.type == HB_U1) {
      int g = 1;  // run of single-qubit gates on distinct bits
      while (g < QPINN_HB_G && o + g < nops && ops[o + g].type == HB_U1) {
        bool distinct = true;
        for (int j = 0; j < g; ++j) distinct &= ops[o + j].a != ops[o + g].a;
        if (!distinct) break;
        ++g;
      }
      if (QPINN_HB_G >= 3 && g == 3) hb_sm_u1_group<3>(t, ops + o, U);
      else if (QPINN_HB_G >= 2 && g == 2) hb_sm_u1_group<2>(t, ops + o, U);
      else hb_sm_u1_group<1>(t, ops + o, U);
      o += g;
    } else if (op.type == HB_CNOT) {
      // a run of CNOTs: new[i] = old[f(i, s)] through the run's tabulated index map
      const int* lut = luts + op.idx;
      const int fs = lut[128 + s];
      cplx<float> v[PER];
#pragma unroll
      for (int r = 0; r < PER; ++r) {
        const int i = threadIdx.x + r * 256;
        v[r] = t[__ldg(lut + (i & 63)) ^ __ldg(lut + 64 + (i >> 6)) ^ fs];
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < PER; ++r) t[threadIdx.x + r * 256] = v[r];
      o += op.b >> 8;
    } else {
      const cplx<float>* ep = ph + (int64_t)op.idx * D + ((int64_t)s << kHbT);
      cplx<float> e[PER];
#pragma unroll
      for (int j = 0; j < PER; ++j) e[j] = ep[threadIdx.x + 256 * j];
#pragma unroll
      for (int j = 0; j < PER; ++j) t[threadIdx.x + 256 * j] = cmul(t[threadIdx.x + 256 * j], e[j]);
      ++o;
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < PER; ++j) x[threadIdx.x + 256 * j] = t[threadIdx.x + 256 * j];
}

// CS pass: thread = (row, low index l); the 2^H amplitudes (s, l) in registers
template <int H>
__device__ __forceinline__ void hb_swap_bit(cplx<float> (&v)[1 << H], int rb, int rc) {
  // swap v[j] <-> v[j | 1 << rb] for j with bit rb clear (and bit rc set when rc >= 0)
#pragma unroll
  for (int j = 0; j < (1 << H); ++j) {
    if (((j >> rb) & 1) == 0 && (rc < 0 || ((j >> rc) & 1))) {
      const cplx<float> a = v[j];
      v[j] = v[j | (1 << rb)];
      v[j | (1 << rb)] = a;
    }
  }
}

template <int H, int RB>
__device__ __forceinline__ void hb_gate_bit(cplx<float> (&v)[1 << H], cplx<float> u00,
                                            cplx<float> u01, cplx<float> u10, cplx<float> u11) {
#pragma unroll
  for (int j = 0; j < (1 << H); ++j) {
    if ((j >> RB) & 1) continue;
    const cplx<float> a = v[j], b = v[j | (1 << RB)];
    v[j] = cmul2(u00, a, u01, b);
    v[j | (1 << RB)] = cmul2(u10, a, u11, b);
  }
}

template <int H>
__global__ void __launch_bounds__(256) hb_cs_pass(int n, int64_t rows, cplx<float>* __restrict__ X,
                                                  const HbOp* __restrict__ ops, int nops,
                                                  const cplx<float>* __restrict__ U,
                                                  const cplx<float>* __restrict__ ph) {
  constexpr int V = 1 << H, TS = 1 << kHbT;
  const int64_t D = (int64_t)1 << n;
  for (int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < rows * TS;
       gid += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = gid >> kHbT;
    const int l = (int)(gid & (TS - 1));
    cplx<float>* x = X + row * D + l;
    cplx<float> v[V];
#pragma unroll
    for (int j = 0; j < V; ++j) v[j] = x[(int64_t)j << kHbT];
    for (int o = 0; o < nops; ++o) {
      const HbOp op = ops[o];
      if (op.type == HB_U1) {
        const cplx<float>* u = U + 4 * op.idx;
        const cplx<float> u00 = u[0], u01 = u[1], u10 = u[2], u11 = u[3];
        const int rb = op.a - kHbT;
        if (rb == 0) hb_gate_bit<H, 0>(v, u00, u01, u10, u11);
        if constexpr (H > 1) if (rb == 1) hb_gate_bit<H, 1>(v, u00, u01, u10, u11);
        if constexpr (H > 2) if (rb == 2) hb_gate_bit<H, 2>(v, u00, u01, u10, u11);
        if constexpr (H > 3) if (rb == 3) hb_gate_bit<H, 3>(v, u00, u01, u10, u11);
      } else if (op.type == HB_CNOT) {
        const int rb = op.b - kHbT;
        if (op.a < kHbT) {  // low control: fixed for this thread
          if ((l >> op.a) & 1) {
#pragma unroll
            for (int q = 0; q < H; ++q)
              if (q == rb) hb_swap_bit<H>(v, q, -1);
          }
        } else {
          const int rc = op.a - kHbT;
#pragma unroll
          for (int q = 0; q < H; ++q)
#pragma unroll
            for (int r = 0; r < H; ++r)
              if (q == rb && r == rc) hb_swap_bit<H>(v, q, r);
        }
      } else {
        const cplx<float>* e = ph + (int64_t)op.idx * D + l;
#pragma unroll
        for (int j = 0; j < V; ++j) v[j] = cmul(v[j], e[(int64_t)j << kHbT]);
      }
    }
#pragma unroll
    for (int j = 0; j < V; ++j) x[(int64_t)j << kHbT] = v[j];
  }
}

struct HbLayout {
  int B;
  size_t U, ph, PT, RP, ops, X, total;
};

HbLayout hb_layout(const qpinn_circuit* c, int64_t B, int nops, int nluts) {
  const size_t D = (size_t)1 << c->n, es = sizeof(cplx<float>);
  HbLayout g{};
  g.B = (int)B;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o += align_up(bytes, 256);
    return at;
  };
  g.U = take(es * 4 * c->n_u1);
  g.ph = take(es * D * c->n_phase);
  g.PT = take(sizeof(float) * 8 * (size_t)B * c->n);
  g.RP = take(8 * (size_t)B * kGbChunks * 4 * c->n);
  g.ops = take(sizeof(HbOp) * (size_t)(nops > 0 ? nops : 1) + sizeof(int) * (size_t)nluts);
  g.X = take(4 * D * (size_t)B * es);
  g.total = o;
  return g;
}

int hb_launch_cs(int h, int n, int64_t rows, cplx<float>* X, const HbOp* ops, int nops,
                 const cplx<float>* U, const cplx<float>* ph, cudaStream_t st) {
  const int64_t threads = rows << kHbT;
  const int grid = (int)((threads + 255) / 256 < (int64_t)num_sms() * 8 ? (threads + 255) / 256
                                                                       : (int64_t)num_sms() * 8);
  switch (h) {
    case 1: hb_cs_pass<1><<<grid, 256, 0, st>>>(n, rows, X, ops, nops, U, ph); break;
    case 2: hb_cs_pass<2><<<grid, 256, 0, st>>>(n, rows, X, ops, nops, U, ph); break;
    case 3: hb_cs_pass<3><<<grid, 256, 0, st>>>(n, rows, X, ops, nops, U, ph); break;
    case 4: hb_cs_pass<4><<<grid, 256, 0, st>>>(n, rows, X, ops, nops, U, ph); break;
    default: return fail(QPINN_ERR_CAPACITY, "multi-gate HBM pass: 13 <= n <= 16");
  }
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

}  // namespace

bool hbm_fwd_supported(const qpinn_circuit* c, int dtype) {
  if (!c || dtype != QPINN_F32 || c->n <= kHbT || c->n > kHbT + 4) return false;
  if (getenv("QPINN_PQC_HBM_MULTIGATE") && atoi(getenv("QPINN_PQC_HBM_MULTIGATE")) == 0) return false;
  return true;
}

// forward with tangents (or value only), several gates per HBM pass (see hb_plan)
int hbm_forward(const qpinn_circuit* c, const KArgs<float>* a, unsigned char* ws, size_t bytes) {
  const PlanDev& p = c->dev;
  const int n = c->n, h = n - kHbT;
  const int64_t D = (int64_t)1 << n;
  const HbPlan plan = hb_plan(c);
  const int nops = (int)plan.ops.size();
  if (getenv("QPINN_VERBOSE")) {
    fprintf(stderr, "[qpinn] multi-gate HBM forward: n = %d, L = %d, %d ops in %d passes:", n,
            c->L, nops, (int)plan.passes.size());
    for (const HbPass& ps : plan.passes) fprintf(stderr, " %s%d", ps.kind == HB_SM ? "S" : "C", ps.nops);
    fprintf(stderr, "\n");
  }
  // largest batch of points that fits the workspace
  int64_t B = a->R < 1024 ? a->R : 1024;
  const int nluts = (int)plan.luts.size();
  while (B > 1 && hb_layout(c, B, nops, nluts).total > bytes) B = B * 3 / 4;
  const HbLayout g = hb_layout(c, B < 1 ? 1 : B, nops, nluts);
  if (bytes < g.total) return fail(QPINN_ERR_CONFIG, "multi-gate HBM PQC: workspace too small");
  cudaStream_t st = a->stream;
  auto* U = (cplx<float>*)(ws + g.U);
  auto* ph = (cplx<float>*)(ws + g.ph);
  auto* PT = (float*)(ws + g.PT);
  auto* RP = (double*)(ws + g.RP);
  auto* dops = (HbOp*)(ws + g.ops);
  auto* X = (cplx<float>*)(ws + g.X);
  auto* dluts = (int*)(dops + nops);
  QPINN_CUDA_CHECK(cudaMemcpyAsync(dops, plan.ops.data(), sizeof(HbOp) * nops,
                                   cudaMemcpyHostToDevice, st));
  if (nluts)
    QPINN_CUDA_CHECK(cudaMemcpyAsync(dluts, plan.luts.data(), sizeof(int) * nluts,
                                     cudaMemcpyHostToDevice, st));
  const int ns = a->tan ? 4 : 1;
  const int ro_smem = 4 * n * 4 * (int)sizeof(double);  // [4 warps][4 n]
  QPINN_CUDA_CHECK(cudaFuncSetAttribute(gb_readout<float>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, ro_smem));
  gb_tables<float><<<64, 256, 0, st>>>(p, a->qp, U, ph);
  if (a->maxabs)
    gb_maxabs<float><<<gb_blocks(a->R * n), kGbThreads, 0, st>>>(a->R * n, a->act, a->maxabs);
  for (int64_t p0 = 0; p0 < a->R; p0 += g.B) {
    const int Bc = (int)(a->R - p0 < g.B ? a->R - p0 : g.B);
    const int64_t rows = (int64_t)Bc * 4;
    gb_point<float><<<gb_blocks(Bc * n), kGbThreads, 0, st>>>(n, a->scale, a->R, p0, Bc, a->act,
                                                              a->tan, PT);
    gb_embed<float><<<gb_blocks(Bc * D), kGbThreads, 0, st>>>(n, Bc, ns, PT, X);
    for (const HbPass& ps : plan.passes) {
      if (ps.kind == HB_SM) {
        hb_sm_pass<<<(unsigned)(rows << h), 256, 0, st>>>(n, X, dops + ps.op0, ps.nops, dluts, U,
                                                          ph);
        QPINN_CUDA_CHECK(cudaGetLastError());
      } else if (int rc = hb_launch_cs(h, n, rows, X, dops + ps.op0, ps.nops, U, ph, st)) {
        return rc;
      }
    }
    gb_readout<float><<<dim3(kGbChunks, Bc), 128, ro_smem, st>>>(n, kGbChunks, ns, X, RP);
    gb_readout_final<float><<<gb_blocks(Bc * n), kGbThreads, 0, st>>>(n, Bc, kGbChunks, ns, p0,
                                                                      a->R, RP, a->z, a->dz);
    QPINN_CUDA_CHECK(cudaGetLastError());
  }
  return QPINN_OK;
}

// number of HBM passes per forward of the multi-gate path (diagnostics)
int hbm_forward_passes(const qpinn_circuit* c) { return (int)hb_plan(c).passes.size(); }

size_t global_adjoint_workspace_bytes(const qpinn_circuit* c, int dtype) {
  if (dtype == QPINN_F64) return gb_layout<double>(c).total;
  // the multi-gate forward reuses this region with batches of ~256 MB of state
  // (1024 points at n = 13), so few launches carry the batch loop
  const size_t g = gb_layout<float>(c).total;
  if (!hbm_fwd_supported(c, dtype)) return g;
  const int64_t B = ((int64_t)256 << 20) / (4 * ((int64_t)8 << c->n));
  const HbPlan plan = hb_plan(c);
  const size_t h = hb_layout(c, B < 1 ? 1 : B, (int)plan.ops.size(), (int)plan.luts.size()).total;
  return h > g ? h : g;
}

template <typename T>
int global_backward(const qpinn_circuit* c, const KArgs<T>* a, unsigned char* ws, size_t bytes) {
  const PlanDev& p = c->dev;
  const int n = c->n, L = c->L;
  const int64_t D = (int64_t)1 << n;
  const int ent = layer_entangler(c);
  if (ent < 0) return fail(QPINN_ERR_CAPACITY, "HBM-regime adjoint needs the standard layer plan");
  const GbLayout g = gb_layout<T>(c);
  if (bytes < g.total) return fail(QPINN_ERR_CONFIG, "HBM-regime adjoint: workspace too small");
  cudaStream_t st = a->stream;
  double* acc = (double*)(ws + g.acc);
  double* part = (double*)(ws + g.part);
  cplx<T>* U = (cplx<T>*)(ws + g.U);
  cplx<T>* ph = (cplx<T>*)(ws + g.ph);
  T* PT = (T*)(ws + g.PT);
  cplx<T>* X = (cplx<T>*)(ws + g.X);
  cplx<T>* A = (cplx<T>*)(ws + g.A);
  cplx<T>* TMP = (cplx<T>*)(ws + g.TMP);
  cplx<T>* CK = (cplx<T>*)(ws + g.CK);
  double* EG = (double*)(ws + g.EG);
  const int n_acc = 8 * p.n_u1 + (int)D * p.n_phase;
  const int eg_smem = 4 * n * 128 * (int)sizeof(double);
  QPINN_CUDA_CHECK(cudaFuncSetAttribute(gb_embed_grad<T>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, eg_smem));
  QPINN_CUDA_CHECK(cudaMemsetAsync(acc, 0, 8 * (size_t)n_acc, st));
  gb_tables<T><<<64, 256, 0, st>>>(p, a->qp, U, ph);
  const int B = g.B;
  const int64_t rows = (int64_t)B * 4;
  const int ob = gb_blocks(rows * (D / 2));
  for (int64_t p0 = 0; p0 < a->R; p0 += B) {
    gb_point<T><<<gb_blocks(B * n), kGbThreads, 0, st>>>(n, a->scale, a->R, p0, B, a->act, a->tan,
                                                         PT);
    gb_embed<T><<<gb_blocks(B * D), kGbThreads, 0, st>>>(n, B, 4, PT, X);
    // forward with layer-boundary checkpoints
    for (int l = 0; l < L; ++l) {
      for (int q = 0; q < n; ++q)
        gb_u1<T><<<ob, kGbThreads, 0, st>>>(n, rows, X, q, U + 4 * (l * n + q), 0);
      QPINN_CUDA_CHECK(cudaMemcpyAsync(CK + (size_t)l * rows * D, X, rows * D * sizeof(cplx<T>),
                                       cudaMemcpyDeviceToDevice, st));
      if (ent == ENT_PERM) {
        gb_perm<T><<<gb_blocks(rows * D), kGbThreads, 0, st>>>(n, rows, X, TMP, p.perm + l * D);
        std::swap(X, TMP);
      } else if (ent == ENT_PHASE) {
        gb_phase<T><<<gb_blocks(rows * D), kGbThreads, 0, st>>>(n, rows, X, ph + l * D, 0);
      }
    }
    gb_seed<T><<<gb_blocks(B * D), kGbThreads, 0, st>>>(n, B, p0, a->R, a->gz, a->gdz, X, A);
    // reverse sweep: only the adjoint is propagated
    for (int l = L - 1; l >= 0; --l) {
      const cplx<T>* xl = CK + (size_t)l * rows * D;
      if (ent == ENT_PERM) {
        gb_perm<T><<<gb_blocks(rows * D), kGbThreads, 0, st>>>(n, rows, A, TMP, p.iperm + l * D);
        std::swap(A, TMP);
      } else if (ent == ENT_PHASE) {
        gb_phase_grad<T><<<gb_blocks(D), kGbThreads, 0, st>>>(n, rows, xl, A, ph + l * D,
                                                               acc + 8 * p.n_u1 + l * D);
        gb_phase<T><<<gb_blocks(rows * D), kGbThreads, 0, st>>>(n, rows, A, ph + l * D, 1);
      }
      for (int q = 0; q < n; ++q) {
        gb_outer<T><<<ob, kGbThreads, 0, st>>>(n, rows, xl, A, q, part);
        gb_sum8<<<1, 32, 0, st>>>(ob, part, acc + 8 * (l * n + q));
      }
      for (int q = 0; q < n; ++q)
        gb_u1<T><<<ob, kGbThreads, 0, st>>>(n, rows, A, q, U + 4 * (l * n + q), 1);
    }
    // embedding gradient against the re-embedded state
    gb_embed<T><<<gb_blocks(B * D), kGbThreads, 0, st>>>(n, B, 1, PT, X);
    gb_embed_grad<T><<<dim3(kGbChunks, B), 128, eg_smem, st>>>(
        n, kGbChunks, PT, X, A, EG);
    gb_embed_final<T><<<gb_blocks(B * n), kGbThreads, 0, st>>>(n, B, kGbChunks, p0, a->R, EG, PT,
                                                                a->tan, a->g_act, a->g_tan);
    QPINN_CUDA_CHECK(cudaGetLastError());
  }
  return pqc_param_grads<T>(c, acc, n, a->qp, a->g_qp, st);
}

// forward in global memory: value-only for any n beyond the register kernels,
// and with tangents where no cluster kernel exists (float64, n = 16)
template <typename T>
int global_forward(const qpinn_circuit* c, const KArgs<T>* a, unsigned char* ws, size_t bytes) {
  const PlanDev& p = c->dev;
  const int n = c->n, L = c->L;
  const int64_t D = (int64_t)1 << n;
  const int ent = layer_entangler(c);
  if (ent < 0) return fail(QPINN_ERR_CAPACITY, "global-memory PQC needs the standard layer plan");
  const GbLayout g = gb_layout<T>(c);
  if (bytes < g.total) return fail(QPINN_ERR_CONFIG, "global-memory PQC: workspace too small");
  cudaStream_t st = a->stream;
  cplx<T>* U = (cplx<T>*)(ws + g.U);
  cplx<T>* ph = (cplx<T>*)(ws + g.ph);
  T* PT = (T*)(ws + g.PT);
  cplx<T>* X = (cplx<T>*)(ws + g.X);
  cplx<T>* TMP = (cplx<T>*)(ws + g.TMP);
  double* RP = (double*)(ws + g.EG);
  const int ns = a->tan ? 4 : 1;
  const int ro_smem = 4 * n * 4 * (int)sizeof(double);  // [4 warps][4 n]
  QPINN_CUDA_CHECK(cudaFuncSetAttribute(gb_readout<T>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, ro_smem));
  gb_tables<T><<<64, 256, 0, st>>>(p, a->qp, U, ph);
  if (a->maxabs)
    gb_maxabs<T><<<gb_blocks(a->R * n), kGbThreads, 0, st>>>(a->R * n, a->act, a->maxabs);
  const int B = g.B;
  const int64_t rows = (int64_t)B * 4;
  const int ob = gb_blocks(rows * (D / 2));
  for (int64_t p0 = 0; p0 < a->R; p0 += B) {
    gb_point<T><<<gb_blocks(B * n), kGbThreads, 0, st>>>(n, a->scale, a->R, p0, B, a->act,
                                                         a->tan, PT);
    gb_embed<T><<<gb_blocks(B * D), kGbThreads, 0, st>>>(n, B, ns, PT, X);
    for (int l = 0; l < L; ++l) {
      for (int q = 0; q < n; ++q)
        gb_u1<T><<<ob, kGbThreads, 0, st>>>(n, rows, X, q, U + 4 * (l * n + q), 0);
      if (ent == ENT_PERM) {
        gb_perm<T><<<gb_blocks(rows * D), kGbThreads, 0, st>>>(n, rows, X, TMP, p.perm + l * D);
        std::swap(X, TMP);
      } else if (ent == ENT_PHASE) {
        gb_phase<T><<<gb_blocks(rows * D), kGbThreads, 0, st>>>(n, rows, X, ph + l * D, 0);
      }
    }
    gb_readout<T><<<dim3(kGbChunks, B), 128, ro_smem, st>>>(n, kGbChunks, ns, X, RP);
    gb_readout_final<T><<<gb_blocks(B * n), kGbThreads, 0, st>>>(n, B, kGbChunks, ns, p0, a->R,
                                                                  RP, a->z, a->dz);
    QPINN_CUDA_CHECK(cudaGetLastError());
  }
  return QPINN_OK;
}

template int global_forward<float>(const qpinn_circuit*, const KArgs<float>*, unsigned char*,
                                   size_t);
template int global_forward<double>(const qpinn_circuit*, const KArgs<double>*, unsigned char*,
                                    size_t);
template int global_backward<float>(const qpinn_circuit*, const KArgs<float>*, unsigned char*,
                                    size_t);
template int global_backward<double>(const qpinn_circuit*, const KArgs<double>*, unsigned char*,
                                     size_t);

}  // namespace qpinn
