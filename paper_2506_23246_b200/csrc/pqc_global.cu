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
#include <algorithm>
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

// embedded state and its tangents (ansatz.py:233-243, :380-390); wire q is bit n-1-q.
// 4 consecutive amplitudes per thread (b0 .. b0 + 3: only the last two wires differ):
// the first n - 2 factors and their tangent terms are shared (n >= 2)
template <typename T>
__global__ void gb_embed4(int n, int B, int nstates, const T* __restrict__ PT,
                          cplx<T>* __restrict__ X) {
  const int64_t D = (int64_t)1 << n, Q = D / 4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < B * Q;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int pb = (int)(i / Q);
    const int64_t b0 = (i % Q) * 4;
    const T* pt = PT + (int64_t)pb * n * 8;
    const int H = n - 2;
    T pre[15];  // prefix products over the shared wires (statically indexed)
    pre[0] = T(1);
#pragma unroll
    for (int q = 0; q < 14; ++q) {
      if (q < H) {
        const int bit = (b0 >> (n - 1 - q)) & 1;
        pre[q + 1] = pre[q] * (bit ? pt[q * 8 + 1] : pt[q * 8]);
      } else {
        pre[q + 1] = pre[q];
      }
    }
    const T P = pre[14];
    T tk[3] = {T(0), T(0), T(0)}, suf = T(1);
#pragma unroll
    for (int q = 13; q >= 0; --q) {
      if (q < H) {
        const int bit = (b0 >> (n - 1 - q)) & 1;
        const T df = bit ? T(0.5) * pt[q * 8] : T(-0.5) * pt[q * 8 + 1];
        const T rest = pre[q] * suf;
#pragma unroll
        for (int k = 0; k < 3; ++k) tk[k] += pt[q * 8 + 4 + k] * df * rest;
        suf *= bit ? pt[q * 8 + 1] : pt[q * 8];
      }
    }
    // the last two wires a = H (bit 1 of b - b0), c = H + 1 (bit 0)
    const T* pa = pt + H * 8;
    const T* pc = pa + 8;
    const T fa[2] = {pa[0], pa[1]}, fc[2] = {pc[0], pc[1]};
    const T da[2] = {T(-0.5) * pa[1], T(0.5) * pa[0]}, dc[2] = {T(-0.5) * pc[1], T(0.5) * pc[0]};
    T m[4][4];  // [state][amplitude]
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int ia = e >> 1, ic = e & 1;
      m[0][e] = P * fa[ia] * fc[ic];
#pragma unroll
      for (int k = 0; k < 3; ++k)
        m[k + 1][e] = tk[k] * fa[ia] * fc[ic] + pa[4 + k] * da[ia] * P * fc[ic] +
                      pc[4 + k] * dc[ic] * P * fa[ia];
    }
    const int pop = __popcll(b0);
    for (int s = 0; s < nstates; ++s) {
      cplx<T> o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int ph = (pop + __popc(e)) & 3;  // (-i)^popcount(b0 + e)
        const T v = m[s][e];
        o[e] = {ph == 0 ? v : ph == 2 ? -v : T(0), ph == 1 ? -v : ph == 3 ? v : T(0)};
      }
      cplx<T>* dst = X + ((int64_t)pb * 4 + s) * D + b0;
#pragma unroll
      for (int e = 0; e < 4; ++e) dst[e] = o[e];
    }
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
  // per-thread partial sums, a fixed warp-shuffle tree and a fixed cross-warp
  // order (deterministic); dynamic shared memory [warps][4 n]
  extern __shared__ double eg_red[];
  const int64_t D = (int64_t)1 << n;
  const int pb = blockIdx.y;
  const T* pt = PT + (int64_t)pb * n * 8;
  const cplx<T>* phi = PHI + (int64_t)pb * 4 * D;  // state 0 of the re-embedded batch
  const cplx<T>* ab = A + (int64_t)pb * 4 * D;
  T acc[4 * 16];
#pragma unroll
  for (int j = 0; j < 4 * 16; ++j) acc[j] = T(0);
  const int64_t per = (D + chunks - 1) / chunks;
  const int64_t b0 = blockIdx.x * per, b1 = b0 + per < D ? b0 + per : D;
  for (int64_t b = b0 + threadIdx.x; b < b1; b += blockDim.x) {
    const cplx<T> phib = ab[b];
    cplx<T> eta = {T(-0.5) * phib.im, T(0.5) * phib.re};  // (i/2) phibar
    cplx<T> mb[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) mb[k] = ab[(k + 1) * D + b];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      if (q < n) {
        const int64_t f = b ^ ((int64_t)1 << (n - 1 - q));
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const cplx<T> m = ab[(k + 1) * D + f];
          const T wk = T(0.25) * __ldg(pt + q * 8 + 4 + k);
          eta.re -= wk * m.re;
          eta.im -= wk * m.im;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      if (q < n) {
        const cplx<T> y = phi[b ^ ((int64_t)1 << (n - 1 - q))];
        acc[q] += eta.re * y.re + eta.im * y.im;  // Re(conj(eta) y)
#pragma unroll
        for (int k = 0; k < 3; ++k)  // (i/2) mu = (-mu.im/2, mu.re/2); Re(conj(that) y)
          acc[16 + k * 16 + q] += T(-0.5) * mb[k].im * y.re + T(0.5) * mb[k].re * y.im;
      }
    }
  }
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int j = 0; j < 4 * 16; ++j) {
    T v = acc[j];
    for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    acc[j] = v;
  }
  if (lane == 0)
#pragma unroll
    for (int g = 0; g < 4; ++g)
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (q < n) eg_red[wp * 4 * n + g * n + q] = (double)acc[g * 16 + q];
  __syncthreads();
  for (int j = threadIdx.x; j < 4 * n; j += blockDim.x) {
    double t = 0.0;
    for (int i = 0; i < nw; ++i) t += eg_red[i * 4 * n + j];
    egp[((int64_t)pb * chunks + blockIdx.x) * 4 * n + j] = t;
  }
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
  T plain[4] = {T(0), T(0), T(0), T(0)};
  const int lowb = (int)((b0 + threadIdx.x) & 127);  // b's low 7 bits (blockDim = 128)
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
    // the wires on the 7 low bits of b are fixed per thread (b advances by 128): their
    // sums are the thread's plain sums, signed once after the loop
#pragma unroll
    for (int k = 0; k < 4; ++k) plain[k] += v[k];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      if (q < n - 7) {
        const bool neg = (b >> (n - 1 - q)) & 1;
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k * 16 + q] += neg ? -v[k] : v[k];
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    if (q >= n - 7 && q < n) {
      const bool neg = (lowb >> (n - 1 - q)) & 1;
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[k * 16 + q] = neg ? -plain[k] : plain[k];
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
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (q < n) ro_red[w * 4 * n + k * n + q] = (double)acc[k * 16 + q];
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

// ---- several gates per HBM pass (fp32, 9 <= n <= 16; the default from n = 11-13) -------
// The one-pass-per-gate kernels above stream the [B][4][D] states through HBM once per
// gate.  Here the basis index is split as b = (s, l): the top h = n - kHbT bits s
// (wires 0 .. h-1) and the low kHbT bits l (for n <= kHbT: h = 0, the tile is the
// whole state and every pass is an SM pass).  Two pass kinds each apply a run of ops in
// one read + write of the state:
//   SM pass: one CTA per (row, s) holds the 2^kHbT amplitudes of that slice in
//            shared memory -- gates on low wires, CNOTs whose target is a low wire
//            (a high control is fixed per slice), phase diagonals;
//   CS pass: one thread per (row, l) holds the 2^h amplitudes (s, l) in registers --
//            gates on high wires, CNOTs whose target is a high wire (a low control
//            is fixed per thread), phase diagonals.
// The CNOT runs are kept as individual CNOTs (qpinn_circuit::cnot_ct): a CNOT is
// local to the pass kind of its TARGET wire.  A host scheduler places every op (in
// circuit order) into the earliest pass of its kind that follows every op it does not
// commute with, so a strongly-entangling layer costs one SM and one CS pass instead
// of n + 1 gate passes (plus one per CNOT run).
//
// The adjoint (hbm_backward) uses the same passes: a forward that checkpoints the
// states after every layer's single-qubit gates (a copy after the segment that ends
// there), the seeds, then a reverse op sequence per layer l = L-1 .. 0:
//   entangler(l)^dagger (CNOTs in reverse order | the conjugate phase),
//   OUTER_q: the post-gate outer product M'_q = sum conj(abar) x_l of every wire q
//            from the boundary adjoint and checkpoint (gates of a layer commute, so
//            each is the layer's last, as the layer kernels' K2),
//   U_q^dagger for every wire q,
// scheduled like the forward: OUTER ops commute only with each other, so a layer
// costs about two passes.  OUTER partials are reduced per CTA and then across CTAs
// in a fixed order (deterministic).
constexpr int kHbT = 12;  // low bits per SM tile: 2^12 complex = 32 KB of shared memory
// the forward (no checkpoint tile) may use 2^13-amplitude tiles (64 KB): at n = 13 the
// whole circuit runs in SM passes, and from n = 14 one wire fewer goes to CS passes
constexpr int kHbTmax = 13;
#ifndef QPINN_HB_OUTER2
#define QPINN_HB_OUTER2 1
#endif
constexpr bool kHbOuter2 = QPINN_HB_OUTER2;  // OUTER ops two per sweep in SM passes
enum { HB_U1 = 0, HB_CNOT = 1, HB_PHASE = 2, HB_OUTER = 3 };
enum { HB_SM = 0, HB_CS = 1, HB_ANY = 2 };
struct HbOp {
  // U1: a = bit, b = dagger, idx = u1 index;  CNOT: a = control bit, b = target bit
  // (| run length << 8 at an SM run head, whose idx is then its table offset);
  // PHASE: b = conjugate, idx = phase step;  OUTER: a = bit, idx = u1 index (acc slot)
  int type, a, b, idx;
};
struct HbPass {
  int kind, op0, nops;
  int ck;         // forward with checkpoints: copy the state to checkpoint ck after this pass
  int layer;      // OUTER passes: the checkpoint layer they read (-1: none)
  int phase_grad; // reverse: the phase-step gradient to take before this pass (-1: none)
  int n_outer;    // OUTER ops in this pass
};
struct HbPlan {
  std::vector<HbOp> ops;
  std::vector<HbPass> passes;
  std::vector<int> luts;  // per CNOT run of an SM pass: [64 low | 256 high | 16 slice] index maps
  int T = kHbT;           // low (tile) bits of this plan's SM passes
};
constexpr int kHbLut = 64 + 256 + 16;

struct HbSOp {  // an op being scheduled
  HbOp op;
  int kind;
  std::vector<int> wires;
  int layer;
  bool barrier;  // must start a fresh pass (a phase step whose gradient is taken first)
};

bool hb_commute(const HbSOp& x, const HbSOp& y) {
  auto has = [](const std::vector<int>& v, int w) {
    for (int e : v)
      if (e == w) return true;
    return false;
  };
  if (x.op.type == HB_OUTER || y.op.type == HB_OUTER)
    return x.op.type == HB_OUTER && y.op.type == HB_OUTER;  // reads the adjoint as it is
  if (x.op.type == HB_PHASE && y.op.type == HB_PHASE) return true;
  if (x.op.type == HB_PHASE || y.op.type == HB_PHASE) {
    const HbSOp& ph = x.op.type == HB_PHASE ? x : y;
    const HbSOp& o = x.op.type == HB_PHASE ? y : x;
    if (o.op.type == HB_U1) return !has(ph.wires, o.wires[0]);
    return !has(ph.wires, o.wires[1]);  // a diagonal commutes with CNOT unless it reads the target
  }
  if (x.op.type == HB_U1 && y.op.type == HB_U1) return x.wires[0] != y.wires[0];
  if (x.op.type == HB_U1 || y.op.type == HB_U1) {
    const HbSOp& u = x.op.type == HB_U1 ? x : y;
    const HbSOp& cn = x.op.type == HB_U1 ? y : x;
    return !has(cn.wires, u.wires[0]);
  }
  return x.wires[1] != y.wires[0] && x.wires[0] != y.wires[1];  // CNOT, CNOT
}

// earliest-legal-pass list scheduling of an op sequence; appends to plan
void hb_schedule(const std::vector<HbSOp>& seq, HbPlan& plan) {
  std::vector<int> kinds;
  std::vector<std::vector<int>> members;
  std::vector<int> pgrad;
  for (int i = 0; i < (int)seq.size(); ++i) {
    int kstar = -1;
    for (int k = 0; k < (int)members.size(); ++k)
      for (int j : members[k])
        if (!hb_commute(seq[j], seq[i])) kstar = k;
    int k;
    if (seq[i].barrier) {
      k = (int)members.size();
      kinds.push_back(HB_SM);
      members.emplace_back();
      pgrad.push_back(seq[i].op.idx);
    } else {
      k = kstar < 0 ? 0 : kstar;
      if (seq[i].kind == HB_ANY) {
        if (members.empty()) {
          kinds.push_back(HB_SM);
          members.emplace_back();
          pgrad.push_back(-1);
        }
      } else {
        // an OUTER op reads its layer's checkpoint tile: one layer per pass (with
        // h = 0 every op is of SM kind and consecutive layers would share a pass)
        auto other_layer = [&](int kk) {
          if (seq[i].op.type != HB_OUTER) return false;
          for (int j : members[kk])
            if (seq[j].op.type == HB_OUTER && seq[j].layer != seq[i].layer) return true;
          return false;
        };
        while (k < (int)members.size() && (kinds[k] != seq[i].kind || other_layer(k))) ++k;
        if (k == (int)members.size()) {
          kinds.push_back(seq[i].kind);
          members.emplace_back();
          pgrad.push_back(-1);
        }
      }
    }
    members[k].push_back(i);
  }
  for (size_t k = 0; k < members.size(); ++k) {
    HbPass ps{kinds[k], (int)plan.ops.size(), (int)members[k].size(), -1, -1, pgrad[k], 0};
    for (int j : members[k]) {
      plan.ops.push_back(seq[j].op);
      if (seq[j].op.type == HB_OUTER) {
        ps.layer = seq[j].layer;
        ++ps.n_outer;
      }
    }
    plan.passes.push_back(ps);
  }
}

// A run of CNOTs in an SM pass is one GF(2)-linear index map on the 12 low bits (plus
// the slice bits as fixed controls): new[i] = old[f(i, s)] with f = g_first o ... o
// g_last, g(j) = j ^ (bit_c(j) << t), tabulated as f(i, s) = lo[i & 63] ^ hi[i >> 6] ^ sl[s]
void hb_tabulate(HbPlan& plan) {
  const int T = plan.T;
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
      auto f = [&](int i, int sl) {
        int j = i;
        for (int q = e - 1; q >= o; --q) {
          const HbOp& c = plan.ops[q];
          const int on = c.a >= T ? (sl >> (c.a - T)) & 1 : (j >> c.a) & 1;
          j ^= on << (c.b & 0xff);
        }
        return j;
      };
      const int off = (int)plan.luts.size();
      plan.luts.resize(off + kHbLut, 0);
      int* lo = plan.luts.data() + off;
      int* hi = lo + 64;
      int* sl = hi + 256;
      for (int v = 0; v < 64; ++v) lo[v] = f(v, 0);
      for (int v = 0; v < 256; ++v) hi[v] = f(v << 6, 0);
      for (int v = 0; v < 16; ++v) sl[v] = f(0, v);
      plan.ops[o].idx = off;
      plan.ops[o].b = (plan.ops[o].b & 0xff) | ((e - o) << 8);
      o = e;
    }
  }
}

// the fused plan as per-layer op lists (u1 ops, entangler ops) in circuit order
struct HbLayerOps {
  std::vector<HbSOp> u1, ent;
};

std::vector<HbLayerOps> hb_layers(const qpinn_circuit* c, int T) {
  const int n = c->n, h = n - T;
  std::vector<HbLayerOps> layers(c->L);
  const int n_steps = (int)c->steps.size() / 3;
  int l = 0, in_layer = 0;
  for (int i = 0; i < n_steps; ++i) {
    const int type = c->steps[3 * i], wire = c->steps[3 * i + 1], idx = c->steps[3 * i + 2];
    if (type == STEP_U1) {
      if (in_layer == n) {  // a layer without an entangler step ended
        ++l;
        in_layer = 0;
      }
      layers[l].u1.push_back({{HB_U1, n - 1 - wire, 0, idx}, wire < h ? HB_CS : HB_SM, {wire}, l,
                              false});
      ++in_layer;
    } else if (type == STEP_PERM) {
      for (int j = c->cnot_off[idx]; j < c->cnot_off[idx + 1]; ++j) {
        const int cw = c->cnot_ct[2 * j], tw = c->cnot_ct[2 * j + 1];
        layers[l].ent.push_back({{HB_CNOT, n - 1 - cw, n - 1 - tw, 0}, tw < h ? HB_CS : HB_SM,
                                 {cw, tw}, l, false});
      }
      ++l;
      in_layer = 0;
    } else {
      std::vector<int> ws;
      for (int k = c->phase_off[idx]; k < c->phase_off[idx + 1]; ++k) {
        ws.push_back(c->pairs[3 * k]);
        ws.push_back(c->pairs[3 * k + 1]);
      }
      layers[l].ent.push_back({{HB_PHASE, 0, 0, idx}, HB_ANY, ws, l, false});
      ++l;
      in_layer = 0;
    }
  }
  return layers;
}

// forward (no checkpoints): the whole circuit as one schedule
// the forward's tile bits (profiles/r02/hb_forward_tile_bits.txt): at n = 13 one
// 2^13-amplitude tile (64 KB, 3 CTAs/SM) holds the whole state, so every op runs in SM
// passes (strongly L = 4: 18.3 -> 12.5 ms, cross_mesh 15.2 -> 12.5 ms at 8192 points);
// at n = 14 a whole-state 2^14 tile (128 KB, one CTA/SM) pays for CNOT entanglers
// (strongly L = 8: 34.7 -> 28.3 ms, CNOT mesh 33.8 -> 20.9 ms at 4096 points) but not for
// the phase / no entangler (13-bit tiles, within 5 %); from n = 15 the 12-bit tiles (with
// CS passes at 4 CTAs/SM) are as fast or faster.  QPINN_HB_FWD_T overrides (9..14).
int hb_fwd_tbits(const qpinn_circuit* c) {
  static const int env = [] {
    const char* e = getenv("QPINN_HB_FWD_T");
    return e ? atoi(e) : 0;
  }();
  const int n = c->n;
  int def = kHbT;
  if (n == 13) def = 13;
  if (n == 14) def = layer_entangler(c) == ENT_PERM ? 14 : 13;
  const int t = env >= 9 && env <= 14 ? env : def;
  return n < t ? n : t;
}

HbPlan hb_plan(const qpinn_circuit* c, int T) {
  std::vector<HbSOp> seq;
  for (const HbLayerOps& lo : hb_layers(c, T)) {
    seq.insert(seq.end(), lo.u1.begin(), lo.u1.end());
    seq.insert(seq.end(), lo.ent.begin(), lo.ent.end());
  }
  HbPlan plan;
  plan.T = T;
  hb_schedule(seq, plan);
  hb_tabulate(plan);
  return plan;
}

// adjoint: forward segments ending at each layer's checkpoint, then the reverse sweep
struct HbBwdPlan {
  HbPlan fwd, rev;
};

// the adjoint's tile bits: at n = 13 the whole state per tile too (state + checkpoint
// tiles: 128 KB, one CTA per SM): strongly L = 4 71.7 -> 59.6 ms, cross_mesh 70.6 ->
// 65.7 ms at 8192 points (profiles/r02/hb_forward_tile_bits.txt).  QPINN_HB_BWD_T
// overrides (9..13; 13-bit adjoint tiles only where they hold the whole state)
int hb_bwd_tbits(int n) {
  static const int env = [] {
    const char* e = getenv("QPINN_HB_BWD_T");
    return e ? atoi(e) : 0;
  }();
  const int def = n == kHbTmax ? kHbTmax : kHbT;
  const int t = env >= 9 && env <= kHbTmax && (env <= kHbT || n <= kHbTmax) ? env : def;
  return n < t ? n : t;
}

HbBwdPlan hb_plan_bwd(const qpinn_circuit* c) {
  // the forward segments carry no checkpoint tile: they take the forward's tile bits
  const int Tf = hb_fwd_tbits(c), T = hb_bwd_tbits(c->n);
  const std::vector<HbLayerOps> flayers = hb_layers(c, Tf);
  const std::vector<HbLayerOps> layers = hb_layers(c, T);
  const int L = (int)layers.size();
  HbBwdPlan bp;
  bp.fwd.T = Tf;
  bp.rev.T = T;
  for (int l = 0; l <= L; ++l) {  // segment l: entangler(l-1), u1(l); checkpoint l after it
    std::vector<HbSOp> seq;
    if (l > 0) seq.insert(seq.end(), flayers[l - 1].ent.begin(), flayers[l - 1].ent.end());
    if (l < L) seq.insert(seq.end(), flayers[l].u1.begin(), flayers[l].u1.end());
    if (seq.empty()) continue;
    hb_schedule(seq, bp.fwd);
    if (l < L) bp.fwd.passes.back().ck = l;
  }
  std::vector<HbSOp> seq;
  for (int l = L - 1; l >= 0; --l) {
    for (int j = (int)layers[l].ent.size() - 1; j >= 0; --j) {
      HbSOp e = layers[l].ent[j];
      if (e.op.type == HB_PHASE) {
        e.op.b = 1;        // conjugate phase
        e.barrier = true;  // its parameter gradient is taken from the adjoint just before
      }
      seq.push_back(e);
    }
    for (const HbSOp& u : layers[l].u1) {
      HbSOp o = u;
      o.op.type = HB_OUTER;
      seq.push_back(o);
    }
    for (const HbSOp& u : layers[l].u1) {
      HbSOp d = u;
      d.op.b = 1;  // U^dagger
      seq.push_back(d);
    }
  }
  hb_schedule(seq, bp.rev);
  hb_tabulate(bp.fwd);
  hb_tabulate(bp.rev);
  return bp;
}

__device__ __forceinline__ int hb_insert0(int k, int bit) {
  return ((k >> bit) << (bit + 1)) | (k & ((1 << bit) - 1));
}

__device__ __forceinline__ void hb_load_u(const cplx<float>* __restrict__ U, const HbOp& op,
                                          cplx<float> (&u)[4]) {
  const cplx<float>* g = U + 4 * op.idx;
  if (op.b) {  // U^dagger
    u[0] = {g[0].re, -g[0].im};
    u[1] = {g[2].re, -g[2].im};
    u[2] = {g[1].re, -g[1].im};
    u[3] = {g[3].re, -g[3].im};
  } else {
    u[0] = g[0];
    u[1] = g[1];
    u[2] = g[2];
    u[3] = g[3];
  }
}

// the CTA's 8 outer-product sums (fixed shuffle tree, fixed warp order) -> part[slot]
__device__ __forceinline__ void hb_outer_commit(float (&m)[8], double* __restrict__ red,
                                                double* __restrict__ part) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    for (int s = 16; s >= 1; s >>= 1) m[k] += __shfl_xor_sync(0xffffffffu, m[k], s);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < 8; ++k) red[w * 8 + k] = (double)m[k];
  __syncthreads();
  if (threadIdx.x < 8) {
    double v = 0.0;
    for (int i = 0; i < nw; ++i) v += red[i * 8 + threadIdx.x];
    part[threadIdx.x] = v;
  }
}

// SM pass: CTA = (row, slice s); ops on the 2^kHbT low-bit amplitudes in shared memory.
// Runs of up to QPINN_HB_G single-qubit gates on distinct bits are applied together
// (one barrier per run), and a run of CNOTs is one gather through its tabulated index
// map.  OUTER ops read the checkpoint tile xc (loaded into a second buffer).
template <int G, int T>
__device__ __forceinline__ void hb_sm_u1_group(cplx<float>* t, const HbOp* op,
                                               const cplx<float>* __restrict__ U) {
  constexpr int TS = 1 << T, M = 1 << G;
  int bits[G], sorted[G];
  cplx<float> u[G][4];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    bits[g] = op[g].a;
    sorted[g] = op[g].a;
    hb_load_u(U, op[g], u[g]);
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
template <int T>
__global__ void __launch_bounds__(256, T >= 14 ? 1 : T >= 13 ? 3 : QPINN_HB_MINB)
hb_sm_pass(int n, cplx<float>* __restrict__ X, const cplx<float>* __restrict__ XC,
           const HbOp* __restrict__ ops, int nops, const int* __restrict__ luts,
           const cplx<float>* __restrict__ U, const cplx<float>* __restrict__ ph,
           double* __restrict__ part) {
  constexpr int TS = 1 << T, PER = TS / 256;
  extern __shared__ __align__(16) unsigned char hb_smem[];
  auto* t = (cplx<float>*)hb_smem;
  auto* tx = t + TS;  // checkpoint tile (OUTER passes)
  __shared__ double red[8 * 8];
  const int h = n - T;
  const int64_t D = (int64_t)1 << n;
  const int64_t row = blockIdx.x >> h;
  const int s = blockIdx.x & ((1 << h) - 1);
  cplx<float>* x = X + row * D + ((int64_t)s << T);
  // all of a chunk's loads in flight before its shared-memory stores (chunks of up
  // to 16 amplitudes per thread keep the registers bounded for 2^13 tiles)
  constexpr int CH = PER < 16 ? PER : 16;
#pragma unroll
  for (int j0 = 0; j0 < PER; j0 += CH) {
    cplx<float> r[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) r[j] = x[threadIdx.x + 256 * (j0 + j)];
#pragma unroll
    for (int j = 0; j < CH; ++j) t[threadIdx.x + 256 * (j0 + j)] = r[j];
  }
  if (XC) {
    const cplx<float>* xc = XC + row * D + ((int64_t)s << T);
#pragma unroll
    for (int j0 = 0; j0 < PER; j0 += CH) {
      cplx<float> r[CH];
#pragma unroll
      for (int j = 0; j < CH; ++j) r[j] = xc[threadIdx.x + 256 * (j0 + j)];
#pragma unroll
      for (int j = 0; j < CH; ++j) tx[threadIdx.x + 256 * (j0 + j)] = r[j];
    }
  }
  __syncthreads();
  int o = 0, slot = 0;
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
      if (QPINN_HB_G >= 3 && g == 3) hb_sm_u1_group<3, T>(t, ops + o, U);
      else if (QPINN_HB_G >= 2 && g == 2) hb_sm_u1_group<2, T>(t, ops + o, U);
      else hb_sm_u1_group<1, T>(t, ops + o, U);
      o += g;
    } else if (op.type == HB_CNOT) {
      // a run of CNOTs: new[i] = old[f(i, s)] through the run's tabulated index map
      const int* lut = luts + op.idx;
      const int fs = lut[320 + s];  // [64 low | 256 high | 16 slice]
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
    } else if (op.type == HB_OUTER) {  // M' = sum over pairs on bit a of conj(abar) x
      // two OUTER ops on distinct bits share one sweep over both tiles (QPINN_HB_OUTER2)
      const bool two = kHbOuter2 && o + 1 < nops && ops[o + 1].type == HB_OUTER &&
                       ops[o + 1].a != op.a;
      float m[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      float m2[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (two) {
        const int b0 = op.a, b1 = ops[o + 1].a;
        const int lo = b0 < b1 ? b0 : b1, hi = b0 < b1 ? b1 : b0;
        for (int k = threadIdx.x; k < TS / 4; k += blockDim.x) {
          const int i00 = hb_insert0(hb_insert0(k, lo), hi);
          const int i10 = i00 | (1 << b0), i01 = i00 | (1 << b1), i11 = i10 | (1 << b1);
          const cplx<float> a00 = t[i00], a10 = t[i10], a01 = t[i01], a11 = t[i11];
          const cplx<float> x00 = tx[i00], x10 = tx[i10], x01 = tx[i01], x11 = tx[i11];
          // bit b0: pairs (00, 10) and (01, 11)
          cmac_c(m[0], m[1], a00, x00);
          cmac_c(m[2], m[3], a00, x10);
          cmac_c(m[4], m[5], a10, x00);
          cmac_c(m[6], m[7], a10, x10);
          cmac_c(m[0], m[1], a01, x01);
          cmac_c(m[2], m[3], a01, x11);
          cmac_c(m[4], m[5], a11, x01);
          cmac_c(m[6], m[7], a11, x11);
          // bit b1: pairs (00, 01) and (10, 11)
          cmac_c(m2[0], m2[1], a00, x00);
          cmac_c(m2[2], m2[3], a00, x01);
          cmac_c(m2[4], m2[5], a01, x00);
          cmac_c(m2[6], m2[7], a01, x01);
          cmac_c(m2[0], m2[1], a10, x10);
          cmac_c(m2[2], m2[3], a10, x11);
          cmac_c(m2[4], m2[5], a11, x10);
          cmac_c(m2[6], m2[7], a11, x11);
        }
      } else {
        for (int k = threadIdx.x; k < TS / 2; k += blockDim.x) {
          const int i0 = hb_insert0(k, op.a), i1 = i0 | (1 << op.a);
          const cplx<float> a0 = t[i0], a1 = t[i1], x0 = tx[i0], x1 = tx[i1];
          cmac_c(m[0], m[1], a0, x0);
          cmac_c(m[2], m[3], a0, x1);
          cmac_c(m[4], m[5], a1, x0);
          cmac_c(m[6], m[7], a1, x1);
        }
      }
      hb_outer_commit(m, red, part + ((int64_t)slot * gridDim.x + blockIdx.x) * 8);
      ++slot;
      if (two) {
        hb_outer_commit(m2, red, part + ((int64_t)slot * gridDim.x + blockIdx.x) * 8);
        ++slot;
      }
      o += two ? 2 : 1;
    } else {
      const cplx<float>* ep = ph + (int64_t)op.idx * D + ((int64_t)s << T);
#pragma unroll
      for (int j0 = 0; j0 < PER; j0 += CH) {
        cplx<float> e[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          e[j] = ep[threadIdx.x + 256 * (j0 + j)];
          if (op.b) e[j].im = -e[j].im;
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int ii = threadIdx.x + 256 * (j0 + j);
          t[ii] = cmul(t[ii], e[j]);
        }
      }
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
__device__ __forceinline__ void hb_gate_bit(cplx<float> (&v)[1 << H], const cplx<float> (&u)[4]) {
#pragma unroll
  for (int j = 0; j < (1 << H); ++j) {
    if ((j >> RB) & 1) continue;
    const cplx<float> a = v[j], b = v[j | (1 << RB)];
    v[j] = cmul2(u[0], a, u[1], b);
    v[j | (1 << RB)] = cmul2(u[2], a, u[3], b);
  }
}

template <int H, int RB>
__device__ __forceinline__ void hb_outer_bit(const cplx<float> (&v)[1 << H],
                                             const cplx<float> (&xv)[1 << H], float (&m)[8]) {
#pragma unroll
  for (int j = 0; j < (1 << H); ++j) {
    if ((j >> RB) & 1) continue;
    const int j1 = j | (1 << RB);
    cmac_c(m[0], m[1], v[j], xv[j]);
    cmac_c(m[2], m[3], v[j], xv[j1]);
    cmac_c(m[4], m[5], v[j1], xv[j]);
    cmac_c(m[6], m[7], v[j1], xv[j1]);
  }
}

template <int H, bool XOUT, int T>
__global__ void __launch_bounds__(256) hb_cs_pass(int n, int64_t rows, cplx<float>* __restrict__ X,
                                                  const cplx<float>* __restrict__ XC,
                                                  const HbOp* __restrict__ ops, int nops,
                                                  const cplx<float>* __restrict__ U,
                                                  const cplx<float>* __restrict__ ph,
                                                  double* __restrict__ part, int n_outer) {
  constexpr int V = 1 << H, TS = 1 << T;
  __shared__ double red[8 * 8];
  const int64_t D = (int64_t)1 << n;
  float mo[XOUT ? 4 : 1][8];  // per-thread outer sums of this pass's OUTER ops (<= H of them)
#pragma unroll
  for (int i = 0; i < (XOUT ? 4 : 1); ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) mo[i][k] = 0.f;
  for (int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < rows * TS;
       gid += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = gid >> T;
    const int l = (int)(gid & (TS - 1));
    cplx<float>* x = X + row * D + l;
    cplx<float> v[V];
#pragma unroll
    for (int j = 0; j < V; ++j) v[j] = x[(int64_t)j << T];
    cplx<float> xv[XOUT ? V : 1];
    if constexpr (XOUT) {
      const cplx<float>* xc = XC + row * D + l;
#pragma unroll
      for (int j = 0; j < V; ++j) xv[j] = xc[(int64_t)j << T];
    }
    int slot = 0;
    for (int o = 0; o < nops; ++o) {
      const HbOp op = ops[o];
      if (op.type == HB_U1) {
        cplx<float> u[4];
        hb_load_u(U, op, u);
        const int rb = op.a - T;
        if (rb == 0) hb_gate_bit<H, 0>(v, u);
        if constexpr (H > 1) if (rb == 1) hb_gate_bit<H, 1>(v, u);
        if constexpr (H > 2) if (rb == 2) hb_gate_bit<H, 2>(v, u);
        if constexpr (H > 3) if (rb == 3) hb_gate_bit<H, 3>(v, u);
      } else if (op.type == HB_CNOT) {
        const int rb = (op.b & 0xff) - T;
        if (op.a < T) {  // low control: fixed for this thread
          if ((l >> op.a) & 1) {
#pragma unroll
            for (int q = 0; q < H; ++q)
              if (q == rb) hb_swap_bit<H>(v, q, -1);
          }
        } else {
          const int rc = op.a - T;
#pragma unroll
          for (int q = 0; q < H; ++q)
#pragma unroll
            for (int r = 0; r < H; ++r)
              if (q == rb && r == rc) hb_swap_bit<H>(v, q, r);
        }
      } else if (op.type == HB_OUTER) {
        if constexpr (XOUT) {
          const int rb = op.a - T;
#pragma unroll
          for (int sl = 0; sl < 4; ++sl) {
            if (sl != slot) continue;
            if (rb == 0) hb_outer_bit<H, 0>(v, xv, mo[sl]);
            if constexpr (H > 1) if (rb == 1) hb_outer_bit<H, 1>(v, xv, mo[sl]);
            if constexpr (H > 2) if (rb == 2) hb_outer_bit<H, 2>(v, xv, mo[sl]);
            if constexpr (H > 3) if (rb == 3) hb_outer_bit<H, 3>(v, xv, mo[sl]);
          }
          ++slot;
        }
      } else {
        const cplx<float>* e = ph + (int64_t)op.idx * D + l;
#pragma unroll
        for (int j = 0; j < V; ++j) {
          cplx<float> ej = e[(int64_t)j << T];
          if (op.b) ej.im = -ej.im;
          v[j] = cmul(v[j], ej);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < V; ++j) x[(int64_t)j << T] = v[j];
  }
  if constexpr (XOUT) {
    for (int sl = 0; sl < n_outer; ++sl) {
      float m[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) m[k] = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i == sl)
#pragma unroll
          for (int k = 0; k < 8; ++k) m[k] = mo[i][k];
      hb_outer_commit(m, red, part + ((int64_t)sl * gridDim.x + blockIdx.x) * 8);
    }
  }
}

// phase-step gradient sums (as gb_phase_grad) parallel over row chunks too:
// part[c][b] = sum over chunk c's rows of Im(conj(a) x e), then acc[b] += sum_c in order
__global__ void hb_phase_grad_part(int n, int64_t rows, int64_t per, const cplx<float>* __restrict__ X,
                                   const cplx<float>* __restrict__ A,
                                   const cplx<float>* __restrict__ ph, double* __restrict__ part) {
  const int64_t D = (int64_t)1 << n;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= D) return;
  const cplx<float> e = ph[b];
  const int64_t r0 = blockIdx.y * per, r1 = r0 + per < rows ? r0 + per : rows;
  double v = 0.0;
  for (int64_t r = r0; r < r1; ++r) {
    const cplx<float> xp = cmul(X[r * D + b], e), a = A[r * D + b];
    v += (double)(a.im * xp.re - a.re * xp.im);
  }
  part[blockIdx.y * D + b] = v;
}

__global__ void hb_phase_grad_sum(int n, int chunks, const double* __restrict__ part,
                                  double* __restrict__ acc) {
  const int64_t D = (int64_t)1 << n;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < D;
       b += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int c = 0; c < chunks; ++c) v += part[c * D + b];
    acc[b] += v;
  }
}

// acc[8 idx + k] += sum over the pass's CTAs of its partials, in CTA order per lane,
// then a fixed shuffle tree (one CTA per OUTER op of the pass)
__global__ void hb_outer_reduce(const HbOp* __restrict__ ops, int nops, int nctas,
                                const double* __restrict__ part, double* __restrict__ acc) {
  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int slot = -1, idx = 0;
  for (int o = 0, sl = 0; o < nops; ++o)
    if (ops[o].type == HB_OUTER) {
      if (sl == blockIdx.x) {
        slot = sl;
        idx = ops[o].idx;
      }
      ++sl;
    }
  if (slot < 0) return;
  double v = 0.0;
  for (int c = lane; c < nctas; c += 32) v += part[((int64_t)slot * nctas + c) * 8 + k];
  for (int s = 16; s >= 1; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
  if (lane == 0) acc[8 * idx + k] += v;
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

int hb_cs_grid(int64_t rows, int T) {
  const int64_t threads = rows << T;
  const int64_t b = (threads + 255) / 256, cap = (int64_t)num_sms() * 8;
  return (int)(b < cap ? b : cap);
}

int hb_launch_cs(int h, int T, int n, int64_t rows, cplx<float>* X, const cplx<float>* XC,
                 const HbOp* ops, int nops, const cplx<float>* U, const cplx<float>* ph,
                 double* part, int n_outer, cudaStream_t st) {
  const int grid = hb_cs_grid(rows, T);
#define QPINN_HB_CS(H, TT)                                                                   \
  (XC ? hb_cs_pass<H, true, TT><<<grid, 256, 0, st>>>(n, rows, X, XC, ops, nops, U, ph,      \
                                                      part, n_outer)                        \
      : hb_cs_pass<H, false, TT><<<grid, 256, 0, st>>>(n, rows, X, XC, ops, nops, U, ph,     \
                                                       part, 0))
  if (T == kHbT) {
    switch (h) {
      case 1: QPINN_HB_CS(1, kHbT); break;
      case 2: QPINN_HB_CS(2, kHbT); break;
      case 3: QPINN_HB_CS(3, kHbT); break;
      case 4: QPINN_HB_CS(4, kHbT); break;
      default: return fail(QPINN_ERR_CAPACITY, "multi-gate HBM pass: 13 <= n <= 16");
    }
  } else if (T == kHbTmax && !XC) {  // the forward's larger tiles
    switch (h) {
      case 1: hb_cs_pass<1, false, kHbTmax><<<grid, 256, 0, st>>>(n, rows, X, XC, ops, nops, U, ph, part, 0); break;
      case 2: hb_cs_pass<2, false, kHbTmax><<<grid, 256, 0, st>>>(n, rows, X, XC, ops, nops, U, ph, part, 0); break;
      case 3: hb_cs_pass<3, false, kHbTmax><<<grid, 256, 0, st>>>(n, rows, X, XC, ops, nops, U, ph, part, 0); break;
      default: return fail(QPINN_ERR_CAPACITY, "multi-gate HBM pass: 14 <= n <= 16 at 13-bit tiles");
    }
  } else if (T == 14 && !XC) {  // 2^14-amplitude forward tiles
    switch (h) {
      case 1: hb_cs_pass<1, false, 14><<<grid, 256, 0, st>>>(n, rows, X, XC, ops, nops, U, ph, part, 0); break;
      case 2: hb_cs_pass<2, false, 14><<<grid, 256, 0, st>>>(n, rows, X, XC, ops, nops, U, ph, part, 0); break;
      default: return fail(QPINN_ERR_CAPACITY, "multi-gate HBM pass: 15 <= n <= 16 at 14-bit tiles");
    }
  } else {
    return fail(QPINN_ERR_CAPACITY, "multi-gate HBM pass: tile bits");
  }
#undef QPINN_HB_CS
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

// one pass of a plan on the batch's states (SM or CS kind)
int hb_run_pass(const HbPass& ps, int n, int tb, int64_t rows, cplx<float>* X,
                const cplx<float>* XC, const HbOp* dops, const int* dluts, const cplx<float>* U,
                const cplx<float>* ph, double* part, double* acc, cudaStream_t st) {
  const int h = n - tb;
  const HbOp* ops = dops + ps.op0;
  int nctas;
  if (ps.kind == HB_SM) {
    nctas = (int)(rows << h);
    const int smem = (XC ? 2 : 1) * (1 << tb) * (int)sizeof(cplx<float>);
    switch (tb) {
#define QPINN_HB_SM(T)                                                                       \
  case T:                                                                                    \
    hb_sm_pass<T><<<(unsigned)nctas, 256, smem, st>>>(n, X, XC, ops, ps.nops, dluts, U, ph, \
                                                      part);                                \
    break;
      QPINN_HB_SM(9)
      QPINN_HB_SM(10)
      QPINN_HB_SM(11)
      QPINN_HB_SM(12)
      QPINN_HB_SM(13)
      QPINN_HB_SM(14)
#undef QPINN_HB_SM
      default: return fail(QPINN_ERR_CAPACITY, "multi-gate HBM pass: 9 <= n <= 16");
    }
    QPINN_CUDA_CHECK(cudaGetLastError());
  } else {
    nctas = hb_cs_grid(rows, tb);
    if (int rc = hb_launch_cs(h, tb, n, rows, X, XC, ops, ps.nops, U, ph, part, ps.n_outer, st))
      return rc;
  }
  if (ps.n_outer) {
    hb_outer_reduce<<<ps.n_outer, 256, 0, st>>>(ops, ps.nops, nctas, part, acc);
    QPINN_CUDA_CHECK(cudaGetLastError());
  }
  return QPINN_OK;
}

}  // namespace

namespace {
// smallest n routed to the multi-gate passes; below it the CTA kernels of pqc_big.cu
// are faster (n = 9..12 both ways: profiles/r02/config5_hbm_vs_cta.txt); QPINN_PQC_HBM_{FWD,BWD}_MIN
// override it, QPINN_PQC_HBM_MULTIGATE=0 turns the path off
bool hbm_supported(const qpinn_circuit* c, int dtype, const char* env, int min_n) {
  if (!c || dtype != QPINN_F32 || c->n < 9 || c->n > kHbT + 4) return false;
  if (getenv("QPINN_PQC_HBM_MULTIGATE") && atoi(getenv("QPINN_PQC_HBM_MULTIGATE")) == 0) return false;
  if (getenv(env)) min_n = atoi(getenv(env));
  return c->n >= min_n && layer_entangler(c) >= 0;
}
}  // namespace

// Whole-state tiles (n <= 12) against the CTA kernels of pqc_big.cu, config 5
// (profiles/r02/config5_hbm_vs_cta.txt): the adjoint is 1.2-4x faster from n = 12 for
// every entangler and at n = 11 with CNOT entanglers or L = 1 (phase and no-entangler
// adjoints at L >= 4 stay 10-20% faster on the CTA kernels); the n = 12 forward is
// 1.6-1.7x faster with CNOT entanglers and L >= 2 and 1.03-1.08x with any entangler at
// L = 8 (phase / none at L = 4: 0.95-1.0x, L = 1: 0.7-0.9x, kept on the CTA kernels);
// n <= 10 stays on the CTA kernels both ways.
bool hbm_fwd_supported(const qpinn_circuit* c, int dtype) {
  const bool n12 = c && ((c->L >= 2 && layer_entangler(c) == ENT_PERM) || c->L >= 8);
  return hbm_supported(c, dtype, "QPINN_PQC_HBM_FWD_MIN", n12 ? 12 : 13);
}

bool hbm_bwd_supported(const qpinn_circuit* c, int dtype) {
  return hbm_supported(c, dtype, "QPINN_PQC_HBM_BWD_MIN",
                       c && (c->L == 1 || layer_entangler(c) == ENT_PERM) ? 11 : 12);
}

namespace {
// points per batch: ~1 GB of adjoint state (X, A, L checkpoints), ~256 MB of forward state
int64_t hb_bwd_bcap(int n) { return std::max<int64_t>(256, (int64_t)1 << (22 - n)); }
// blocks per point of the readout / embedding gradient: >= 1024 amplitudes each
int hb_chunks(int n) { return n <= 10 ? 1 : std::min(kGbChunks, 1 << (n - 10)); }
int64_t hb_fwd_bcap(int n) { return std::max<int64_t>(1024, (int64_t)1 << (22 - n)); }
}  // namespace

// dynamic shared memory limits of the SM-pass instances (state tile, plus the
// checkpoint tile where it is used: 12- and 13-bit adjoint tiles)
int hb_set_smem_limits() {
  const int es = (int)sizeof(cplx<float>);
  QPINN_CUDA_CHECK(cudaFuncSetAttribute(hb_sm_pass<12>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * es << 12));
  QPINN_CUDA_CHECK(cudaFuncSetAttribute(hb_sm_pass<13>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * es << 13));
  QPINN_CUDA_CHECK(cudaFuncSetAttribute(hb_sm_pass<14>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, es << 14));
  return QPINN_OK;
}

// forward with tangents (or value only), several gates per HBM pass (see hb_plan)
int hbm_forward(const qpinn_circuit* c, const KArgs<float>* a, unsigned char* ws, size_t bytes) {
  const PlanDev& p = c->dev;
  const int n = c->n;
  const int64_t D = (int64_t)1 << n;
  const HbPlan plan = hb_plan(c, hb_fwd_tbits(c));
  const int nops = (int)plan.ops.size();
  if (getenv("QPINN_VERBOSE")) {
    fprintf(stderr, "[qpinn] multi-gate HBM forward: n = %d, L = %d, %d ops in %d passes:", n,
            c->L, nops, (int)plan.passes.size());
    for (const HbPass& ps : plan.passes) fprintf(stderr, " %s%d", ps.kind == HB_SM ? "S" : "C", ps.nops);
    fprintf(stderr, "\n");
  }
  // largest batch of points that fits the workspace
  int64_t B = std::min<int64_t>(a->R, hb_fwd_bcap(n));
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
  auto* dluts = (int*)(dops + nops);
  auto* X = (cplx<float>*)(ws + g.X);
  QPINN_CUDA_CHECK(cudaMemcpyAsync(dops, plan.ops.data(), sizeof(HbOp) * nops,
                                   cudaMemcpyHostToDevice, st));
  if (nluts)
    QPINN_CUDA_CHECK(cudaMemcpyAsync(dluts, plan.luts.data(), sizeof(int) * nluts,
                                     cudaMemcpyHostToDevice, st));
  const int ns = a->tan ? 4 : 1;
  const int chunks = hb_chunks(n);
  const int ro_smem = 4 * n * 4 * (int)sizeof(double);  // [4 warps][4 n]
  if (int rc = hb_set_smem_limits()) return rc;
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
    gb_embed4<float><<<gb_blocks(Bc * D / 4), kGbThreads, 0, st>>>(n, Bc, ns, PT, X);
    for (const HbPass& ps : plan.passes)
      if (int rc = hb_run_pass(ps, n, plan.T, rows, X, nullptr, dops, dluts, U, ph, nullptr,
                               nullptr, st))
        return rc;
    gb_readout<float><<<dim3(chunks, Bc), 128, ro_smem, st>>>(n, chunks, ns, X, RP);
    gb_readout_final<float><<<gb_blocks(Bc * n), kGbThreads, 0, st>>>(n, Bc, chunks, ns, p0,
                                                                      a->R, RP, a->z, a->dz);
    QPINN_CUDA_CHECK(cudaGetLastError());
  }
  return QPINN_OK;
}

// number of HBM passes per forward of the multi-gate path (diagnostics)
int hbm_forward_passes(const qpinn_circuit* c) {
  return (int)hb_plan(c, hb_fwd_tbits(c)).passes.size();
}

namespace {

struct HbBwdLayout {
  int B;
  size_t acc, U, ph, PT, EG, ops, part, X, A, CK, total;
};

HbBwdLayout hb_bwd_layout(const qpinn_circuit* c, int64_t B, int nops, int nluts) {
  const size_t D = (size_t)1 << c->n, es = sizeof(cplx<float>);
  HbBwdLayout g{};
  g.B = (int)B;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o += align_up(bytes, 256);
    return at;
  };
  const int64_t rows = 4 * B;
  const int64_t max_ctas =
      std::max<int64_t>(rows << (c->n - hb_bwd_tbits(c->n)), (int64_t)num_sms() * 8);
  g.acc = take(8 * (8 * (size_t)c->n_u1 + D * c->n_phase));
  g.U = take(es * 4 * c->n_u1);
  g.ph = take(es * D * c->n_phase);
  g.PT = take(sizeof(float) * 8 * (size_t)B * c->n);
  g.EG = take(8 * (size_t)B * kGbChunks * 4 * c->n);
  g.ops = take(sizeof(HbOp) * (size_t)(nops > 0 ? nops : 1) + sizeof(int) * (size_t)nluts);
  g.part = take(std::max<size_t>(8 * 8 * (size_t)c->n * max_ctas, 8 * 32 * D));
  g.X = take(4 * D * (size_t)B * es);
  g.A = take(4 * D * (size_t)B * es);
  g.CK = take((size_t)c->L * 4 * D * (size_t)B * es);
  g.total = o;
  return g;
}

}  // namespace

// adjoint backward, several gates per HBM pass (see hb_plan_bwd)
int hbm_backward(const qpinn_circuit* c, const KArgs<float>* a, unsigned char* ws, size_t bytes) {
  const PlanDev& p = c->dev;
  const int n = c->n, L = c->L;
  const int64_t D = (int64_t)1 << n;
  const HbBwdPlan bp = hb_plan_bwd(c);
  // one op / lut array: forward plan first, reverse plan after it
  std::vector<HbOp> ops = bp.fwd.ops;
  std::vector<int> luts = bp.fwd.luts;
  const int rev_op0 = (int)ops.size(), rev_lut0 = (int)luts.size();
  for (HbOp op : bp.rev.ops) {
    if (op.type == HB_CNOT && (op.b >> 8)) op.idx += rev_lut0;  // run head: table offset
    ops.push_back(op);
  }
  luts.insert(luts.end(), bp.rev.luts.begin(), bp.rev.luts.end());
  const int nops = (int)ops.size(), nluts = (int)luts.size();
  if (getenv("QPINN_VERBOSE"))
    fprintf(stderr, "[qpinn] multi-gate HBM adjoint: n = %d, L = %d, %d forward + %d reverse passes\n",
            n, L, (int)bp.fwd.passes.size(), (int)bp.rev.passes.size());
  int64_t B = std::min<int64_t>(a->R, hb_bwd_bcap(n));
  while (B > 1 && hb_bwd_layout(c, B, nops, nluts).total > bytes) B = B * 3 / 4;
  const HbBwdLayout g = hb_bwd_layout(c, B < 1 ? 1 : B, nops, nluts);
  if (bytes < g.total) return fail(QPINN_ERR_CONFIG, "multi-gate HBM adjoint: workspace too small");
  cudaStream_t st = a->stream;
  auto* acc = (double*)(ws + g.acc);
  auto* U = (cplx<float>*)(ws + g.U);
  auto* ph = (cplx<float>*)(ws + g.ph);
  auto* PT = (float*)(ws + g.PT);
  auto* EG = (double*)(ws + g.EG);
  auto* dops = (HbOp*)(ws + g.ops);
  auto* dluts = (int*)(dops + nops);
  auto* part = (double*)(ws + g.part);
  auto* X = (cplx<float>*)(ws + g.X);
  auto* A = (cplx<float>*)(ws + g.A);
  auto* CK = (cplx<float>*)(ws + g.CK);
  QPINN_CUDA_CHECK(cudaMemcpyAsync(dops, ops.data(), sizeof(HbOp) * nops, cudaMemcpyHostToDevice,
                                   st));
  if (nluts)
    QPINN_CUDA_CHECK(cudaMemcpyAsync(dluts, luts.data(), sizeof(int) * nluts,
                                     cudaMemcpyHostToDevice, st));
  const int n_acc = 8 * p.n_u1 + (int)D * p.n_phase;
  QPINN_CUDA_CHECK(cudaMemsetAsync(acc, 0, 8 * (size_t)n_acc, st));
  const int eg_smem = 4 * n * 4 * (int)sizeof(double);  // [4 warps][4 n]
  const int chunks = hb_chunks(n);
  QPINN_CUDA_CHECK(cudaFuncSetAttribute(gb_embed_grad<float>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, eg_smem));
  if (int rc = hb_set_smem_limits()) return rc;
  gb_tables<float><<<64, 256, 0, st>>>(p, a->qp, U, ph);
  for (int64_t p0 = 0; p0 < a->R; p0 += g.B) {
    const int Bc = (int)(a->R - p0 < g.B ? a->R - p0 : g.B);
    const int64_t rows = (int64_t)Bc * 4;
    const size_t ckl = (size_t)rows * D;  // one layer's checkpoint
    gb_point<float><<<gb_blocks(Bc * n), kGbThreads, 0, st>>>(n, a->scale, a->R, p0, Bc, a->act,
                                                              a->tan, PT);
    gb_embed4<float><<<gb_blocks(Bc * D / 4), kGbThreads, 0, st>>>(n, Bc, 4, PT, X);
    for (const HbPass& ps : bp.fwd.passes) {  // forward, checkpointing every layer boundary
      if (int rc = hb_run_pass(ps, n, bp.fwd.T, rows, X, nullptr, dops, dluts, U, ph, nullptr,
                               nullptr, st))
        return rc;
      if (ps.ck >= 0)
        QPINN_CUDA_CHECK(cudaMemcpyAsync(CK + ps.ck * ckl, X, ckl * sizeof(cplx<float>),
                                         cudaMemcpyDeviceToDevice, st));
    }
    gb_seed<float><<<gb_blocks(Bc * D), kGbThreads, 0, st>>>(n, Bc, p0, a->R, a->gz, a->gdz, X, A);
    for (const HbPass& pr : bp.rev.passes) {
      HbPass ps = pr;
      ps.op0 += rev_op0;
      if (ps.phase_grad >= 0) {  // Im<abar, i pmat x'> sums of this phase step, per basis state
        const int l = ps.phase_grad;
        const int chunks = (int)std::min<int64_t>(32, rows);
        const int64_t per = (rows + chunks - 1) / chunks;
        hb_phase_grad_part<<<dim3((unsigned)((D + 255) / 256), chunks), 256, 0, st>>>(
            n, rows, per, CK + l * ckl, A, ph + (size_t)l * D, part);
        hb_phase_grad_sum<<<gb_blocks(D), kGbThreads, 0, st>>>(n, chunks, part,
                                                              acc + 8 * p.n_u1 + (size_t)l * D);
      }
      const cplx<float>* xc = ps.layer >= 0 ? CK + ps.layer * ckl : nullptr;
      if (int rc = hb_run_pass(ps, n, bp.rev.T, rows, A, xc, dops, dluts, U, ph, part, acc, st))
        return rc;
    }
    gb_embed4<float><<<gb_blocks(Bc * D / 4), kGbThreads, 0, st>>>(n, Bc, 1, PT, X);
    gb_embed_grad<float><<<dim3(chunks, Bc), 128, eg_smem, st>>>(n, chunks, PT, X, A, EG);
    gb_embed_final<float><<<gb_blocks(Bc * n), kGbThreads, 0, st>>>(n, Bc, chunks, p0, a->R,
                                                                    EG, PT, a->tan, a->g_act,
                                                                    a->g_tan);
    QPINN_CUDA_CHECK(cudaGetLastError());
  }
  return pqc_param_grads<float>(c, acc, n, a->qp, a->g_qp, st);
}

size_t hbm_bwd_workspace_bytes(const qpinn_circuit* c, int64_t rows) {
  const HbBwdPlan bp = hb_plan_bwd(c);
  const int nops = (int)(bp.fwd.ops.size() + bp.rev.ops.size());
  const int nluts = (int)(bp.fwd.luts.size() + bp.rev.luts.size());
  // ~1 GB of batch state: X, A and L checkpoints per point (no more points than rows)
  const int64_t per = (int64_t)(2 + c->L) * 4 * ((int64_t)8 << c->n);
  int64_t B = ((int64_t)1 << 30) / per;
  B = std::min<int64_t>(B, hb_bwd_bcap(c->n));
  if (rows >= 0) B = std::min<int64_t>(B, rows);
  B = B < 1 ? 1 : B;
  return hb_bwd_layout(c, B, nops, nluts).total;
}

size_t global_adjoint_workspace_bytes(const qpinn_circuit* c, int dtype, int64_t rows) {
  if (dtype == QPINN_F64) return gb_layout<double>(c).total;
  // the multi-gate forward reuses this region with batches of ~256 MB of state
  // (1024 points at n = 13), so few launches carry the batch loop; both passes size
  // their batch to the call's rows when that is smaller
  const size_t g = gb_layout<float>(c).total;
  size_t h = 0;
  if (hbm_fwd_supported(c, dtype)) {
    int64_t B = ((int64_t)256 << 20) / (4 * ((int64_t)8 << c->n));
    B = std::min<int64_t>(B, hb_fwd_bcap(c->n));
    if (rows >= 0) B = std::min<int64_t>(B, rows);
    const HbPlan plan = hb_plan(c, hb_fwd_tbits(c));
    h = hb_layout(c, B < 1 ? 1 : B, (int)plan.ops.size(), (int)plan.luts.size()).total;
  }
  if (hbm_bwd_supported(c, dtype)) h = std::max(h, hbm_bwd_workspace_bytes(c, rows));
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
  const int eg_smem = 4 * n * 4 * (int)sizeof(double);  // [4 warps][4 n]
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
    gb_embed4<T><<<gb_blocks(B * D / 4), kGbThreads, 0, st>>>(n, B, 4, PT, X);
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
    gb_embed4<T><<<gb_blocks(B * D / 4), kGbThreads, 0, st>>>(n, B, 1, PT, X);
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
    gb_embed4<T><<<gb_blocks(B * D / 4), kGbThreads, 0, st>>>(n, B, ns, PT, X);
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
