// K1 / K2 as tensor-core GEMMs: the transfer-matrix formulation of the PQC.
//
// The circuit after the embedding is one fixed unitary per step, so the
// reference's default path (quantum_layer_forward via="matrix",
// ansatz.py:300-338) builds its transfer matrix once and maps every embedded
// state through it.  Here that matrix is built on the device by running the
// circuit on the D basis states (one CTA per basis row), and the map itself
// is a real GEMM on the tcgen05 tensor cores (3xTF32, tc_gemm.cu):
//
//   rows of B:   B[j] = circuit(e_j)                     (complex [D][D])
//   W          = [[Br, Bi], [-Bi, Br]]                    (real [2D][2D])
//   W'         = W with rows b, D+b folded by the embedding phase (tr_wmat)  [D][2D]
//   Psi        = m W'        with m = the real magnitudes of phi per state row
//                [4R][2D]    ([4R][D]), rows s R + p (s = 0: phi, 1..3: d phi/dx,y,t)
//
// For n = 7 that is 2 (4 2 D^2) flops per point instead of the gate-by-gate
// 2.4e5, but at tensor-core rate.  The backward is the GEMM's backward:
//   Abar  = seeds(Psi, dL/dz, dL/ddz)                     (qpinn_oracle.pqc_backward)
//   dL/dm = Abar W'^T  -> the embedding gradient, per point
//   dL/dW' = m^T Abar (deterministic split-K)  -> adjoint of the rows of B
//   the circuit's adjoint on the D basis rows (one CTA per row, checkpointed
//   at the layer boundaries like K2) -> the gate-space sums -> dL/dqparams.
// Float32 only (the GEMM is 3xTF32); chosen for 5 <= n <= 8 and n = 9, 10 at L >= 4:
// the folded map costs 8 D^2 FLOP per point against ~5 n L D for the gate sweep, but at
// tensor-core rate (n = 8: 1.4-7.5x faster than the layer kernels; n = 9, 10 at
// L >= 4: 1.2-3.3x faster than the CTA kernels for K1 + K2; profiles/r02).
#include <cstdlib>
#include <mutex>

#include "pqc_layer.h"
#include "tc_gemm.cuh"
#include "tc_gemm.h"

namespace qpinn {

namespace {

constexpr int kTrThreads = 64;  // circuit kernels: amplitude pairs strided over 64 threads
constexpr int kTrMaxN = 10;     // transfer-matrix path: n <= 10

// u1 matrices [n_u1][4] and phase diagonals [n_phase][D] (as gb_tables, pqc_global.cu)
__global__ void tr_tables(PlanDev p, const float* __restrict__ qp, cplx<float>* __restrict__ U,
                          cplx<float>* __restrict__ ph) {
  const int D = 1 << p.n;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int i = tid; i < p.n_u1; i += nt) {
    const int kind = p.u1[i * 4];
    double th[3] = {0, 0, 0};
    for (int j = 0; j < u1_nslots(kind); ++j) th[j] = (double)qp[p.u1[i * 4 + 1 + j]];
    double M[8];
    u1_matrix_d(kind, th, M);
    for (int e = 0; e < 4; ++e) U[i * 4 + e] = {float(M[2 * e]), float(M[2 * e + 1])};
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
    ph[i] = {float(cp), float(sp)};
  }
}

__device__ __forceinline__ void pair_index(int k, int pos, int& i0, int& i1) {
  i0 = ((k >> pos) << (pos + 1)) | (k & ((1 << pos) - 1));
  i1 = i0 | (1 << pos);
}

// B[j] = circuit(e_j); CK[l][j] = the state after layer l's single-qubit gates
template <int NQ>  // the circuit's qubit count: shared-memory rows of 2^NQ amplitudes
__global__ void __launch_bounds__(kTrThreads) tr_circuit_fwd(
    int n, int L, int ent, const cplx<float>* __restrict__ U, const cplx<float>* __restrict__ ph,
    const uint16_t* __restrict__ perm, cplx<float>* __restrict__ B, cplx<float>* __restrict__ CK) {
  __shared__ cplx<float> s[2][1 << NQ];
  const int D = 1 << n, j = blockIdx.x, t = threadIdx.x;
  int cur = 0;
  for (int b = t; b < D; b += kTrThreads) s[0][b] = {b == j ? 1.f : 0.f, 0.f};
  __syncthreads();
  for (int l = 0; l < L; ++l) {
    for (int q = 0; q < n; ++q) {
      const cplx<float>* u = U + 4 * (l * n + q);
      for (int k = t; k < D / 2; k += kTrThreads) {
        int i0, i1;
        pair_index(k, n - 1 - q, i0, i1);
        const cplx<float> a = s[cur][i0], c = s[cur][i1];
        s[cur][i0] = cmul2(u[0], a, u[1], c);
        s[cur][i1] = cmul2(u[2], a, u[3], c);
      }
      __syncthreads();
    }
    if (CK)
      for (int b = t; b < D; b += kTrThreads) CK[((size_t)l * D + j) * D + b] = s[cur][b];
    if (ent == ENT_PERM) {
      for (int b = t; b < D; b += kTrThreads) s[cur ^ 1][b] = s[cur][perm[l * D + b]];
      cur ^= 1;
    } else if (ent == ENT_PHASE) {
      for (int b = t; b < D; b += kTrThreads) s[cur][b] = cmul(s[cur][b], ph[l * D + b]);
    }
    __syncthreads();
  }
  for (int b = t; b < D; b += kTrThreads) B[(size_t)j * D + b] = s[cur][b];
}

template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* red /* [2][NV] */) {
#pragma unroll
  for (int e = 0; e < NV; ++e)
    for (int m = 16; m >= 1; m >>= 1) v[e] += __shfl_xor_sync(0xffffffffu, v[e], m);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
    for (int e = 0; e < NV; ++e) red[w * NV + e] = v[e];
  __syncthreads();
  for (int e = 0; e < NV; ++e) v[e] = red[e] + red[NV + e];  // fixed order: warp 0 + warp 1
  __syncthreads();
}

// reverse sweep for basis row j from the adjoint of B[j]: per gate the 2x2
// post-gate outer product M'_ab = sum conj(abar_a) x_b (gates of one layer
// commute, so each is the layer's last), per phase layer Im(conj(abar) x');
// per-row partials, reduced over rows in fixed order by tr_reduce
template <int NQ>  // the circuit's qubit count (register sums: 8 per qubit)
__global__ void __launch_bounds__(kTrThreads) tr_circuit_bwd(
    int n, int L, int ent, const cplx<float>* __restrict__ U, const cplx<float>* __restrict__ ph,
    const uint16_t* __restrict__ iperm, const cplx<float>* __restrict__ Abar,
    const cplx<float>* __restrict__ CK, double* __restrict__ part_u1,
    double* __restrict__ part_ph) {
  __shared__ cplx<float> s[2][1 << NQ];
  __shared__ double red[2 * 8 * NQ];
  const int D = 1 << n, j = blockIdx.x, t = threadIdx.x, n_u1 = n * L;
  int cur = 0;
  for (int b = t; b < D; b += kTrThreads) s[0][b] = Abar[(size_t)j * D + b];
  __syncthreads();
  for (int l = L - 1; l >= 0; --l) {
    const cplx<float>* xl = CK + ((size_t)l * D + j) * D;
    if (ent == ENT_PERM) {
      for (int b = t; b < D; b += kTrThreads) s[cur ^ 1][b] = s[cur][iperm[l * D + b]];
      cur ^= 1;
      __syncthreads();
    } else if (ent == ENT_PHASE) {
      for (int b = t; b < D; b += kTrThreads) {
        const cplx<float> e = ph[l * D + b], xp = cmul(xl[b], e), a = s[cur][b];
        part_ph[((size_t)j * L + l) * D + b] = (double)(a.im * xp.re - a.re * xp.im);
        s[cur][b] = cmul(a, cplx<float>{e.re, -e.im});
      }
      __syncthreads();
    }
    // all of the layer's outer products from the same (adjoint, checkpoint) pair,
    // then one block reduction for the layer (8 n sums)
    double m[8 * NQ];
#pragma unroll
    for (int e = 0; e < 8 * NQ; ++e) m[e] = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      if (q < n) {
        for (int k = t; k < D / 2; k += kTrThreads) {
          int i0, i1;
          pair_index(k, n - 1 - q, i0, i1);
          const cplx<float> x0 = xl[i0], x1 = xl[i1], a0 = s[cur][i0], a1 = s[cur][i1];
          float f[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          cmac_c(f[0], f[1], a0, x0);
          cmac_c(f[2], f[3], a0, x1);
          cmac_c(f[4], f[5], a1, x0);
          cmac_c(f[6], f[7], a1, x1);
#pragma unroll
          for (int e = 0; e < 8; ++e) m[8 * q + e] += (double)f[e];
        }
      }
    }
    block_sum<8 * NQ>(m, red);
    for (int t2 = t; t2 < 8 * n; t2 += kTrThreads) {
      // m is uniform after the sum: pick entry t2 without dynamic register indexing
      double v = 0.0;
#pragma unroll
      for (int e = 0; e < 8 * NQ; ++e)
        if (e == t2) v = m[e];
      part_u1[((size_t)j * n_u1 + l * n) * 8 + t2] = v;
    }
    for (int q = 0; q < n; ++q) {
      const cplx<float>* u = U + 4 * (l * n + q);
      const cplx<float> d00 = {u[0].re, -u[0].im}, d01 = {u[2].re, -u[2].im},
                        d10 = {u[1].re, -u[1].im}, d11 = {u[3].re, -u[3].im};
      for (int k = t; k < D / 2; k += kTrThreads) {
        int i0, i1;
        pair_index(k, n - 1 - q, i0, i1);
        const cplx<float> a = s[cur][i0], c = s[cur][i1];
        s[cur][i0] = cmul2(d00, a, d01, c);
        s[cur][i1] = cmul2(d10, a, d11, c);
      }
      __syncthreads();
    }
  }
}

// acc[i] = sum over the D basis rows of the partials, in row order
__global__ void tr_reduce(int D, int n_u1, int n_ph, const double* __restrict__ part_u1,
                          const double* __restrict__ part_ph, double* __restrict__ acc) {
  // one warp per entry: lane-strided row sums, then a fixed xor tree (deterministic)
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= 8 * n_u1 + n_ph) return;
  const bool u1 = i < 8 * n_u1;
  const double* src = u1 ? part_u1 + i : part_ph + (i - 8 * n_u1);
  const size_t stride = u1 ? (size_t)8 * n_u1 : (size_t)n_ph;
  double v = 0.0;
  for (int j = lane; j < D; j += 32) v += src[(size_t)j * stride];
  for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  if (lane == 0) acc[i] = v;
}

// phase of embedded amplitude b: (-i)^popcount(b) = (pr, pi)
__device__ __forceinline__ void embed_phase(int b, float& pr, float& pi) {
  const int ph = __popc(b) & 3;
  pr = ph == 0 ? 1.f : ph == 2 ? -1.f : 0.f;
  pi = ph == 1 ? -1.f : ph == 3 ? 1.f : 0.f;
}

// Every embedded row (state or tangent) is phi_b = p_b m_b with a real
// magnitude m_b and the point-independent phase p_b = (-i)^popcount(b), so in
// the real-block form [Re phi | Im phi] half of the 2D entries are zero in a
// fixed pattern.  The map is therefore applied to the D magnitudes only:
//   W'[b][c] = Re p_b W[b][c] + Im p_b W[D + b][c],   W = [[Br, Bi], [-Bi, Br]]
//   Psi = m W'   (K = D instead of 2D),   dL/dm = Abar W'^T   (N = D),
//   dL/dW' = m^T Abar   (D x 2D),   dL/dW[b] = Re p_b dL/dW'[b], dL/dW[D+b] = Im p_b dL/dW'[b]
// which halves all three transfer GEMMs and the embedded-state traffic.
// Wt [2D][D] = W'^T (forward GEMM operand) and W [D][2D] = W' (backward operand).
// W' and W'^T go straight out as the tf32 hi / lo pairs the map's GEMMs take (W: hi
// [D][2D] then lo; Wt: hi [2D][D] then lo), so no GEMM splits them again
__global__ void tr_wmat(int n, const cplx<float>* __restrict__ B, float* __restrict__ W,
                        float* __restrict__ Wt) {
  const int D = 1 << n, D2 = 2 * D;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < D * D2; i += gridDim.x * blockDim.x) {
    const int r = i / D2, c = i % D2;  // W'[r][c]
    const cplx<float> b = B[(size_t)r * D + (c % D)];
    const float top = c < D ? b.re : b.im;    // W[r][c]
    const float bot = c < D ? -b.im : b.re;   // W[D + r][c]
    float pr, pi;
    embed_phase(r, pr, pi);
    const float v = pr * top + pi * bot;
    const float hi = tc::rna_tf32(v), lo = tc::rna_tf32(v - hi);
    W[i] = hi;
    W[(size_t)D * D2 + i] = lo;
    Wt[(size_t)c * D + r] = hi;
    Wt[(size_t)D * D2 + (size_t)c * D + r] = lo;
  }
}

// complex adjoint of the rows of B from dL/dW' [D][2D] (see tr_wmat):
// dL/dBr = gW11 + gW22, dL/dBi = gW12 - gW21 on the expanded dL/dW
__global__ void tr_gb(int n, const float* __restrict__ gW, cplx<float>* __restrict__ Ab) {
  const int D = 1 << n, D2 = 2 * D;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < D * D; i += gridDim.x * blockDim.x) {
    const int j = i / D, k = i % D;
    float pr, pi;
    embed_phase(j, pr, pi);
    const float g0 = gW[(size_t)j * D2 + k], g1 = gW[(size_t)j * D2 + D + k];
    Ab[i] = {pr * g0 + pi * g1, pr * g1 - pi * g0};
  }
}

// ---- per-point kernels: 8 warps per block, kPB points per block iteration ----
// The per-qubit angle data of a block's points is staged once into shared
// memory with coalesced loads (one DRAM round trip per kPB points); each warp
// then owns one point at a time, lane l holding the amplitudes b = l + 32 j.
constexpr int kPB = 64;
constexpr int kAng = 10;  // c, s, s1, dth_x, dth_y, dth_z, s2 tan_x, s2 tan_y, s2 tan_z, -

template <int NQ>
__device__ __forceinline__ void stage_angles(int scale, int64_t R, int64_t p0,
                                             const float* __restrict__ act,
                                             const float* __restrict__ tan, float* ang,
                                             float& amax) {
  for (int i = threadIdx.x; i < kPB * NQ; i += blockDim.x) {
    const int64_t p = p0 + i / NQ;
    const int q = i % NQ;
    float c = 1.f, sn = 0.f, s1 = 0.f, s2 = 0.f, tv[3] = {0.f, 0.f, 0.f};
    if (p < R) {
      float a = act[p * NQ + q];
      amax = fmaxf(amax, fabsf(a));
      a = fminf(fmaxf(a, -1.f), 1.f);
      half_angle<float>(scale, a, c, sn, s1, s2);
      if (tan)
        for (int k = 0; k < 3; ++k) tv[k] = tan[((int64_t)k * R + p) * NQ + q];
    }
    float* o = ang + i * kAng;
    o[0] = c;
    o[1] = sn;
    o[2] = s1;
    for (int k = 0; k < 3; ++k) {
      o[3 + k] = s1 * tv[k];
      o[6 + k] = s2 * tv[k];
    }
  }
}

template <int NQ>
struct PointAngles {
  float c[NQ], s[NQ], d[3][NQ];
};

template <int NQ>
__device__ __forceinline__ void read_angles(const float* ang, PointAngles<NQ>& pa) {
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    pa.c[q] = ang[q * kAng];
    pa.s[q] = ang[q * kAng + 1];
#pragma unroll
    for (int k = 0; k < 3; ++k) pa.d[k][q] = ang[q * kAng + 3 + k];
  }
}

// embedded amplitude of basis state b and its x/y/t tangents (ansatz.py:233-243,
// :380-390; wire q is bit NQ-1-q), before the (-i)^popcount phase
template <int NQ>
__device__ __forceinline__ void embed_amp(const PointAngles<NQ>& pa, int b, bool tangents,
                                          float& m0, float (&mk)[3]) {
  float pre[NQ + 1];
  pre[0] = 1.f;
#pragma unroll
  for (int q = 0; q < NQ; ++q) pre[q + 1] = pre[q] * (((b >> (NQ - 1 - q)) & 1) ? pa.s[q] : pa.c[q]);
  m0 = pre[NQ];
  mk[0] = mk[1] = mk[2] = 0.f;
  if (!tangents) return;
  float suf = 1.f;
#pragma unroll
  for (int q = NQ - 1; q >= 0; --q) {
    const bool bit = (b >> (NQ - 1 - q)) & 1;
    const float df = bit ? 0.5f * pa.c[q] : -0.5f * pa.s[q];
    const float rest = pre[q] * suf;
#pragma unroll
    for (int k = 0; k < 3; ++k) mk[k] += pa.d[k][q] * df * rest;
    suf *= bit ? pa.s[q] : pa.c[q];
  }
}

// embed_amp for the 4 amplitudes b0 .. b0 + 3 (b0 % 4 == 0: only the last two wires
// differ): the first NQ - 2 factors, and their tangent terms, are shared
template <int NQ>
__device__ __forceinline__ void embed_amp4(const PointAngles<NQ>& pa, int b0, bool tangents,
                                           float (&m0)[4], float (&mk)[4][3]) {
  constexpr int H = NQ - 2;
  float pre[H + 1];
  pre[0] = 1.f;
#pragma unroll
  for (int q = 0; q < H; ++q) pre[q + 1] = pre[q] * (((b0 >> (NQ - 1 - q)) & 1) ? pa.s[q] : pa.c[q]);
  const float P = pre[H];
  // the last two wires: factor f(bit) and derivative factor df(bit) (as embed_amp)
  const float fa[2] = {pa.c[H], pa.s[H]}, fb[2] = {pa.c[H + 1], pa.s[H + 1]};
  const float da[2] = {-0.5f * pa.s[H], 0.5f * pa.c[H]}, db[2] = {-0.5f * pa.s[H + 1], 0.5f * pa.c[H + 1]};
#pragma unroll
  for (int e = 0; e < 4; ++e) m0[e] = P * fa[e >> 1] * fb[e & 1];
#pragma unroll
  for (int e = 0; e < 4; ++e) mk[e][0] = mk[e][1] = mk[e][2] = 0.f;
  if (!tangents) return;
  float T[3] = {0.f, 0.f, 0.f};  // sum over the shared wires of d_kq df_q prod_{q' != q} f_q'
  float suf = 1.f;
#pragma unroll
  for (int q = H - 1; q >= 0; --q) {
    const bool bit = (b0 >> (NQ - 1 - q)) & 1;
    const float df = bit ? 0.5f * pa.c[q] : -0.5f * pa.s[q];
    const float rest = pre[q] * suf;
#pragma unroll
    for (int k = 0; k < 3; ++k) T[k] += pa.d[k][q] * df * rest;
    suf *= bit ? pa.s[q] : pa.c[q];
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int ia = e >> 1, ib = e & 1;
#pragma unroll
    for (int k = 0; k < 3; ++k)
      mk[e][k] = T[k] * fa[ia] * fb[ib] + pa.d[k][H] * da[ia] * P * fb[ib] +
                 pa.d[k][H + 1] * db[ib] * P * fa[ia];
  }
}

// lane l ends with the warp total of value index l (recursive halving, 31 shuffles)
__device__ __forceinline__ void reduce_scatter32(float* v);

// NV <= 64 per-lane values -> warp totals: value e on lane e % 32 of half e / 32
// (h[0] = values 0..31, h[1] = 32..63); total of value e for any lane via warp_value
template <int NV>
struct Scatter {
  static constexpr int H = NV <= 32 ? 1 : 2;
  float h[H];
};
template <int NV>
__device__ __forceinline__ Scatter<NV> reduce_scatter(float* v) {
  Scatter<NV> r;
  reduce_scatter32(v);
  r.h[0] = v[0];
  if constexpr (NV > 32) {
    reduce_scatter32(v + 32);
    r.h[1] = v[32];
  }
  return r;
}
template <int NV>
__device__ __forceinline__ float warp_value(const Scatter<NV>& r, int e) {
  const float a = __shfl_sync(0xffffffffu, r.h[0], e & 31);
  if constexpr (NV > 32) {
    const float b = __shfl_sync(0xffffffffu, r.h[1], e & 31);
    return e >= 32 ? b : a;
  }
  return a;
}

__device__ __forceinline__ void reduce_scatter32(float* v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    const bool up = lane & m;
#pragma unroll
    for (int i = 0; i < m; ++i) {
      const float send = up ? v[i] : v[i + m];
      const float keep = up ? v[i + m] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
  }
}

template <typename F>
__device__ __forceinline__ void for_points(int64_t R, F&& body) {
  // block iteration over kPB-point groups; warp w takes points w, w + 8, ...
  for (int64_t p0 = (int64_t)blockIdx.x * kPB; p0 < R; p0 += (int64_t)gridDim.x * kPB)
    body(p0);
}

// Phi rows: the magnitudes m_b of the embedded state and its tangents (D per row)
#ifndef QPINN_TR_EMB_MINB
#define QPINN_TR_EMB_MINB 4
#endif
template <int NQ>
__global__ void __launch_bounds__(256, NQ >= 9 ? 1 : NQ >= 8 ? 2 : QPINN_TR_EMB_MINB) tr_embed(int scale, int64_t R, const float* __restrict__ act,
                                                const float* __restrict__ tan,
                                                float* __restrict__ Phi,
                                                unsigned long long* __restrict__ maxabs) {
  constexpr int D = 1 << NQ;
  __shared__ float ang[kPB * NQ * kAng];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float amax = 0.f;
  for_points(R, [&](int64_t p0) {
    stage_angles<NQ>(scale, R, p0, act, tan, ang, amax);
    __syncthreads();
    for (int pl = w; pl < kPB && p0 + pl < R; pl += 8) {
      const int64_t p = p0 + pl;
      PointAngles<NQ> pa;
      read_angles<NQ>(ang + pl * NQ * kAng, pa);
      if constexpr (D >= 128) {  // 4 consecutive amplitudes per lane: 16-byte stores
#pragma unroll(NQ >= 10 ? 2 : D / 128)
        for (int b0 = 4 * lane; b0 < D; b0 += 128) {
          float m0[4], mk[4][3];
          embed_amp4<NQ>(pa, b0, tan != nullptr, m0, mk);
          // magnitudes: the phase (-i)^popcount(b) lives in W' (tr_wmat)
          *reinterpret_cast<float4*>(Phi + p * D + b0) = make_float4(m0[0], m0[1], m0[2], m0[3]);
          if (tan)
#pragma unroll
            for (int k = 0; k < 3; ++k)
              *reinterpret_cast<float4*>(Phi + ((int64_t)(k + 1) * R + p) * D + b0) =
                  make_float4(mk[0][k], mk[1][k], mk[2][k], mk[3][k]);
        }
      } else {
#pragma unroll
        for (int b = lane; b < D; b += 32) {
          float m0, mk[3];
          embed_amp<NQ>(pa, b, tan != nullptr, m0, mk);
          Phi[p * D + b] = m0;
          if (tan)
            for (int k = 0; k < 3; ++k) Phi[((int64_t)(k + 1) * R + p) * D + b] = mk[k];
        }
      }
    }
    __syncthreads();
  });
  if (maxabs) {
    for (int m = 16; m >= 1; m >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, m));
    if (lane == 0) atomic_max_abs(maxabs, amax);
  }
}

// z_q = sum_b |psi_b|^2 s_bq, dz_kq = sum_b 2 Re(conj(psi_b) dpsi_kb) s_bq (qsim.py:369-381)
#ifndef QPINN_TR_RD_MINB
#define QPINN_TR_RD_MINB 1
#endif
template <int NQ>
__global__ void __launch_bounds__(256, QPINN_TR_RD_MINB) tr_readout(int64_t R, int ns, const float* __restrict__ Psi,
                                                  float* __restrict__ z, float* __restrict__ dz) {
  constexpr int D = 1 << NQ, D2 = 2 * D;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < R; p += nw) {
    constexpr int NV = 4 * NQ, NA = NV <= 32 ? 32 : 64;
    float acc[NA];
#pragma unroll
    for (int e = 0; e < NA; ++e) acc[e] = 0.f;
#pragma unroll
    for (int b = lane; b < D; b += 32) {
      const float pr = Psi[p * D2 + b], pi = Psi[p * D2 + D + b];
      float v[4];
      v[0] = pr * pr + pi * pi;
#pragma unroll
      for (int k = 1; k < 4; ++k) {
        if (k < ns) {
          const float* row = Psi + ((int64_t)k * R + p) * D2;
          v[k] = 2.f * (pr * row[b] + pi * row[D + b]);
        } else {
          v[k] = 0.f;
        }
      }
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const bool neg = (b >> (NQ - 1 - q)) & 1;
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k * NQ + q] += neg ? -v[k] : v[k];
      }
    }
    const Scatter<NV> sc = reduce_scatter<NV>(acc);
#pragma unroll
    for (int hh = 0; hh < Scatter<NV>::H; ++hh) {
      const int e = lane + 32 * hh, k = e / NQ, q = e % NQ;
      if (e >= NV) continue;
      if (k == 0) z[p * NQ + q] = sc.h[hh];
      else if (k < ns) dz[((int64_t)(k - 1) * R + p) * NQ + q] = sc.h[hh];
    }
  }
}

// adjoint seeds as real-block rows:
// lambda = 2 w psi + 2 sum_k v_k dpsi_k, mu_k = 2 v_k psi
#ifndef QPINN_TR_SD_MINB
#define QPINN_TR_SD_MINB 1
#endif
template <int NQ>
__global__ void __launch_bounds__(256, QPINN_TR_SD_MINB) tr_seed(int64_t R, const float* __restrict__ gz,
                                               const float* __restrict__ gdz,
                                               const float* __restrict__ Psi,
                                               float* __restrict__ Abar) {
  constexpr int D = 1 << NQ, D2 = 2 * D;
  __shared__ float sg[kPB][4][NQ];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for_points(R, [&](int64_t p0) {
    for (int i = threadIdx.x; i < kPB * NQ; i += blockDim.x) {
      const int64_t p = p0 + i / NQ;
      const int q = i % NQ;
      const bool ok = p < R;
      sg[i / NQ][0][q] = ok ? gz[p * NQ + q] : 0.f;
      for (int k = 0; k < 3; ++k) sg[i / NQ][k + 1][q] = ok ? gdz[((int64_t)k * R + p) * NQ + q] : 0.f;
    }
    __syncthreads();
    for (int pl = w; pl < kPB && p0 + pl < R; pl += 8) {
      const int64_t p = p0 + pl;
#pragma unroll
      for (int b = lane; b < D; b += 32) {
        float wv[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const bool neg = (b >> (NQ - 1 - q)) & 1;
#pragma unroll
          for (int k = 0; k < 4; ++k) wv[k] += neg ? -sg[pl][k][q] : sg[pl][k][q];
        }
        const float pr = Psi[p * D2 + b], pi = Psi[p * D2 + D + b];
        float lr = 2.f * wv[0] * pr, li = 2.f * wv[0] * pi;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const float* row = Psi + ((int64_t)(k + 1) * R + p) * D2;
          lr += 2.f * wv[k + 1] * row[b];
          li += 2.f * wv[k + 1] * row[D + b];
          float* o = Abar + ((int64_t)(k + 1) * R + p) * D2;
          o[b] = 2.f * wv[k + 1] * pr;
          o[D + b] = 2.f * wv[k + 1] * pi;
        }
        Abar[p * D2 + b] = lr;
        Abar[p * D2 + D + b] = li;
      }
    }
    __syncthreads();
  });
}

// value of register j at the partner index b ^ bit(q) (lane bits: shuffle; j bits: register)
template <int NQ, int J>
__device__ __forceinline__ float flip_get(const float (&v)[J], int j, int q) {
  const int pos = NQ - 1 - q;
  if (pos < 5) return __shfl_xor_sync(0xffffffffu, v[j], 1 << pos);
  return v[j ^ (1 << (pos - 5))];
}

// embedding gradient (qpinn_oracle.pqc_backward):
//   eta = (i/2) phibar - 1/4 sum_q X_q nu_q,  nu_q = sum_k dth_kq mu_k
//   g_th[q] = Re sum conj(eta) X_q phi, g_dth[k][q] = Re sum conj((i/2) mu_k) X_q phi
// phibar, mu_k = p_b x the rows of dL/dm; phi = p_b m is re-embedded in registers;
// with the common phase p_b factored out the sums are real (see the kernel body)
#ifndef QPINN_TR_EG_MINB
#define QPINN_TR_EG_MINB 4  // 64 registers, no spills: 58 vs 63 us at 3 (real-arithmetic version)
#endif
template <int NQ>
__global__ void __launch_bounds__(256, NQ >= 9 ? 1 : NQ >= 8 ? 2 : QPINN_TR_EG_MINB) tr_embed_grad(int scale, int64_t R,
                                                     const float* __restrict__ act,
                                                     const float* __restrict__ tan,
                                                     const float* __restrict__ gPhi,
                                                     float* __restrict__ g_act,
                                                     float* __restrict__ g_tan) {
  constexpr int D = 1 << NQ, J = D / 32;
  __shared__ float ang[kPB * NQ * kAng];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float amax = 0.f;
  for_points(R, [&](int64_t p0) {
    stage_angles<NQ>(scale, R, p0, act, tan, ang, amax);
    __syncthreads();
    // loop exit through a warp vote: provably warp-uniform, so the shuffles below
    // compile to plain SHFL (no WARPSYNC / ENDCOLLECTIVE divergence wrappers)
    for (int pl = w; __all_sync(0xffffffffu, pl < kPB && p0 + pl < R); pl += 8) {
      const int64_t p = p0 + pl;
      const float* pang = ang + pl * NQ * kAng;
      PointAngles<NQ> pa;
      read_angles<NQ>(pang, pa);
      // Every factor here is p_b x real (phi_b = p_b m_b, phibar_b = p_b dL/dm_b,
      // p_b = (-i)^popcount(b)), so the complex formulas reduce to real ones on the
      // magnitudes (sigma_q(b) = +1 if wire q is set in b, else -1):
      //   nu_q(b)  = sum_k dth_kq g_k(b)                      (g_k = dL/dm of tangent row k)
      //   eta(b)   = g_0(b) / 2 - 1/4 sum_q sigma_q(b) nu_q(b ^ q)
      //   g_th[q]  = sum_b sigma_q(b) eta(b) m(b ^ q),  g_dth[k][q] = 1/2 sum_b sigma_q(b) g_k(b) m(b ^ q)
      constexpr int NV = 4 * NQ, NA = NV <= 32 ? 32 : 64;
      float acc[NA];
#pragma unroll
      for (int e = 0; e < NA; ++e) acc[e] = 0.f;
      if constexpr (J >= 32) {
        // 32 amplitudes per lane: only the adjoint rows one at a time stay in registers
        // (flips are linear, so nu's flip is the sum of the rows' flips; the rows are
        // re-read from L1/L2 for the outer products)
        const float* grow = gPhi + p * D + lane;
        const int64_t rs = R * D;
        float m[J], et[J];
#pragma unroll
        for (int j = 0; j < J; ++j) {
          float mk[3];
          embed_amp<NQ>(pa, lane + 32 * j, false, m[j], mk);
          et[j] = 0.5f * grow[32 * j];
        }
        for (int k = 0; k < 3; ++k) {
          float gk[J];
#pragma unroll
          for (int j = 0; j < J; ++j) gk[j] = grow[(k + 1) * rs + 32 * j];
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const float dq = 0.25f * pang[q * kAng + 3 + k];  // pa.d[k][q] (k not unrolled)
#pragma unroll
            for (int j = 0; j < J; ++j) {
              const float f = dq * flip_get<NQ, J>(gk, j, q);
              et[j] += ((lane + 32 * j) >> (NQ - 1 - q)) & 1 ? -f : f;
            }
          }
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
          for (int j = 0; j < J; ++j) {
            const float mf = flip_get<NQ, J>(m, j, q);
            const float y = ((lane + 32 * j) >> (NQ - 1 - q)) & 1 ? mf : -mf;
            acc[q] = fmaf(et[j], y, acc[q]);
          }
        for (int k = 0; k < 3; ++k) {
          float gk[J];
#pragma unroll
          for (int j = 0; j < J; ++j) gk[j] = grow[(k + 1) * rs + 32 * j];
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            float a = 0.f;
#pragma unroll
            for (int j = 0; j < J; ++j) {
              const float mf = flip_get<NQ, J>(m, j, q);
              a = fmaf(gk[j], ((lane + 32 * j) >> (NQ - 1 - q)) & 1 ? mf : -mf, a);
            }
            // acc index NQ + k NQ + q with k a loop variable: select without local memory
#pragma unroll
            for (int kk = 0; kk < 3; ++kk)
              if (kk == k) acc[NQ + kk * NQ + q] += a;
          }
        }
      } else {
      float m[J], et[J], g[4][J];
#pragma unroll
      for (int r = 0; r < 4; ++r)  // all the point's loads in flight before any use
#pragma unroll
        for (int j = 0; j < J; ++j) g[r][j] = gPhi[((int64_t)r * R + p) * D + lane + 32 * j];
#pragma unroll
      for (int j = 0; j < J; ++j) {
        float mk[3];
        embed_amp<NQ>(pa, lane + 32 * j, false, m[j], mk);
        et[j] = 0.5f * g[0][j];
      }
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        float nu[J];
#pragma unroll
        for (int j = 0; j < J; ++j)
          nu[j] = pa.d[0][q] * g[1][j] + pa.d[1][q] * g[2][j] + pa.d[2][q] * g[3][j];
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const float f = 0.25f * flip_get<NQ, J>(nu, j, q);
          et[j] += ((lane + 32 * j) >> (NQ - 1 - q)) & 1 ? -f : f;
        }
      }
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const float mf = flip_get<NQ, J>(m, j, q);
          const float y = ((lane + 32 * j) >> (NQ - 1 - q)) & 1 ? mf : -mf;
          acc[q] = fmaf(et[j], y, acc[q]);
#pragma unroll
          for (int k = 0; k < 3; ++k) acc[NQ + k * NQ + q] = fmaf(g[k + 1][j], y, acc[NQ + k * NQ + q]);
        }
      }
      }
      // value v on lane v % 32 of half v / 32: g_th[q] = value q, g_dth[k][q] = NQ + k NQ + q
      const Scatter<NV> sc = reduce_scatter<NV>(acc);
      const int q = lane < NQ ? lane : 0;
      float gd[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) gd[k] = 0.5f * warp_value<NV>(sc, NQ + k * NQ + q);
      const float gth = warp_value<NV>(sc, q);
      if (lane < NQ) {
        const float* a = pang + q * kAng;
        float ga = gth * a[2];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          ga += gd[k] * a[6 + k];
          g_tan[((int64_t)k * R + p) * NQ + q] = gd[k] * a[2];
        }
        g_act[p * NQ + q] = ga;
      }
    }
    __syncthreads();
  });
}

struct TrLayout {
  size_t U, ph, B, CK, Ab, W, Wt, gW, pu, pp, acc, g3, wg, BUF1, BUF2, total;
};

TrLayout tr_layout(const qpinn_circuit* c, int64_t R) {
  const size_t D = (size_t)1 << c->n, D2 = 2 * D, cs = sizeof(cplx<float>);
  TrLayout t{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o += align_up(bytes, 256);
    return at;
  };
  t.U = take(cs * 4 * c->n_u1);
  t.ph = take(cs * D * c->n_phase);
  t.B = take(cs * D * D);
  t.CK = take(cs * D * D * c->L);
  t.Ab = take(cs * D * D);
  t.W = take(4 * D2 * D2);
  t.Wt = take(4 * D2 * D2);
  t.gW = take(4 * D2 * D2);
  t.pu = take(8 * D * 8 * (size_t)c->n_u1);
  t.pp = take(8 * D * D * c->n_phase);
  t.acc = take(8 * (8 * (size_t)c->n_u1 + D * c->n_phase));
  t.g3 = take(tc::gemm3_workspace_bytes((int)D2, (int)D2));
  t.wg = take(tc::wgrad_workspace_bytes(4 * R, (int)D2, (int)D2));
  t.BUF1 = take(4 * (size_t)R * D2 * 4);
  t.BUF2 = take(4 * (size_t)R * D2 * 4);
  t.total = o;
  return t;
}

int grid_points(int64_t R) {  // 8 warps per block, kPB points per block iteration
  const int64_t b = (R + kPB - 1) / kPB, cap = (int64_t)num_sms() * 8;
  return (int)(b < 1 ? 1 : b > cap ? cap : b);
}

// The circuit's device tables: u1 matrices, phase diagonals, the layer
// checkpoints of the basis rows, W (backward operand) and W^T (forward operand).
struct TrCircuit {
  cplx<float>* U;
  cplx<float>* ph;
  cplx<float>* CK;
  float* W;   // W' [D][2D] tf32 hi, then lo
  float* Wt;  // W'^T [2D][D] tf32 hi, then lo
};

// the split operands of the map's GEMMs: B = W'^T [2D, D] (forward), B = W' [D, 2D]
inline tc::Wsplit split_wt(const TrCircuit& cc, int D) {
  return tc::Wsplit{cc.Wt, cc.Wt + (size_t)2 * D * D, D};
}
inline tc::Wsplit split_w(const TrCircuit& cc, int D) {
  return tc::Wsplit{cc.W, cc.W + (size_t)2 * D * D, 2 * D};
}

// hand-off layout (after the forward with tangents): [Psi | Phi | W | CK | U | ph]
struct TrHandoff {
  size_t psi, phi, W, CK, U, ph, total;
};

TrHandoff tr_handoff(const qpinn_circuit* c, int64_t R) {
  const size_t D = (size_t)1 << c->n, D2 = 2 * D, cs = sizeof(cplx<float>);
  TrHandoff h{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o += align_up(bytes, 256);
    return at;
  };
  h.psi = take(4 * (size_t)R * D2 * 4);
  h.phi = take(4 * (size_t)R * D * 4);
  h.W = take(2 * 4 * D * D2);  // tf32 hi / lo
  h.CK = take(cs * D * D * c->L);
  h.U = take(cs * 4 * c->n_u1);
  h.ph = take(cs * D * c->n_phase);
  h.total = o;
  return h;
}

// B = the circuit on the basis rows (with the layer checkpoints), then W / W^T
int build_transfer(const qpinn_circuit* c, const float* qp, const TrCircuit& tc_,
                   cplx<float>* B, cudaStream_t st) {
  const PlanDev& p = c->dev;
  const int n = c->n, D = 1 << n;
  const int ent = layer_entangler(c);
  tr_tables<<<32, 256, 0, st>>>(p, qp, tc_.U, tc_.ph);
  switch (n) {  // rows of 2^n amplitudes in shared memory
#define QPINN_TR_CF(NN)                                                                  \
  case NN:                                                                               \
    tr_circuit_fwd<NN><<<D, kTrThreads, 0, st>>>(n, c->L, ent, tc_.U, tc_.ph, p.perm, B, \
                                                 tc_.CK);                                \
    break;
    QPINN_TR_CF(5) QPINN_TR_CF(6) QPINN_TR_CF(7) QPINN_TR_CF(8) QPINN_TR_CF(9) QPINN_TR_CF(10)
#undef QPINN_TR_CF
    default: return fail(QPINN_ERR_CAPACITY, "transfer PQC covers 5 <= n <= 10");
  }
  tr_wmat<<<(2 * D * D + 255) / 256, 256, 0, st>>>(n, B, tc_.W, tc_.Wt);
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

// side stream per device for the backward's weight-gradient chain (fork/join
// through events, so it is captured as a parallel branch of the step's CUDA graph)
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream g_side[64];
std::mutex g_side_mu;

// *out = nullptr (serial fallback) when the stream and events do not exist yet
// and `st` is being captured (creating them would invalidate the capture)
int side_stream(cudaStream_t st, SideStream** out) {
  int dev = 0;
  QPINN_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_side_mu);
  SideStream& ss = g_side[dev & 63];
  *out = nullptr;
  if (!ss.s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    QPINN_CUDA_CHECK(cudaStreamIsCapturing(st, &cs));
    if (cs != cudaStreamCaptureStatusNone) return QPINN_OK;
    QPINN_CUDA_CHECK(cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking));
    QPINN_CUDA_CHECK(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming));
    QPINN_CUDA_CHECK(cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming));
  }
  *out = &ss;
  return QPINN_OK;
}

// A fork of `st` onto the side stream that every return path joins back (errors
// included): a graph capture never ends with an unjoined fork, and an eager caller
// never gets control back while side work still runs.  fork() returns the side
// stream, or `st` itself when there is none (serial fallback).
struct ForkJoin {
  SideStream* side = nullptr;
  cudaStream_t st = nullptr;
  int fork(cudaStream_t main, cudaStream_t* out) {
    st = main;
    *out = main;
    static const bool serial = getenv("QPINN_SERIAL_BWD") != nullptr;  // A/B switch
    if (serial) return QPINN_OK;
    if (int rc = side_stream(main, &side)) return rc;
    if (!side) return QPINN_OK;
    QPINN_CUDA_CHECK(cudaEventRecord(side->fork, main));
    QPINN_CUDA_CHECK(cudaStreamWaitEvent(side->s, side->fork, 0));
    *out = side->s;
    return QPINN_OK;
  }
  ~ForkJoin() {
    if (side) {
      cudaEventRecord(side->join, side->s);
      cudaStreamWaitEvent(st, side->join, 0);
    }
  }
};

// QPINN_TR_FUSED_READOUT=0: the separate tr_readout pass (A/B experiments)
bool fused_readout_off() {
  static const bool off = [] {
    const char* e = getenv("QPINN_TR_FUSED_READOUT");
    return e && atoi(e) == 0;
  }();
  return off;
}

TrCircuit ws_circuit(unsigned char* ws, const TrLayout& t) {
  return {(cplx<float>*)(ws + t.U), (cplx<float>*)(ws + t.ph), (cplx<float>*)(ws + t.CK),
          (float*)(ws + t.W), (float*)(ws + t.Wt)};
}

template <int NQ>
int fwd_n(const qpinn_circuit* c, const KArgs<float>* a, unsigned char* ws, const TrLayout& t) {
  constexpr int D = 1 << NQ, D2 = 2 * D;
  cudaStream_t st = a->stream;
  const bool handoff = a->states && a->tan;
  auto* hs = (unsigned char*)a->states;
  const TrHandoff h = tr_handoff(c, a->R);
  TrCircuit cc = ws_circuit(ws, t);
  if (handoff) {  // the backward reuses the circuit tables, checkpoints and W
    cc.U = (cplx<float>*)(hs + h.U);
    cc.ph = (cplx<float>*)(hs + h.ph);
    cc.CK = (cplx<float>*)(hs + h.CK);
    cc.W = (float*)(hs + h.W);
  }
  auto* Psi = a->states ? (float*)(hs + h.psi) : (float*)(ws + t.BUF2);
  auto* Phi = handoff ? (float*)(hs + h.phi) : (float*)(ws + t.BUF1);
  const int ns = a->tan ? 4 : 1;
  {
    // the circuit's transfer map depends on qparams only: it is built on the side
    // stream while the points are embedded, and joined before the map's GEMM
    ForkJoin fj;
    cudaStream_t s2;
    if (int rc = fj.fork(st, &s2)) return rc;
    if (int rc = build_transfer(c, a->qp, cc, (cplx<float>*)(ws + t.B), s2)) return rc;
    tr_embed<NQ><<<grid_points(a->R), 256, 0, st>>>(a->scale, a->R, a->act, a->tan, Phi,
                                                    a->maxabs);
    QPINN_CUDA_CHECK(cudaGetLastError());
  }
  if (NQ == 7 && ns == 4 && !fused_readout_off()) {  // map + readout in one tensor-core pass
    const tc::Wsplit wt = split_wt(cc, D);
    return tc::gemm3_readout(a->R, Phi, cc.Wt, Psi, a->z, a->dz, ws + t.g3,
                             tc::gemm3_workspace_bytes(D2, D2), st, &wt);
  }
  const tc::Wsplit wt = split_wt(cc, D);
  if (int rc = tc::gemm3(ns * a->R, D2, D, Phi, D, cc.Wt, D, Psi, D2, ws + t.g3,
                         tc::gemm3_workspace_bytes(D2, D2), st, &wt))
    return rc;
  tr_readout<NQ><<<grid_points(a->R), 256, 0, st>>>(a->R, ns, Psi, a->z, a->dz);
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

template <int NQ>
int bwd_n(const qpinn_circuit* c, const KArgs<float>* a, unsigned char* ws, const TrLayout& t) {
  constexpr int D = 1 << NQ, D2 = 2 * D;
  cudaStream_t st = a->stream;
  const PlanDev& p = c->dev;
  const int ent = layer_entangler(c), L = c->L, n_u1 = c->n_u1;
  auto* Abar = (float*)(ws + t.BUF1);
  auto* G = (float*)(ws + t.BUF2);
  const int gp = grid_points(a->R);
  const float* Psi;
  const float* Phi;
  TrCircuit cc = ws_circuit(ws, t);
  if (a->states) {  // hand-off of the matching forward
    auto* hs = (unsigned char*)a->states;
    const TrHandoff h = tr_handoff(c, a->R);
    Psi = (const float*)(hs + h.psi);
    Phi = (const float*)(hs + h.phi);
    cc.U = (cplx<float>*)(hs + h.U);
    cc.ph = (cplx<float>*)(hs + h.ph);
    cc.CK = (cplx<float>*)(hs + h.CK);
    cc.W = (float*)(hs + h.W);
  } else {  // replay the forward map: Phi into BUF1, Psi into BUF2
    if (int rc = build_transfer(c, a->qp, cc, (cplx<float>*)(ws + t.B), st)) return rc;
    tr_embed<NQ><<<gp, 256, 0, st>>>(a->scale, a->R, a->act, a->tan, Abar, nullptr);
    QPINN_CUDA_CHECK(cudaGetLastError());
    const tc::Wsplit wt = split_wt(cc, D);
    if (int rc = tc::gemm3(4 * a->R, D2, D, Abar, D, cc.Wt, D, G, D2, ws + t.g3,
                           tc::gemm3_workspace_bytes(D2, D2), st, &wt))
      return rc;
    Psi = G;
    Phi = nullptr;  // re-embedded after the embedding gradient
  }
  tr_seed<NQ><<<gp, 256, 0, st>>>(a->R, a->gz, a->gdz, Psi, Abar);
  QPINN_CUDA_CHECK(cudaGetLastError());
  // the weight-gradient chain (dL/dW' -> adjoint on the basis rows -> dL/dqparams)
  // needs only m and Abar: with the hand-off it runs on a side stream, overlapping
  // the dL/dm GEMM and the embedding gradient (the replay path reuses G for m, so
  // it stays serial)
  auto weight_chain = [&](cudaStream_t s2) -> int {
    if (int rc = tc::wgrad(4 * a->R, D, D2, Phi, D, Abar, D2, (float*)(ws + t.gW), ws + t.wg,
                           tc::wgrad_workspace_bytes(4 * a->R, D2, D2), s2))
      return rc;
    auto* Ab = (cplx<float>*)(ws + t.Ab);
    tr_gb<<<(D * D + 255) / 256, 256, 0, s2>>>(NQ, (const float*)(ws + t.gW), Ab);
    auto* pu = (double*)(ws + t.pu);
    auto* pp = (double*)(ws + t.pp);
    auto* acc = (double*)(ws + t.acc);
    tr_circuit_bwd<NQ><<<D, kTrThreads, 0, s2>>>(NQ, L, ent, cc.U, cc.ph, p.iperm, Ab, cc.CK, pu, pp);
    const int n_ph = D * c->n_phase, n_acc = 8 * n_u1 + n_ph;
    tr_reduce<<<(n_acc + 7) / 8, 256, 0, s2>>>(D, n_u1, n_ph, pu, pp, acc);
    QPINN_CUDA_CHECK(cudaGetLastError());
    return pqc_param_grads<float>(c, acc, NQ, a->qp, a->g_qp, s2);
  };
  // with the hand-off the weight chain forks onto the side stream (joined on every
  // return path, errors included: it writes g_qp)
  ForkJoin fj;
  cudaStream_t s2 = st;
  if (Phi)
    if (int rc = fj.fork(st, &s2)) return rc;
  const bool side = s2 != st;
  // dL/dm = Abar W'^T  (D per row)
  const tc::Wsplit wsp = split_w(cc, D);
  if (int rc = tc::gemm3(4 * a->R, D, D2, Abar, D2, cc.W, D2, G, D, ws + t.g3,
                         tc::gemm3_workspace_bytes(D2, D2), st, &wsp))
    return rc;
  if (side)
    if (int rc = weight_chain(s2)) return rc;
  tr_embed_grad<NQ><<<gp, 256, 0, st>>>(a->scale, a->R, a->act, a->tan, G, a->g_act, a->g_tan);
  QPINN_CUDA_CHECK(cudaGetLastError());
  if (side) return QPINN_OK;  // joined by `fj`
  // replay path: re-embed m into G once the embedding gradient has read it
  tr_embed<NQ><<<gp, 256, 0, st>>>(a->scale, a->R, a->act, a->tan, G, nullptr);
  Phi = G;
  QPINN_CUDA_CHECK(cudaGetLastError());
  return weight_chain(st);
}

}  // namespace

bool transfer_supported(const qpinn_circuit* c, int dtype) {
  return c && dtype == QPINN_F32 && c->n >= 5 && c->n <= kTrMaxN && layer_entangler(c) >= 0;
}

// the default (variant 0) path: the transfer map up to n = 8, and at n = 9, 10 from
// L = 4 (its cost does not grow with L; at 2^16 points K1 + K2 take 8.6 ms at n = 9 and
// 30 ms at n = 10 against the CTA kernels' 14-16 / 33-38 ms at L = 4 and 24-28 / 56-64
// ms at L = 8; at L = 1 the CTA kernels win, 6.5-7.1 / 16-18 ms;
// profiles/r02/config5_n9_transfer_vs_cta.txt, config5_n10_transfer_vs_cta.txt)
bool transfer_default(const qpinn_circuit* c, int dtype) {
  return transfer_supported(c, dtype) && (c->n <= 8 || c->L >= 4);
}

size_t transfer_state_bytes(const qpinn_circuit* c, int64_t R) {
  return R <= 0 ? 0 : tr_handoff(c, R).total;
}

size_t transfer_workspace_bytes(const qpinn_circuit* c, int64_t R) {
  return tr_layout(c, R < 1 ? 1 : R).total;
}

int transfer_forward(const qpinn_circuit* c, const KArgs<float>* a, unsigned char* ws,
                     size_t bytes) {
  const TrLayout t = tr_layout(c, a->R);
  if (bytes < t.total) return fail(QPINN_ERR_CONFIG, "transfer PQC: workspace too small");
  switch (c->n) {
    case 5: return fwd_n<5>(c, a, ws, t);
    case 6: return fwd_n<6>(c, a, ws, t);
    case 7: return fwd_n<7>(c, a, ws, t);
    case 8: return fwd_n<8>(c, a, ws, t);
    case 9: return fwd_n<9>(c, a, ws, t);
    case 10: return fwd_n<10>(c, a, ws, t);
    default: return fail(QPINN_ERR_CAPACITY, "transfer PQC covers 5 <= n <= 10");
  }
}

int transfer_backward(const qpinn_circuit* c, const KArgs<float>* a, unsigned char* ws,
                      size_t bytes) {
  const TrLayout t = tr_layout(c, a->R);
  if (bytes < t.total) return fail(QPINN_ERR_CONFIG, "transfer PQC: workspace too small");
  switch (c->n) {
    case 5: return bwd_n<5>(c, a, ws, t);
    case 6: return bwd_n<6>(c, a, ws, t);
    case 7: return bwd_n<7>(c, a, ws, t);
    case 8: return bwd_n<8>(c, a, ws, t);
    case 9: return bwd_n<9>(c, a, ws, t);
    case 10: return bwd_n<10>(c, a, ws, t);
    default: return fail(QPINN_ERR_CAPACITY, "transfer PQC covers 5 <= n <= 10");
  }
}

}  // namespace qpinn
