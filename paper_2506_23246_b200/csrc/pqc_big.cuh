// Large-register PQC kernels (n = 9 .. 16): one thread-block CLUSTER per point.
//
// Same per-point algorithm as the register kernels (pqc_layer.cu): closed-form
// embedding, layer loop of single-qubit steps + entangler, Z readout, adjoint
// backward with per-gate outer products.  The statevector of one
// point no longer fits one warp, so amplitude index bits are spread over
//     (CTA rank in cluster : CB) (warp : WB) (lane : LB) (register : AB)
// with the 4 states (psi, dpsi/dx, dpsi/dy, dpsi/dt) in lanes (LB = 3) as
// before.  A gate on a
//   * register wire is pure FMA,
//   * lane wire is one shfl.xor per amplitude,
//   * warp wire exchanges through shared memory (one buffer per CTA),
//   * CTA wire exchanges through DISTRIBUTED shared memory across the cluster
//     (up to 16 CTAs at n = 16, non-portable cluster size).
// Fused CNOT runs are gathers through the same buffers; CRZ-mesh phases come
// from a per-call table in global memory.  The backward re-runs the forward
// (a state hand-off would be 2^n x 32 B per point), then sweeps back with the
// state and its adjoint in the same lane.  Parameter-gradient partials are
// per cluster, reduced in fixed order (deterministic).
#include <cooperative_groups.h>

#pragma once
#include "pqc_layer.h"

namespace cg = cooperative_groups;

namespace qpinn {

// BWD kernels hold state + adjoint (2 x A complex per thread, ~255 registers):
// at most 8 warps per CTA.  Forward kernels: at most 16 warps, 32 only where a
// 16-CTA cluster is not enough (n = 16).
template <typename T, int N, int NSL, bool BWD = false>
struct BigGeo {
  static constexpr int AB = sizeof(T) == 8 ? 3 : 4;
  static constexpr int A = 1 << AB;
  static constexpr int LB = NSL == 4 ? 3 : 5;
  static constexpr int G = 1 << LB;
  static constexpr int REST = N - AB - LB;
  static constexpr int MAXWB = BWD ? 3 : (REST > 8 ? 5 : 4);
  static constexpr int WB = REST < MAXWB ? REST : MAXWB;
  static constexpr int CB = REST - WB;
  static constexpr int W = 1 << WB, C = 1 << CB, D = 1 << N;
  static constexpr int THREADS = 32 * W;
  static constexpr int HB = CB + WB + LB;  // bits above the register bits
  static_assert(REST >= 0, "big kernels start above the register regime");
};

// cluster-wide barrier (falls back to the block barrier for one-CTA clusters)
template <int CB>
__device__ __forceinline__ void csync() {
  if constexpr (CB > 0) cg::this_cluster().sync();
  else __syncthreads();
}

template <int CB, typename P>
__device__ __forceinline__ P* remote(P* local, int rank) {
  if constexpr (CB > 0) return cg::this_cluster().map_shared_rank(local, rank);
  else return local;
}

// exchange-based single-qubit step: partner amplitude lives in another warp
// (mask on the warp bits) or another CTA (mask on the rank bits)
template <typename T, typename Geo, bool CTA_WIRE>
__device__ __forceinline__ void gate_exchange(cplx<T> (&st)[Geo::A], cplx<T>* buf, int tid,
                                              int rank, int mask, bool beta, cplx<T> u00,
                                              cplx<T> u01, cplx<T> u10, cplx<T> u11) {
  constexpr int A = Geo::A, TH = Geo::THREADS;
#pragma unroll
  for (int r = 0; r < A; ++r) buf[r * TH + tid] = st[r];
  if constexpr (CTA_WIRE) csync<Geo::CB>();
  else __syncthreads();
  const cplx<T>* src = CTA_WIRE ? remote<Geo::CB>(buf, rank ^ mask) : buf;
  const int ptid = CTA_WIRE ? tid : (tid ^ (mask << 5));
  const cplx<T> cs = beta ? u11 : u00, cp = beta ? u10 : u01;
#pragma unroll
  for (int r = 0; r < A; ++r) st[r] = cmul2(cs, st[r], cp, src[r * TH + ptid]);
  if constexpr (CTA_WIRE) csync<Geo::CB>();
  else __syncthreads();
}

// read the partner's A amplitudes (other warp or other CTA) into p
template <typename T, typename Geo, bool CTA_WIRE>
__device__ __forceinline__ void exchange_read(const cplx<T> (&v)[Geo::A], cplx<T> (&p)[Geo::A],
                                              cplx<T>* buf, int tid, int rank, int mask) {
  constexpr int A = Geo::A, TH = Geo::THREADS;
#pragma unroll
  for (int r = 0; r < A; ++r) buf[r * TH + tid] = v[r];
  if constexpr (CTA_WIRE) csync<Geo::CB>();
  else __syncthreads();
  const cplx<T>* src = CTA_WIRE ? remote<Geo::CB>(buf, rank ^ mask) : buf;
  const int ptid = CTA_WIRE ? tid : (tid ^ (mask << 5));
#pragma unroll
  for (int r = 0; r < A; ++r) p[r] = src[r * TH + ptid];
  if constexpr (CTA_WIRE) csync<Geo::CB>();
  else __syncthreads();
}

// permutation gather new[b] = old[perm[b]] over the cluster; table entries
// are source indices, stored in the layout ((c W + w) A + r) G + gl
template <typename T, typename Geo>
__device__ __forceinline__ void gather(cplx<T> (&st)[Geo::A], cplx<T>* buf, int tid, int rank,
                                       int w, int sidx, int gl, const uint32_t* __restrict__ tab) {
  constexpr int A = Geo::A, TH = Geo::THREADS, G = Geo::G, W = Geo::W, AB = Geo::AB,
                LB = Geo::LB, N0 = Geo::HB + Geo::AB;
#pragma unroll
  for (int r = 0; r < A; ++r) buf[r * TH + tid] = st[r];
  csync<Geo::CB>();
#pragma unroll
  for (int r = 0; r < A; ++r) {
    const uint32_t b = tab[((rank * W + w) * A + r) * G + gl];
    const int c2 = (int)(b >> (N0 - Geo::CB)) & (Geo::C - 1);
    const int w2 = (int)(b >> (AB + LB)) & (W - 1);
    const int g2 = (int)(b >> AB) & (G - 1);
    const int r2 = (int)b & (A - 1);
    const cplx<T>* src = remote<Geo::CB>(buf, c2);
    st[r] = src[r2 * TH + w2 * 32 + sidx * G + g2];
  }
  csync<Geo::CB>();
}

template <typename T, int AB>
__device__ __forceinline__ void rot_left(cplx<T> (&v)[1 << AB]) {  // new[r] = old[rotr(r)]
  constexpr int A = 1 << AB;
  cplx<T> t[A];
#pragma unroll
  for (int r = 0; r < A; ++r) t[r] = v[((r >> 1) | ((r & 1) << (AB - 1))) & (A - 1)];
#pragma unroll
  for (int r = 0; r < A; ++r) v[r] = t[r];
}

// one full layer of single-qubit steps, wires 0 .. N-1 in order
template <typename T, typename Geo>
__device__ __forceinline__ void layer_fwd(cplx<T> (&st)[Geo::A], const cplx<T>* Ul, cplx<T>* buf,
                                          int tid, int rank, int w, int gl) {
  constexpr int CB = Geo::CB, WB = Geo::WB, LB = Geo::LB, AB = Geo::AB;
  for (int q = 0; q < CB; ++q) {
    const int m = 1 << (CB - 1 - q);
    const cplx<T>* U = Ul + 4 * q;
    gate_exchange<T, Geo, true>(st, buf, tid, rank, m, rank & m, U[0], U[1], U[2], U[3]);
  }
  for (int q = 0; q < WB; ++q) {
    const int m = 1 << (WB - 1 - q);
    const cplx<T>* U = Ul + 4 * (CB + q);
    gate_exchange<T, Geo, false>(st, buf, tid, rank, m, w & m, U[0], U[1], U[2], U[3]);
  }
  cplx<T>(&s1)[1][Geo::A] = *reinterpret_cast<cplx<T>(*)[1][Geo::A]>(&st[0]);
  for (int q = 0; q < LB; ++q) {
    const int lb = LB - 1 - q;
    const cplx<T>* U = Ul + 4 * (CB + WB + q);
    gate_lane<T, Geo::A, 1>(s1, 1 << lb, (gl >> lb) & 1, U[0], U[1], U[2], U[3]);
  }
  for (int i = 0; i < AB; ++i) {
    const cplx<T>* U = Ul + 4 * (CB + WB + LB + i);
    gate_reg<AB - 1, T, Geo::A, 1>(s1, U[0], U[1], U[2], U[3]);
    if constexpr (AB > 1) rot_left<T, AB>(st);
  }
}

template <typename T, typename Geo, int ENT>
__device__ __forceinline__ void entangle_fwd(cplx<T> (&st)[Geo::A], int l, cplx<T>* buf, int tid,
                                             int rank, int w, int sidx, int gl,
                                             const uint32_t* perm, const cplx<T>* ph) {
  constexpr int A = Geo::A, G = Geo::G, W = Geo::W;
  if constexpr (ENT == ENT_PERM) {
    gather<T, Geo>(st, buf, tid, rank, w, sidx, gl, perm + (size_t)l * Geo::D);
  } else if constexpr (ENT == ENT_PHASE) {
    const cplx<T>* p = ph + (size_t)l * Geo::D;
#pragma unroll
    for (int r = 0; r < A; ++r) st[r] = cmul(st[r], p[((rank * W + w) * A + r) * G + gl]);
  }
}

// per-call tables for the big kernels: u1 matrices, layout-ordered permutation
// source indices and phase diagonals
template <typename T, int N, int NSL, bool BWD = false>
__global__ void big_prepare(PlanDev p, const T* __restrict__ qp, cplx<T>* __restrict__ U,
                            uint32_t* __restrict__ perm, cplx<T>* __restrict__ ph) {
  using Gm = BigGeo<T, N, NSL, BWD>;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int i = tid; i < p.n_u1; i += nt) {
    const int kind = p.u1[i * 4];
    double th[3] = {0, 0, 0};
    for (int j = 0; j < u1_nslots(kind); ++j) th[j] = (double)qp[p.u1[i * 4 + 1 + j]];
    double M[8];
    u1_matrix_d(kind, th, M);
    for (int e = 0; e < 4; ++e) U[i * 4 + e] = {T(M[2 * e]), T(M[2 * e + 1])};
  }
  constexpr int D = Gm::D, AB = Gm::AB, LB = Gm::LB, A = Gm::A, G = Gm::G;
  // layout index of basis state b = (c, w, gl, r)
  auto lay_big = [](int b) {
    const int r = b & (A - 1), gl = (b >> AB) & (G - 1), cw = b >> (AB + LB);
    return (cw * A + r) * G + gl;
  };
  for (int i = tid; i < p.n_perm * D; i += nt) {
    const int st = i / D, b = i % D;
    perm[(size_t)st * D + lay_big(b)] = (uint32_t)p.perm[i];
  }
  for (int i = tid; i < p.n_phase * D; i += nt) {
    const int st = i / D, b = i % D;
    double phi = 0.0;
    for (int k = p.phase_off[st]; k < p.phase_off[st + 1]; ++k) {
      const int c = p.pairs[3 * k], t = p.pairs[3 * k + 1], s = p.pairs[3 * k + 2];
      const int on = (b >> (N - 1 - c)) & 1, tb = (b >> (N - 1 - t)) & 1;
      phi += on * (tb - 0.5) * (double)qp[s];
    }
    double sp, cp;
    sincos(phi, &sp, &cp);
    ph[(size_t)st * D + lay_big(b)] = {T(cp), T(sp)};
  }
}

template <typename T, int N, int NSL, bool BWD = false>
__global__ void big_prepare_inverse(PlanDev p, uint32_t* __restrict__ iperm) {
  using Gm = BigGeo<T, N, NSL, BWD>;
  constexpr int D = Gm::D, AB = Gm::AB, LB = Gm::LB, A = Gm::A, G = Gm::G;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int i = tid; i < p.n_perm * D; i += nt) {
    const int st = i / D, b = i % D;
    const int r = b & (A - 1), gl = (b >> AB) & (G - 1), cw = b >> (AB + LB);
    iperm[(size_t)st * D + (cw * A + r) * G + gl] = (uint32_t)p.iperm[i];
  }
}

// readout reduce: out[q] (this thread's state) summed over the point's threads of
// the same state; result valid in CTA 0, warp 0
template <typename T, typename Geo, int NSTATE, int N>
__device__ __forceinline__ void reduce_point(T (&out)[N], T* red, int tid, int w, int sidx,
                                             int rank) {
  constexpr int G = Geo::G, W = Geo::W;
#pragma unroll
  for (int m = 1; m < G; m <<= 1)
#pragma unroll
    for (int q = 0; q < N; ++q) out[q] += __shfl_xor_sync(0xffffffffu, out[q], m);
  // red: [W][NSTATE][N] per CTA, then CTA 0 gathers the cluster
  if ((tid & (G - 1)) == 0)
#pragma unroll
    for (int q = 0; q < N; ++q) red[(w * NSTATE + sidx) * N + q] = out[q];
  csync<Geo::CB>();
  if (rank == 0 && w == 0) {
#pragma unroll
    for (int q = 0; q < N; ++q) {
      T v = T(0);
      for (int c = 0; c < Geo::C; ++c) {
        const T* rr = remote<Geo::CB>(red, c);
        for (int ww = 0; ww < W; ++ww) v += rr[(ww * NSTATE + sidx) * N + q];
      }
      out[q] = v;
    }
  }
  csync<Geo::CB>();
}

template <typename T, int N, int NSL, int ENT>
__global__ void __launch_bounds__(BigGeo<T, N, NSL>::THREADS, 1) pqc_forward_big(PlanDev plan, const cplx<T>* __restrict__ Ug,
                                const uint32_t* __restrict__ perm, const cplx<T>* __restrict__ ph,
                                int n_layers, int scale, int64_t R, const T* __restrict__ act,
                                const T* __restrict__ act_tan, T* __restrict__ z,
                                T* __restrict__ dz, unsigned long long* __restrict__ maxabs) {
  using Gm = BigGeo<T, N, NSL>;
  constexpr int AB = Gm::AB, A = Gm::A, G = Gm::G, TH = Gm::THREADS, LB = Gm::LB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx<T>* buf = (cplx<T>*)smem_raw;                                // [A][TH]
  cplx<T>* sU = buf + (size_t)A * TH;                               // [n_u1][4]
  T* red = (T*)(sU + 4 * plan.n_u1);                                // [W][NSL][N]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int sidx = NSL == 4 ? lane / G : 0, gl = lane & (G - 1);
  int rank = 0;
  if constexpr (Gm::CB > 0) rank = (int)cg::this_cluster().block_rank();
  for (int i = tid; i < 4 * plan.n_u1; i += TH) sU[i] = Ug[i];
  __syncthreads();
  const int64_t cid = blockIdx.x / Gm::C, ncl = gridDim.x / Gm::C;
  const int hi = (rank << (Gm::WB + LB)) | (w << LB) | gl;  // upper index bits of this thread
  T amax = T(0);
  for (int64_t s = cid; s < R; s += ncl) {
    T c[N], sn[N], dth[N], s1[N], s2[N];
    load_point_fast<T, N>(scale, act, act_tan, R, s, true, NSL == 4 ? sidx - 1 : -1, c, sn, dth,
                          s1, s2, amax);
    cplx<T> st[A];
    embed<T, N, AB>(c, sn, dth, sidx > 0, hi, st);
    for (int l = 0; l < n_layers; ++l) {
      layer_fwd<T, Gm>(st, sU + 4 * N * l, buf, tid, rank, w, gl);
      entangle_fwd<T, Gm, ENT>(st, l, buf, tid, rank, w, sidx, gl, perm, ph);
    }
    T out[N], tot = T(0);
#pragma unroll
    for (int q = 0; q < N; ++q) out[q] = T(0);
#pragma unroll
    for (int r = 0; r < A; ++r) {
      T v;
      if constexpr (NSL == 4) {
        const cplx<T> p = {__shfl_sync(0xffffffffu, st[r].re, gl),
                           __shfl_sync(0xffffffffu, st[r].im, gl)};
        v = sidx == 0 ? p.re * p.re + p.im * p.im : T(2) * (p.re * st[r].re + p.im * st[r].im);
      } else {
        v = st[r].re * st[r].re + st[r].im * st[r].im;
      }
      tot += v;
#pragma unroll
      for (int qi = 0; qi < AB; ++qi) {
        if ((r >> (AB - 1 - qi)) & 1) out[N - AB + qi] -= v;
        else out[N - AB + qi] += v;
      }
    }
#pragma unroll
    for (int q = 0; q < N - AB; ++q) out[q] = ((hi >> (N - AB - 1 - q)) & 1) ? -tot : tot;
    reduce_point<T, Gm, NSL, N>(out, red, tid, w, sidx, rank);
    if (rank == 0 && w == 0) {
#pragma unroll
      for (int q = 0; q < N; ++q) {
        if ((q % G) != gl) continue;
        if (sidx == 0) z[s * N + q] = out[q];
        else dz[((int64_t)(sidx - 1) * R + s) * N + q] = out[q];
      }
    }
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, m));
  if (lane == 0 && maxabs) atomic_max_abs(maxabs, amax);
}

// ---- K2 big ------------------------------------------------------------------------------------
template <typename T, int AB>
__device__ __forceinline__ void rot_right(cplx<T> (&v)[1 << AB]) {  // new[r] = old[rotl(r)]
  constexpr int A = 1 << AB;
  cplx<T> t[A];
#pragma unroll
  for (int r = 0; r < A; ++r) t[r] = v[((r << 1) | (r >> (AB - 1))) & (A - 1)];
#pragma unroll
  for (int r = 0; r < A; ++r) v[r] = t[r];
}

// reverse step on register bit 0 (caller rotates the next wire into bit 0)
template <typename T, int A>
__device__ __forceinline__ void gate_bwd_bit0(cplx<T> (&x)[A], cplx<T> (&a)[A], const cplx<T>* U,
                                              T* acc, int lane) {
  const cplx<T> h00 = {U[0].re, -U[0].im}, h01 = {U[2].re, -U[2].im};
  const cplx<T> h10 = {U[1].re, -U[1].im}, h11 = {U[3].re, -U[3].im};
  T m[8] = {T(0), T(0), T(0), T(0), T(0), T(0), T(0), T(0)};
#pragma unroll
  for (int r = 0; r < A; r += 2) {
    const cplx<T> x0 = x[r], x1 = x[r + 1], a0 = a[r], a1 = a[r + 1];
    cmac_c(m[0], m[1], a0, x0);
    cmac_c(m[2], m[3], a0, x1);
    cmac_c(m[4], m[5], a1, x0);
    cmac_c(m[6], m[7], a1, x1);
    x[r] = cmul2(h00, x0, h01, x1);
    x[r + 1] = cmul2(h10, x0, h11, x1);
    a[r] = cmul2(h00, a0, h01, a1);
    a[r + 1] = cmul2(h10, a0, h11, a1);
  }
  const T v = warp_reduce8(m, lane);
  if ((lane & 3) == 0) acc[lane >> 2] += v;
}

// reverse single-qubit step with a partner in another warp / CTA: exchange x and
// a (sequentially through one buffer), un-compute both, accumulate M'
template <typename T, typename Geo, int KIND>  // KIND 0 CTA wire, 1 warp wire, 2 lane wire
__device__ __forceinline__ void gate_bwd_x(cplx<T> (&x)[Geo::A], cplx<T> (&a)[Geo::A],
                                           cplx<T>* buf, int tid, int rank, int mask, bool beta,
                                           const cplx<T>* U, T* acc, int lane) {
  constexpr int A = Geo::A, TH = Geo::THREADS;
  const cplx<T> h00 = {U[0].re, -U[0].im}, h01 = {U[2].re, -U[2].im};
  const cplx<T> h10 = {U[1].re, -U[1].im}, h11 = {U[3].re, -U[3].im};
  const cplx<T> cs = beta ? h11 : h00, cp = beta ? h10 : h01;
  cplx<T> xp[A], ap[A];
  if constexpr (KIND == 2) {
#pragma unroll
    for (int r = 0; r < A; ++r) {
      xp[r] = shfl_xor_c(x[r], mask);
      ap[r] = shfl_xor_c(a[r], mask);
    }
  } else {
    const cplx<T>* src = KIND == 0 ? remote<Geo::CB>(buf, rank ^ mask) : buf;
    const int ptid = KIND == 0 ? tid : (tid ^ (mask << 5));
#pragma unroll
    for (int r = 0; r < A; ++r) buf[r * TH + tid] = x[r];
    if constexpr (KIND == 0) csync<Geo::CB>(); else __syncthreads();
#pragma unroll
    for (int r = 0; r < A; ++r) xp[r] = src[r * TH + ptid];
    if constexpr (KIND == 0) csync<Geo::CB>(); else __syncthreads();
#pragma unroll
    for (int r = 0; r < A; ++r) buf[r * TH + tid] = a[r];
    if constexpr (KIND == 0) csync<Geo::CB>(); else __syncthreads();
#pragma unroll
    for (int r = 0; r < A; ++r) ap[r] = src[r * TH + ptid];
    if constexpr (KIND == 0) csync<Geo::CB>(); else __syncthreads();
  }
  T ms_re = 0, ms_im = 0, mc_re = 0, mc_im = 0;
#pragma unroll
  for (int r = 0; r < A; ++r) {
    cmac_c(ms_re, ms_im, a[r], x[r]);
    cmac_c(mc_re, mc_im, a[r], xp[r]);
    x[r] = cmul2(cs, x[r], cp, xp[r]);
    a[r] = cmul2(cs, a[r], cp, ap[r]);
  }
  T m[8];
  m[0] = beta ? T(0) : ms_re; m[1] = beta ? T(0) : ms_im;
  m[2] = beta ? T(0) : mc_re; m[3] = beta ? T(0) : mc_im;
  m[6] = beta ? ms_re : T(0); m[7] = beta ? ms_im : T(0);
  m[4] = beta ? mc_re : T(0); m[5] = beta ? mc_im : T(0);
  const T v = warp_reduce8(m, lane);
  if ((lane & 3) == 0) acc[lane >> 2] += v;
}

template <typename T, int N, int ENT>
__global__ void __launch_bounds__(BigGeo<T, N, 4, true>::THREADS, 1) pqc_backward_big(PlanDev plan, const cplx<T>* __restrict__ Ug,
                                 const uint32_t* __restrict__ perm, const uint32_t* __restrict__ iperm,
                                 const cplx<T>* __restrict__ ph, int n_layers, int scale, int64_t R,
                                 const T* __restrict__ act, const T* __restrict__ act_tan,
                                 const T* __restrict__ gz, const T* __restrict__ gdz,
                                 T* __restrict__ g_act, T* __restrict__ g_act_tan,
                                 double* __restrict__ partial) {
  using Gm = BigGeo<T, N, 4, true>;
  constexpr int AB = Gm::AB, A = Gm::A, G = Gm::G, TH = Gm::THREADS, LB = Gm::LB, W = Gm::W,
                D = Gm::D;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx<T>* buf = (cplx<T>*)smem_raw;                 // [A][TH]
  cplx<T>* sU = buf + (size_t)A * TH;                // [n_u1][4]
  T* red = (T*)(sU + 4 * plan.n_u1);                 // [W][4][N]
  T* accU = red + W * 4 * N;                         // [W][8 n_u1]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int sidx = lane / G, gl = lane & (G - 1);
  int rank = 0;
  if constexpr (Gm::CB > 0) rank = (int)cg::this_cluster().block_rank();
  for (int i = tid; i < 4 * plan.n_u1; i += TH) sU[i] = Ug[i];
  for (int i = tid; i < W * 8 * plan.n_u1; i += TH) accU[i] = T(0);
  __syncthreads();
  const int64_t cid = blockIdx.x / Gm::C, ncl = gridDim.x / Gm::C;
  const int hi = (rank << (Gm::WB + LB)) | (w << LB) | gl;
  T* myacc = accU + (size_t)w * 8 * plan.n_u1;
  // phase-gradient accumulators p_b of this cluster, natural index order (double)
  double* pacc = partial + (size_t)cid * (8 * plan.n_u1 + (size_t)D * plan.n_phase) + 8 * plan.n_u1;
  if (ENT == ENT_PHASE) {
    for (int i = (rank * TH + tid); i < D * plan.n_phase; i += Gm::C * TH) pacc[i] = 0.0;
  }
  csync<Gm::CB>();
  for (int64_t s = cid; s < R; s += ncl) {
    T c[N], sn[N], dth[N], s1v[N], s2v[N], amax_unused = T(0);
    load_point_fast<T, N>(scale, act, act_tan, R, s, true, sidx - 1, c, sn, dth, s1v, s2v,
                          amax_unused);
    cplx<T> x[A], a[A];
    embed<T, N, AB>(c, sn, dth, sidx > 0, hi, x);
    for (int l = 0; l < n_layers; ++l) {  // forward replay
      layer_fwd<T, Gm>(x, sU + 4 * N * l, buf, tid, rank, w, gl);
      entangle_fwd<T, Gm, ENT>(x, l, buf, tid, rank, w, sidx, gl, perm, ph);
    }
    // seeds
    T gsel[N];
#pragma unroll
    for (int q = 0; q < N; ++q)
      gsel[q] = sidx == 0 ? gz[s * N + q] : gdz[((int64_t)(sidx - 1) * R + s) * N + q];
    T wl = T(0);
#pragma unroll
    for (int q = 0; q < N - AB; ++q) wl += ((hi >> (N - AB - 1 - q)) & 1) ? -gsel[q] : gsel[q];
#pragma unroll
    for (int r = 0; r < A; ++r) {
      T wv = wl;
#pragma unroll
      for (int qi = 0; qi < AB; ++qi)
        wv += ((r >> (AB - 1 - qi)) & 1) ? -gsel[N - AB + qi] : gsel[N - AB + qi];
      wv *= T(2);
      const cplx<T> p = {__shfl_sync(0xffffffffu, x[r].re, gl), __shfl_sync(0xffffffffu, x[r].im, gl)};
      cplx<T> t = {wv * x[r].re, wv * x[r].im};
#pragma unroll
      for (int m = G; m < 4 * G; m <<= 1) {
        t.re += __shfl_xor_sync(0xffffffffu, t.re, m);
        t.im += __shfl_xor_sync(0xffffffffu, t.im, m);
      }
      a[r] = sidx == 0 ? t : cplx<T>{wv * p.re, wv * p.im};
    }
    // reverse sweep
    for (int l = n_layers - 1; l >= 0; --l) {
      if constexpr (ENT == ENT_PERM) {
        gather<T, Gm>(x, buf, tid, rank, w, sidx, gl, iperm + (size_t)l * D);
        gather<T, Gm>(a, buf, tid, rank, w, sidx, gl, iperm + (size_t)l * D);
      } else if constexpr (ENT == ENT_PHASE) {
        const cplx<T>* p = ph + (size_t)l * D;
        double* pa = pacc + (size_t)l * D;
#pragma unroll
        for (int r = 0; r < A; ++r) {
          T pv = a[r].im * x[r].re - a[r].re * x[r].im;
#pragma unroll
          for (int mk = G; mk < 4 * G; mk <<= 1) pv += __shfl_xor_sync(0xffffffffu, pv, mk);
          if (sidx == 0) pa[((hi << AB) | r)] += (double)pv;  // natural index b
          const cplx<T> pe = p[((rank * W + w) * A + r) * G + gl];
          const cplx<T> e = {pe.re, -pe.im};
          x[r] = cmul(x[r], e);
          a[r] = cmul(a[r], e);
        }
      }
      const cplx<T>* Ul = sU + 4 * N * l;
      T* accl = myacc + 8 * N * l;
      // register wires, last first: rotate right so wire N-1-i sits at bit 0
      for (int i = 0; i < AB; ++i) {
        const int q = N - 1 - i;
        gate_bwd_bit0<T, A>(x, a, Ul + 4 * q, accl + 8 * q, lane);
        rot_right<T, AB>(x);
        rot_right<T, AB>(a);
      }
      for (int qq = LB - 1; qq >= 0; --qq) {
        const int q = Gm::CB + Gm::WB + qq;
        const int lm = 1 << (LB - 1 - qq);
        gate_bwd_x<T, Gm, 2>(x, a, buf, tid, rank, lm, gl & lm, Ul + 4 * q, accl + 8 * q, lane);
      }
      for (int qq = Gm::WB - 1; qq >= 0; --qq) {
        const int q = Gm::CB + qq;
        const int m = 1 << (Gm::WB - 1 - qq);
        gate_bwd_x<T, Gm, 1>(x, a, buf, tid, rank, m, w & m, Ul + 4 * q, accl + 8 * q, lane);
      }
      for (int q = Gm::CB - 1; q >= 0; --q) {
        const int m = 1 << (Gm::CB - 1 - q);
        gate_bwd_x<T, Gm, 0>(x, a, buf, tid, rank, m, rank & m, Ul + 4 * q, accl + 8 * q, lane);
      }
    }
    // embedding gradient: x <- phi (closed form); a = phibar (state 0) or mu_k.
    // rho = sum_q dth_q X_q a (own state's tangent row; zero in state-0 lanes)
    embed<T, N, AB>(c, sn, dth, false, hi, x);
    cplx<T> rho[A];
#pragma unroll
    for (int r = 0; r < A; ++r) rho[r] = {T(0), T(0)};
    {
      cplx<T> ap[A];
      for (int q = 0; q < Gm::CB; ++q) {  // CTA wires: partner via DSMEM
        exchange_read<T, Gm, true>(a, ap, buf, tid, rank, 1 << (Gm::CB - 1 - q));
#pragma unroll
        for (int r = 0; r < A; ++r) { rho[r].re += dth[q] * ap[r].re; rho[r].im += dth[q] * ap[r].im; }
      }
      for (int q = 0; q < Gm::WB; ++q) {  // warp wires: partner via shared memory
        exchange_read<T, Gm, false>(a, ap, buf, tid, rank, 1 << (Gm::WB - 1 - q));
        const T d = dth[Gm::CB + q];
#pragma unroll
        for (int r = 0; r < A; ++r) { rho[r].re += d * ap[r].re; rho[r].im += d * ap[r].im; }
      }
      for (int q = 0; q < LB; ++q) {  // lane wires
        const int lm = 1 << (LB - 1 - q);
        const T d = dth[Gm::CB + Gm::WB + q];
#pragma unroll
        for (int r = 0; r < A; ++r) {
          const cplx<T> p = shfl_xor_c(a[r], lm);
          rho[r].re += d * p.re;
          rho[r].im += d * p.im;
        }
      }
#pragma unroll
      for (int qi = 0; qi < AB; ++qi) {  // register wires
        const int S = 1 << (AB - 1 - qi);
        const T d = dth[N - AB + qi];
#pragma unroll
        for (int r = 0; r < A; ++r) { rho[r].re += d * a[r ^ S].re; rho[r].im += d * a[r ^ S].im; }
      }
    }
    // gt[q] = Re<(i/2) phibar - 1/4 sum_k rho_k, X_q phi>,  gd[q] = Re<(i/2) mu_k, X_q phi>
    T gt[N], gd[N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
      gt[q] = T(0);
      gd[q] = T(0);
      cplx<T> y[A];
      constexpr int nh = N - AB;
      if (q >= nh) {
#pragma unroll
        for (int r = 0; r < A; ++r) y[r] = x[r ^ (1 << (N - 1 - q))];
      } else {
        embed<T, N, AB>(c, sn, dth, false, hi ^ (1 << (nh - 1 - q)), y);
      }
#pragma unroll
      for (int r = 0; r < A; ++r) {
        const T half = T(0.5) * (a[r].re * y[r].im - a[r].im * y[r].re);
        if (sidx == 0) gt[q] += half;
        else {
          gt[q] -= T(0.25) * (rho[r].re * y[r].re + rho[r].im * y[r].im);
          gd[q] += half;
        }
      }
    }
    reduce_point<T, Gm, 4, N>(gt, red, tid, w, sidx, rank);
    reduce_point<T, Gm, 4, N>(gd, red, tid, w, sidx, rank);
    if (rank == 0 && w == 0) {
      T gtot[N], gk[3][N];
#pragma unroll
      for (int q = 0; q < N; ++q) {
        T v = gt[q];
#pragma unroll
        for (int m = G; m < 4 * G; m <<= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
        gtot[q] = v;
#pragma unroll
        for (int k = 0; k < 3; ++k) gk[k][q] = __shfl_sync(0xffffffffu, gd[q], (k + 1) * G + gl);
      }
#pragma unroll
      for (int q = 0; q < N; ++q) {
        if ((q % G) != gl) continue;
        if (sidx == 0) {
          T ga = gtot[q] * s1v[q];
#pragma unroll
          for (int k = 0; k < 3; ++k) ga += gk[k][q] * s2v[q] * act_tan[((int64_t)k * R + s) * N + q];
          g_act[s * N + q] = ga;
        } else {
          g_act_tan[((int64_t)(sidx - 1) * R + s) * N + q] = gd[q] * s1v[q];
        }
      }
    }
  }
  // u1 partials: warps (fixed order) -> this CTA (double, smem) -> cluster rank order
  __syncthreads();
  double* dacc = (double*)buf;  // the exchange buffer is free now
  for (int i = tid; i < 8 * plan.n_u1; i += TH) {
    double v = 0.0;
    for (int ww = 0; ww < W; ++ww) v += (double)accU[(size_t)ww * 8 * plan.n_u1 + i];
    dacc[i] = v;
  }
  csync<Gm::CB>();
  if (rank == 0) {
    double* row = partial + (size_t)cid * (8 * plan.n_u1 + (size_t)D * plan.n_phase);
    for (int i = tid; i < 8 * plan.n_u1; i += TH) {
      double v = 0.0;
      for (int cc = 0; cc < Gm::C; ++cc) v += remote<Gm::CB>(dacc, cc)[i];
      row[i] = v;
    }
  }
  csync<Gm::CB>();
}

// ---- launchers -------------------------------------------------------------------------------
template <typename T, int N, int NSL, bool BWD>
static size_t big_smem(const PlanDev& p, bool bwd) {
  using Gm = BigGeo<T, N, NSL, BWD>;
  size_t o = sizeof(cplx<T>) * Gm::A * Gm::THREADS + sizeof(cplx<T>) * 4 * p.n_u1;
  o += sizeof(T) * Gm::W * NSL * N;
  if (bwd) o += sizeof(T) * Gm::W * 8 * p.n_u1;
  return align_up(o, 16);
}

struct BigTables {
  void* U;
  uint32_t* perm;
  uint32_t* iperm;
  void* ph;
};

template <typename T, int N>
static BigTables big_tables(const qpinn_circuit* c, unsigned char* base) {
  const size_t D = (size_t)1 << N;
  BigTables t;
  size_t o = 0;
  t.U = base + o; o = align_up(o + sizeof(cplx<T>) * 4 * c->n_u1, 256);
  t.perm = (uint32_t*)(base + o); o = align_up(o + 4 * D * c->n_perm, 256);
  t.iperm = (uint32_t*)(base + o); o = align_up(o + 4 * D * c->n_perm, 256);
  t.ph = base + o;
  return t;
}

template <typename K, typename... Args>
static int launch_cluster(K kern, int grid, int threads, size_t smem, int C, cudaStream_t st,
                          Args... args) {
  QPINN_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (C > 8) QPINN_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  QPINN_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, args...));
  return QPINN_OK;
}

template <typename T, int N, int NSL, bool BWD>
static int big_cluster_count(void* kern, size_t smem, int64_t R) {
  using Gm = BigGeo<T, N, NSL, BWD>;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Gm::THREADS, smem);
  if (occ < 1) occ = 1;
  int64_t clusters = ((int64_t)num_sms() * occ) / Gm::C;
  if (clusters < 1) clusters = 1;
  if (clusters > R) clusters = R;
  return (int)clusters;
}

template <typename T, int N, int ENT>
static int big_fwd(const qpinn_circuit* c, const KArgs<T>* a) {
  constexpr int NSL = 4;
  using Gm = BigGeo<T, N, NSL>;
  const PlanDev& p = c->dev;
  BigTables tb = big_tables<T, N>(c, a->tables);
  big_prepare<T, N, NSL><<<64, 256, 0, a->stream>>>(p, a->qp, (cplx<T>*)tb.U, tb.perm, (cplx<T>*)tb.ph);
  QPINN_CUDA_CHECK(cudaGetLastError());
  const size_t smem = big_smem<T, N, NSL, false>(p, false);
  if (smem > 227 * 1024) return fail(QPINN_ERR_CAPACITY, "big PQC kernel exceeds shared memory");
  auto kern = pqc_forward_big<T, N, NSL, ENT>;
  QPINN_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int ncl = big_cluster_count<T, N, NSL, false>((void*)kern, smem, a->R);
  const T* tan = a->tan;
  T* dz = a->dz;
  return launch_cluster(kern, ncl * Gm::C, Gm::THREADS, smem, Gm::C, a->stream, p,
                        (const cplx<T>*)tb.U, (const uint32_t*)tb.perm, (const cplx<T>*)tb.ph,
                        c->L, a->scale, a->R, a->act, tan, a->z, dz, a->maxabs);
}

template <typename T, int N, int ENT>
static int big_bwd(const qpinn_circuit* c, const KArgs<T>* a) {
  using Gm = BigGeo<T, N, 4, true>;
  const PlanDev& p = c->dev;
  BigTables tb = big_tables<T, N>(c, a->tables);
  big_prepare<T, N, 4, true><<<64, 256, 0, a->stream>>>(p, a->qp, (cplx<T>*)tb.U, tb.perm,
                                                        (cplx<T>*)tb.ph);
  QPINN_CUDA_CHECK(cudaGetLastError());
  if (c->n_perm) {  // inverse tables: layout-ordered sources of the inverse permutation
    big_prepare_inverse<T, N, 4, true><<<64, 256, 0, a->stream>>>(p, tb.iperm);
    QPINN_CUDA_CHECK(cudaGetLastError());
  }
  const size_t smem = big_smem<T, N, 4, true>(p, true);
  if (smem > 227 * 1024) return fail(QPINN_ERR_CAPACITY, "big PQC kernel exceeds shared memory");
  auto kern = pqc_backward_big<T, N, ENT>;
  QPINN_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int ncl = big_cluster_count<T, N, 4, true>((void*)kern, smem, a->R);
  if (int rc = launch_cluster(kern, ncl * Gm::C, Gm::THREADS, smem, Gm::C, a->stream, p,
                              (const cplx<T>*)tb.U, (const uint32_t*)tb.perm,
                              (const uint32_t*)tb.iperm, (const cplx<T>*)tb.ph, c->L, a->scale,
                              a->R, a->act, a->tan, a->gz, a->gdz, a->g_act, a->g_tan, a->partial))
    return rc;
  return pqc_finish_grads_ab<T>(c, ncl, a, c->n);  // phase accumulators in natural order
}

template <typename T, int N>
int big_n(bool fwd, int ent, const qpinn_circuit* c, const KArgs<T>* a) {
  if (fwd) {
    if (!a->tan) return fail(QPINN_ERR_CAPACITY, "value-only evaluation needs n <= 8");
    if (ent == ENT_PERM) return big_fwd<T, N, ENT_PERM>(c, a);
    if (ent == ENT_PHASE) return big_fwd<T, N, ENT_PHASE>(c, a);
    return big_fwd<T, N, ENT_NONE>(c, a);
  }
  if constexpr (BigGeo<T, N, 4, true>::CB <= 4) {
    if (ent == ENT_PERM) return big_bwd<T, N, ENT_PERM>(c, a);
    if (ent == ENT_PHASE) return big_bwd<T, N, ENT_PHASE>(c, a);
    return big_bwd<T, N, ENT_NONE>(c, a);
  }
  return fail(QPINN_ERR_CAPACITY, "adjoint beyond the cluster-resident range (HBM regime)");
}

}  // namespace qpinn
