// Layer-loop K1 / K2: the production PQC kernels for every ansatz.
//
// All six ansatze of build_circuit (ansatz.py:178-204) have the same layer
// shape after fusion (ansatz.py:117-156): one single-qubit step (Rot, RX or
// the fused RX.RZ) on each wire 0..n-1 in order, then at most one entangler
// step, a CNOT-run permutation (basic, strongly, cross_mesh_cnot) or a CRZ-mesh
// phase diagonal (cross_mesh, cross_mesh_2rot).  These kernels loop over the
// layers at run time and unroll the wires at compile time: the wire ->
// lane/register mapping, shuffle masks and register pairings are constants,
// there is no per-gate dispatch and the loop-carried state only has to be
// re-homed once per layer.  The body stays ~20 KB of SASS, inside the L1.5
// instruction cache (a fully unrolled circuit does not: warps then stall on
// instruction fetch).  Numerics, lane geometry and the deterministic
// reductions are those of the generic kernels in pqc.cu, which remain the
// cross-check (kernel variant 1).  The hand-off differs: K1 stores the state
// at every layer boundary (after the single-qubit gates), so K2 never
// un-computes the state and only propagates the adjoint (see K2).
#include "pqc_layer.h"

namespace qpinn {

template <typename T>
__device__ __forceinline__ cplx<T> conj(cplx<T> a) {
  return {a.re, -a.im};
}

// post-gate outer product M'_ij = sum conj(a_i) x_j of the single-qubit step on
// the wire held by register bit RB, summed over the warp into acc[0..7]
template <typename T, int A, int RB>
__device__ __forceinline__ void outer_reg(const cplx<T> (&x)[A], const cplx<T> (&a)[A],
                                          T* __restrict__ acc, int lane) {
  constexpr int S = 1 << RB;
  T m[8] = {T(0), T(0), T(0), T(0), T(0), T(0), T(0), T(0)};
#pragma unroll
  for (int r = 0; r < A; ++r) {
    if (r & S) continue;
    const int r1 = r | S;
    cmac_c(m[0], m[1], a[r], x[r]);
    cmac_c(m[2], m[3], a[r], x[r1]);
    cmac_c(m[4], m[5], a[r1], x[r]);
    cmac_c(m[6], m[7], a[r1], x[r1]);
  }
  const T v = warp_reduce8(m, lane);
  if ((lane & 3) == 0) acc[lane >> 2] += v;
}

// the same for a lane wire (run-time lane mask lm: one code copy serves all
// lane wires, which keeps K2's hot loop inside the instruction cache)
template <typename T, int A>
__device__ __forceinline__ void outer_lane(const cplx<T> (&x)[A], const cplx<T> (&a)[A],
                                           T* __restrict__ acc, int lm, int gl, int lane) {
  const bool beta = gl & lm;
  T ms_re = 0, ms_im = 0, mc_re = 0, mc_im = 0;
#pragma unroll
  for (int r = 0; r < A; ++r) {
    const cplx<T> xp = shfl_xor_c(x[r], lm);
    cmac_c(ms_re, ms_im, a[r], x[r]);
    cmac_c(mc_re, mc_im, a[r], xp);
  }
  // own row i: beta = 0 -> M'(0,0), M'(0,1); beta = 1 -> M'(1,1), M'(1,0)
  T m[8];
  m[0] = beta ? T(0) : ms_re; m[1] = beta ? T(0) : ms_im;
  m[2] = beta ? T(0) : mc_re; m[3] = beta ? T(0) : mc_im;
  m[6] = beta ? ms_re : T(0); m[7] = beta ? ms_im : T(0);
  m[4] = beta ? mc_re : T(0); m[5] = beta ? mc_im : T(0);
  const T v = warp_reduce8(m, lane);
  if ((lane & 3) == 0) acc[lane >> 2] += v;
}

// new[r] = old[r with its high and low AB/2-bit halves swapped] (an involution)
template <typename T, int AB>
__device__ __forceinline__ void swap_halves(cplx<T> (&v)[1 << AB]) {
  constexpr int A = 1 << AB, H = AB / 2, HM = (1 << H) - 1;
  cplx<T> t[A];
#pragma unroll
  for (int r = 0; r < A; ++r) t[r] = v[((r & HM) << H) | (r >> H)];
#pragma unroll
  for (int r = 0; r < A; ++r) v[r] = t[r];
}

// new[r] = old[rotr(r)]: after AB rotations the layout is back to the original
template <typename T, int AB>
__device__ __forceinline__ void rotate_regs_left(cplx<T> (&v)[1 << AB]) {
  constexpr int A = 1 << AB;
  cplx<T> t[A];
#pragma unroll
  for (int r = 0; r < A; ++r) t[r] = v[((r >> 1) | ((r & 1) << (AB - 1))) & (A - 1)];
#pragma unroll
  for (int r = 0; r < A; ++r) v[r] = t[r];
}

// reduce-scatter of K values over the lanes that differ in mask bits M, M/2, .., G:
// at each level a lane keeps the half its mask bit selects and adds the
// partner's copy of it; the survivors (sums over all those lanes) go to
// acc[(rbase + i) G + gl]
template <int M, int G, typename T, int K>
__device__ __forceinline__ void reduce_scatter_acc(const T (&v)[K], int lane, T* __restrict__ acc,
                                                   int gl, int rbase) {
  if constexpr (M < G) {
#pragma unroll
    for (int i = 0; i < K; ++i) acc[(rbase + i) * G + gl] += v[i];
  } else {
    static_assert(K >= 2, "reduce-scatter needs at least two values per level");
    const bool up = lane & M;
    T nv[K / 2];
#pragma unroll
    for (int i = 0; i < K / 2; ++i) {
      const T send = up ? v[i] : v[i + K / 2];
      const T keep = up ? v[i + K / 2] : v[i];
      nv[i] = keep + __shfl_xor_sync(0xffffffffu, send, M);
    }
    reduce_scatter_acc<M / 2, G, T, K / 2>(nv, lane, acc, gl, rbase + (up ? K / 2 : 0));
  }
}

// K1 -> K2 hand-off: the 4 states of point s after the single-qubit gates of
// layer l (before its entangler), register pairs innermost so that one
// 16-byte (fp32) store / load per lane moves two amplitudes and a warp
// instruction touches 32 consecutive pairs:
//   states[(((s L + l) A/2 + r/2) 4G + sidx G + gl) 2 + (r & 1)]
template <int G, int A>
__device__ __forceinline__ int64_t boundary_offset(int64_t s, int n_layers, int l) {
  return ((s * n_layers + l) * (A / 2)) * (4 * G) * 2;
}
__device__ __forceinline__ void st_pair(cplx<float>* p, cplx<float> a, cplx<float> b) {
  *reinterpret_cast<float4*>(p) = make_float4(a.re, a.im, b.re, b.im);
}
__device__ __forceinline__ void st_pair(cplx<double>* p, cplx<double> a, cplx<double> b) {
  p[0] = a;
  p[1] = b;
}
__device__ __forceinline__ void ld_pair(const cplx<float>* p, cplx<float>& a, cplx<float>& b) {
  const float4 v = __ldg(reinterpret_cast<const float4*>(p));
  a = {v.x, v.y};
  b = {v.z, v.w};
}
__device__ __forceinline__ void ld_pair(const cplx<double>* p, cplx<double>& a,
                                        cplx<double>& b) {
  const double2 u = __ldg(reinterpret_cast<const double2*>(p));
  const double2 v = __ldg(reinterpret_cast<const double2*>(p + 1));
  a = {u.x, u.y};
  b = {v.x, v.y};
}

#ifndef QPINN_K1_MINB
#define QPINN_K1_MINB 5
#endif
#ifndef QPINN_K2_MINB
#define QPINN_K2_MINB 2
#endif

// ---- K1 -----------------------------------------------------------------------------------
template <typename T, int N, int NSL, int ENT>
__global__ void __launch_bounds__(kThreads, sizeof(T) == 4 && N <= 7 ? QPINN_K1_MINB : 1)
pqc_forward_layer(PlanDev plan, const unsigned char* __restrict__ tables, int n_layers, int scale,
                  int64_t R, const T* __restrict__ act, const T* __restrict__ act_tan,
                  const T* __restrict__ qp, T* __restrict__ z,
                  T* __restrict__ dz, cplx<T>* __restrict__ states,
                  unsigned long long* __restrict__ maxabs, cplx<T>* __restrict__ coh) {
  using Gm = Geo<T, N, NSL>;
  constexpr int AB = Gm::AB, A = Gm::A, LB = Gm::LB, G = Gm::G, LPP = Gm::LPP, SPW = Gm::SPW,
                D = Gm::D;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warps = blockDim.x >> 5;
  Smem<T> sm;
  smem_layout<T, N, AB>(plan, warps, false, &sm, smem_raw);
  copy_tables<T>(tables, table_bytes<T, N>(plan, false), smem_raw, sm.acc, 0);
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pw = lane / LPP, sidx = (lane / G) % NSL, gl = lane & (G - 1);
  const int lane_hi = lane >> LB;
  const int psi_lane = pw * LPP + gl;
  cplx<T>* buf = sm.buf + warp * 32 * A;
  T amax = T(0);
  const int64_t per_block = (int64_t)warps * SPW;
  const int64_t stride = (int64_t)gridDim.x * per_block;
  for (int64_t base = (int64_t)blockIdx.x * per_block; base < R; base += stride) {
    const int64_t s = base + warp * SPW + pw;
    const bool valid = s < R;
    T c[N], sn[N], dth[N], s1[N], s2[N];
    load_point_lanes<T, N, LPP>(scale, act, act_tan, R, s, valid, sidx - 1, lane, c, sn, dth, s1, s2,
                                amax);
    cplx<T> st[1][A];
    embed<T, N, AB>(c, sn, dth, sidx > 0, gl, st[0]);
    for (int l = 0; l < n_layers; ++l) {
      const cplx<T>* Ul = sm.U + 4 * N * l;
      for (int q = 0; q < LB; ++q) {  // lane wires, one shared copy
        const int lb = LB - 1 - q;
        const cplx<T>* U = Ul + 4 * q;
        gate_lane<T, A, 1>(st, 1 << lb, (gl >> lb) & 1, U[0], U[1], U[2], U[3]);
      }
      // register wires LB .. N-1 (bits AB-1 .. 0).  Gates of one layer commute,
      // so with AB = 4 two gate copies (bits 3, 2) plus a half-swap of
      // the register index cover all wires: fewer moves than single-bit rotation
      // and far less code than unrolling every wire.
#ifndef QPINN_K1_UNROLL_REG
#define QPINN_K1_UNROLL_REG 0
#endif
      if constexpr (AB == 4 && QPINN_K1_UNROLL_REG) {  // every register wire its own copy
        static_for<0, AB>([&](auto qi_) {
          constexpr int qi = decltype(qi_)::value;
          const cplx<T>* U = Ul + 4 * (LB + qi);
          gate_reg<AB - 1 - qi, T, A, 1>(st, U[0], U[1], U[2], U[3]);
        });
      } else if constexpr (AB == 4) {
        for (int i = 0; i < AB; i += 2) {
          const cplx<T>* U = Ul + 4 * (LB + i);
          gate_reg<AB - 1, T, A, 1>(st, U[0], U[1], U[2], U[3]);
          gate_reg<AB - 2, T, A, 1>(st, U[4], U[5], U[6], U[7]);
          swap_halves<T, AB>(st[0]);
        }
      } else {
        for (int i = 0; i < AB; ++i) {
          const cplx<T>* U = Ul + 4 * (LB + i);
          gate_reg<AB - 1, T, A, 1>(st, U[0], U[1], U[2], U[3]);
          if constexpr (AB > 1) rotate_regs_left<T, AB>(st[0]);
        }
      }
      if (NSL == 4 && states != nullptr && valid) {  // layer-boundary hand-off for K2
        cplx<T>* sp = states + boundary_offset<G, A>(s, n_layers, l) + 2 * (sidx * G + gl);
#pragma unroll
        for (int r = 0; r < A; r += 2) st_pair(sp + r * 4 * G, st[0][r], st[0][r + 1]);
      }
      if constexpr (ENT == ENT_PERM) {
        permute<T, A, G, 1>(st, sm.pt + l * D, buf, gl, lane_hi);
      } else if constexpr (ENT == ENT_PHASE) {
        const cplx<T>* ph = sm.ph + l * D;
#pragma unroll
        for (int r = 0; r < A; ++r) st[0][r] = cmul(st[0][r], ph[r * G + gl]);
      }
    }
    T out[N], tot = T(0);
#pragma unroll
    for (int q = 0; q < N; ++q) out[q] = T(0);
#pragma unroll
    for (int r = 0; r < A; ++r) {
      T v;
      if constexpr (NSL == 4) {
        const cplx<T> p = {__shfl_sync(0xffffffffu, st[0][r].re, psi_lane),
                           __shfl_sync(0xffffffffu, st[0][r].im, psi_lane)};
        v = sidx == 0 ? p.re * p.re + p.im * p.im
                      : T(2) * (p.re * st[0][r].re + p.im * st[0][r].im);
      } else {
        v = st[0][r].re * st[0][r].re + st[0][r].im * st[0][r].im;
      }
      tot += v;
#pragma unroll
      for (int qi = 0; qi < AB; ++qi) {
        if ((r >> (AB - 1 - qi)) & 1) out[LB + qi] -= v;
        else out[LB + qi] += v;
      }
    }
#pragma unroll
    for (int q = 0; q < LB; ++q) out[q] = ((gl >> (LB - 1 - q)) & 1) ? -tot : tot;
#pragma unroll
    for (int m = 1; m < G; m <<= 1)
#pragma unroll
      for (int q = 0; q < N; ++q) out[q] += __shfl_xor_sync(0xffffffffu, out[q], m);
    if (valid) {
#pragma unroll
      for (int q = 0; q < N; ++q) {
        if ((q % G) != gl) continue;
        if (sidx == 0) z[s * N + q] = out[q];
        else dz[((int64_t)(sidx - 1) * R + s) * N + q] = out[q];
      }
    }
    if constexpr (NSL == 1) {
      // Meyer-Wallach probe (qsim.py:384-406): rho_k's coherence
      // c_k = sum_{b: bit_k = 0} psi_b conj(psi_{b ^ bit_k}); its diagonal is (1 +- z_k)/2
      if (coh != nullptr) {
        T cre[N], cim[N];
#pragma unroll
        for (int q = 0; q < N; ++q) cre[q] = cim[q] = T(0);
        static_for<0, AB>([&](auto rb_) {
          constexpr int RB = decltype(rb_)::value, S = 1 << RB, q = N - 1 - RB;
#pragma unroll
          for (int r = 0; r < A; ++r) {
            if (r & S) continue;
            const cplx<T> a = st[0][r], b = st[0][r | S];
            cre[q] += a.re * b.re + a.im * b.im;
            cim[q] += a.im * b.re - a.re * b.im;
          }
        });
#pragma unroll
        for (int q = 0; q < LB; ++q) {
          const int lm = 1 << (LB - 1 - q);
          const T w = (gl & lm) ? T(0) : T(1);
#pragma unroll
          for (int r = 0; r < A; ++r) {
            const cplx<T> a = st[0][r], b = shfl_xor_c(st[0][r], lm);
            cre[q] += w * (a.re * b.re + a.im * b.im);
            cim[q] += w * (a.im * b.re - a.re * b.im);
          }
        }
#pragma unroll
        for (int m = 1; m < G; m <<= 1)
#pragma unroll
          for (int q = 0; q < N; ++q) {
            cre[q] += __shfl_xor_sync(0xffffffffu, cre[q], m);
            cim[q] += __shfl_xor_sync(0xffffffffu, cim[q], m);
          }
        if (valid && gl == 0)
#pragma unroll
          for (int q = 0; q < N; ++q) coh[s * N + q] = cplx<T>{cre[q], cim[q]};
      }
    }
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, m));
  if (lane == 0 && maxabs) atomic_max_abs(maxabs, amax);
}

// ---- K2 -----------------------------------------------------------------------------------
template <typename T, int N, int ENT>
__global__ void __launch_bounds__(kThreads, sizeof(T) == 4 && N <= 7 ? QPINN_K2_MINB : 1)
pqc_backward_layer(PlanDev plan, const unsigned char* __restrict__ tables, int n_layers,
                   int scale, int64_t R, const T* __restrict__ act,
                   const T* __restrict__ act_tan, const T* __restrict__ qp,
                   const cplx<T>* __restrict__ states, const T* __restrict__ gz,
                   const T* __restrict__ gdz, T* __restrict__ g_act, T* __restrict__ g_act_tan,
                   double* __restrict__ partial) {
  using Gm = Geo<T, N, 4>;
  constexpr int AB = Gm::AB, A = Gm::A, LB = Gm::LB, G = Gm::G, LPP = Gm::LPP, SPW = Gm::SPW,
                D = Gm::D;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warps = blockDim.x >> 5;
  Smem<T> sm;
  smem_layout<T, N, AB>(plan, warps, true, &sm, smem_raw);
  copy_tables<T>(tables, table_bytes<T, N>(plan, true), smem_raw, sm.acc,
                 (size_t)warps * (8 * plan.n_u1 + (size_t)D * plan.n_phase));
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pw = lane / LPP, sidx = (lane / G) % 4, gl = lane & (G - 1);
  const int lane_hi = lane >> LB;
  const int psi_lane = pw * LPP + gl;
  cplx<T>* buf = sm.buf + warp * 2 * 32 * A;
  const int n_acc = 8 * plan.n_u1 + D * plan.n_phase;
  T* accU = sm.acc + (size_t)warp * n_acc;
  T* accP = accU + 8 * plan.n_u1;
  const int64_t per_block = (int64_t)warps * SPW;
  const int64_t stride = (int64_t)gridDim.x * per_block;
  for (int64_t base = (int64_t)blockIdx.x * per_block; base < R; base += stride) {
    const int64_t s = base + warp * SPW + pw;
    const bool valid = s < R;
    cplx<T> xa[2][A];  // [0] this lane's layer-boundary state, [1] its adjoint
    cplx<T>(&x1)[1][A] = reinterpret_cast<cplx<T>(&)[1][A]>(xa[0]);
    cplx<T>(&a1)[1][A] = reinterpret_cast<cplx<T>(&)[1][A]>(xa[1]);
    const cplx<T>* sp0 =
        states + boundary_offset<G, A>(valid ? s : 0, n_layers, 0) + 2 * (sidx * G + gl);
    auto load_boundary = [&](int l) {
      const cplx<T>* sp = sp0 + (int64_t)l * (4 * D);
#pragma unroll
      for (int r = 0; r < A; r += 2) {
        ld_pair(sp + r * 4 * G, xa[0][r], xa[0][r + 1]);
        if (!valid) xa[0][r] = xa[0][r + 1] = cplx<T>{T(0), T(0)};
      }
    };
    // final state = last entangler applied to the last boundary
    load_boundary(n_layers - 1);
    if constexpr (ENT == ENT_PERM) {
      permute<T, A, G, 1>(x1, sm.pt + (n_layers - 1) * D, buf, gl, lane_hi);
    } else if constexpr (ENT == ENT_PHASE) {
      const cplx<T>* ph = sm.ph + (n_layers - 1) * D;
#pragma unroll
      for (int r = 0; r < A; ++r) xa[0][r] = cmul(xa[0][r], ph[r * G + gl]);
    }
    // adjoint seeds: lambda = 2 w psi + 2 sum_k v_k dpsi_k, mu_k = 2 v_k psi
    T gsel[N];
#pragma unroll
    for (int q = 0; q < N; ++q)
      gsel[q] = !valid ? T(0) : sidx == 0 ? gz[s * N + q]
                                          : gdz[((int64_t)(sidx - 1) * R + s) * N + q];
    T wl = T(0);
#pragma unroll
    for (int q = 0; q < LB; ++q) wl += ((gl >> (LB - 1 - q)) & 1) ? -gsel[q] : gsel[q];
#pragma unroll
    for (int r = 0; r < A; ++r) {
      T w = wl;
#pragma unroll
      for (int qi = 0; qi < AB; ++qi)
        w += ((r >> (AB - 1 - qi)) & 1) ? -gsel[LB + qi] : gsel[LB + qi];
      w *= T(2);
      const cplx<T> p = {__shfl_sync(0xffffffffu, xa[0][r].re, psi_lane),
                         __shfl_sync(0xffffffffu, xa[0][r].im, psi_lane)};
      cplx<T> t = {w * xa[0][r].re, w * xa[0][r].im};
#pragma unroll
      for (int m = G; m < 4 * G; m <<= 1) {
        t.re += __shfl_xor_sync(0xffffffffu, t.re, m);
        t.im += __shfl_xor_sync(0xffffffffu, t.im, m);
      }
      xa[1][r] = sidx == 0 ? t : cplx<T>{w * p.re, w * p.im};
    }
    // reverse sweep over layers
    // Single-qubit gates of one layer act on distinct wires and commute, so
    // each may be taken as the layer's last: its post-gate state is the stored
    // boundary x_l and its post-gate adjoint the adjoint a_l at that boundary.
    // Every M'_q of the layer is then an outer product of (a_l, x_l) and only
    // the adjoint is propagated (a <- U_q^dagger a); no state is un-computed.
    for (int l = n_layers - 1; l >= 0; --l) {
      load_boundary(l);
      if constexpr (ENT == ENT_PERM) {
        permute<T, A, G, 1>(a1, sm.pti + l * D, buf, gl, lane_hi);
      } else if constexpr (ENT == ENT_PHASE) {
        const cplx<T>* ph = sm.ph + l * D;
        T* acc = accP + l * D;
        if constexpr (A >= 32 / G) {
          // the D-wide phase gradient summed over the lanes sharing gl by a
          // reduce-scatter: every lane ends up owning A / (32 / G) sums
          T pv[A];
#pragma unroll
          for (int r = 0; r < A; ++r) {
            const cplx<T> e = ph[r * G + gl];
            const cplx<T> xp = cmul(xa[0][r], e);  // post-entangler state
            pv[r] = xa[1][r].im * xp.re - xa[1][r].re * xp.im;
            xa[1][r] = cmul(xa[1][r], cplx<T>{e.re, -e.im});
          }
          reduce_scatter_acc<16, G, T, A>(pv, lane, acc, gl, 0);
        } else {
#pragma unroll
          for (int r = 0; r < A; ++r) {
            const cplx<T> e = ph[r * G + gl];
            const cplx<T> xp = cmul(xa[0][r], e);
            T pv = xa[1][r].im * xp.re - xa[1][r].re * xp.im;
#pragma unroll
            for (int mk = G; mk < 32; mk <<= 1) pv += __shfl_xor_sync(0xffffffffu, pv, mk);
            if (lane_hi == 0) acc[r * G + gl] += pv;
            xa[1][r] = cmul(xa[1][r], cplx<T>{e.re, -e.im});
          }
        }
      }
      const cplx<T>* Ul = sm.U + 4 * N * l;
      T* accl = accU + 8 * N * l;
      // outer products: register wires (compile-time pairings), then lane wires
      static_for<0, AB>([&](auto rb_) {
        constexpr int RB = decltype(rb_)::value;
        outer_reg<T, A, RB>(xa[0], xa[1], accl + 8 * (N - 1 - RB), lane);
      });
      for (int q = 0; q < LB; ++q)
        outer_lane<T, A>(xa[0], xa[1], accl + 8 * q, 1 << (LB - 1 - q), gl, lane);
      // adjoint propagation through every U_q^dagger
      static_for<0, AB>([&](auto rb_) {
        constexpr int RB = decltype(rb_)::value;
        const cplx<T>* U = Ul + 4 * (N - 1 - RB);
        gate_reg<RB, T, A, 1>(a1, conj(U[0]), conj(U[2]), conj(U[1]), conj(U[3]));
      });
      for (int q = 0; q < LB; ++q) {
        const cplx<T>* U = Ul + 4 * q;
        const int lb = LB - 1 - q;
        gate_lane<T, A, 1>(a1, 1 << lb, (gl >> lb) & 1, conj(U[0]), conj(U[2]), conj(U[1]),
                           conj(U[3]));
      }
    }
    // embedding gradient: xa[1] = phibar (s = 0) or mu_k (s = k+1); the point's
    // angles are loaded only now, so they are not live across the layer loop
    T c[N], sn[N], dth[N], s1v[N], s2v[N], amax_unused = T(0);
    load_point_lanes<T, N, LPP>(scale, act, act_tan, R, s, valid, sidx - 1, lane, c, sn, dth,
                                s1v, s2v, amax_unused);
    embed<T, N, AB>(c, sn, dth, false, gl, xa[0]);
    cplx<T> rho[A];
#pragma unroll
    for (int r = 0; r < A; ++r) rho[r] = {T(0), T(0)};
#pragma unroll
    for (int q = 0; q < LB; ++q) {
      const int lm = 1 << (LB - 1 - q);
#pragma unroll
      for (int r = 0; r < A; ++r) {
        const cplx<T> p = shfl_xor_c(xa[1][r], lm);
        rho[r].re += dth[q] * p.re;
        rho[r].im += dth[q] * p.im;
      }
    }
#pragma unroll
    for (int qi = 0; qi < AB; ++qi) {
      const int Sm = 1 << (AB - 1 - qi);
#pragma unroll
      for (int r = 0; r < A; ++r) {
        rho[r].re += dth[LB + qi] * xa[1][r ^ Sm].re;
        rho[r].im += dth[LB + qi] * xa[1][r ^ Sm].im;
      }
    }
    // H_q = Im sum conj(xa1) X_q phi, P_q = Re sum conj(rho) X_q phi (rho = 0 in
    // the psi lanes, whose dtheta is 0): g_theta = H/2 (psi) or -P/4, g_dtheta = H/2
    T gt[N], gd[N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
      T H = T(0), P = T(0);
#pragma unroll
      for (int r = 0; r < A; ++r) {
        cplx<T> y;
        if (q < LB) y = shfl_xor_c(xa[0][r], 1 << (LB - 1 - q));
        else y = xa[0][r ^ (1 << (N - 1 - q))];
        H = fma(xa[1][r].re, y.im, H);
        H = fma(-xa[1][r].im, y.re, H);
        P = fma(rho[r].re, y.re, P);
        P = fma(rho[r].im, y.im, P);
      }
      gt[q] = (sidx == 0 ? T(0.5) * H : T(0)) - T(0.25) * P;
      gd[q] = sidx == 0 ? T(0) : T(0.5) * H;
    }
#pragma unroll
    for (int m = 1; m < G; m <<= 1)
#pragma unroll
      for (int q = 0; q < N; ++q) {
        gt[q] += __shfl_xor_sync(0xffffffffu, gt[q], m);
        gd[q] += __shfl_xor_sync(0xffffffffu, gd[q], m);
      }
#pragma unroll
    for (int m = G; m < 4 * G; m <<= 1)
#pragma unroll
      for (int q = 0; q < N; ++q) gt[q] += __shfl_xor_sync(0xffffffffu, gt[q], m);
    T gk[3][N];
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int q = 0; q < N; ++q)
        gk[k][q] = __shfl_sync(0xffffffffu, gd[q], pw * LPP + (k + 1) * G + gl);
    if (valid) {
#pragma unroll
      for (int q = 0; q < N; ++q) {
        if ((q % G) != gl) continue;
        if (sidx == 0) {
          T ga = gt[q] * s1v[q];
#pragma unroll
          for (int k = 0; k < 3; ++k)
            ga += gk[k][q] * s2v[q] * act_tan[((int64_t)k * R + s) * N + q];
          g_act[s * N + q] = ga;
        } else {
          g_act_tan[((int64_t)(sidx - 1) * R + s) * N + q] = gd[q] * s1v[q];
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_acc; i += blockDim.x) {
    double v = 0.0;
    for (int w = 0; w < warps; ++w) v += (double)sm.acc[(size_t)w * n_acc + i];
    partial[(size_t)blockIdx.x * n_acc + i] = v;
  }
}

// ---- launch ---------------------------------------------------------------------------------
#ifdef QPINN_LAYER_DEFINE_ENTANGLER
int layer_entangler(const qpinn_circuit* c) {
  // the plan must be [n u1 on wires 0..n-1, entangler?] x L (ansatz.py:178-204)
  const int n = c->n, L = c->L;
  const int n_steps = (int)c->steps.size() / 3;
  int ent = ENT_NONE;
  if (c->n_perm) ent = ENT_PERM;
  if (c->n_phase) ent = ENT_PHASE;
  if (c->n_perm && c->n_phase) return -1;
  const int per = n + (ent == ENT_NONE ? 0 : 1);
  if (c->n_u1 != n * L || n_steps != per * L) return -1;
  for (int l = 0; l < L; ++l) {
    for (int q = 0; q < n; ++q) {
      const int* s = &c->steps[3 * (l * per + q)];
      if (s[0] != STEP_U1 || s[1] != q || s[2] != l * n + q) return -1;
    }
    if (ent != ENT_NONE) {
      const int* s = &c->steps[3 * (l * per + n)];
      if (s[0] != (ent == ENT_PERM ? STEP_PERM : STEP_PHASE) || s[2] != l) return -1;
    }
  }
  return ent;
}
#endif

template <typename T, int N>
static int prepare(const qpinn_circuit* c, const KArgs<T>* a) {
  pqc_prepare_tables<T, N><<<4, 128, 0, a->stream>>>(c->dev, a->qp, a->tables);
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

template <typename T, int N, int ENT>
static int layer_fwd(const qpinn_circuit* c, const KArgs<T>* a) {
  const PlanDev& p = c->dev;
  if (int rc = prepare<T, N>(c, a)) return rc;
  const size_t smem = smem_layout<T, N, Geo<T, N, 4>::AB>(p, kThreads / 32, false, nullptr, nullptr);
  if (smem > 227 * 1024) return fail(QPINN_ERR_CAPACITY, "PQC plan tables exceed shared memory");
  auto go = [&](auto kern, int spw) -> int {
    QPINN_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem);
    const int grid = pqc_grid(a->R, spw, occ > 0 ? occ : 1);
    kern<<<grid, kThreads, smem, a->stream>>>(p, a->tables, c->L, a->scale, a->R, a->act, a->tan,
                                              a->qp, a->z, a->dz, (cplx<T>*)a->states, a->maxabs,
                                              (cplx<T>*)a->coh);
    QPINN_CUDA_CHECK(cudaGetLastError());
    return QPINN_OK;
  };
  if (a->tan) return go(pqc_forward_layer<T, N, 4, ENT>, Geo<T, N, 4>::SPW);
  return go(pqc_forward_layer<T, N, 1, ENT>, Geo<T, N, 1>::SPW);
}

template <typename T, int N, int ENT>
static int layer_bwd(const qpinn_circuit* c, const KArgs<T>* a) {
  using Gm = Geo<T, N, 4>;
  const PlanDev& p = c->dev;
  const size_t smem = smem_layout<T, N, Gm::AB>(p, kThreads / 32, true, nullptr, nullptr);
  if (smem > 227 * 1024) return fail(QPINN_ERR_CAPACITY, "PQC plan tables exceed shared memory");
  if (int rc = prepare<T, N>(c, a)) return rc;
  auto kern = pqc_backward_layer<T, N, ENT>;
  QPINN_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem);
  if (occ > kMaxBlocksPerSm) occ = kMaxBlocksPerSm;
  const int grid = pqc_grid(a->R, Gm::SPW, occ > 0 ? occ : 1);
  kern<<<grid, kThreads, smem, a->stream>>>(p, a->tables, c->L, a->scale, a->R, a->act, a->tan, a->qp,
                                            (const cplx<T>*)a->states, a->gz, a->gdz, a->g_act,
                                            a->g_tan, a->partial);
  QPINN_CUDA_CHECK(cudaGetLastError());
  return pqc_finish_grads<T>(c, grid, a);
}

template <typename T, int N>
static int layer_n(bool fwd, int ent, const qpinn_circuit* c, const KArgs<T>* a) {
  if (fwd) {
    if (ent == ENT_PERM) return layer_fwd<T, N, ENT_PERM>(c, a);
    if (ent == ENT_PHASE) return layer_fwd<T, N, ENT_PHASE>(c, a);
    return layer_fwd<T, N, ENT_NONE>(c, a);
  }
  if (!a->states) return KERNEL_NONE;  // no hand-off: the generic kernel replays the circuit
  if (ent == ENT_PERM) return layer_bwd<T, N, ENT_PERM>(c, a);
  if (ent == ENT_PHASE) return layer_bwd<T, N, ENT_PHASE>(c, a);
  return layer_bwd<T, N, ENT_NONE>(c, a);
}

template <typename T>
int layer_dispatch(bool fwd, const qpinn_circuit* c, const KArgs<T>* a) {
  const int ent = layer_entangler(c);
  if (ent < 0) return KERNEL_NONE;
  switch (c->n) {
    case 1: return layer_n<T, 1>(fwd, ent, c, a);
    case 2: return layer_n<T, 2>(fwd, ent, c, a);
    case 3: return layer_n<T, 3>(fwd, ent, c, a);
    case 4: return layer_n<T, 4>(fwd, ent, c, a);
    case 5: return layer_n<T, 5>(fwd, ent, c, a);
    case 6: return layer_n<T, 6>(fwd, ent, c, a);
    case 7: return layer_n<T, 7>(fwd, ent, c, a);
    case 8:
      if constexpr (sizeof(T) == 4) return layer_n<T, 8>(fwd, ent, c, a);
      return KERNEL_NONE;
    default: return KERNEL_NONE;
  }
}

}  // namespace qpinn
