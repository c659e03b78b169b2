// K1 / K2: per-point statevector PQC with forward-mode x/y/t tangents and its
// adjoint-differentiation backward, register-resident on sm_100a.
//
// Reference path (qpinn, pure numpy): quantum_layer_forward
// (ansatz.py:341-400) builds the embedded product state (ansatz.py:233-243)
// and its tangent states (ansatz.py:380-390), pushes all of them through the
// ansatz transfer matrix (ansatz.py:284-293, :392-394) and reads <Z_q>
// (qsim.py:369-381); gradients come from the reverse tape (tape.py:118-148).
//
// Here every collocation point is simulated gate by gate in registers.
// Lane geometry ("states in lanes"): a point owns NSL x G lanes, NSL = 4
// states (psi, d psi/dx, d psi/dy, d psi/dt) times G = 2^LB lanes per state;
// each lane holds A = 2^AB amplitudes of ONE state (n = 7: G = 8, A = 16, one
// point per warp).  Amplitude b = gl * A + r, so wires 0..LB-1 are lane bits
// (a gate needs one shfl.xor per amplitude) and wires LB..n-1 are register
// bits (pure FMA).  All four states see the same gate sequence, so the gate
// coefficients are warp-uniform.  Keeping one state per lane keeps register
// use low (occupancy hides the FMA/shuffle latencies) and only 3 of 7 wires
// at n = 7 need shuffles.
//   * the embedded state and its tangents are closed form (magnitude product
//     x (-i)^popcount), no gate sweep needed;
//   * fused CNOT runs go through a per-warp shared-memory permutation, fused
//     CRZ meshes are one diagonal phase table per step (built per block);
//   * the readout fetches psi from the state-0 lane and reduces over the
//     state's lane group with butterfly shuffles.
// K2 takes the final states from K1 (or recomputes them), seeds the adjoints
// from dL/dz, dL/d(dz), walks the plan backwards un-computing
// the state and propagating its adjoint in the same lane, and accumulates
// the per-gate 2x2 outer products (post-gate form M' = sum conj(abar) x') per
// warp in shared memory; the per-point embedding gradient applies X_q to the
// starting state.  Parameter gradients are reduced warp -> block -> grid in a
// fixed order (run-to-run deterministic) in float64.
#include <cmath>
#include <cstring>
#include <mutex>

#include "pqc_layer.h"

namespace qpinn {

// ---- K1: forward + tangents ---------------------------------------------------------
template <typename T, int N, int NSL>
__global__ void __launch_bounds__(kThreads)
pqc_forward_kernel(PlanDev plan, const __grid_constant__ StepTable steps, int scale, int64_t R,
                   const T* __restrict__ act,
                   const T* __restrict__ act_tan, const T* __restrict__ qp, T* __restrict__ z,
                   T* __restrict__ dz, cplx<T>* __restrict__ states,
                   unsigned long long* __restrict__ maxabs) {
  using Gm = Geo<T, N, NSL>;
  constexpr int AB = Gm::AB, A = Gm::A, LB = Gm::LB, G = Gm::G, LPP = Gm::LPP, SPW = Gm::SPW,
                D = Gm::D;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warps = blockDim.x >> 5;
  Smem<T> sm;
  smem_layout<T, N, AB>(plan, warps, false, &sm, smem_raw);
  prologue<T, N, AB, G>(plan, qp, sm, false, warps);
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pw = lane / LPP, sidx = (lane / G) % NSL, gl = lane & (G - 1);
  const int lane_hi = lane >> LB;
  const int psi_lane = pw * LPP + gl;  // state-0 lane with the same gl
  cplx<T>* buf = sm.buf + warp * 32 * A;
  const int n_steps = steps.n;
  T amax = T(0);
  // block-uniform trip count (the loop bound must not depend on threadIdx, or
  // every shuffle inside gets a divergence/collective wrapper)
  const int64_t per_block = (int64_t)warps * SPW;
  const int64_t stride = (int64_t)gridDim.x * per_block;
  for (int64_t base = (int64_t)blockIdx.x * per_block; base < R; base += stride) {
    const int64_t s = base + warp * SPW + pw;
    const bool valid = s < R;
    T c[N], sn[N], dth[N], s1[N], s2[N];
    load_point<T, N>(scale, act, act_tan, R, s, valid, sidx - 1, c, sn, dth, s1, s2, amax);
    cplx<T> st[1][A];
    embed<T, N, AB>(c, sn, dth, sidx > 0, gl, st[0]);
    for (int si = 0; si < n_steps; ++si) {
      const int h = steps.s[si].x, idx = steps.s[si].y;
      const int type = h & 3, wire = (h >> 2) - 1;
      if (type == STEP_U1) {
        const cplx<T>* U = sm.U + 4 * idx;
        apply_u1<T, N, AB, 1>(st, wire, gl, U[0], U[1], U[2], U[3]);
      } else if (type == STEP_PERM) {
        permute<T, A, G, 1>(st, sm.pt + idx * D, buf, gl, lane_hi);
      } else {
        const cplx<T>* ph = sm.ph + idx * D;
#pragma unroll
        for (int r = 0; r < A; ++r) st[0][r] = cmul(st[0][r], ph[r * G + gl]);
      }
    }
    if (NSL == 4 && states != nullptr && valid) {  // hand-off for K2
      cplx<T>* sp = states + s * (4 * D) + sidx * D;
#pragma unroll
      for (int r = 0; r < A; ++r) sp[r * G + gl] = st[0][r];
    }
    // readout: z_q = sum_b s_bq |psi_b|^2 ; dz_kq = sum_b s_bq 2 Re(conj(psi_b) dpsi_kb)
    T out[N], tot = T(0);
#pragma unroll
    for (int q = 0; q < N; ++q) out[q] = T(0);
#pragma unroll
    for (int r = 0; r < A; ++r) {
      T v;
      if (NSL == 4) {
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
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, m));
  if (lane == 0 && maxabs) atomic_max_abs(maxabs, amax);
}

// ---- K2: adjoint backward -------------------------------------------------------------

template <typename T, int N>
__global__ void __launch_bounds__(kThreads)
pqc_backward_kernel(PlanDev plan, const __grid_constant__ StepTable steps, int scale, int64_t R,
                    const T* __restrict__ act,
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
  prologue<T, N, AB, G>(plan, qp, sm, true, warps);
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pw = lane / LPP, sidx = (lane / G) % 4, gl = lane & (G - 1);
  const int lane_hi = lane >> LB;
  const int psi_lane = pw * LPP + gl;
  cplx<T>* buf = sm.buf + warp * 2 * 32 * A;
  const int n_acc = 8 * plan.n_u1 + D * plan.n_phase;
  T* accU = sm.acc + (size_t)warp * n_acc;
  T* accP = accU + 8 * plan.n_u1;
  const int n_steps = steps.n;
  // block-uniform trip count (the loop bound must not depend on threadIdx, or
  // every shuffle inside gets a divergence/collective wrapper)
  const int64_t per_block = (int64_t)warps * SPW;
  const int64_t stride = (int64_t)gridDim.x * per_block;
  for (int64_t base = (int64_t)blockIdx.x * per_block; base < R; base += stride) {
    const int64_t s = base + warp * SPW + pw;
    const bool valid = s < R;
    T c[N], sn[N], dth[N], s1v[N], s2v[N], amax_unused = T(0);
    load_point<T, N>(scale, act, act_tan, R, s, valid, sidx - 1, c, sn, dth, s1v, s2v,
                     amax_unused);
    // xa[0] = this lane's state x, xa[1] = its adjoint
    cplx<T> xa[2][A];
    if (states != nullptr) {  // final states from K1
      const cplx<T>* sp = states + (valid ? s : 0) * (4 * D) + sidx * D;
#pragma unroll
      for (int r = 0; r < A; ++r) xa[0][r] = valid ? sp[r * G + gl] : cplx<T>{T(0), T(0)};
    } else {
      embed<T, N, AB>(c, sn, dth, sidx > 0, gl, xa[0]);
      for (int si = 0; si < n_steps; ++si) {
        const int h = steps.s[si].x, idx = steps.s[si].y;
        const int type = h & 3, wire = (h >> 2) - 1;
        cplx<T>(&x1)[1][A] = *reinterpret_cast<cplx<T>(*)[1][A]>(&xa[0][0]);
        if (type == STEP_U1) {
          const cplx<T>* U = sm.U + 4 * idx;
          apply_u1<T, N, AB, 1>(x1, wire, gl, U[0], U[1], U[2], U[3]);
        } else if (type == STEP_PERM) {
          permute<T, A, G, 1>(x1, sm.pt + idx * D, buf, gl, lane_hi);
        } else {
          const cplx<T>* ph = sm.ph + idx * D;
#pragma unroll
          for (int r = 0; r < A; ++r) xa[0][r] = cmul(xa[0][r], ph[r * G + gl]);
        }
      }
    }
    // adjoint seeds: lambda = 2 w psi + 2 sum_k v_k dpsi_k (state 0), mu_k = 2 v_k psi.
    // This lane's sign-weighted cotangent row: g_z (s = 0) or g_dz[k] (s = k+1).
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
      for (int qi = 0; qi < AB; ++qi) w += ((r >> (AB - 1 - qi)) & 1) ? -gsel[LB + qi] : gsel[LB + qi];
      w *= T(2);
      const cplx<T> p = {__shfl_sync(0xffffffffu, xa[0][r].re, psi_lane),
                         __shfl_sync(0xffffffffu, xa[0][r].im, psi_lane)};
      // lambda contribution of this lane: 2 w psi (s = 0) or 2 v_k dpsi_k (s = k+1)
      cplx<T> t = {w * xa[0][r].re, w * xa[0][r].im};
#pragma unroll
      for (int m = G; m < 4 * G; m <<= 1) {
        t.re += __shfl_xor_sync(0xffffffffu, t.re, m);
        t.im += __shfl_xor_sync(0xffffffffu, t.im, m);
      }
      xa[1][r] = sidx == 0 ? t : cplx<T>{w * p.re, w * p.im};
    }
    // reverse sweep
    for (int si = n_steps - 1; si >= 0; --si) {
      const int h = steps.s[si].x, idx = steps.s[si].y;
      const int type = h & 3, wire = (h >> 2) - 1;
      if (type == STEP_U1) {
        const cplx<T>* U = sm.U + 4 * idx;
        const cplx<T> h00 = {U[0].re, -U[0].im}, h01 = {U[2].re, -U[2].im};
        const cplx<T> h10 = {U[1].re, -U[1].im}, h11 = {U[3].re, -U[3].im};
        T m[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) m[e] = T(0);
        if (wire < LB) {
          const int lb = LB - 1 - wire;
          const bool beta = (gl >> lb) & 1;
          const cplx<T> cs = beta ? h11 : h00, cp = beta ? h10 : h01;
          T ms_re = 0, ms_im = 0, mc_re = 0, mc_im = 0;
#pragma unroll
          for (int r = 0; r < A; ++r) {
            const cplx<T> xs = xa[0][r], as = xa[1][r];
            const cplx<T> xp = shfl_xor_c(xs, 1 << lb), ap = shfl_xor_c(as, 1 << lb);
            cmac_c(ms_re, ms_im, as, xs);
            cmac_c(mc_re, mc_im, as, xp);
            xa[0][r] = cmul2(cs, xs, cp, xp);
            xa[1][r] = cmul2(cs, as, cp, ap);
          }
          // M'[i][j] with i the own row: beta = 0 -> (0,0),(0,1); beta = 1 -> (1,1),(1,0)
          if (!beta) { m[0] = ms_re; m[1] = ms_im; m[2] = mc_re; m[3] = mc_im; }
          else { m[6] = ms_re; m[7] = ms_im; m[4] = mc_re; m[5] = mc_im; }
        } else {
          const int rb = N - 1 - wire;
#pragma unroll
          for (int bsel = 0; bsel < AB; ++bsel) {
            if (bsel != rb) continue;
#pragma unroll
            for (int r = 0; r < A; ++r) {
              if (r & (1 << bsel)) continue;
              const int r1 = r | (1 << bsel);
              const cplx<T> x0 = xa[0][r], x1 = xa[0][r1], a0 = xa[1][r], a1 = xa[1][r1];
              cmac_c(m[0], m[1], a0, x0);
              cmac_c(m[2], m[3], a0, x1);
              cmac_c(m[4], m[5], a1, x0);
              cmac_c(m[6], m[7], a1, x1);
              xa[0][r] = cmul2(h00, x0, h01, x1);
              xa[0][r1] = cmul2(h10, x0, h11, x1);
              xa[1][r] = cmul2(h00, a0, h01, a1);
              xa[1][r1] = cmul2(h10, a0, h11, a1);
            }
          }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) m[e] = warp_sum(m[e]);
        if (lane < 8) {
          T v = m[0];
#pragma unroll
          for (int e = 1; e < 8; ++e) v = (lane == e) ? m[e] : v;
          accU[idx * 8 + lane] += v;
        }
      } else if (type == STEP_PERM) {
        permute<T, A, G, 2>(xa, sm.pti + idx * D, buf, gl, lane_hi);
      } else {
        const cplx<T>* ph = sm.ph + idx * D;
        T* acc = accP + idx * D;
#pragma unroll
        for (int r = 0; r < A; ++r) {
          T pv = xa[1][r].im * xa[0][r].re - xa[1][r].re * xa[0][r].im;
#pragma unroll
          for (int mk = G; mk < 32; mk <<= 1) pv += __shfl_xor_sync(0xffffffffu, pv, mk);
          if (lane_hi == 0) acc[r * G + gl] += pv;
          const cplx<T> e = {ph[r * G + gl].re, -ph[r * G + gl].im};
          xa[0][r] = cmul(xa[0][r], e);
          xa[1][r] = cmul(xa[1][r], e);
        }
      }
    }
    // embedding gradient.  xa[1] = phibar (s = 0) or mu_k (s = k+1).
    // xa[0] <- phi (recomputed exactly); rho = sum_q dth_kq X_q mu_k in lanes k.
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
      const int S = 1 << (AB - 1 - qi);
#pragma unroll
      for (int r = 0; r < A; ++r) {
        rho[r].re += dth[LB + qi] * xa[1][r ^ S].re;
        rho[r].im += dth[LB + qi] * xa[1][r ^ S].im;
      }
    }
    // gt[q]  : partial of dL/dtheta_q  = Re<(i/2) phibar - 1/4 sum_k rho_k, X_q phi>
    // gd[q]  : partial of dL/ddtheta_kq = Re<(i/2) mu_k, X_q phi>   (lanes of state k)
    T gt[N], gd[N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
      gt[q] = T(0);
      gd[q] = T(0);
#pragma unroll
      for (int r = 0; r < A; ++r) {
        cplx<T> y;
        if (q < LB) y = shfl_xor_c(xa[0][r], 1 << (LB - 1 - q));
        else y = xa[0][r ^ (1 << (N - 1 - q))];
        // Re<(i/2) a, y> = 1/2 (a.re y.im - a.im y.re)
        const T half = T(0.5) * (xa[1][r].re * y.im - xa[1][r].im * y.re);
        if (sidx == 0) gt[q] += half;
        else {
          gt[q] -= T(0.25) * (rho[r].re * y.re + rho[r].im * y.im);
          gd[q] += half;
        }
      }
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
    // gather gd of states 1..3 into every lane of the point
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
  // block partial: sum the per-warp accumulators in warp order (float64)
  for (int i = threadIdx.x; i < n_acc; i += blockDim.x) {
    double v = 0.0;
    for (int w = 0; w < warps; ++w) v += (double)sm.acc[(size_t)w * n_acc + i];
    partial[(size_t)blockIdx.x * n_acc + i] = v;
  }
}

// grid-level reduction of block partials (fixed order)
__global__ void pqc_reduce_partials(const double* __restrict__ partial, int blocks, int n_acc,
                                    double* __restrict__ tot) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_acc) return;
  double v = 0.0;
  for (int b = 0; b < blocks; ++b) v += partial[(size_t)b * n_acc + i];
  tot[i] = v;
}

// gate-space gradients -> parameter slots of the u1 steps
template <typename T>
__global__ void pqc_u1_grads(PlanDev p, const T* __restrict__ qp, const double* __restrict__ tot,
                             T* __restrict__ g_qp) {
  // one thread per (gate, parameter slot): the double-precision trig of a gate's
  // matrix and derivative runs in parallel over its slots
  for (int it = blockIdx.x * blockDim.x + threadIdx.x; it < 3 * p.n_u1;
       it += gridDim.x * blockDim.x) {
    const int i = it / 3, jslot = it % 3;
    const int kind = p.u1[i * 4];
    double th[3] = {0, 0, 0};
    const int ns = u1_nslots(kind);
    if (jslot >= ns) continue;
    for (int j = 0; j < ns; ++j) th[j] = (double)qp[p.u1[i * 4 + 1 + j]];
    double U[8];
    u1_matrix_d(kind, th, U);
    const double* Mp = tot + 8 * i;  // M'[i][j'] = sum conj(abar_i) x'_j'
    // M = M' conj(U): M_ij = sum_j' M'_ij' conj(U_j'j)
    double M[8];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        double re = 0, im = 0;
        for (int k = 0; k < 2; ++k) {
          const double mr = Mp[(a * 2 + k) * 2], mi = Mp[(a * 2 + k) * 2 + 1];
          const double ur = U[(k * 2 + b) * 2], ui = -U[(k * 2 + b) * 2 + 1];
          re += mr * ur - mi * ui;
          im += mr * ui + mi * ur;
        }
        M[(a * 2 + b) * 2] = re;
        M[(a * 2 + b) * 2 + 1] = im;
      }
    {
      const int j = jslot;
      double dU[8];
      u1_dmatrix_d(kind, th, j, dU);
      double g = 0.0;  // Re sum_ij dU_ij M_ij
      for (int e = 0; e < 4; ++e) g += dU[2 * e] * M[2 * e] - dU[2 * e + 1] * M[2 * e + 1];
      g_qp[p.u1[i * 4 + 1 + j]] = T(g);
    }
  }
}

// ... and of the CRZ-mesh phase steps (accumulators stored at lay(b))
template <typename T>
__global__ void pqc_phase_grads(PlanDev p, int ab, const double* __restrict__ tot,
                                T* __restrict__ g_qp) {
  const int D = 1 << p.n;
  const int G = 1 << (p.n - ab);
  const double* accP = tot + 8 * p.n_u1;
  for (int st = 0; st < p.n_phase; ++st) {
    for (int k = p.phase_off[st] + threadIdx.x; k < p.phase_off[st + 1]; k += blockDim.x) {
      const int c = p.pairs[3 * k], t = p.pairs[3 * k + 1], s = p.pairs[3 * k + 2];
      double g = 0.0;
      for (int b = 0; b < D; ++b) {
        const int on = (b >> (p.n - 1 - c)) & 1, tb = (b >> (p.n - 1 - t)) & 1;
        if (on) g += (tb - 0.5) * accP[st * D + (b & ((1 << ab) - 1)) * G + (b >> ab)];
      }
      g_qp[s] = T(g);
    }
  }
}

// ---- host launchers -------------------------------------------------------------------
template <typename K>
static int occupancy_blocks(K kernel, size_t smem) {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, kThreads, smem);
  return nb > 0 ? nb : 1;
}

static int grid_for(int64_t R, int spw, int occ) {
  const int64_t per_block = (int64_t)(kThreads / 32) * spw;
  int64_t need = (R + per_block - 1) / per_block;
  int64_t cap = (int64_t)num_sms() * occ;
  int64_t g = need < cap ? need : cap;
  return (int)(g < 1 ? 1 : g);
}

static std::mutex g_attr_mu;

static int step_table(const qpinn_circuit* c, StepTable* t) {
  const int n = (int)c->steps.size() / 3;
  if (n > kMaxKSteps) return fail(QPINN_ERR_CAPACITY, "fused plan longer than the kernel step table");
  t->n = n;
  for (int i = 0; i < n; ++i)
    t->s[i] = make_int2(c->steps[3 * i] | ((c->steps[3 * i + 1] + 1) << 2), c->steps[3 * i + 2]);
  return QPINN_OK;
}

template <typename T, int N>
static int launch_forward(qpinn_circuit* c, int scale, int64_t R, const T* act, const T* tan,
                          const T* qp, T* z, T* dz, void* states, unsigned long long* maxabs,
                          cudaStream_t stream) {
  const PlanDev& p = c->dev;
  StepTable steps;
  if (int rc = step_table(c, &steps)) return rc;
  auto run = [&](auto kern, int ab, int spw, bool bwd_layout) -> int {
    (void)ab;
    const size_t smem = smem_layout<T, N, Geo<T, N, 4>::AB>(p, kThreads / 32, bwd_layout,
                                                            nullptr, nullptr);
    if (smem > 227 * 1024) return fail(QPINN_ERR_CAPACITY, "PQC plan tables exceed shared memory");
    {
      std::lock_guard<std::mutex> lk(g_attr_mu);
      QPINN_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem));
    }
    const int grid = grid_for(R, spw, occupancy_blocks(kern, smem));
    kern<<<grid, kThreads, smem, stream>>>(p, steps, scale, R, act, tan, qp, z, dz,
                                           (cplx<T>*)states, maxabs);
    QPINN_CUDA_CHECK(cudaGetLastError());
    return QPINN_OK;
  };
  if (tan) return run(pqc_forward_kernel<T, N, 4>, Geo<T, N, 4>::AB, Geo<T, N, 4>::SPW, false);
  return run(pqc_forward_kernel<T, N, 1>, Geo<T, N, 1>::AB, Geo<T, N, 1>::SPW, false);
}

template <typename T, int N>
static int launch_backward(qpinn_circuit* c, int scale, int64_t R, const T* act, const T* tan,
                           const T* qp, const void* states, const T* gz, const T* gdz, T* g_act,
                           T* g_tan, T* g_qp, double* partial, double* tot, cudaStream_t stream) {
  using Gm = Geo<T, N, 4>;
  const PlanDev& p = c->dev;
  StepTable steps;
  if (int rc = step_table(c, &steps)) return rc;
  const size_t smem = smem_layout<T, N, Gm::AB>(p, kThreads / 32, true, nullptr, nullptr);
  if (smem > 227 * 1024) return fail(QPINN_ERR_CAPACITY, "PQC plan tables exceed shared memory");
  auto kern = pqc_backward_kernel<T, N>;
  {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    QPINN_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
  }
  int occ = occupancy_blocks(kern, smem);
  if (occ > kMaxBlocksPerSm) occ = kMaxBlocksPerSm;
  const int grid = grid_for(R, Gm::SPW, occ);
  kern<<<grid, kThreads, smem, stream>>>(p, steps, scale, R, act, tan, qp, (const cplx<T>*)states,
                                         gz, gdz, g_act, g_tan, partial);
  QPINN_CUDA_CHECK(cudaGetLastError());
  KArgs<T> a{scale, R, act, tan, qp, nullptr, nullptr, nullptr, nullptr, gz, gdz, g_act, g_tan,
             g_qp, partial, tot, stream, nullptr};
  return pqc_finish_grads<T>(c, grid, &a);
}

int pqc_grid(int64_t R, int spw, int occ) { return grid_for(R, spw, occ); }

// fixed-order grid reduction of the block partials, then gate-space -> slots
template <typename T>
int pqc_finish_grads(const qpinn_circuit* c, int grid, const KArgs<T>* a) {
  const int ab = c->n <= 4 ? c->n : (c->n - 3 > 4 ? c->n - 3 : 4);  // Geo::AB
  return pqc_finish_grads_ab<T>(c, grid, a, ab);
}

template <typename T>
int pqc_finish_grads_ab(const qpinn_circuit* c, int grid, const KArgs<T>* a, int ab) {
  const PlanDev& p = c->dev;
  const int n_acc = 8 * p.n_u1 + (1 << p.n) * p.n_phase;
  if (n_acc > 0) {
    pqc_reduce_partials<<<(n_acc + 255) / 256, 256, 0, a->stream>>>(a->partial, grid, n_acc, a->tot);
    QPINN_CUDA_CHECK(cudaGetLastError());
  }
  pqc_u1_grads<T><<<p.n_u1 > 0 ? (3 * p.n_u1 + 127) / 128 : 1, 128, 0, a->stream>>>(p, a->qp, a->tot, a->g_qp);
  QPINN_CUDA_CHECK(cudaGetLastError());
  if (p.n_phase) {
    pqc_phase_grads<T><<<1, 256, 0, a->stream>>>(p, ab, a->tot, a->g_qp);
    QPINN_CUDA_CHECK(cudaGetLastError());
  }
  return QPINN_OK;
}
template <typename T>
int pqc_param_grads(const qpinn_circuit* c, const double* tot, int ab, const T* qp, T* g_qp,
                    cudaStream_t st) {
  pqc_u1_grads<T><<<c->dev.n_u1 > 0 ? (3 * c->dev.n_u1 + 127) / 128 : 1, 128, 0, st>>>(c->dev, qp, tot, g_qp);
  QPINN_CUDA_CHECK(cudaGetLastError());
  if (c->dev.n_phase) {
    pqc_phase_grads<T><<<1, 256, 0, st>>>(c->dev, ab, tot, g_qp);
    QPINN_CUDA_CHECK(cudaGetLastError());
  }
  return QPINN_OK;
}
template int pqc_param_grads<float>(const qpinn_circuit*, const double*, int, const float*,
                                    float*, cudaStream_t);
template int pqc_param_grads<double>(const qpinn_circuit*, const double*, int, const double*,
                                     double*, cudaStream_t);

template int pqc_finish_grads<float>(const qpinn_circuit*, int, const KArgs<float>*);
template int pqc_finish_grads<double>(const qpinn_circuit*, int, const KArgs<double>*);
template int pqc_finish_grads_ab<float>(const qpinn_circuit*, int, const KArgs<float>*, int);
template int pqc_finish_grads_ab<double>(const qpinn_circuit*, int, const KArgs<double>*, int);

// runtime n -> template instantiation
#define QPINN_DISPATCH_N(MAXN, N_RT, CALL)                                         \
  switch (N_RT) {                                                                  \
    case 1: if constexpr (1 <= MAXN) { constexpr int NN = 1; return CALL; } break; \
    case 2: if constexpr (2 <= MAXN) { constexpr int NN = 2; return CALL; } break; \
    case 3: if constexpr (3 <= MAXN) { constexpr int NN = 3; return CALL; } break; \
    case 4: if constexpr (4 <= MAXN) { constexpr int NN = 4; return CALL; } break; \
    case 5: if constexpr (5 <= MAXN) { constexpr int NN = 5; return CALL; } break; \
    case 6: if constexpr (6 <= MAXN) { constexpr int NN = 6; return CALL; } break; \
    case 7: if constexpr (7 <= MAXN) { constexpr int NN = 7; return CALL; } break; \
    case 8: if constexpr (8 <= MAXN) { constexpr int NN = 8; return CALL; } break; \
    default: break;                                                                \
  }

// workspace: [0,256) running max|a| (u64 double bits) | block partials | totals
static size_t n_acc_of(const qpinn_circuit* c) {
  return 8 * (size_t)c->n_u1 + ((size_t)1 << c->n) * c->n_phase;
}
static size_t partial_bytes(const qpinn_circuit* c) {
  return align_up(sizeof(double) * n_acc_of(c) * (size_t)num_sms() * kMaxBlocksPerSm, 256);
}
static size_t tables_bytes_bound(const qpinn_circuit* c) {  // any dtype
  const size_t D = (size_t)1 << c->n;
  return align_up(16 * (4 * (size_t)c->n_u1 + D * c->n_phase) + 4 * D * c->n_perm + 1024, 256);
}

// workspace carve-up of the cluster regime (must match big_workspace_bytes)
static void big_ws(const qpinn_circuit* c, void* ws, double** partial, double** tot,
                   unsigned char** tables) {
  const size_t n_acc = n_acc_of(c), rows = (size_t)num_sms() * 2;
  char* base = (char*)ws + 256;
  *partial = (double*)base;
  base += align_up(8 * n_acc * rows, 256);
  *tot = (double*)base;
  base += align_up(8 * n_acc, 256);
  *tables = (unsigned char*)base;
}

// The reference domain rule (ansatz.py:51-58) as device flags, so a
// data-parallel step can carry it through its one all-reduce and veto Adam:
// out[0] = 1 if max|a| - 1 > 1e-12 (DomainError), out[1] = 1 if max|a| > 1
// (clamped, or the error), out[2] = max|a|; the running maximum is reset.
__global__ void pqc_domain_flags(unsigned long long* maxabs, double* out) {
  const unsigned long long bits = *maxabs;
  double m;
  memcpy(&m, &bits, 8);
  const double over = m - 1.0;
  out[0] = over > 1e-12 ? 1.0 : 0.0;
  out[1] = over > 0.0 ? 1.0 : 0.0;
  out[2] = m;
  *maxabs = 0ull;
}

}  // namespace qpinn

using namespace qpinn;

extern "C" {

int qpinn_circuit_set_kernel_variant(qpinn_circuit* c, int variant) {
  if (!c || variant < 0 || variant > 3) return fail(QPINN_ERR_CONFIG, "bad kernel variant");
  c->variant = variant;
  return QPINN_OK;
}

int qpinn_circuit_specialized(const qpinn_circuit* c) {
  return c && layer_entangler(c) >= 0 ? 1 : 0;
}

int qpinn_pqc_max_qubits(int dtype) {
  return dtype == QPINN_F64 ? max_qubits<double>() : max_qubits<float>();
}

static size_t small_ws_bytes(const qpinn_circuit* c) {
  return 256 + partial_bytes(c) + align_up(sizeof(double) * n_acc_of(c), 256) +
         tables_bytes_bound(c);
}

// the transfer-matrix kernels (pqc_transfer.cu): variant 2, and the default for
// float32 n = 5..8 (measured with the phase-folded map, 2^16 points, L = 4,
// K1 + K2: n = 7 0.69 ms vs 1.74 ms for the layer kernels, n = 6 0.41 vs 0.82,
// n = 5 0.32 vs 0.37-0.39; profiles/r01/transfer_vs_layer_folded.txt; n = 8 at
// 2^17 points: 3.7 vs 13.2 ms, profiles/r02/config5_n8_transfer_vs_layer.txt)
static bool use_transfer(const qpinn_circuit* c, int dtype) {
  if (c->variant == 2) return transfer_supported(c, dtype);
  return c->variant == 0 && transfer_default(c, dtype);
}

int qpinn_pqc_regime(const qpinn_circuit* c, int dtype, int backward) {
  if (!c) return -1;
  if (use_transfer(c, dtype)) return 2;
  if (c->n <= qpinn_pqc_max_qubits(dtype))
    return (c->variant == 0 || c->variant == 3) && layer_entangler(c) >= 0 ? 0 : 1;
  if (backward) {
    if (hbm_bwd_supported(c, dtype)) return 4;
    return big_bwd_supported(c, dtype) ? 3 : 5;
  }
  if (hbm_fwd_supported(c, dtype)) return 4;
  return big_fwd_supported(c, dtype) ? 3 : 5;
}

int qpinn_pqc_uses_transfer(const qpinn_circuit* c, int dtype) {
  return c && use_transfer(c, dtype) ? 1 : 0;
}

size_t qpinn_pqc_workspace_bytes(const qpinn_circuit* c, int dtype, int64_t rows) {
  if (!c) return 0;
  // the transfer-matrix kernels: up to n = 8 whatever the variant, beyond that (where
  // their staging is GBs at large batches) only when the current variant selects them
  // -- query the size after qpinn_circuit_set_kernel_variant
  size_t t = 0;
  if (c->n <= qpinn_pqc_max_qubits(dtype) ? transfer_supported(c, dtype) : use_transfer(c, dtype))
    t = small_ws_bytes(c) + transfer_workspace_bytes(c, rows);
  if (c->n > qpinn_pqc_max_qubits(dtype)) {
    const size_t b = align_up(big_workspace_bytes(c, dtype), 256) +
                     global_adjoint_workspace_bytes(c, dtype, rows);
    return b > t ? b : t;
  }
  const size_t b = small_ws_bytes(c);
  return b > t ? b : t;
}

size_t qpinn_pqc_state_bytes(const qpinn_circuit* c, int dtype, int64_t rows) {
  if (!c || rows < 0) return 0;
  // layer-loop kernels: the 4 states at each of the L layer boundaries;
  // generic kernels: the 4 final states (fits inside the former)
  const size_t per = 4 * ((size_t)1 << c->n) * 2 * (dtype == QPINN_F64 ? 8 : 4);
  const bool layer = c->n <= qpinn_pqc_max_qubits(dtype) && layer_entangler(c) >= 0;
  const size_t b = (size_t)rows * per * (layer && c->L > 1 ? (size_t)c->L : 1);
  // the transfer-matrix hand-off (Psi, Phi, W, checkpoints, tables): up to n = 8 for
  // any variant, beyond that only when the current variant selects the transfer map
  const bool tr = c->n <= qpinn_pqc_max_qubits(dtype) ? transfer_supported(c, dtype)
                                                       : use_transfer(c, dtype);
  if (!tr) return b;
  const size_t t = transfer_state_bytes(c, rows);
  return t > b ? t : b;
}

static int check_common(const qpinn_circuit* c, int dtype, int scale, int64_t rows,
                        size_t ws_bytes, size_t need) {
  if (!c) return fail(QPINN_ERR_CONFIG, "null circuit");
  if (dtype != QPINN_F32 && dtype != QPINN_F64) return fail(QPINN_ERR_CONFIG, "bad dtype");
  if (scale < 0 || scale > 4) return fail(QPINN_ERR_CONFIG, "unknown scale kind");
  if (rows < 0) return fail(QPINN_ERR_INVALID_BATCH, "negative row count");
  if (ws_bytes < need) return fail(QPINN_ERR_CONFIG, "workspace too small");
  return QPINN_OK;
}

int qpinn_pqc_forward(const qpinn_circuit* cc, int dtype, int scale, int64_t rows,
                      const void* act_val, const void* act_tan, const void* qparams, void* z,
                      void* dz, void* states, void* workspace, size_t workspace_bytes,
                      void* stream) {
  qpinn_circuit* c = const_cast<qpinn_circuit*>(cc);
  int rc = check_common(c, dtype, scale, rows, workspace_bytes,
                        qpinn_pqc_workspace_bytes(c, dtype, rows));
  if (rc) return rc;
  if ((act_tan == nullptr) != (dz == nullptr))
    return fail(QPINN_ERR_CONFIG, "act_tan and dz must both be given or both be NULL");
  const int n = c->n;
  rc = ensure_device_plan(c);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  auto* maxabs = (unsigned long long*)workspace;  // running max, reset by domain_check
  if (n > qpinn_pqc_max_qubits(dtype) && !use_transfer(c, dtype)) {  // cluster kernels (pqc_big.cu)
    if (rows == 0) return QPINN_OK;
    double* partial;
    double* tot;
    unsigned char* tables;
    big_ws(c, workspace, &partial, &tot, &tables);
    if (hbm_fwd_supported(c, dtype)) {  // several gates per HBM pass (pqc_global.cu)
      const size_t off = align_up(big_workspace_bytes(c, dtype), 256);
      KArgs<float> a{scale, rows, (const float*)act_val, (const float*)act_tan,
                     (const float*)qparams, (float*)z, (float*)dz, nullptr, maxabs, nullptr,
                     nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, st, nullptr};
      return hbm_forward(c, &a, (unsigned char*)workspace + off,
                         workspace_bytes > off ? workspace_bytes - off : 0);
    }
    if (!act_tan || !big_fwd_supported(c, dtype)) {  // global-memory forward (pqc_global.cu)
      const size_t off = align_up(big_workspace_bytes(c, dtype), 256);
      unsigned char* gws = (unsigned char*)workspace + off;
      const size_t gbytes = workspace_bytes > off ? workspace_bytes - off : 0;
      if (dtype == QPINN_F32) {
        KArgs<float> a{scale, rows, (const float*)act_val, (const float*)act_tan,
                       (const float*)qparams, (float*)z, (float*)dz, nullptr, maxabs, nullptr,
                       nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, st, nullptr};
        return global_forward<float>(c, &a, gws, gbytes);
      }
      KArgs<double> a{scale, rows, (const double*)act_val, (const double*)act_tan,
                      (const double*)qparams, (double*)z, (double*)dz, nullptr, maxabs, nullptr,
                      nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, st, nullptr};
      return global_forward<double>(c, &a, gws, gbytes);
    }
    if (dtype == QPINN_F32) {
      KArgs<float> a{scale, rows, (const float*)act_val, (const float*)act_tan, (const float*)qparams,
                     (float*)z, (float*)dz, nullptr, maxabs, nullptr, nullptr, nullptr, nullptr,
                     nullptr, partial, tot, st, tables};
      return big_dispatch<float>(true, c, &a);
    }
    KArgs<double> a{scale, rows, (const double*)act_val, (const double*)act_tan,
                    (const double*)qparams, (double*)z, (double*)dz, nullptr, maxabs, nullptr,
                    nullptr, nullptr, nullptr, nullptr, partial, tot, st, tables};
    return big_dispatch<double>(true, c, &a);
  }
  unsigned char* tables = (unsigned char*)workspace + 256 + partial_bytes(c) +
                          align_up(sizeof(double) * n_acc_of(c), 256);
  if (rows == 0) return QPINN_OK;
  if (use_transfer(c, dtype)) {
    KArgs<float> a{scale, rows, (const float*)act_val, (const float*)act_tan,
                   (const float*)qparams, (float*)z, (float*)dz, states, maxabs, nullptr,
                   nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, st, nullptr};
    const size_t off = small_ws_bytes(c);
    return transfer_forward(c, &a, (unsigned char*)workspace + off, workspace_bytes - off);
  }
  if (c->variant == 0 || c->variant == 3) {  // layer-loop kernels for every standard plan
    if (dtype == QPINN_F32) {
      KArgs<float> a{scale, rows, (const float*)act_val, (const float*)act_tan,
                        (const float*)qparams, (float*)z, (float*)dz, states, maxabs,
                        nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, st, tables};
      rc = layer_dispatch<float>(true, c, &a);
    } else {
      KArgs<double> a{scale, rows, (const double*)act_val, (const double*)act_tan,
                         (const double*)qparams, (double*)z, (double*)dz, states, maxabs,
                         nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, st, tables};
      rc = layer_dispatch<double>(true, c, &a);
    }
    if (rc != KERNEL_NONE) return rc;
  }
  if (dtype == QPINN_F32) {
    QPINN_DISPATCH_N(8, n, (launch_forward<float, NN>(c, scale, rows, (const float*)act_val,
                                                      (const float*)act_tan, (const float*)qparams,
                                                      (float*)z, (float*)dz, states, maxabs, st)));
  } else {
    QPINN_DISPATCH_N(7, n, (launch_forward<double, NN>(c, scale, rows, (const double*)act_val,
                                                       (const double*)act_tan,
                                                       (const double*)qparams, (double*)z,
                                                       (double*)dz, states, maxabs, st)));
  }
  return fail(QPINN_ERR_CAPACITY, "unsupported n_qubits");
}

int qpinn_pqc_backward(const qpinn_circuit* cc, int dtype, int scale, int64_t rows,
                       const void* act_val, const void* act_tan, const void* qparams,
                       const void* states, const void* g_z, const void* g_dz, void* g_act_val,
                       void* g_act_tan, void* g_qparams, void* workspace, size_t workspace_bytes,
                       void* stream) {
  qpinn_circuit* c = const_cast<qpinn_circuit*>(cc);
  const size_t need = qpinn_pqc_workspace_bytes(c, dtype, rows);
  int rc = check_common(c, dtype, scale, rows, workspace_bytes, need);
  if (rc) return rc;
  if (!act_tan || !g_z || !g_dz || !g_act_val || !g_act_tan || !g_qparams)
    return fail(QPINN_ERR_CONFIG, "backward needs tangents and all gradient buffers");
  const int n = c->n;
  rc = ensure_device_plan(c);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (n > qpinn_pqc_max_qubits(dtype) && !use_transfer(c, dtype)) {  // cluster kernels, forward replayed
    if (rows == 0) {
      QPINN_CUDA_CHECK(cudaMemsetAsync(g_qparams, 0,
                                       (dtype == QPINN_F64 ? 8 : 4) * (size_t)c->n_params, st));
      return QPINN_OK;
    }
    double* bp;
    double* bt;
    unsigned char* btab;
    big_ws(c, workspace, &bp, &bt, &btab);
    if (hbm_bwd_supported(c, dtype)) {  // several gates per HBM pass (pqc_global.cu)
      const size_t off = align_up(big_workspace_bytes(c, dtype), 256);
      KArgs<float> a{scale, rows, (const float*)act_val, (const float*)act_tan,
                     (const float*)qparams, nullptr, nullptr, nullptr, nullptr,
                     (const float*)g_z, (const float*)g_dz, (float*)g_act_val,
                     (float*)g_act_tan, (float*)g_qparams, nullptr, nullptr, st, nullptr};
      return hbm_backward(c, &a, (unsigned char*)workspace + off,
                          workspace_bytes > off ? workspace_bytes - off : 0);
    }
    if (!big_bwd_supported(c, dtype)) {  // HBM regime (pqc_global.cu)
      const size_t off = align_up(big_workspace_bytes(c, dtype), 256);
      unsigned char* gws = (unsigned char*)workspace + off;
      const size_t gbytes = workspace_bytes > off ? workspace_bytes - off : 0;
      if (dtype == QPINN_F32) {
        KArgs<float> a{scale, rows, (const float*)act_val, (const float*)act_tan,
                       (const float*)qparams, nullptr, nullptr, nullptr, nullptr,
                       (const float*)g_z, (const float*)g_dz, (float*)g_act_val,
                       (float*)g_act_tan, (float*)g_qparams, nullptr, nullptr, st, nullptr};
        return global_backward<float>(c, &a, gws, gbytes);
      }
      KArgs<double> a{scale, rows, (const double*)act_val, (const double*)act_tan,
                      (const double*)qparams, nullptr, nullptr, nullptr, nullptr,
                      (const double*)g_z, (const double*)g_dz, (double*)g_act_val,
                      (double*)g_act_tan, (double*)g_qparams, nullptr, nullptr, st, nullptr};
      return global_backward<double>(c, &a, gws, gbytes);
    }
    if (dtype == QPINN_F32) {
      KArgs<float> a{scale, rows, (const float*)act_val, (const float*)act_tan,
                     (const float*)qparams, nullptr, nullptr, nullptr, nullptr, (const float*)g_z,
                     (const float*)g_dz, (float*)g_act_val, (float*)g_act_tan, (float*)g_qparams,
                     bp, bt, st, btab};
      return big_dispatch<float>(false, c, &a);
    }
    KArgs<double> a{scale, rows, (const double*)act_val, (const double*)act_tan,
                    (const double*)qparams, nullptr, nullptr, nullptr, nullptr,
                    (const double*)g_z, (const double*)g_dz, (double*)g_act_val,
                    (double*)g_act_tan, (double*)g_qparams, bp, bt, st, btab};
    return big_dispatch<double>(false, c, &a);
  }
  double* partial = (double*)((char*)workspace + 256);
  double* tot = (double*)((char*)workspace + 256 + partial_bytes(c));
  unsigned char* tables = (unsigned char*)workspace + 256 + partial_bytes(c) +
                          align_up(sizeof(double) * n_acc_of(c), 256);
  if (rows == 0) {
    QPINN_CUDA_CHECK(cudaMemsetAsync(g_qparams, 0,
                                     (dtype == QPINN_F64 ? 8 : 4) * (size_t)c->n_params, st));
    return QPINN_OK;
  }
  if (use_transfer(c, dtype)) {
    KArgs<float> a{scale, rows, (const float*)act_val, (const float*)act_tan,
                   (const float*)qparams, nullptr, nullptr, const_cast<void*>(states), nullptr,
                   (const float*)g_z, (const float*)g_dz, (float*)g_act_val, (float*)g_act_tan,
                   (float*)g_qparams, nullptr, nullptr, st, nullptr};
    const size_t off = small_ws_bytes(c);
    return transfer_backward(c, &a, (unsigned char*)workspace + off, workspace_bytes - off);
  }
  if (c->variant == 0 || c->variant == 3) {
    if (dtype == QPINN_F32) {
      KArgs<float> a{scale, rows, (const float*)act_val, (const float*)act_tan,
                        (const float*)qparams, nullptr, nullptr, const_cast<void*>(states),
                        nullptr, (const float*)g_z, (const float*)g_dz, (float*)g_act_val,
                        (float*)g_act_tan, (float*)g_qparams, partial, tot, st, tables};
      rc = layer_dispatch<float>(false, c, &a);
    } else {
      KArgs<double> a{scale, rows, (const double*)act_val, (const double*)act_tan,
                         (const double*)qparams, nullptr, nullptr, const_cast<void*>(states),
                         nullptr, (const double*)g_z, (const double*)g_dz, (double*)g_act_val,
                         (double*)g_act_tan, (double*)g_qparams, partial, tot, st, tables};
      rc = layer_dispatch<double>(false, c, &a);
    }
    if (rc != KERNEL_NONE) return rc;
  }
  if (dtype == QPINN_F32) {
    QPINN_DISPATCH_N(8, n, (launch_backward<float, NN>(
                               c, scale, rows, (const float*)act_val, (const float*)act_tan,
                               (const float*)qparams, states, (const float*)g_z,
                               (const float*)g_dz, (float*)g_act_val, (float*)g_act_tan,
                               (float*)g_qparams, partial, tot, st)));
  } else {
    QPINN_DISPATCH_N(7, n, (launch_backward<double, NN>(
                               c, scale, rows, (const double*)act_val, (const double*)act_tan,
                               (const double*)qparams, states, (const double*)g_z,
                               (const double*)g_dz, (double*)g_act_val, (double*)g_act_tan,
                               (double*)g_qparams, partial, tot, st)));
  }
  return fail(QPINN_ERR_CAPACITY, "unsupported n_qubits");
}

int qpinn_pqc_forward_probe(const qpinn_circuit* cc, int dtype, int scale, int64_t rows,
                            const void* act_val, const void* qparams, void* z, void* coh,
                            void* workspace, size_t workspace_bytes, void* stream) {
  qpinn_circuit* c = const_cast<qpinn_circuit*>(cc);
  int rc = check_common(c, dtype, scale, rows, workspace_bytes,
                        qpinn_pqc_workspace_bytes(c, dtype, rows));
  if (rc) return rc;
  if (!z || !coh) return fail(QPINN_ERR_CONFIG, "probe needs z and coh");
  if (c->n > qpinn_pqc_max_qubits(dtype) || layer_entangler(c) < 0)
    return fail(QPINN_ERR_CAPACITY, "the entanglement probe needs the layer-loop kernels "
                                    "(standard ansatz, n <= 8 fp32 / 7 fp64)");
  rc = ensure_device_plan(c);
  if (rc) return rc;
  if (rows == 0) return QPINN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  auto* maxabs = (unsigned long long*)workspace;
  unsigned char* tables = (unsigned char*)workspace + 256 + partial_bytes(c) +
                          align_up(sizeof(double) * n_acc_of(c), 256);
  if (dtype == QPINN_F32) {
    KArgs<float> a{scale, rows, (const float*)act_val, nullptr, (const float*)qparams, (float*)z,
                   nullptr, nullptr, maxabs, nullptr, nullptr, nullptr, nullptr, nullptr,
                   nullptr, nullptr, st, tables, (float*)coh};
    rc = layer_dispatch<float>(true, c, &a);
  } else {
    KArgs<double> a{scale, rows, (const double*)act_val, nullptr, (const double*)qparams,
                    (double*)z, nullptr, nullptr, maxabs, nullptr, nullptr, nullptr, nullptr,
                    nullptr, nullptr, nullptr, st, tables, (double*)coh};
    rc = layer_dispatch<double>(true, c, &a);
  }
  return rc == KERNEL_NONE ? fail(QPINN_ERR_CAPACITY, "probe: no layer kernel") : rc;
}

int qpinn_pqc_domain_fetch(const void* workspace, void* host_dst, void* stream) {
  if (!workspace || !host_dst) return fail(QPINN_ERR_CONFIG, "domain fetch: null pointer");
  QPINN_CUDA_CHECK(cudaMemcpyAsync(host_dst, workspace, 8, cudaMemcpyDeviceToHost,
                                   (cudaStream_t)stream));
  QPINN_CUDA_CHECK(cudaMemsetAsync(const_cast<void*>(workspace), 0, 8, (cudaStream_t)stream));
  return QPINN_OK;
}

int qpinn_pqc_domain_flags(const void* workspace, double* flags_dev, void* stream) {
  if (!workspace || !flags_dev) return fail(QPINN_ERR_CONFIG, "domain flags: null pointer");
  pqc_domain_flags<<<1, 1, 0, (cudaStream_t)stream>>>(
      (unsigned long long*)const_cast<void*>(workspace), flags_dev);
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

int qpinn_pqc_domain_check(const void* workspace, void* stream, double* max_abs, int* clamped) {
  unsigned long long bits = 0;
  QPINN_CUDA_CHECK(cudaStreamSynchronize((cudaStream_t)stream));
  QPINN_CUDA_CHECK(cudaMemcpy(&bits, workspace, 8, cudaMemcpyDeviceToHost));
  QPINN_CUDA_CHECK(cudaMemset(const_cast<void*>(workspace), 0, 8));
  double m;
  memcpy(&m, &bits, 8);
  if (max_abs) *max_abs = m;
  const double over = m - 1.0;
  if (clamped) *clamped = (over > 0.0 && over <= 1e-12) ? 1 : 0;
  if (over > 1e-12) return fail(QPINN_ERR_DOMAIN, "scale input exceeds [-1, 1]");
  return QPINN_OK;
}

}  // extern "C"
