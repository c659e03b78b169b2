// K1 / K2: per-point statevector PQC with forward-mode x/y/t tangents and its
// adjoint-differentiation backward, register-resident on sm_100a.
//
// Reference path (qpinn, pure numpy): quantum_layer_forward
// (ansatz.py:341-400) builds the embedded product state (ansatz.py:233-243)
// and its tangent states (ansatz.py:380-390), pushes all of them through the
// ansatz transfer matrix (ansatz.py:284-293, :392-394) and reads <Z_q>
// (qsim.py:369-381); gradients come from the reverse tape (tape.py:118-148).
//
// Here every collocation point is simulated gate by gate in registers:
//   * a group of G = 2^LB lanes owns one point; each lane holds A = 2^AB
//     amplitudes of each of the NS states (value + 3 tangents, plus 4
//     adjoint states in K2).  Amplitude b = lane_in_group * A + r, so wires
//     0..LB-1 are lane bits (gates need one shfl.xor per amplitude) and
//     wires LB..n-1 are register bits (gates are pure FMA);
//   * the embedded state and its tangents are written in closed form
//     (magnitude product x (-i)^popcount), no gate sweep needed;
//   * fused CNOT runs go through a per-warp shared-memory permutation, fused
//     CRZ meshes are one diagonal phase table per step (built per block);
//   * the readout reduces over the lane group with butterfly shuffles.
// K2 re-runs the forward, seeds the adjoints from dL/dz, dL/d(dz)
// (SURVEY 8.A), walks the plan backwards un-computing the 4 forward states
// and propagating the 4 adjoint states, and accumulates per-gate 2x2
// outer products (post-gate form M' = sum conj(abar) x') per warp in shared
// memory; the per-point embedding gradient uses X_q applications on the
// starting state.  Parameter gradients are reduced warp -> block -> grid in
// a fixed order (run-to-run deterministic) in float64.
#include <cmath>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace qpinn {

constexpr double kPi = 3.14159265358979323846;

__device__ __forceinline__ void sincos_(float x, float* s, float* c) { sincosf(x, s, c); }
__device__ __forceinline__ void sincos_(double x, double* s, double* c) { sincos(x, s, c); }

// ---- lane/register geometry --------------------------------------------------
template <typename T, bool BWD>
struct AbBase;
template <>
struct AbBase<float, false> { static constexpr int v = 3; };
template <>
struct AbBase<float, true> { static constexpr int v = 3; };
template <>
struct AbBase<double, false> { static constexpr int v = 2; };
template <>
struct AbBase<double, true> { static constexpr int v = 2; };

template <typename T, bool BWD>
constexpr int max_qubits() { return AbBase<T, BWD>::v + 5; }

template <typename T, int N, bool BWD>
struct Geo {
  static constexpr int AB = N < AbBase<T, BWD>::v ? N : AbBase<T, BWD>::v;
  static constexpr int A = 1 << AB;
  static constexpr int LB = N - AB;
  static constexpr int G = 1 << LB;
  static constexpr int SPW = 32 / G;
  static constexpr int D = 1 << N;
  static_assert(LB <= 5, "register regime holds at most 32 lanes per point");
};

constexpr int kThreads = 128;  // 4 warps per block

// shared-memory layout index of basis state b ("lane-fastest"): conflict-free
// for the group's A x G amplitudes.
template <int AB, int G>
__host__ __device__ __forceinline__ int lay(int b) {
  return (b & ((1 << AB) - 1)) * G + (b >> AB);
}

// ---- scaling: theta = S(a), S'(a), S''(a)  (ansatz.py:44-67, ops.py:181-192) -
template <typename T>
__device__ __forceinline__ void scale_fn(int kind, T a, T& th, T& s1, T& s2) {
  const T pi = T(kPi);
  switch (kind) {
    case QPINN_SCALE_NONE:
      th = a; s1 = T(1); s2 = T(0);
      break;
    case QPINN_SCALE_PI:
      th = a * pi; s1 = pi; s2 = T(0);
      break;
    case QPINN_SCALE_BIAS:
      th = (a + T(1)) * (pi / T(2)); s1 = pi / T(2); s2 = T(0);
      break;
    default: {
      const T om = (T(1) - a) * (T(1) + a);
      const T r = sqrt(om);
      if (kind == QPINN_SCALE_ASIN) {
        th = asin(a) + pi / T(2); s1 = T(1) / r; s2 = a / (om * r);
      } else {
        th = acos(a); s1 = T(-1) / r; s2 = -a / (om * r);
      }
    }
  }
}

// ---- gate matrices (qsim.py:274-316), evaluated in float64 -------------------
__device__ inline void u1_matrix_d(int kind, const double* th, double U[8]) {
  double c, s;
  switch (kind) {
    case U1_ROT: {  // RZ(c) RY(b) RZ(a)  (qsim.py:294-305)
      double p = (th[0] + th[2]) * 0.5, m = (th[0] - th[2]) * 0.5;
      double cb = cos(th[1] * 0.5), sb = sin(th[1] * 0.5);
      double cp = cos(p), sp = sin(p), cm = cos(m), sm = sin(m);
      U[0] = cp * cb; U[1] = -(sp * cb);
      U[2] = -(cm * sb); U[3] = -(sm * sb);
      U[4] = cm * sb; U[5] = -(sm * sb);
      U[6] = cp * cb; U[7] = sp * cb;
      break;
    }
    case U1_RXRZ: {  // RZ(b) RX(a)  (qsim.py:308-316)
      double ca = cos(th[0] * 0.5), sa = sin(th[0] * 0.5);
      double cb = cos(th[1] * 0.5), sb = sin(th[1] * 0.5);
      U[0] = cb * ca; U[1] = -(sb * ca);
      U[2] = -(sb * sa); U[3] = -(cb * sa);
      U[4] = sb * sa; U[5] = -(cb * sa);
      U[6] = cb * ca; U[7] = sb * ca;
      break;
    }
    case U1_RX:
      c = cos(th[0] * 0.5); s = sin(th[0] * 0.5);
      U[0] = c; U[1] = 0; U[2] = 0; U[3] = -s; U[4] = 0; U[5] = -s; U[6] = c; U[7] = 0;
      break;
    case U1_RY:
      c = cos(th[0] * 0.5); s = sin(th[0] * 0.5);
      U[0] = c; U[1] = 0; U[2] = -s; U[3] = 0; U[4] = s; U[5] = 0; U[6] = c; U[7] = 0;
      break;
    default:  // RZ
      c = cos(th[0] * 0.5); s = sin(th[0] * 0.5);
      U[0] = c; U[1] = -s; U[2] = 0; U[3] = 0; U[4] = 0; U[5] = 0; U[6] = c; U[7] = s;
  }
}

__device__ inline int u1_nslots(int kind) {
  return kind == U1_ROT ? 3 : kind == U1_RXRZ ? 2 : 1;
}

// complex 2x2 product C = A B on interleaved [re, im] x 4 arrays
__device__ inline void m2mul(const double* A, const double* B, double* C) {
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) {
      double re = 0, im = 0;
      for (int k = 0; k < 2; ++k) {
        double ar = A[(i * 2 + k) * 2], ai = A[(i * 2 + k) * 2 + 1];
        double br = B[(k * 2 + j) * 2], bi = B[(k * 2 + j) * 2 + 1];
        re += ar * br - ai * bi;
        im += ar * bi + ai * br;
      }
      C[(i * 2 + j) * 2] = re;
      C[(i * 2 + j) * 2 + 1] = im;
    }
}
__device__ inline void rx_d(double t, bool deriv, double* M) {
  double c = cos(t * 0.5), s = sin(t * 0.5);
  if (!deriv) {
    double v[8] = {c, 0, 0, -s, 0, -s, c, 0};
    for (int i = 0; i < 8; ++i) M[i] = v[i];
  } else {
    double v[8] = {-0.5 * s, 0, 0, -0.5 * c, 0, -0.5 * c, -0.5 * s, 0};
    for (int i = 0; i < 8; ++i) M[i] = v[i];
  }
}
__device__ inline void ry_d(double t, bool deriv, double* M) {
  double c = cos(t * 0.5), s = sin(t * 0.5);
  if (!deriv) {
    double v[8] = {c, 0, -s, 0, s, 0, c, 0};
    for (int i = 0; i < 8; ++i) M[i] = v[i];
  } else {
    double v[8] = {-0.5 * s, 0, -0.5 * c, 0, 0.5 * c, 0, -0.5 * s, 0};
    for (int i = 0; i < 8; ++i) M[i] = v[i];
  }
}
__device__ inline void rz_d(double t, bool deriv, double* M) {
  double c = cos(t * 0.5), s = sin(t * 0.5);
  if (!deriv) {
    double v[8] = {c, -s, 0, 0, 0, 0, c, s};
    for (int i = 0; i < 8; ++i) M[i] = v[i];
  } else {  // d/dt diag(e^{-it/2}, e^{it/2}) = diag(-i/2 e^{-it/2}, i/2 e^{it/2})
    double v[8] = {-0.5 * s, -0.5 * c, 0, 0, 0, 0, -0.5 * s, 0.5 * c};
    for (int i = 0; i < 8; ++i) M[i] = v[i];
  }
}
// dU/d(slot j) of a fused u1 step
__device__ inline void u1_dmatrix_d(int kind, const double* th, int j, double* dU) {
  double A[8], B[8], C[8], T1[8];
  switch (kind) {
    case U1_ROT:  // RZ(c) RY(b) RZ(a)
      rz_d(th[2], j == 2, A);
      ry_d(th[1], j == 1, B);
      rz_d(th[0], j == 0, C);
      m2mul(A, B, T1);
      m2mul(T1, C, dU);
      break;
    case U1_RXRZ:  // RZ(b) RX(a)
      rz_d(th[1], j == 1, A);
      rx_d(th[0], j == 0, B);
      m2mul(A, B, dU);
      break;
    case U1_RX: rx_d(th[0], true, dU); break;
    case U1_RY: ry_d(th[0], true, dU); break;
    default: rz_d(th[0], true, dU);
  }
}

// ---- block prologue: gate matrices, phase tables, permutation tables --------
template <typename T, int N, int AB>
struct Smem {
  cplx<T>* U;         // [n_u1][4]
  cplx<T>* ph;        // [n_phase][D] at lay(b)
  uint16_t* pt;       // [n_perm][D]  lay(perm[b]) at lay(b)
  uint16_t* pti;      // [n_perm][D]  lay(iperm[b]) at lay(b)
  int* steps;         // [n_steps][2]
  cplx<T>* buf;       // per-warp permutation buffer [warps][32 * A]
  T* acc;             // K2: per-warp gradient accumulators [warps][n_acc]
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

template <typename T, int N, int AB>
__host__ __device__ inline size_t smem_layout(const PlanDev& p, int warps, bool bwd,
                                              Smem<T, N, AB>* out, unsigned char* base) {
  constexpr int D = 1 << N;
  constexpr int A = 1 << AB;
  size_t o = 0;
  size_t oU = o; o = align_up(o + sizeof(cplx<T>) * 4 * p.n_u1, 16);
  size_t oPh = o; o = align_up(o + sizeof(cplx<T>) * (size_t)D * p.n_phase, 16);
  size_t oPt = o; o = align_up(o + 2 * (size_t)D * p.n_perm, 16);
  size_t oPti = o; o = align_up(o + (bwd ? 2 * (size_t)D * p.n_perm : 0), 16);
  size_t oSt = o; o = align_up(o + 8 * (size_t)p.n_steps, 16);
  size_t oBuf = o; o = align_up(o + sizeof(cplx<T>) * 32 * A * (size_t)warps, 16);
  size_t oAcc = o;
  if (bwd) o = align_up(o + sizeof(T) * (size_t)warps * (8 * p.n_u1 + (size_t)D * p.n_phase), 16);
  if (out) {
    out->U = (cplx<T>*)(base + oU);
    out->ph = (cplx<T>*)(base + oPh);
    out->pt = (uint16_t*)(base + oPt);
    out->pti = (uint16_t*)(base + oPti);
    out->steps = (int*)(base + oSt);
    out->buf = (cplx<T>*)(base + oBuf);
    out->acc = (T*)(base + oAcc);
  }
  return o;
}

template <typename T, int N, int AB, int G>
__device__ void prologue(const PlanDev& p, const T* __restrict__ qp, const Smem<T, N, AB>& sm,
                         bool bwd, int warps) {
  constexpr int D = 1 << N;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < p.n_u1; i += nt) {
    const int kind = p.u1[i * 4];
    double th[3] = {0, 0, 0};
    for (int j = 0; j < u1_nslots(kind); ++j) th[j] = (double)qp[p.u1[i * 4 + 1 + j]];
    double U[8];
    u1_matrix_d(kind, th, U);
    for (int e = 0; e < 4; ++e) sm.U[i * 4 + e] = {T(U[2 * e]), T(U[2 * e + 1])};
  }
  for (int i = tid; i < p.n_phase * D; i += nt) {
    const int st = i / D, b = i % D;
    double phi = 0.0;
    for (int k = p.phase_off[st]; k < p.phase_off[st + 1]; ++k) {
      const int c = p.pairs[3 * k], t = p.pairs[3 * k + 1], s = p.pairs[3 * k + 2];
      const int on = (b >> (N - 1 - c)) & 1, tb = (b >> (N - 1 - t)) & 1;
      phi += on * (tb - 0.5) * (double)qp[s];  // qsim.py:212-225, ansatz.py:259-265
    }
    sm.ph[st * D + lay<AB, G>(b)] = {T(cos(phi)), T(sin(phi))};
  }
  for (int i = tid; i < p.n_perm * D; i += nt) {
    const int st = i / D, b = i % D;
    sm.pt[st * D + lay<AB, G>(b)] = (uint16_t)lay<AB, G>(p.perm[i]);
    if (bwd) sm.pti[st * D + lay<AB, G>(b)] = (uint16_t)lay<AB, G>(p.iperm[i]);
  }
  for (int i = tid; i < p.n_steps; i += nt) {
    sm.steps[2 * i] = p.steps[3 * i] | ((p.steps[3 * i + 1] + 1) << 2);
    sm.steps[2 * i + 1] = p.steps[3 * i + 2];
  }
  if (bwd) {
    const size_t nacc = (size_t)warps * (8 * p.n_u1 + (size_t)D * p.n_phase);
    for (size_t i = tid; i < nacc; i += nt) sm.acc[i] = T(0);
  }
}

// ---- per-point embedding: product state and tangents (ansatz.py:233-243,
//      :380-390) in closed form ------------------------------------------------
template <typename T, int N, int AB, int NT>
__device__ __forceinline__ void embed(const T (&c)[N], const T (&sn)[N], const T (&dth)[3][N],
                                      int gl, cplx<T> (&st)[1 + NT][1 << AB]) {
  constexpr int A = 1 << AB, LB = N - AB;
  // lane wires: forward-mode product over the lane bits
  T mL = T(1), dL[3] = {T(0), T(0), T(0)};
#pragma unroll
  for (int q = 0; q < LB; ++q) {
    const int bit = (gl >> (LB - 1 - q)) & 1;
    const T f = bit ? sn[q] : c[q];
    const T df = bit ? T(0.5) * c[q] : T(-0.5) * sn[q];
#pragma unroll
    for (int k = 0; k < NT; ++k) dL[k] = dL[k] * f + mL * dth[k][q] * df;
    mL *= f;
  }
  // register wires: doubling, wire LB is the most significant register bit
  st[0][0].re = T(1);
#pragma unroll
  for (int k = 0; k < NT; ++k) st[1 + k][0].re = T(0);
#pragma unroll
  for (int qi = 0; qi < AB; ++qi) {
    const int q = LB + qi;
#pragma unroll
    for (int i = (1 << qi) - 1; i >= 0; --i) {
      const T m = st[0][i].re;
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        const T d = st[1 + k][i].re;
        st[1 + k][2 * i + 1].re = d * sn[q] + m * dth[k][q] * (T(0.5) * c[q]);
        st[1 + k][2 * i].re = d * c[q] + m * dth[k][q] * (T(-0.5) * sn[q]);
      }
      st[0][2 * i + 1].re = m * sn[q];
      st[0][2 * i].re = m * c[q];
    }
  }
  const int popL = __popc(gl);
#pragma unroll
  for (int r = 0; r < A; ++r) {
    const int ph = (popL + __popc(r)) & 3;  // (-i)^popcount
    const T mr = st[0][r].re;
    T mags[1 + NT];
    mags[0] = mL * mr;
#pragma unroll
    for (int k = 0; k < NT; ++k) mags[1 + k] = dL[k] * mr + mL * st[1 + k][r].re;
#pragma unroll
    for (int j = 0; j < 1 + NT; ++j) {
      const T m = mags[j];
      st[j][r].re = (ph == 0) ? m : (ph == 2) ? -m : T(0);
      st[j][r].im = (ph == 1) ? -m : (ph == 3) ? m : T(0);
    }
  }
}

// ---- gate application --------------------------------------------------------
template <int RB, typename T, int A, int NS>
__device__ __forceinline__ void gate_reg(cplx<T> (&st)[NS][A], cplx<T> u00, cplx<T> u01,
                                         cplx<T> u10, cplx<T> u11) {
#pragma unroll
  for (int r = 0; r < A; ++r) {
    if (r & (1 << RB)) continue;
    const int r1 = r | (1 << RB);
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      const cplx<T> a0 = st[j][r], a1 = st[j][r1];
      st[j][r] = cmul2(u00, a0, u01, a1);
      st[j][r1] = cmul2(u10, a0, u11, a1);
    }
  }
}

template <typename T, int A, int NS>
__device__ __forceinline__ void gate_lane(cplx<T> (&st)[NS][A], int lm, bool beta, cplx<T> u00,
                                          cplx<T> u01, cplx<T> u10, cplx<T> u11) {
  const cplx<T> cs = beta ? u11 : u00, cp = beta ? u10 : u01;
#pragma unroll
  for (int r = 0; r < A; ++r)
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      const cplx<T> p = shfl_xor_c(st[j][r], lm);
      st[j][r] = cmul2(cs, st[j][r], cp, p);
    }
}

template <typename T, int N, int AB, int NS>
__device__ __forceinline__ void apply_u1(cplx<T> (&st)[NS][1 << AB], int wire, int gl,
                                         cplx<T> u00, cplx<T> u01, cplx<T> u10, cplx<T> u11) {
  constexpr int LB = N - AB, A = 1 << AB;
  if (wire < LB) {
    const int lb = LB - 1 - wire;
    gate_lane<T, A, NS>(st, 1 << lb, (gl >> lb) & 1, u00, u01, u10, u11);
  } else {
    const int rb = N - 1 - wire;
    if (rb == 0) gate_reg<0, T, A, NS>(st, u00, u01, u10, u11);
    if constexpr (AB > 1) if (rb == 1) gate_reg<1, T, A, NS>(st, u00, u01, u10, u11);
    if constexpr (AB > 2) if (rb == 2) gate_reg<2, T, A, NS>(st, u00, u01, u10, u11);
    if constexpr (AB > 3) if (rb == 3) gate_reg<3, T, A, NS>(st, u00, u01, u10, u11);
  }
}

// new[b] = old[table[b]] through the warp's shared buffer, one state at a time
template <typename T, int A, int G, int SPW, int NS>
__device__ __forceinline__ void permute(cplx<T> (&st)[NS][A], const uint16_t* tab, cplx<T>* buf,
                                        int gl, int grp) {
#pragma unroll
  for (int j = 0; j < NS; ++j) {
#pragma unroll
    for (int r = 0; r < A; ++r) buf[(r * G + gl) * SPW + grp] = st[j][r];
    __syncwarp();
#pragma unroll
    for (int r = 0; r < A; ++r) st[j][r] = buf[tab[r * G + gl] * SPW + grp];
    __syncwarp();
  }
}

// ---- readout (qsim.py:369-381; tangent readout ansatz.py:395-399) ------------
template <typename T, int N, int AB, int NT>
__device__ __forceinline__ void readout(const cplx<T> (&st)[1 + NT][1 << AB], int gl,
                                        T (&out)[1 + NT][N]) {
  constexpr int A = 1 << AB, LB = N - AB, G = 1 << LB;
  T tot[1 + NT];
#pragma unroll
  for (int k = 0; k <= NT; ++k) {
    tot[k] = T(0);
#pragma unroll
    for (int q = 0; q < N; ++q) out[k][q] = T(0);
  }
#pragma unroll
  for (int r = 0; r < A; ++r) {
    T v[1 + NT];
    v[0] = st[0][r].re * st[0][r].re + st[0][r].im * st[0][r].im;
#pragma unroll
    for (int k = 0; k < NT; ++k)
      v[1 + k] = T(2) * (st[0][r].re * st[1 + k][r].re + st[0][r].im * st[1 + k][r].im);
#pragma unroll
    for (int k = 0; k <= NT; ++k) {
      tot[k] += v[k];
#pragma unroll
      for (int qi = 0; qi < AB; ++qi) {
        if ((r >> (AB - 1 - qi)) & 1) out[k][LB + qi] -= v[k];
        else out[k][LB + qi] += v[k];
      }
    }
  }
#pragma unroll
  for (int q = 0; q < LB; ++q) {
    const bool neg = (gl >> (LB - 1 - q)) & 1;
#pragma unroll
    for (int k = 0; k <= NT; ++k) out[k][q] = neg ? -tot[k] : tot[k];
  }
#pragma unroll
  for (int m = 1; m < G; m <<= 1)
#pragma unroll
    for (int k = 0; k <= NT; ++k)
#pragma unroll
      for (int q = 0; q < N; ++q) out[k][q] += __shfl_xor_sync(0xffffffffu, out[k][q], m);
}

template <typename T>
__device__ __forceinline__ void atomic_max_abs(unsigned long long* dst, T v) {
  atomicMax(dst, (unsigned long long)__double_as_longlong((double)v));
}

// ---- K1: forward + tangents ----------------------------------------------------
template <typename T, int N, bool TAN>
__global__ void __launch_bounds__(kThreads)
pqc_forward_kernel(PlanDev plan, int scale, int64_t R, const T* __restrict__ act,
                   const T* __restrict__ act_tan, const T* __restrict__ qp, T* __restrict__ z,
                   T* __restrict__ dz, unsigned long long* __restrict__ maxabs) {
  using Gm = Geo<T, N, false>;
  constexpr int AB = Gm::AB, A = Gm::A, LB = Gm::LB, G = Gm::G, SPW = Gm::SPW;
  constexpr int NT = TAN ? 3 : 0, NS = 1 + NT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warps = blockDim.x >> 5;
  Smem<T, N, AB> sm;
  smem_layout<T, N, AB>(plan, warps, false, &sm, smem_raw);
  prologue<T, N, AB, G>(plan, qp, sm, false, warps);
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane >> LB, gl = lane & (G - 1);
  cplx<T>* buf = sm.buf + warp * 32 * A;
  const int n_steps = plan.n_steps;
  T amax = T(0);
  const int64_t stride = (int64_t)gridDim.x * warps * SPW;
  for (int64_t base = ((int64_t)blockIdx.x * warps + warp) * SPW; base < R; base += stride) {
    const int64_t s = base + grp;
    const bool valid = s < R;
    T c[N], sn[N], dth[3][N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
      T a = valid ? act[s * N + q] : T(0);
      amax = fmax(amax, fabs(a));
      a = fmin(fmax(a, T(-1)), T(1));
      T th, s1, s2;
      scale_fn<T>(scale, a, th, s1, s2);
      sincos_(th * T(0.5), &sn[q], &c[q]);
#pragma unroll
      for (int k = 0; k < 3; ++k)
        dth[k][q] = (TAN && valid) ? s1 * act_tan[((int64_t)k * R + s) * N + q] : T(0);
    }
    cplx<T> st[NS][A];
    embed<T, N, AB, NT>(c, sn, dth, gl, st);
    for (int si = 0; si < n_steps; ++si) {
      const int h = sm.steps[2 * si], idx = sm.steps[2 * si + 1];
      const int type = h & 3, wire = (h >> 2) - 1;
      if (type == STEP_U1) {
        const cplx<T>* U = sm.U + 4 * idx;
        apply_u1<T, N, AB, NS>(st, wire, gl, U[0], U[1], U[2], U[3]);
      } else if (type == STEP_PERM) {
        permute<T, A, G, SPW, NS>(st, sm.pt + idx * Gm::D, buf, gl, grp);
      } else {
        const cplx<T>* ph = sm.ph + idx * Gm::D;
#pragma unroll
        for (int r = 0; r < A; ++r) {
          const cplx<T> e = ph[r * G + gl];
#pragma unroll
          for (int j = 0; j < NS; ++j) st[j][r] = cmul(st[j][r], e);
        }
      }
    }
    T out[NS][N];
    readout<T, N, AB, NT>(st, gl, out);
    if (valid) {
#pragma unroll
      for (int v = 0; v < NS * N; ++v) {
        if ((v % G) != gl) continue;
        const int k = v / N, q = v % N;
        if (k == 0) z[s * N + q] = out[0][q];
        else dz[((int64_t)(k - 1) * R + s) * N + q] = out[k][q];
      }
    }
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, m));
  if (lane == 0 && maxabs) atomic_max_abs(maxabs, amax);
}

// ---- K2: adjoint backward ----------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}

template <typename T, int N>
__global__ void __launch_bounds__(kThreads)
pqc_backward_kernel(PlanDev plan, int scale, int64_t R, const T* __restrict__ act,
                    const T* __restrict__ act_tan, const T* __restrict__ qp,
                    const T* __restrict__ gz, const T* __restrict__ gdz, T* __restrict__ g_act,
                    T* __restrict__ g_act_tan, double* __restrict__ partial) {
  using Gm = Geo<T, N, true>;
  constexpr int AB = Gm::AB, A = Gm::A, LB = Gm::LB, G = Gm::G, SPW = Gm::SPW, D = Gm::D;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warps = blockDim.x >> 5;
  Smem<T, N, AB> sm;
  smem_layout<T, N, AB>(plan, warps, true, &sm, smem_raw);
  prologue<T, N, AB, G>(plan, qp, sm, true, warps);
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane >> LB, gl = lane & (G - 1);
  cplx<T>* buf = sm.buf + warp * 32 * A;
  const int n_acc = 8 * plan.n_u1 + D * plan.n_phase;
  T* accU = sm.acc + (size_t)warp * n_acc;
  T* accP = accU + 8 * plan.n_u1;
  const int n_steps = plan.n_steps;
  const int64_t stride = (int64_t)gridDim.x * warps * SPW;
  for (int64_t base = ((int64_t)blockIdx.x * warps + warp) * SPW; base < R; base += stride) {
    const int64_t s = base + grp;
    const bool valid = s < R;
    T c[N], sn[N], dth[3][N], s1v[N], s2v[N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
      T a = valid ? act[s * N + q] : T(0);
      a = fmin(fmax(a, T(-1)), T(1));
      T th;
      scale_fn<T>(scale, a, th, s1v[q], s2v[q]);
      sincos_(th * T(0.5), &sn[q], &c[q]);
#pragma unroll
      for (int k = 0; k < 3; ++k)
        dth[k][q] = valid ? s1v[q] * act_tan[((int64_t)k * R + s) * N + q] : T(0);
    }
    cplx<T> x[4][A];
    embed<T, N, AB, 3>(c, sn, dth, gl, x);
    // forward replay
    for (int si = 0; si < n_steps; ++si) {
      const int h = sm.steps[2 * si], idx = sm.steps[2 * si + 1];
      const int type = h & 3, wire = (h >> 2) - 1;
      if (type == STEP_U1) {
        const cplx<T>* U = sm.U + 4 * idx;
        apply_u1<T, N, AB, 4>(x, wire, gl, U[0], U[1], U[2], U[3]);
      } else if (type == STEP_PERM) {
        permute<T, A, G, SPW, 4>(x, sm.pt + idx * D, buf, gl, grp);
      } else {
        const cplx<T>* ph = sm.ph + idx * D;
#pragma unroll
        for (int r = 0; r < A; ++r) {
          const cplx<T> e = ph[r * G + gl];
#pragma unroll
          for (int j = 0; j < 4; ++j) x[j][r] = cmul(x[j][r], e);
        }
      }
    }
    // adjoint seeds: lambda = 2 w psi + 2 sum_k v_k dpsi_k, mu_k = 2 v_k psi
    T gv[4][N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
      gv[0][q] = valid ? gz[s * N + q] : T(0);
#pragma unroll
      for (int k = 0; k < 3; ++k) gv[1 + k][q] = valid ? gdz[((int64_t)k * R + s) * N + q] : T(0);
    }
    T wl[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      wl[k] = T(0);
#pragma unroll
      for (int q = 0; q < LB; ++q) wl[k] += ((gl >> (LB - 1 - q)) & 1) ? -gv[k][q] : gv[k][q];
    }
    cplx<T> ad[4][A];
#pragma unroll
    for (int r = 0; r < A; ++r) {
      T w[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        w[k] = wl[k];
#pragma unroll
        for (int qi = 0; qi < AB; ++qi)
          w[k] += ((r >> (AB - 1 - qi)) & 1) ? -gv[k][LB + qi] : gv[k][LB + qi];
        w[k] *= T(2);
      }
      cplx<T> l;
      l.re = w[0] * x[0][r].re + w[1] * x[1][r].re + w[2] * x[2][r].re + w[3] * x[3][r].re;
      l.im = w[0] * x[0][r].im + w[1] * x[1][r].im + w[2] * x[2][r].im + w[3] * x[3][r].im;
      ad[0][r] = l;
#pragma unroll
      for (int k = 0; k < 3; ++k) ad[1 + k][r] = {w[1 + k] * x[0][r].re, w[1 + k] * x[0][r].im};
    }
    // reverse sweep
    for (int si = n_steps - 1; si >= 0; --si) {
      const int h = sm.steps[2 * si], idx = sm.steps[2 * si + 1];
      const int type = h & 3, wire = (h >> 2) - 1;
      if (type == STEP_U1) {
        const cplx<T>* U = sm.U + 4 * idx;
        // U^dagger
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
          for (int r = 0; r < A; ++r)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const cplx<T> xp = shfl_xor_c(x[j][r], 1 << lb);
              const cplx<T> ap = shfl_xor_c(ad[j][r], 1 << lb);
              const cplx<T> xs = x[j][r], as = ad[j][r];
              const cplx<T> t1 = cmulc(as, xs), t2 = cmulc(as, xp);
              ms_re += t1.re; ms_im += t1.im; mc_re += t2.re; mc_im += t2.im;
              x[j][r] = cmul2(cs, xs, cp, xp);
              ad[j][r] = cmul2(cs, as, cp, ap);
            }
          // M'[i][j] (i = own row, j = column): beta=0 -> (0,0),(0,1); beta=1 -> (1,1),(1,0)
          if (!beta) { m[0] = ms_re; m[1] = ms_im; m[2] = mc_re; m[3] = mc_im; }
          else { m[6] = ms_re; m[7] = ms_im; m[4] = mc_re; m[5] = mc_im; }
        } else {
          const int rb = N - 1 - wire;
#pragma unroll
          for (int r = 0; r < A; ++r) {
            // runtime register bit: handled by a predicated, fully unrolled pair loop
#pragma unroll
            for (int bsel = 0; bsel < AB; ++bsel) {
              if (bsel != rb) continue;
              if (r & (1 << bsel)) continue;
              const int r1 = r | (1 << bsel);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const cplx<T> x0 = x[j][r], x1 = x[j][r1], a0 = ad[j][r], a1 = ad[j][r1];
                cplx<T> t;
                t = cmulc(a0, x0); m[0] += t.re; m[1] += t.im;
                t = cmulc(a0, x1); m[2] += t.re; m[3] += t.im;
                t = cmulc(a1, x0); m[4] += t.re; m[5] += t.im;
                t = cmulc(a1, x1); m[6] += t.re; m[7] += t.im;
                x[j][r] = cmul2(h00, x0, h01, x1);
                x[j][r1] = cmul2(h10, x0, h11, x1);
                ad[j][r] = cmul2(h00, a0, h01, a1);
                ad[j][r1] = cmul2(h10, a0, h11, a1);
              }
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
        permute<T, A, G, SPW, 4>(x, sm.pti + idx * D, buf, gl, grp);
        permute<T, A, G, SPW, 4>(ad, sm.pti + idx * D, buf, gl, grp);
      } else {
        const cplx<T>* ph = sm.ph + idx * D;
        T* acc = accP + idx * D;
#pragma unroll
        for (int r = 0; r < A; ++r) {
          T pv = T(0);
#pragma unroll
          for (int j = 0; j < 4; ++j) pv += ad[j][r].im * x[j][r].re - ad[j][r].re * x[j][r].im;
#pragma unroll
          for (int m = G; m < 32; m <<= 1) pv += __shfl_xor_sync(0xffffffffu, pv, m);
          if (grp == 0) acc[r * G + gl] += pv;
          const cplx<T> e = {ph[r * G + gl].re, -ph[r * G + gl].im};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            x[j][r] = cmul(x[j][r], e);
            ad[j][r] = cmul(ad[j][r], e);
          }
        }
      }
    }
    // embedding gradient: phibar = ad[0], mu_k = ad[1+k]
    embed<T, N, AB, 0>(c, sn, dth, gl, *reinterpret_cast<cplx<T>(*)[1][A]>(&x[0][0]));
    // rho_k = sum_q dth_kq X_q mu_k  -> x[1+k]
#pragma unroll
    for (int r = 0; r < A; ++r)
#pragma unroll
      for (int k = 0; k < 3; ++k) x[1 + k][r] = {T(0), T(0)};
#pragma unroll
    for (int q = 0; q < LB; ++q) {
      const int lm = 1 << (LB - 1 - q);
#pragma unroll
      for (int r = 0; r < A; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const cplx<T> p = shfl_xor_c(ad[1 + k][r], lm);
          x[1 + k][r].re += dth[k][q] * p.re;
          x[1 + k][r].im += dth[k][q] * p.im;
        }
    }
#pragma unroll
    for (int qi = 0; qi < AB; ++qi) {
      const int S = 1 << (AB - 1 - qi);
#pragma unroll
      for (int r = 0; r < A; ++r)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          x[1 + k][r].re += dth[k][LB + qi] * ad[1 + k][r ^ S].re;
          x[1 + k][r].im += dth[k][LB + qi] * ad[1 + k][r ^ S].im;
        }
    }
    // eta = (i/2) phibar - 1/4 sum_k rho_k  -> ad[0]
#pragma unroll
    for (int r = 0; r < A; ++r) {
      const T er = T(-0.5) * ad[0][r].im - T(0.25) * (x[1][r].re + x[2][r].re + x[3][r].re);
      const T ei = T(0.5) * ad[0][r].re - T(0.25) * (x[1][r].im + x[2][r].im + x[3][r].im);
      ad[0][r] = {er, ei};
    }
    // g_theta_q = Re<eta, X_q phi>, g_dtheta_kq = Re<(i/2) mu_k, X_q phi>
    T gt[4][N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
#pragma unroll
      for (int k = 0; k < 4; ++k) gt[k][q] = T(0);
      const bool lanew = q < LB;
#pragma unroll
      for (int r = 0; r < A; ++r) {
        cplx<T> y;
        if (lanew) {
          y = shfl_xor_c(x[0][r], 1 << (LB - 1 - q));
        } else {
          y = x[0][r ^ (1 << (N - 1 - q))];
        }
        gt[0][q] += ad[0][r].re * y.re + ad[0][r].im * y.im;
#pragma unroll
        for (int k = 0; k < 3; ++k)
          gt[1 + k][q] += T(0.5) * (ad[1 + k][r].re * y.im - ad[1 + k][r].im * y.re);
      }
    }
#pragma unroll
    for (int m = 1; m < G; m <<= 1)
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int q = 0; q < N; ++q) gt[k][q] += __shfl_xor_sync(0xffffffffu, gt[k][q], m);
    if (valid) {
#pragma unroll
      for (int v = 0; v < 4 * N; ++v) {
        if ((v % G) != gl) continue;
        const int k = v / N, q = v % N;
        if (k == 0) {
          T ga = gt[0][q] * s1v[q];
#pragma unroll
          for (int kk = 0; kk < 3; ++kk)
            ga += gt[1 + kk][q] * s2v[q] * act_tan[((int64_t)kk * R + s) * N + q];
          g_act[s * N + q] = ga;
        } else {
          g_act_tan[((int64_t)(k - 1) * R + s) * N + q] = gt[k][q] * s1v[q];
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

// grid-level reduction of block partials (fixed order), then gate-space
// gradients -> parameter slots
__global__ void pqc_reduce_partials(const double* __restrict__ partial, int blocks, int n_acc,
                                    double* __restrict__ tot) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_acc) return;
  double v = 0.0;
  for (int b = 0; b < blocks; ++b) v += partial[(size_t)b * n_acc + i];
  tot[i] = v;
}

template <typename T, int AB, int G>
__global__ void pqc_param_grads(PlanDev p, const T* __restrict__ qp, const double* __restrict__ tot,
                                T* __restrict__ g_qp) {
  const int D = 1 << p.n;
  const double* accP = tot + 8 * p.n_u1;
  for (int i = threadIdx.x; i < p.n_u1; i += blockDim.x) {
    const int kind = p.u1[i * 4];
    double th[3] = {0, 0, 0};
    const int ns = u1_nslots(kind);
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
    for (int j = 0; j < ns; ++j) {
      double dU[8];
      u1_dmatrix_d(kind, th, j, dU);
      double g = 0.0;  // Re sum_ij dU_ij M_ij
      for (int e = 0; e < 4; ++e) g += dU[2 * e] * M[2 * e] - dU[2 * e + 1] * M[2 * e + 1];
      g_qp[p.u1[i * 4 + 1 + j]] = T(g);
    }
  }
  for (int st = 0; st < p.n_phase; ++st) {
    for (int k = p.phase_off[st] + threadIdx.x; k < p.phase_off[st + 1]; k += blockDim.x) {
      const int c = p.pairs[3 * k], t = p.pairs[3 * k + 1], s = p.pairs[3 * k + 2];
      double g = 0.0;
      for (int b = 0; b < D; ++b) {
        const int on = (b >> (p.n - 1 - c)) & 1, tb = (b >> (p.n - 1 - t)) & 1;
        if (on) g += (tb - 0.5) * accP[st * D + lay<AB, G>(b)];
      }
      g_qp[s] = T(g);
    }
  }
}

// ---- host launchers -------------------------------------------------------------
struct LaunchInfo {
  int grid;
  size_t smem;
};

template <typename K>
static int occupancy_blocks(K kernel, size_t smem) {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, kThreads, smem);
  return nb > 0 ? nb : 1;
}

template <typename T, int N, bool BWD>
static size_t smem_bytes(const PlanDev& p) {
  using Gm = Geo<T, N, BWD>;
  return smem_layout<T, N, Gm::AB>(p, kThreads / 32, BWD, nullptr, nullptr);
}

template <typename T, int N, bool BWD>
static int grid_for(int64_t R, size_t smem, void* kernel_ptr, int occ) {
  using Gm = Geo<T, N, BWD>;
  const int64_t per_block = (int64_t)(kThreads / 32) * Gm::SPW;
  int64_t need = (R + per_block - 1) / per_block;
  int64_t cap = (int64_t)num_sms() * occ;
  int64_t g = need < cap ? need : cap;
  return (int)(g < 1 ? 1 : g);
}

static std::mutex g_attr_mu;

template <typename T, int N>
static int launch_forward(qpinn_circuit* c, int scale, int64_t R, const T* act, const T* tan,
                          const T* qp, T* z, T* dz, unsigned long long* maxabs,
                          cudaStream_t stream) {
  const PlanDev& p = c->dev;
  const size_t smem = smem_bytes<T, N, false>(p);
  if (smem > 227 * 1024) return fail(QPINN_ERR_CAPACITY, "PQC plan tables exceed shared memory");
  auto kern = tan ? pqc_forward_kernel<T, N, true> : pqc_forward_kernel<T, N, false>;
  {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    QPINN_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
  }
  const int occ = occupancy_blocks(kern, smem);
  const int grid = grid_for<T, N, false>(R, smem, (void*)kern, occ);
  kern<<<grid, kThreads, smem, stream>>>(p, scale, R, act, tan, qp, z, dz, maxabs);
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

template <typename T, int N>
static int backward_grid(qpinn_circuit* c, int64_t R, size_t* smem_out) {
  const size_t smem = smem_bytes<T, N, true>(c->dev);
  *smem_out = smem;
  auto kern = pqc_backward_kernel<T, N>;
  {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  const int occ = occupancy_blocks(kern, smem);
  return grid_for<T, N, true>(R, smem, (void*)kern, occ);
}

template <typename T, int N>
static int launch_backward(qpinn_circuit* c, int scale, int64_t R, const T* act, const T* tan,
                           const T* qp, const T* gz, const T* gdz, T* g_act, T* g_tan, T* g_qp,
                           double* partial, double* tot, cudaStream_t stream) {
  using Gm = Geo<T, N, true>;
  const PlanDev& p = c->dev;
  size_t smem = 0;
  const int grid = backward_grid<T, N>(c, R, &smem);
  if (smem > 227 * 1024) return fail(QPINN_ERR_CAPACITY, "PQC plan tables exceed shared memory");
  const int n_acc = 8 * p.n_u1 + Gm::D * p.n_phase;
  pqc_backward_kernel<T, N><<<grid, kThreads, smem, stream>>>(p, scale, R, act, tan, qp, gz, gdz,
                                                              g_act, g_tan, partial);
  QPINN_CUDA_CHECK(cudaGetLastError());
  if (n_acc > 0) {
    pqc_reduce_partials<<<(n_acc + 255) / 256, 256, 0, stream>>>(partial, grid, n_acc, tot);
    QPINN_CUDA_CHECK(cudaGetLastError());
  }
  pqc_param_grads<T, Gm::AB, Gm::G><<<1, 256, 0, stream>>>(p, qp, tot, g_qp);
  QPINN_CUDA_CHECK(cudaGetLastError());
  return QPINN_OK;
}

// runtime n -> template instantiation
#define QPINN_DISPATCH_N(MAXN, N_RT, CALL)                       \
  switch (N_RT) {                                                \
    case 1: if constexpr (1 <= MAXN) { constexpr int NN = 1; return CALL; } break; \
    case 2: if constexpr (2 <= MAXN) { constexpr int NN = 2; return CALL; } break; \
    case 3: if constexpr (3 <= MAXN) { constexpr int NN = 3; return CALL; } break; \
    case 4: if constexpr (4 <= MAXN) { constexpr int NN = 4; return CALL; } break; \
    case 5: if constexpr (5 <= MAXN) { constexpr int NN = 5; return CALL; } break; \
    case 6: if constexpr (6 <= MAXN) { constexpr int NN = 6; return CALL; } break; \
    case 7: if constexpr (7 <= MAXN) { constexpr int NN = 7; return CALL; } break; \
    case 8: if constexpr (8 <= MAXN) { constexpr int NN = 8; return CALL; } break; \
    case 9: if constexpr (9 <= MAXN) { constexpr int NN = 9; return CALL; } break; \
    default: break;                                              \
  }

// workspace: [0,256) max|a| (u64 double bits) | [256, ...) block partials | totals
template <typename T>
static size_t workspace_for(qpinn_circuit* c, int64_t R) {
  const int n = c->n;
  if (n > max_qubits<T, true>()) return 256;
  const size_t n_acc = 8 * (size_t)c->n_u1 + ((size_t)1 << n) * c->n_phase;
  // grid cap: every SM at the maximum residency the backward kernel can reach
  const size_t blocks = (size_t)num_sms() * 16;
  (void)R;
  return 256 + align_up(sizeof(double) * n_acc * blocks, 256) + align_up(sizeof(double) * n_acc, 256);
}

}  // namespace qpinn

using namespace qpinn;

extern "C" {

int qpinn_pqc_max_qubits(int dtype) {
  return dtype == QPINN_F64 ? max_qubits<double, true>() : max_qubits<float, true>();
}

size_t qpinn_pqc_workspace_bytes(const qpinn_circuit* c, int dtype, int64_t rows) {
  if (!c) return 0;
  return dtype == QPINN_F64 ? workspace_for<double>(const_cast<qpinn_circuit*>(c), rows)
                            : workspace_for<float>(const_cast<qpinn_circuit*>(c), rows);
}

static int check_common(const qpinn_circuit* c, int dtype, int scale, int64_t rows, size_t ws_bytes,
                        size_t need) {
  if (!c) return fail(QPINN_ERR_CONFIG, "null circuit");
  if (dtype != QPINN_F32 && dtype != QPINN_F64) return fail(QPINN_ERR_CONFIG, "bad dtype");
  if (scale < 0 || scale > 4) return fail(QPINN_ERR_CONFIG, "unknown scale kind");
  if (rows < 0) return fail(QPINN_ERR_INVALID_BATCH, "negative row count");
  if (ws_bytes < need) return fail(QPINN_ERR_CONFIG, "workspace too small");
  return QPINN_OK;
}

int qpinn_pqc_forward(const qpinn_circuit* cc, int dtype, int scale, int64_t rows,
                      const void* act_val, const void* act_tan, const void* qparams, void* z,
                      void* dz, void* workspace, size_t workspace_bytes, void* stream) {
  qpinn_circuit* c = const_cast<qpinn_circuit*>(cc);
  int rc = check_common(c, dtype, scale, rows, workspace_bytes, 256);
  if (rc) return rc;
  if ((act_tan == nullptr) != (dz == nullptr))
    return fail(QPINN_ERR_CONFIG, "act_tan and dz must both be given or both be NULL");
  const int n = c->n;
  const int maxn = dtype == QPINN_F64 ? max_qubits<double, false>() : max_qubits<float, false>();
  if (n > maxn) return fail(QPINN_ERR_CAPACITY, "n_qubits beyond the register-resident kernels");
  rc = ensure_device_plan(c);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  auto* maxabs = (unsigned long long*)workspace;  // running max, reset by domain_check
  if (rows == 0) return QPINN_OK;
  if (dtype == QPINN_F32) {
    QPINN_DISPATCH_N(8, n, (launch_forward<float, NN>(c, scale, rows, (const float*)act_val,
                                                      (const float*)act_tan, (const float*)qparams,
                                                      (float*)z, (float*)dz, maxabs, st)));
  } else {
    QPINN_DISPATCH_N(7, n, (launch_forward<double, NN>(c, scale, rows, (const double*)act_val,
                                                       (const double*)act_tan,
                                                       (const double*)qparams, (double*)z,
                                                       (double*)dz, maxabs, st)));
  }
  return fail(QPINN_ERR_CAPACITY, "unsupported n_qubits");
}

int qpinn_pqc_backward(const qpinn_circuit* cc, int dtype, int scale, int64_t rows,
                       const void* act_val, const void* act_tan, const void* qparams,
                       const void* g_z, const void* g_dz, void* g_act_val, void* g_act_tan,
                       void* g_qparams, void* workspace, size_t workspace_bytes, void* stream) {
  qpinn_circuit* c = const_cast<qpinn_circuit*>(cc);
  const size_t need = qpinn_pqc_workspace_bytes(c, dtype, rows);
  int rc = check_common(c, dtype, scale, rows, workspace_bytes, need);
  if (rc) return rc;
  if (!act_tan || !g_z || !g_dz || !g_act_val || !g_act_tan || !g_qparams)
    return fail(QPINN_ERR_CONFIG, "backward needs tangents and all gradient buffers");
  const int n = c->n;
  if (n > qpinn_pqc_max_qubits(dtype))
    return fail(QPINN_ERR_CAPACITY, "n_qubits beyond the register-resident kernels");
  rc = ensure_device_plan(c);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t n_acc = 8 * (size_t)c->n_u1 + ((size_t)1 << n) * c->n_phase;
  double* partial = (double*)((char*)workspace + 256);
  double* tot = (double*)((char*)workspace + 256 +
                          align_up(sizeof(double) * n_acc * (size_t)num_sms() * 16, 256));
  if (rows == 0) {
    QPINN_CUDA_CHECK(cudaMemsetAsync(g_qparams, 0,
                                     (dtype == QPINN_F64 ? 8 : 4) * (size_t)c->n_params, st));
    return QPINN_OK;
  }
  if (dtype == QPINN_F32) {
    QPINN_DISPATCH_N(8, n, (launch_backward<float, NN>(
                               c, scale, rows, (const float*)act_val, (const float*)act_tan,
                               (const float*)qparams, (const float*)g_z, (const float*)g_dz,
                               (float*)g_act_val, (float*)g_act_tan, (float*)g_qparams, partial,
                               tot, st)));
  } else {
    QPINN_DISPATCH_N(7, n, (launch_backward<double, NN>(
                               c, scale, rows, (const double*)act_val, (const double*)act_tan,
                               (const double*)qparams, (const double*)g_z, (const double*)g_dz,
                               (double*)g_act_val, (double*)g_act_tan, (double*)g_qparams, partial,
                               tot, st)));
  }
  return fail(QPINN_ERR_CAPACITY, "unsupported n_qubits");
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
