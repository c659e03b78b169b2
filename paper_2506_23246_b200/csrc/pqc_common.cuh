// Device helpers shared by the generic (runtime-plan) and the compile-time
// specialised PQC kernels: lane geometry, shared-memory tables, the
// closed-form embedding, gate application and the point loader.
#pragma once
#include <utility>

#include "gates.cuh"

namespace qpinn {

// ---- lane geometry -----------------------------------------------------------------
// AB register bits per lane: n <= 4 -> all in registers; else max(4, n - 3),
// so that one state of a point spans at most 8 lanes.
template <typename T, int N, int NSL>
struct Geo {
  static constexpr int AB = N <= 4 ? N : (N - 3 > 4 ? N - 3 : 4);
  static constexpr int A = 1 << AB;
  static constexpr int LB = N - AB;
  static constexpr int G = 1 << LB;
  static constexpr int LPP = NSL * G;  // lanes per point
  static constexpr int SPW = 32 / LPP;  // points per warp
  static constexpr int D = 1 << N;
  static_assert(LPP <= 32, "one point must fit in a warp");
};

template <typename T>
constexpr int max_qubits() { return sizeof(T) == 8 ? 7 : 8; }

constexpr int kThreads = 128;  // 4 warps per block

// shared-memory / hand-off layout index of basis state b within one state
template <int AB, int G>
__host__ __device__ __forceinline__ int lay(int b) {
  return (b & ((1 << AB) - 1)) * G + (b >> AB);
}

// ---- fused step list as a by-value kernel parameter --------------------------------
// Step descriptors live in the constant bank, so the per-step dispatch is
// provably warp-uniform: no divergence barriers around the shuffles.
constexpr int kMaxKSteps = 256;
struct StepTable {
  int n;
  int2 s[kMaxKSteps];  // {type | (wire + 1) << 2, table index}
};

// ---- block prologue: gate matrices, phase tables, permutation tables --------
template <typename T>
struct Smem {
  cplx<T>* U;     // [n_u1][4]
  cplx<T>* ph;    // [n_phase][D] at lay(b)
  uint16_t* pt;   // [n_perm][D]  lay(perm[b]) at lay(b)
  uint16_t* pti;  // [n_perm][D]  lay(iperm[b]) at lay(b)
  cplx<T>* buf;   // per-warp permutation buffer [warps][2][32 * A]
  T* acc;         // K2: per-warp gradient accumulators [warps][n_acc]
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

template <typename T, int N, int AB>
__host__ __device__ inline size_t smem_layout(const PlanDev& p, int warps, bool bwd, Smem<T>* out,
                                              unsigned char* base) {
  constexpr int D = 1 << N;
  constexpr int A = 1 << AB;
  size_t o = 0;
  size_t oU = o; o = align_up(o + sizeof(cplx<T>) * 4 * p.n_u1, 16);
  size_t oPh = o; o = align_up(o + sizeof(cplx<T>) * (size_t)D * p.n_phase, 16);
  size_t oPt = o; o = align_up(o + 2 * (size_t)D * p.n_perm, 16);
  size_t oPti = o; o = align_up(o + (bwd ? 2 * (size_t)D * p.n_perm : 0), 16);
  size_t oBuf = o; o = align_up(o + sizeof(cplx<T>) * 32 * A * (bwd ? 2 : 1) * (size_t)warps, 16);
  size_t oAcc = o;
  if (bwd) o = align_up(o + sizeof(T) * (size_t)warps * (8 * p.n_u1 + (size_t)D * p.n_phase), 16);
  if (out) {
    out->U = (cplx<T>*)(base + oU);
    out->ph = (cplx<T>*)(base + oPh);
    out->pt = (uint16_t*)(base + oPt);
    out->pti = (uint16_t*)(base + oPti);
    out->buf = (cplx<T>*)(base + oBuf);
    out->acc = (T*)(base + oAcc);
  }
  return o;
}

template <typename T, int N, int AB, int G>
__device__ void prologue(const PlanDev& p, const T* __restrict__ qp, const Smem<T>& sm, bool bwd,
                         int warps) {
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
  if (bwd) {
    const size_t nacc = (size_t)warps * (8 * p.n_u1 + (size_t)D * p.n_phase);
    for (size_t i = tid; i < nacc; i += nt) sm.acc[i] = T(0);
  }
}

// ---- per-point embedding (ansatz.py:233-243, :380-390) in closed form --------
// State s of the point: s = 0 -> phi = prod_q RX(theta_q)|0>; s = k+1 ->
// d phi/dx_k = sum_q dtheta_kq d phi/dtheta_q.  Every amplitude is a real
// magnitude times (-i)^popcount(b); the tangent replaces one factor by its
// derivative (forward-mode product rule), which leaves the phase unchanged.
template <typename T, int N, int AB>
__device__ __forceinline__ void embed(const T (&c)[N], const T (&sn)[N], const T (&dth)[N],
                                      bool tangent, int gl, cplx<T> (&st)[1 << AB]) {
  constexpr int A = 1 << AB, LB = N - AB;
  T mL = T(1), dL = T(0);
#pragma unroll
  for (int q = 0; q < LB; ++q) {
    const int bit = (gl >> (LB - 1 - q)) & 1;
    const T f = bit ? sn[q] : c[q];
    const T df = bit ? T(0.5) * c[q] : T(-0.5) * sn[q];
    dL = dL * f + mL * dth[q] * df;
    mL *= f;
  }
  // register wires by doubling (wire LB is the most significant register bit);
  // magnitudes in .re, their tangent in .im
  st[0].re = T(1);
  st[0].im = T(0);
#pragma unroll
  for (int qi = 0; qi < AB; ++qi) {
    const int q = LB + qi;
#pragma unroll
    for (int i = (1 << qi) - 1; i >= 0; --i) {
      const T m = st[i].re, d = st[i].im;
      st[2 * i + 1].im = d * sn[q] + m * dth[LB + qi] * (T(0.5) * c[q]);
      st[2 * i].im = d * c[q] + m * dth[LB + qi] * (T(-0.5) * sn[q]);
      st[2 * i + 1].re = m * sn[q];
      st[2 * i].re = m * c[q];
    }
  }
  const int popL = __popc(gl);
#pragma unroll
  for (int r = 0; r < A; ++r) {
    const int ph = (popL + __popc(r)) & 3;  // (-i)^popcount
    const T m = tangent ? dL * st[r].re + mL * st[r].im : mL * st[r].re;
    st[r].re = (ph == 0) ? m : (ph == 2) ? -m : T(0);
    st[r].im = (ph == 1) ? -m : (ph == 3) ? m : T(0);
  }
}

// ---- gate application (NR register-resident arrays sharing one gate) ----------
template <int RB, typename T, int A, int NR>
__device__ __forceinline__ void gate_reg(cplx<T> (&st)[NR][A], cplx<T> u00, cplx<T> u01,
                                         cplx<T> u10, cplx<T> u11) {
#pragma unroll
  for (int r = 0; r < A; ++r) {
    if (r & (1 << RB)) continue;
    const int r1 = r | (1 << RB);
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const cplx<T> a0 = st[j][r], a1 = st[j][r1];
      st[j][r] = cmul2(u00, a0, u01, a1);
      st[j][r1] = cmul2(u10, a0, u11, a1);
    }
  }
}

template <typename T, int A, int NR>
__device__ __forceinline__ void gate_lane(cplx<T> (&st)[NR][A], int lm, bool beta, cplx<T> u00,
                                          cplx<T> u01, cplx<T> u10, cplx<T> u11) {
  const cplx<T> cs = beta ? u11 : u00, cp = beta ? u10 : u01;
#pragma unroll
  for (int r = 0; r < A; ++r)
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const cplx<T> p = shfl_xor_c(st[j][r], lm);
      st[j][r] = cmul2(cs, st[j][r], cp, p);
    }
}

template <typename T, int N, int AB, int NR>
__device__ __forceinline__ void apply_u1(cplx<T> (&st)[NR][1 << AB], int wire, int gl, cplx<T> u00,
                                         cplx<T> u01, cplx<T> u10, cplx<T> u11) {
  constexpr int LB = N - AB, A = 1 << AB;
  if (wire < LB) {
    const int lb = LB - 1 - wire;
    gate_lane<T, A, NR>(st, 1 << lb, (gl >> lb) & 1, u00, u01, u10, u11);
  } else {
    const int rb = N - 1 - wire;
    if (rb == 0) gate_reg<0, T, A, NR>(st, u00, u01, u10, u11);
    if constexpr (AB > 1) if (rb == 1) gate_reg<1, T, A, NR>(st, u00, u01, u10, u11);
    if constexpr (AB > 2) if (rb == 2) gate_reg<2, T, A, NR>(st, u00, u01, u10, u11);
    if constexpr (AB > 3) if (rb == 3) gate_reg<3, T, A, NR>(st, u00, u01, u10, u11);
    if constexpr (AB > 4) if (rb == 4) gate_reg<4, T, A, NR>(st, u00, u01, u10, u11);
  }
}

// new[b] = old[table[b]] through the warp's shared buffer; every lane moves
// its own state's A amplitudes (lane-fastest layout: conflict-free writes)
template <typename T, int A, int G, int NR>
__device__ __forceinline__ void permute(cplx<T> (&st)[NR][A], const uint16_t* tab, cplx<T>* buf,
                                        int gl, int lane_hi) {
  constexpr int W = 32 / G;  // lanes sharing one gl
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    cplx<T>* bj = buf + j * 32 * A;
#pragma unroll
    for (int r = 0; r < A; ++r) bj[(r * G + gl) * W + lane_hi] = st[j][r];
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < A; ++r) {
    const int src = tab[r * G + gl] * W + lane_hi;
#pragma unroll
    for (int j = 0; j < NR; ++j) st[j][r] = buf[j * 32 * A + src];
  }
  __syncwarp();
}

template <typename T>
__device__ __forceinline__ void atomic_max_abs(unsigned long long* dst, T v) {
  atomicMax(dst, (unsigned long long)__double_as_longlong((double)v));
}

// loads a, theta, cos/sin(theta/2), S', S'' and the lane's own tangent row
template <typename T, int N>
__device__ __forceinline__ void load_point(int scale, const T* __restrict__ act,
                                           const T* __restrict__ act_tan, int64_t R, int64_t s,
                                           bool valid, int k_own, T (&c)[N], T (&sn)[N],
                                           T (&dth)[N], T (&s1)[N], T (&s2)[N], T& amax) {
#pragma unroll
  for (int q = 0; q < N; ++q) {
    T a = valid ? act[s * N + q] : T(0);
    amax = fmax(amax, fabs(a));
    a = fmin(fmax(a, T(-1)), T(1));
    T th;
    scale_fn<T>(scale, a, th, s1[q], s2[q]);
    sincos_(th * T(0.5), &sn[q], &c[q]);
    dth[q] = (valid && k_own >= 0) ? s1[q] * act_tan[((int64_t)k_own * R + s) * N + q] : T(0);
  }
}

// cos(theta/2), sin(theta/2), S'(a), S''(a) of the scaled embedding angle
// theta = S(a) (ansatz.py:44-67) without inverse trig: for acos/asin the
// half-angle cosines are exactly sqrt((1 +- a)/2) (theta in [0, pi]); the
// linear scalings use sincospi, whose argument reduction is trivial.
__device__ __forceinline__ void sincospi_(float x, float* s, float* c) { sincospif(x, s, c); }
__device__ __forceinline__ void sincospi_(double x, double* s, double* c) { sincospi(x, s, c); }

template <typename T>
__device__ __forceinline__ void half_angle(int kind, T a, T& c, T& s, T& s1, T& s2) {
  const T om = (T(1) - a) * (T(1) + a);
  const T rt = sqrt(om);
  if (kind == QPINN_SCALE_ACOS || kind == QPINN_SCALE_ASIN) {
    const T cp = sqrt((T(1) + a) * T(0.5)), cm = sqrt((T(1) - a) * T(0.5));
    const bool ac = kind == QPINN_SCALE_ACOS;
    c = ac ? cp : cm;           // acos: cos(th/2) = sqrt((1+a)/2); asin: sqrt((1-a)/2)
    s = ac ? cm : cp;
    s1 = (ac ? T(-1) : T(1)) / rt;
    s2 = (ac ? -a : a) / (om * rt);
  } else {
    // none: th/2 = a/2; pi: th/2 = pi a/2; bias: th/2 = pi (a+1)/4
    const T x = kind == QPINN_SCALE_NONE ? a * T(0.5 / kPi)
              : kind == QPINN_SCALE_PI ? a * T(0.5) : (a + T(1)) * T(0.25);
    sincospi_(x, &s, &c);
    s1 = kind == QPINN_SCALE_NONE ? T(1) : kind == QPINN_SCALE_PI ? T(kPi) : T(0.5 * kPi);
    s2 = T(0);
  }
}

template <typename T, int N>
__device__ __forceinline__ void load_point_fast(int scale, const T* __restrict__ act,
                                                const T* __restrict__ act_tan, int64_t R,
                                                int64_t s, bool valid, int k_own, T (&c)[N],
                                                T (&sn)[N], T (&dth)[N], T (&s1)[N], T (&s2)[N],
                                                T& amax) {
#pragma unroll
  for (int q = 0; q < N; ++q) {
    T a = valid ? act[s * N + q] : T(0);
    amax = fmax(amax, fabs(a));
    a = fmin(fmax(a, T(-1)), T(1));
    half_angle<T>(scale, a, c[q], sn[q], s1[q], s2[q]);
    dth[q] = (valid && k_own >= 0) ? s1[q] * act_tan[((int64_t)k_own * R + s) * N + q] : T(0);
  }
}

// load_point_fast with the per-qubit transcendental work spread over the
// point's lanes: lane j < N of the point evaluates qubit j once and the values
// are broadcast with shuffles (the 4G lanes of a point otherwise repeat the
// same N square roots and divisions).  Needs LPP >= N lanes per point (true
// with tangents, NSL = 4); otherwise every lane evaluates every qubit.
template <typename T, int N, int LPP>
__device__ __forceinline__ void load_point_lanes(int scale, const T* __restrict__ act,
                                                 const T* __restrict__ act_tan, int64_t R,
                                                 int64_t s, bool valid, int k_own, int lane,
                                                 T (&c)[N], T (&sn)[N], T (&dth)[N],
                                                 T (&s1)[N], T (&s2)[N], T& amax) {
  if constexpr (LPP < N) {
    load_point_fast<T, N>(scale, act, act_tan, R, s, valid, k_own, c, sn, dth, s1, s2, amax);
    return;
  }
  const int j = lane % LPP, src0 = lane - j;
  T a = (valid && j < N) ? act[s * N + j] : T(0);
  amax = fmax(amax, fabs(a));
  a = fmin(fmax(a, T(-1)), T(1));
  T cj, sj, s1j, s2j;
  half_angle<T>(scale, a, cj, sj, s1j, s2j);
#pragma unroll
  for (int q = 0; q < N; ++q) {
    c[q] = __shfl_sync(0xffffffffu, cj, src0 + q);
    sn[q] = __shfl_sync(0xffffffffu, sj, src0 + q);
    s1[q] = __shfl_sync(0xffffffffu, s1j, src0 + q);
    s2[q] = __shfl_sync(0xffffffffu, s2j, src0 + q);
    dth[q] = (valid && k_own >= 0) ? s1[q] * act_tan[((int64_t)k_own * R + s) * N + q] : T(0);
  }
}

// Per-call gate tables (u1 matrices, phase diagonals, layout-mapped
// permutations) built once by a small kernel into global memory with exactly
// the shared-memory layout of smem_layout(bwd = true); the layer kernels'
// prologue is then a flat copy.
template <typename T, int N>
__global__ void pqc_prepare_tables(PlanDev p, const T* __restrict__ qp,
                                   unsigned char* __restrict__ out) {
  using Gm = Geo<T, N, 4>;
  Smem<T> sm;
  smem_layout<T, N, Gm::AB>(p, 1, true, &sm, out);
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  constexpr int D = Gm::D;
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
    double sp, cp;
    sincos(phi, &sp, &cp);
    sm.ph[st * D + lay<Gm::AB, Gm::G>(b)] = {T(cp), T(sp)};
  }
  for (int i = tid; i < p.n_perm * D; i += nt) {
    const int st = i / D, b = i % D;
    sm.pt[st * D + lay<Gm::AB, Gm::G>(b)] = (uint16_t)lay<Gm::AB, Gm::G>(p.perm[i]);
    sm.pti[st * D + lay<Gm::AB, Gm::G>(b)] = (uint16_t)lay<Gm::AB, Gm::G>(p.iperm[i]);
  }
}

// bytes of the table block (U, ph, pt, pti) = offset of the permutation buffer
template <typename T, int N>
__host__ __device__ inline size_t table_bytes(const PlanDev& p, bool with_inverse) {
  using Gm = Geo<T, N, 4>;
  Smem<T> sm;
  smem_layout<T, N, Gm::AB>(p, 1, true, &sm, nullptr);
  return (size_t)(with_inverse ? (unsigned char*)sm.buf : (unsigned char*)sm.pti) - (size_t)0;
}

// cooperative copy of the prepared tables into shared memory (+ zeroed accumulators)
template <typename T>
__device__ __forceinline__ void copy_tables(const unsigned char* __restrict__ tables, size_t nbytes,
                                            unsigned char* smem, T* acc, size_t n_acc) {
  const int4* src = reinterpret_cast<const int4*>(tables);
  int4* dst = reinterpret_cast<int4*>(smem);
  for (size_t i = threadIdx.x; i < nbytes / 16; i += blockDim.x) dst[i] = src[i];
  for (size_t i = threadIdx.x; i < n_acc; i += blockDim.x) acc[i] = T(0);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}

}  // namespace qpinn

namespace qpinn {

template <int I, int E, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < E) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, E>(f);
  }
}

// 8 values summed over the warp with a reduce-scatter butterfly (9 shuffles);
// afterwards lane l holds the total of value ((l >> 2) & 7)
template <typename T>
__device__ __forceinline__ T warp_reduce8(const T (&m)[8], int lane) {
  T v4[4];
  const bool h16 = lane & 16;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const T send = h16 ? m[i] : m[i + 4];
    v4[i] = (h16 ? m[i + 4] : m[i]) + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  T v2[2];
  const bool h8 = lane & 8;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const T send = h8 ? v4[i] : v4[i + 2];
    v2[i] = (h8 ? v4[i + 2] : v4[i]) + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  const bool h4 = lane & 4;
  T v = (h4 ? v2[1] : v2[0]) + __shfl_xor_sync(0xffffffffu, h4 ? v2[0] : v2[1], 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v;
}

}  // namespace qpinn
