// Gate algebra shared by the PQC kernels: the scaled angle embedding and the
// fused single-qubit step matrices and their parameter derivatives.
#pragma once
#include "common.cuh"

namespace qpinn {

constexpr double kPi = 3.14159265358979323846;

__device__ __forceinline__ void sincos_(float x, float* s, float* c) { sincosf(x, s, c); }
__device__ __forceinline__ void sincos_(double x, double* s, double* c) { sincos(x, s, c); }

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

}  // namespace qpinn
