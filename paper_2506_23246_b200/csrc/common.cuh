// Shared definitions for the QPINN B200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "qpinn_b200.h"

namespace qpinn {

// ---- error plumbing (thread-local message, C ABI returns codes) ------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

#define QPINN_CUDA_CHECK(expr)                                  \
  do {                                                          \
    cudaError_t _e = (expr);                                    \
    if (_e != cudaSuccess) return ::qpinn::cuda_fail(_e, #expr); \
  } while (0)

int num_sms();

// ---- complex helpers -------------------------------------------------------
template <typename T>
struct cplx {
  T re, im;
};

template <typename T>
__device__ __forceinline__ cplx<T> cmul(cplx<T> a, cplx<T> b) {
  return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
// conj(a) * b
template <typename T>
__device__ __forceinline__ cplx<T> cmulc(cplx<T> a, cplx<T> b) {
  return {a.re * b.re + a.im * b.im, a.re * b.im - a.im * b.re};
}
// (re, im) += conj(a) * b as four FMAs (no rounding of the product on its own)
template <typename T>
__device__ __forceinline__ void cmac_c(T& re, T& im, cplx<T> a, cplx<T> b) {
  re = fma(a.re, b.re, re);
  re = fma(a.im, b.im, re);
  im = fma(a.re, b.im, im);
  im = fma(-a.im, b.re, im);
}
// a*x + b*y
template <typename T>
__device__ __forceinline__ cplx<T> cmul2(cplx<T> a, cplx<T> x, cplx<T> b, cplx<T> y) {
  cplx<T> r;
  r.re = fma(a.re, x.re, fma(-a.im, x.im, fma(b.re, y.re, -b.im * y.im)));
  r.im = fma(a.re, x.im, fma(a.im, x.re, fma(b.re, y.im, b.im * y.re)));
  return r;
}
template <typename T>
__device__ __forceinline__ cplx<T> shfl_xor_c(cplx<T> v, int m) {
  return {__shfl_xor_sync(0xffffffffu, v.re, m), __shfl_xor_sync(0xffffffffu, v.im, m)};
}

// ---- circuit plan shared with the device ----------------------------------
enum StepType : int { STEP_U1 = 0, STEP_PERM = 1, STEP_PHASE = 2 };
// u1 kinds of the fused plan (ansatz.py:146-154)
enum U1Kind : int { U1_ROT = 0, U1_RXRZ = 1, U1_RX = 2, U1_RY = 3, U1_RZ = 4 };

constexpr int kMaxSteps = 512;

struct PlanDev {
  int n;          // qubits
  int n_steps;    // fused steps after the embedding layer
  int n_u1, n_perm, n_phase, n_pairs;
  int n_params;
  const int* steps;        // [n_steps][3]: type, wire, table index
  const int* u1;           // [n_u1][4]: kind, slot0, slot1, slot2
  const uint16_t* perm;    // [n_perm][D]: new[j] = old[perm[j]]  (qsim.py:182-195)
  const uint16_t* iperm;   // [n_perm][D]: inverse
  const int* pairs;        // [n_pairs][3]: control, target, slot (qsim.py:212-225)
  const int* phase_off;    // [n_phase + 1] offsets into pairs
};

}  // namespace qpinn

struct qpinn_circuit {
  int kind, n, L, n_params;
  std::string dump, plan_dump;
  // host copies
  std::vector<int> steps, u1, pairs, phase_off;
  std::vector<uint16_t> perm, iperm;
  // the CNOTs of each fused permutation step, in gate order: perm step k holds
  // pairs cnot_ct[2 j], cnot_ct[2 j + 1] (control, target) for cnot_off[k] <= j < cnot_off[k + 1]
  std::vector<int> cnot_ct, cnot_off;
  int n_u1 = 0, n_perm = 0, n_phase = 0;
  int variant = 0;  // 0: specialised kernels when available, 1: generic only
  int device = -1;
  void* dev_block = nullptr;
  qpinn::PlanDev dev{};
};

namespace qpinn {
// Uploads the plan tables to the current device on first use (lazy, so the
// host-side circuit logic needs no GPU).
int ensure_device_plan(qpinn_circuit* c);
}
