// Interface between the PQC launcher (pqc.cu) and the layer-loop kernels
// (pqc_layer.cu).
#pragma once
#include "pqc_common.cuh"

namespace qpinn {

constexpr int KERNEL_NONE = -1;
constexpr int ENT_NONE = 0, ENT_PERM = 1, ENT_PHASE = 2;
constexpr int kMaxBlocksPerSm = 16;  // 128-thread blocks: 2048 / 128

template <typename T>
struct KArgs {
  int scale;
  int64_t R;
  const T* act;
  const T* tan;
  const T* qp;
  T* z;
  T* dz;
  void* states;
  unsigned long long* maxabs;
  const T* gz;
  const T* gdz;
  T* g_act;
  T* g_tan;
  T* g_qp;
  double* partial;
  double* tot;
  cudaStream_t stream;
  unsigned char* tables;  // workspace region for pqc_prepare_tables
  T* coh = nullptr;       // value-only probe: per-qubit coherences [R, n] complex
};

// QPINN_OK / error code, or KERNEL_NONE when the circuit's plan does not have
// the uniform layer shape (the generic kernels then run).
template <typename T>
int layer_dispatch(bool fwd, const qpinn_circuit* c, const KArgs<T>* a);
int layer_entangler(const qpinn_circuit* c);

// provided by pqc.cu
int pqc_grid(int64_t R, int spw, int occ);
template <typename T>
int pqc_finish_grads(const qpinn_circuit* c, int grid, const KArgs<T>* a);
// ab = register bits of the phase-accumulator layout ((b & (2^ab-1)) 2^(n-ab) + (b >> ab));
// ab = n means natural index order
template <typename T>
int pqc_finish_grads_ab(const qpinn_circuit* c, int grid, const KArgs<T>* a, int ab);

// large-n cluster kernels (pqc_big.cu)
template <typename T>
int big_dispatch(bool fwd, const qpinn_circuit* c, const KArgs<T>* a);
size_t big_workspace_bytes(const qpinn_circuit* c, int dtype);
// whether the cluster-resident adjoint covers this circuit (else the HBM regime)
bool big_bwd_supported(const qpinn_circuit* c, int dtype);
// gate-space sums tot [8 n_u1 | D n_phase] -> parameter gradients (pqc.cu)
template <typename T>
int pqc_param_grads(const qpinn_circuit* c, const double* tot, int ab, const T* qp, T* g_qp,
                    cudaStream_t st);
// HBM-regime adjoint (pqc_global.cu)
size_t global_adjoint_workspace_bytes(const qpinn_circuit* c, int dtype, int64_t rows = -1);
template <typename T>
int global_backward(const qpinn_circuit* c, const KArgs<T>* a, unsigned char* ws, size_t bytes);
template <typename T>
int global_forward(const qpinn_circuit* c, const KArgs<T>* a, unsigned char* ws, size_t bytes);
// whether a cluster forward kernel with tangents exists for this circuit
bool big_fwd_supported(const qpinn_circuit* c, int dtype);
// forward with several gates per HBM pass (pqc_global.cu): fp32, 9 <= n <= 16 (the default
// from n = 11-13, see hbm_fwd_supported / hbm_bwd_supported)
bool hbm_fwd_supported(const qpinn_circuit* c, int dtype);
int hbm_forward(const qpinn_circuit* c, const KArgs<float>* a, unsigned char* ws, size_t bytes);
int hbm_forward_passes(const qpinn_circuit* c);
bool hbm_bwd_supported(const qpinn_circuit* c, int dtype);
int hbm_backward(const qpinn_circuit* c, const KArgs<float>* a, unsigned char* ws, size_t bytes);
size_t hbm_bwd_workspace_bytes(const qpinn_circuit* c, int64_t rows = -1);
// transfer-matrix K1 / K2 on the tensor cores (pqc_transfer.cu)
bool transfer_supported(const qpinn_circuit* c, int dtype);
bool transfer_default(const qpinn_circuit* c, int dtype);
size_t transfer_workspace_bytes(const qpinn_circuit* c, int64_t R);
size_t transfer_state_bytes(const qpinn_circuit* c, int64_t R);
int transfer_forward(const qpinn_circuit* c, const KArgs<float>* a, unsigned char* ws, size_t bytes);
int transfer_backward(const qpinn_circuit* c, const KArgs<float>* a, unsigned char* ws,
                      size_t bytes);

}  // namespace qpinn
