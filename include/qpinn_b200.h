/*
 * qpinn_b200.h -- C ABI of the B200-native QPINN hot path.
 *
 * Plain pointers, sizes and enums only: no torch types.  Every device
 * pointer is a CUDA global-memory address on the current device; every
 * `stream` argument is a cudaStream_t passed as void* (NULL = legacy default
 * stream).  Launch functions are asynchronous: they validate arguments on the
 * host, enqueue kernels on `stream` and return; device-side conditions
 * (domain excursions, non-finite gradients) are reported through the
 * status functions below.
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/qpinn):
 *   qpinn_circuit_*        <- ansatz.build_circuit / CircuitSpec (ansatz.py:70-207)
 *   qpinn_pqc_forward      <- ansatz.quantum_layer_forward       (ansatz.py:341-400)
 *   qpinn_pqc_backward     <- the taped backward of the same call
 *                             (tape.py:118-148 through ansatz.py:378-400, qsim.py:122-209)
 *   qpinn_loss_*           <- physics.LossEvaluator.evaluate      (physics.py:334-460)
 *                             and physics.time_bin_weights     (physics.py:172-180)
 *   qpinn_adam_step        <- training.adam_step                  (training.py:101-111)
 */
#ifndef QPINN_B200_H
#define QPINN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the Python host maps them onto the reference exception
 * classes of errors.py:4-37. */
#define QPINN_OK 0
#define QPINN_ERR_CONFIG 1        /* ConfigError        */
#define QPINN_ERR_DOMAIN 2        /* DomainError        */
#define QPINN_ERR_CAPACITY 3      /* CapacityError      */
#define QPINN_ERR_INVALID_GATE 4  /* InvalidGateError   */
#define QPINN_ERR_INVALID_BATCH 5 /* InvalidBatchError  */
#define QPINN_ERR_NONFINITE 6     /* RunAborted         */
#define QPINN_ERR_CUDA 7          /* CUDA runtime failure */

#define QPINN_F32 0
#define QPINN_F64 1

/* AnsatzKind (ansatz.py:27-33), in declaration order */
#define QPINN_ANSATZ_BASIC 0
#define QPINN_ANSATZ_STRONGLY 1
#define QPINN_ANSATZ_CROSS_MESH 2
#define QPINN_ANSATZ_CROSS_MESH_2ROT 3
#define QPINN_ANSATZ_CROSS_MESH_CNOT 4
#define QPINN_ANSATZ_NO_ENTANGLEMENT 5

/* ScaleKind (ansatz.py:36-41) */
#define QPINN_SCALE_NONE 0
#define QPINN_SCALE_PI 1
#define QPINN_SCALE_BIAS 2
#define QPINN_SCALE_ASIN 3
#define QPINN_SCALE_ACOS 4

/* Last error message of the calling thread (static storage). */
const char* qpinn_last_error(void);
/* Library version string. */
const char* qpinn_version(void);

/* ---- circuit (ansatz.py:159-207, fused plan ansatz.py:117-156) ---------- */
typedef struct qpinn_circuit qpinn_circuit;

/* Builds the gate list and fused plan and uploads the plan to the current
 * device.  QPINN_ERR_CONFIG for n_qubits/n_layers < 1 or an entangling
 * ansatz with n_qubits < 2 (ansatz.py:163-166). */
int qpinn_circuit_create(int kind, int n_qubits, int n_layers, qpinn_circuit** out);
void qpinn_circuit_destroy(qpinn_circuit* c);
int qpinn_circuit_param_count(const qpinn_circuit* c);
int qpinn_circuit_n_qubits(const qpinn_circuit* c);
/* CircuitSpec.dump() text (ansatz.py:98-109); returns the required size
 * including the NUL, writes at most `len` bytes. */
size_t qpinn_circuit_dump(const qpinn_circuit* c, char* buf, size_t len);
/* One line per fused step: "u1 <kind> <wire> <slots>" | "perm <p0,p1,...>" |
 * "phases <c:t:slot ...>". */
size_t qpinn_circuit_plan_dump(const qpinn_circuit* c, char* buf, size_t len);
/* Kernel choice for this circuit: 0 (default) uses the transfer-matrix K1/K2
 * for float32 n = 5..8 (and n = 9, 10 from L = 4) and the layer-loop K1/K2 (wires unrolled at compile
 * time) otherwise, when the fused plan has the uniform layer shape every
 * build_circuit ansatz has; 1 forces the generic runtime-plan kernels; 2
 * forces the transfer-matrix kernels (float32, 5 <= n <= 10: the circuit as
 * one [2^(n+1), 2^(n+1)] real map applied on the tensor cores, the
 * reference's via="matrix" formulation, ansatz.py:300-338); 3 forces the
 * layer-loop kernels wherever the plan allows them.  Set it before
 * the forward whose states feed a backward (the two must use the same
 * variant). */
int qpinn_circuit_set_kernel_variant(qpinn_circuit* c, int variant);
/* 1 if the layer-loop kernels apply to this circuit. */
int qpinn_circuit_specialized(const qpinn_circuit* c);
/* 1 if forward/backward run the transfer-matrix kernels for `dtype`. */
int qpinn_pqc_uses_transfer(const qpinn_circuit* c, int dtype);
/* Which kernels a forward (backward = 0, with tangents) or adjoint (backward = 1)
 * of this circuit runs for `dtype` (diagnostics): 0 layer-loop register kernels,
 * 1 generic register kernels, 2 transfer-matrix map, 3 shared-memory / cluster
 * kernels, 4 multi-gate HBM passes, 5 one-pass-per-gate global-memory kernels. */
int qpinn_pqc_regime(const qpinn_circuit* c, int dtype, int backward);
/* Largest n_qubits the register-resident kernels accept for `dtype`. */
int qpinn_pqc_max_qubits(int dtype);

/* ---- PQC forward + tangents (K1) and adjoint backward (K2) -------------- */
/* Device scratch needed by forward/backward for `rows` points (the
 * transfer-matrix kernels stage [4 rows, 2^(n+1)] float32 operands here).
 * Beyond qpinn_pqc_max_qubits the statevectors no longer fit registers: the
 * CTA / cluster kernels hold a point's states in shared memory, and for
 * float32 standard layer plans the multi-gate HBM passes take over (forward
 * from n = 12 with CNOT entanglers and L >= 2, or L >= 8, else from n = 13;
 * adjoint from n = 12, and n = 11 with CNOT entanglers or L = 1), streaming
 * batches of points' states through this scratch: up to ~256 MB for the
 * forward and ~1 GB (states, adjoints, layer checkpoints) for the adjoint.
 * The size depends on the kernel variant: query it (and qpinn_pqc_state_bytes)
 * after qpinn_circuit_set_kernel_variant. */
size_t qpinn_pqc_workspace_bytes(const qpinn_circuit* c, int dtype, int64_t rows);

/* Bytes of the optional state hand-off buffer that lets the backward skip
 * re-running the circuit: 4 states x 2^n amplitudes per row at each of the L
 * layer boundaries for the layer-loop kernels (variant 0), the 4 final states
 * for the generic kernels (variant 1); the transfer-matrix kernels keep the
 * final states and (L >= 2) the embedded states in it.  The content is
 * opaque. */
size_t qpinn_pqc_state_bytes(const qpinn_circuit* c, int dtype, int64_t rows);

/* z[R,n] = <Z_q>, dz[3,R,n] = d<Z_q>/d(x,y,t) of the scaled-angle-embedded
 * circuit; act_val [R,n], act_tan [3,R,n] row-major (act_tan/dz may be NULL
 * for value-only evaluation), qparams [P].  When `states` is not NULL (and
 * tangents are on) psi, d psi/dx,y,t are checkpointed there for
 * qpinn_pqc_backward.  Folds max|act_val| into the workspace's running
 * maximum for qpinn_pqc_domain_check. */
int qpinn_pqc_forward(const qpinn_circuit* c, int dtype, int scale, int64_t rows,
                      const void* act_val, const void* act_tan, const void* qparams,
                      void* z, void* dz, void* states, void* workspace,
                      size_t workspace_bytes, void* stream);

/* Value-only forward for the Meyer-Wallach probe (qsim.py:384-406): z [R,n]
 * and coh [R,n] complex (interleaved re, im) with coh_k = sum over basis
 * states b with bit k = 0 of psi_b conj(psi_{b with bit k set}), the reduced
 * density matrix's off-diagonal (its diagonal is (1 +- z_k)/2).  Standard
 * ansatze with the layer-loop kernels only (n <= 8 fp32, n <= 7 fp64). */
int qpinn_pqc_forward_probe(const qpinn_circuit* c, int dtype, int scale, int64_t rows,
                            const void* act_val, const void* qparams, void* z, void* coh,
                            void* workspace, size_t workspace_bytes, void* stream);

/* Gradients of L(z, dz) given g_z = dL/dz [R,n] and g_dz = dL/d(dz) [3,R,n]:
 * g_act_val [R,n], g_act_tan [3,R,n] and g_qparams [P] (summed over all rows
 * in a fixed, run-to-run deterministic order).  `states` is the buffer a
 * forward on the same inputs filled, or NULL to recompute the circuit.
 * Transfer-matrix path with `states`: part of the work runs on a per-device
 * side stream forked from and joined back into `stream` before the call
 * returns (CUDA-graph capturable once the first call has created it); calls
 * on one device are not to be issued concurrently from several host threads
 * (the reference is single-threaded). */
int qpinn_pqc_backward(const qpinn_circuit* c, int dtype, int scale, int64_t rows,
                       const void* act_val, const void* act_tan, const void* qparams,
                       const void* states, const void* g_z, const void* g_dz,
                       void* g_act_val, void* g_act_tan, void* g_qparams,
                       void* workspace, size_t workspace_bytes, void* stream);

/* Synchronises `stream`, reads (and resets to 0) the running max|act_val| of
 * the forwards launched on this workspace since the last check (a fresh
 * workspace must be zero-filled): QPINN_ERR_DOMAIN if it exceeds 1 by more than 1e-12
 * (ansatz.py:51-58); *clamped = 1 when 0 < excess <= 1e-12 (the kernels
 * clamp those values, as the reference does with a warning). */
int qpinn_pqc_domain_check(const void* workspace, void* stream, double* max_abs,
                           int* clamped);
/* Asynchronous half of the check, for a caller that synchronises anyway: enqueues
 * on `stream` the copy of the running max|act_val| (a double) into `host_dst`
 * (8 bytes, pinned) and its reset; apply the rule above to the value after the
 * caller's own synchronisation (no extra host round trip per step). */
int qpinn_pqc_domain_fetch(const void* workspace, void* host_dst, void* stream);
/* Device-side form of the same rule, for a data-parallel step that carries it
 * through its one all-reduce and vetoes the optimizer on the device: enqueues
 * on `stream` flags_dev[0] = 1.0 if max|act_val| - 1 > 1e-12 (DomainError)
 * else 0, flags_dev[1] = 1.0 if max|act_val| > 1 (clamped or error) else 0,
 * flags_dev[2] = max|act_val|, and resets the running maximum.  Summed over
 * ranks, flags_dev[0] > 0 raises on every rank. */
int qpinn_pqc_domain_flags(const void* workspace, double* flags_dev, void* stream);

/* ---- classical trunk with forward-mode tangents (network.py:133-147, :284-298)
 * periodic map -> frozen RFF -> tanh hidden layers -> tanh adapter, carried as
 * value + d/dx, d/dy, d/dt channels stacked along rows ([4, R, width]) so each
 * layer is ONE GEMM on [4R, in] x [in, out] (tensor cores, FP32-accurate
 * 3xTF32 hi/lo split for float32; DGEMM for float64).  Weights are read from
 * and gradients written to the flat parameter vector at the given offsets. */
typedef struct qpinn_trunk_desc {
  int32_t n_hidden;      /* hidden tanh layers (3 for the hybrid, network.py:188-189) */
  int32_t rff;           /* RFF features F; the first layer reads 2F                 */
  int32_t hidden;        /* hidden width                                             */
  int32_t n_out;         /* adapter width (= n_qubits)                               */
  int64_t off_w[8];      /* flat offset of hidden layer i weights [in, out]          */
  int64_t off_b[8];      /* flat offset of hidden layer i bias [out]                 */
  int64_t off_adapter_w, off_adapter_b, off_tau_raw;
  double t_domain;       /* tau = t_domain * (1 + softplus(tau_raw)) (network.py:292) */
  const void* omega;     /* device [F, 6] frozen RFF projection (dtype)              */
} qpinn_trunk_desc;

size_t qpinn_trunk_workspace_bytes(const qpinn_trunk_desc* d, int dtype, int64_t rows);
/* act [4, R, n_out]: a = tanh(h Wa + ba) and its x/y/t tangents (the PQC
 * input: act_val = act, act_tan = act + R*n_out).  Saves what the backward
 * needs in the workspace. */
int qpinn_trunk_forward(const qpinn_trunk_desc* d, int dtype, int64_t rows, const void* x,
                        const void* y, const void* t, const void* params, void* act,
                        void* workspace, size_t workspace_bytes, void* stream);

/* Value-only trunk for inference and the probes (network.py:310-335): act
 * [R, n] = adapter activations without tangents.  Same descriptor and
 * workspace as the dual forward. */
int qpinn_trunk_forward_value(const qpinn_trunk_desc* d, int dtype, int64_t rows,
                              const void* x, const void* y, const void* t,
                              const void* params, void* act, void* workspace,
                              size_t workspace_bytes, void* stream);
/* Given g_act = dL/d(act) [4, R, n_out] (from qpinn_pqc_backward), writes the
 * gradients of every trunk weight, bias and tau_raw into `grad` (flat layout;
 * overwrites those entries). */
int qpinn_trunk_backward(const qpinn_trunk_desc* d, int dtype, int64_t rows, const void* x,
                         const void* y, const void* t, const void* params, const void* act,
                         const void* g_act, void* grad, void* workspace, size_t workspace_bytes,
                         void* stream);

/* ---- fused Maxwell loss (K4), physics.py:123-187, :334-460 -------------- */
/* Static per-grid description.  The host derives every table with the same
 * numpy expressions as the reference (grid coordinates, permittivity, pulse,
 * time bins, region counts) so the device never re-derives a floating-point
 * bin edge. */
typedef struct qpinn_loss_spec {
  int32_t nx, ny;                /* slice geometry (physics.py:89-98)               */
  int32_t n_local_slices;        /* time slices covered by this call                */
  const int32_t* slice_bin;      /* device [n_local_slices] time bin (physics.py:115-117) */
  const int32_t* slice_is_ic;    /* device [n_local_slices] 1 for the t = 0 slice   */
  const double* eps;             /* device [nx*ny] permittivity (physics.py:45-49)   */
  const double* ic_target;       /* device [nx*ny] E_z(t=0) pulse (physics.py:64-67) */
  int32_t balanced;              /* diel_balanced: res1 split by region (physics.py:144-151) */
  int32_t energy;                /* energy term enabled                             */
  int32_t n_sym;                 /* parity terms (physics.py:194-205)               */
  int32_t sym_field[6];          /* 0 ez, 1 hx, 2 hy                                */
  int32_t sym_axis[6];           /* 0 x-mirror, 1 y-mirror                          */
  double sym_sign[6];            /* +1 penalises f - f_mirror, -1 f + f_mirror      */
  /* 1/count(key, slices of bin m) (0 when the key is unused or the bin empty),
   * keys: 0 res1 | res1_vac, 1 res1_diel, 2 res2, 3 res3 (physics.py:432-450) */
  double inv_count_bin[5][4];
  double inv_count_all[4];       /* 1/count(key, all nt slices) (pooled formula)   */
  double n_total;                /* grid points N (energy/sym normaliser)          */
  double slice_size;             /* nx*ny (IC normaliser)                          */
} qpinn_loss_spec;

/* Loss-sum vector: [bin m][key k] at 4*m + k (20), energy 20, sym 21, ic 22. */
#define QPINN_LOSS_NSUMS 23
size_t qpinn_loss_workspace_bytes(const qpinn_loss_spec* s, int dtype, int64_t rows);

/* Residuals (physics.py:123-128) and every loss term of the fused evaluator
 * (physics.py:352-414) for the rows of `slices` (row r = local slice
 * r / (nx*ny), slice-major), given the head outputs out [R,3] = (E_z, H_x,
 * H_y) and their input jacobians dout [3,R,3] (d/dx, d/dy, d/dt).  With the
 * adaptive weights `weights_dev` [5] (double, device; NULL = the pooled
 * formula) it writes the loss gradient g_out [R,3], g_dout [3,R,3] (dtype) and
 * the raw per-term sums `sums_dev` [QPINN_LOSS_NSUMS] (double; deterministic
 * fixed-order reduction).  See qpinn_loss_head_forward_backward for the
 * variant with the linear head (network.py:302) fused in. */
int qpinn_loss_forward_backward(const qpinn_loss_spec* s, int dtype, int64_t rows,
                                const void* out, const void* dout,
                                const double* weights_dev, void* g_out, void* g_dout,
                                double* sums_dev, void* workspace, size_t workspace_bytes,
                                void* stream);

/* Same loss with the linear head fused in: reads the PQC output z [4, R, W]
 * (value and x/y/t tangents, W <= 16) and the head weights w_out [W, 3],
 * b_out [3] (dtype), and writes dL/dz [4, R, W] plus dL/dw_out, dL/db_out
 * (into g_w_out [3W], g_b_out [3], dtype, deterministic reduction). */
int qpinn_loss_head_forward_backward(const qpinn_loss_spec* s, int dtype, int64_t rows, int width,
                                     const void* z, const void* w_out, const void* b_out,
                                     const double* weights_dev, void* g_z, void* g_w_out,
                                     void* g_b_out, double* sums_dev, void* workspace,
                                     size_t workspace_bytes, void* stream);

/* From (globally reduced) sums: breakdown_dev[10] = phys, ic, sym, energy,
 * total, bin_phys[5] (physics.py:416-426); when `weights_next_dev` is not
 * NULL also time_bin_weights(bin_phys, kappa) into it (physics.py:172-180).
 * `weighted` says whether the sums were taken with adaptive weights
 * `weights_dev` (else the pooled formula). */
int qpinn_loss_finalize(const qpinn_loss_spec* s, const double* sums_dev,
                        const double* weights_dev, int weighted, double kappa,
                        double* breakdown_dev, double* weights_next_dev, void* stream);

/* ---- Adam (training.py:87-111) ------------------------------------------ */
/* If the loss *loss_dev (optional, device double) is non-finite, *flag_dev
 * gets bit 2; if any grad entry is non-finite it gets bit 1; if the optional
 * *veto_dev is non-zero (the step's reduced domain flag, see
 * qpinn_pqc_domain_flags) it gets bit 4; in every case nothing is updated
 * (the reference raises RunAborted before touching its state,
 * training.py:104-105, :363-364, and DomainError in the forward,
 * ansatz.py:51-58).  Otherwise m, v, params are updated
 * in place with bias correction for step t (1-based, i.e. the value of
 * AdamState.t after its increment). */
int qpinn_adam_step(int dtype, int64_t n, void* params, const void* grad, void* m,
                    void* v, int64_t t, double lr, double beta1, double beta2,
                    double eps, const double* loss_dev, const double* veto_dev,
                    int32_t* flag_dev, void* stream);

/* ---- FP32-accurate tensor-core GEMM (the trunk's dense layers) ------------ */
/* C[m,n] = A[m,k] B[n,k]^T in float32 on the tcgen05 TF32 tensor cores with
 * a 3-way hi/lo operand split (FP32-class accuracy).  Row-major, K
 * contiguous; A, B, C 16-byte aligned with lda, ldb multiples of 4; n <= 256.
 * Replaces the dense layers' stacked dual GEMM (ops.py:282-298 on
 * network.py:294-298).  Workspace holds the split B. */
size_t qpinn_gemm_f32_workspace_bytes(int n, int k);
int qpinn_gemm_f32(int64_t m, int n, int k, const void* a, int64_t lda, const void* b,
                   int64_t ldb, void* c, int64_t ldc, void* workspace,
                   size_t workspace_bytes, void* stream);
/* C[m,n] = X[rows,m]^T G[rows,n] (the dense layers' weight gradients, a
 * reduction over all rows): same split-operand tensor-core math, split over
 * row chunks with a fixed-order float64 sum of the chunk partials
 * (run-to-run deterministic).  ldx, ldg multiples of 4. */
size_t qpinn_gemm_f32_atb_workspace_bytes(int64_t rows, int m, int n);
int qpinn_gemm_f32_atb(int64_t rows, int m, int n, const void* x, int64_t ldx, const void* g,
                       int64_t ldg, void* c, void* workspace, size_t workspace_bytes,
                       void* stream);

/* ---- value-only inference head and probe reductions ------ */
/* fields [R, 3] = z [R, n] W_out [n, 3] + b_out (network.py:302). */
int qpinn_head_forward(int dtype, int64_t rows, int n, const void* z, const void* w_out,
                       const void* b_out, void* fields, void* stream);
/* u[t] = dxdy * sum over slice t's `points` rows of 0.5 (eps Ez^2 + Hx^2 + Hy^2)
 * (training.py:187-200, fdtd.py:194-197); fields [n_slices * points, 3], eps
 * [points] and u [n_slices] float64 on the device; fixed-order sums. */
int qpinn_probe_energy(int dtype, int n_slices, int64_t points, const void* fields,
                       const double* eps, double dxdy, double* u, void* stream);
/* sums[2t] = sum (Ez - ref)^2, sums[2t+1] = sum ref^2 over slice t
 * (training.py:203-217); ref [n_slices * points] float64. */
int qpinn_probe_l2(int dtype, int n_slices, int64_t points, const void* fields,
                   const double* ref, double* sums, void* stream);

/* ---- FDTD reference solver (fdtd.py:115-211) ----------------------------- */
/* Yee TEz leapfrog on the periodic [-1,1)^2 cell, float64, `steps` steps of
 * size dt on an nx x ny grid (arrays [ny][nx], x fastest).  ic: 0 Gaussian
 * pulse with pulse = {cx, cy, sx, sy} (host, NULL = centred, unstretched),
 * 1 the analytic plane wave.  Collocated snapshots (Ez, H averaged to the Ez
 * nodes) are written at the host-given increasing step indices into rec_*
 * [n_snaps][ny][nx] (device), and, when `energy` is not NULL, U at each
 * snapshot (fdtd.py:194-197) into energy[n_snaps] (device).  Every update is
 * rounded in the reference's order (no FMA contraction). */
size_t qpinn_fdtd_workspace_bytes(int nx, int ny);
int qpinn_fdtd_run(int nx, int ny, int steps, double dt, int ic, const double* pulse,
                   int dielectric, double eps_r, double slab_x0, const int32_t* snap_steps,
                   int n_snaps, double* rec_ez, double* rec_hx, double* rec_hy,
                   double* energy, void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* QPINN_B200_H */
