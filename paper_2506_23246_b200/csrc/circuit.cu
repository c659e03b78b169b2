// Native circuit construction and fused plan (host side).
//
// Restates ansatz.build_circuit (ansatz.py:159-207) and _build_plan
// (ansatz.py:117-156): the embedding RX layer (slots 0..n-1 of the
// per-point angle vector) is implicit in the kernels' product-state
// prologue; the layer gates are fused into u1 / perm / phases steps exactly
// as the reference fuses them, then uploaded once to the current device.
#include <cstdio>
#include <cstring>
#include <sstream>
#include <vector>

#include "common.cuh"

namespace qpinn {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return QPINN_ERR_CUDA;
}
int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 148;
  }
  return cached[dev];
}

namespace {

struct Gate {
  std::string kind;
  int w0, w1;  // w1 = -1 for single-qubit gates
  int s[3];
  int ns;
  bool embed;
};

std::vector<Gate> build_gates(int kind, int n, int L, int* n_params) {
  std::vector<Gate> g;
  for (int q = 0; q < n; ++q) g.push_back({"RX", q, -1, {q, 0, 0}, 1, true});
  int slot = 0;
  for (int layer = 1; layer <= L; ++layer) {
    if (kind == QPINN_ANSATZ_BASIC || kind == QPINN_ANSATZ_STRONGLY ||
        kind == QPINN_ANSATZ_CROSS_MESH_CNOT || kind == QPINN_ANSATZ_NO_ENTANGLEMENT) {
      for (int q = 0; q < n; ++q) {
        g.push_back({"Rot", q, -1, {slot, slot + 1, slot + 2}, 3, false});
        slot += 3;
      }
    } else if (kind == QPINN_ANSATZ_CROSS_MESH) {
      for (int q = 0; q < n; ++q) g.push_back({"RX", q, -1, {slot++, 0, 0}, 1, false});
    } else {  // CROSS_MESH_2ROT
      for (int q = 0; q < n; ++q) {
        g.push_back({"RX", q, -1, {slot++, 0, 0}, 1, false});
        g.push_back({"RZ", q, -1, {slot++, 0, 0}, 1, false});
      }
    }
    if (kind == QPINN_ANSATZ_BASIC) {
      for (int i = 0; i < n; ++i) g.push_back({"CNOT", i, (i + 1) % n, {0, 0, 0}, 0, false});
    } else if (kind == QPINN_ANSATZ_STRONGLY) {
      int gap = (layer - 1) % (n - 1) + 1;  // ansatz.py:196
      for (int i = 0; i < n; ++i) g.push_back({"CNOT", i, (i + gap) % n, {0, 0, 0}, 0, false});
    } else if (kind == QPINN_ANSATZ_CROSS_MESH_CNOT) {
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
          if (j != i) g.push_back({"CNOT", i, j, {0, 0, 0}, 0, false});
    } else if (kind == QPINN_ANSATZ_CROSS_MESH || kind == QPINN_ANSATZ_CROSS_MESH_2ROT) {
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
          if (j != i) g.push_back({"CRZ", i, j, {slot++, 0, 0}, 1, false});
    }
  }
  *n_params = slot;
  return g;
}

std::string dump_gates(const std::vector<Gate>& gs) {
  std::ostringstream os;
  for (size_t i = 0; i < gs.size(); ++i) {
    const Gate& g = gs[i];
    if (i) os << "\n";
    os << g.kind << " " << g.w0;
    if (g.w1 >= 0) os << "," << g.w1;
    os << " ";
    if (g.ns == 0) {
      os << "-";
    } else {
      os << (g.embed ? "embed:" : "p:");
      for (int k = 0; k < g.ns; ++k) os << (k ? "," : "") << g.s[k];
    }
  }
  return os.str();
}

// new[j] = old[perm[j]] for a CNOT sequence (qsim.py:182-195)
std::vector<uint16_t> cnot_perm(const std::vector<std::pair<int, int>>& cn, int n) {
  int D = 1 << n;
  std::vector<int> perm(D), tmp(D);
  for (int j = 0; j < D; ++j) perm[j] = j;
  for (auto& ct : cn) {
    int c = ct.first, t = ct.second;
    for (int j = 0; j < D; ++j) {
      int on = (j >> (n - 1 - c)) & 1;
      int sigma = on ? (j ^ (1 << (n - 1 - t))) : j;
      tmp[j] = perm[sigma];
    }
    perm.swap(tmp);
  }
  return std::vector<uint16_t>(perm.begin(), perm.end());
}

}  // namespace
int ensure_device_plan(qpinn_circuit* c) {
  int cur = 0;
  QPINN_CUDA_CHECK(cudaGetDevice(&cur));
  if (c->dev_block && c->device == cur) return QPINN_OK;
  if (c->dev_block && c->device != cur)
    return fail(QPINN_ERR_CONFIG, "circuit plan was uploaded to another device");
  auto bytes_of = [](size_t nbytes) { return (nbytes + 255) & ~size_t(255); };
  size_t o_steps = 0;
  size_t o_u1 = o_steps + bytes_of(c->steps.size() * 4 + 4);
  size_t o_perm = o_u1 + bytes_of(c->u1.size() * 4 + 4);
  size_t o_iperm = o_perm + bytes_of(c->perm.size() * 2 + 4);
  size_t o_pairs = o_iperm + bytes_of(c->iperm.size() * 2 + 4);
  size_t o_off = o_pairs + bytes_of(c->pairs.size() * 4 + 4);
  size_t total = o_off + bytes_of(c->phase_off.size() * 4 + 4);
  void* blk = nullptr;
  QPINN_CUDA_CHECK(cudaMalloc(&blk, total));
  char* base = (char*)blk;
  auto up = [&](size_t off, const void* src, size_t nbytes) -> cudaError_t {
    return nbytes ? cudaMemcpy(base + off, src, nbytes, cudaMemcpyHostToDevice) : cudaSuccess;
  };
  cudaError_t e = up(o_steps, c->steps.data(), c->steps.size() * 4);
  if (e == cudaSuccess) e = up(o_u1, c->u1.data(), c->u1.size() * 4);
  if (e == cudaSuccess) e = up(o_perm, c->perm.data(), c->perm.size() * 2);
  if (e == cudaSuccess) e = up(o_iperm, c->iperm.data(), c->iperm.size() * 2);
  if (e == cudaSuccess) e = up(o_pairs, c->pairs.data(), c->pairs.size() * 4);
  if (e == cudaSuccess) e = up(o_off, c->phase_off.data(), c->phase_off.size() * 4);
  if (e != cudaSuccess) {
    cudaFree(blk);
    return cuda_fail(e, "plan upload");
  }
  c->device = cur;
  c->dev_block = blk;
  c->dev.n = c->n;
  c->dev.n_steps = (int)c->steps.size() / 3;
  c->dev.n_u1 = c->n_u1;
  c->dev.n_perm = c->n_perm;
  c->dev.n_phase = c->n_phase;
  c->dev.n_pairs = (int)c->pairs.size() / 3;
  c->dev.n_params = c->n_params;
  c->dev.steps = (const int*)(base + o_steps);
  c->dev.u1 = (const int*)(base + o_u1);
  c->dev.perm = (const uint16_t*)(base + o_perm);
  c->dev.iperm = (const uint16_t*)(base + o_iperm);
  c->dev.pairs = (const int*)(base + o_pairs);
  c->dev.phase_off = (const int*)(base + o_off);
  return QPINN_OK;
}

}  // namespace qpinn

using namespace qpinn;

extern "C" {

const char* qpinn_last_error(void) { return g_err.c_str(); }
const char* qpinn_version(void) { return "qpinn_b200 0.1 (sm_100a)"; }

int qpinn_circuit_create(int kind, int n, int L, qpinn_circuit** out) {
  if (!out) return fail(QPINN_ERR_CONFIG, "null output handle");
  *out = nullptr;
  if (kind < 0 || kind > 5) return fail(QPINN_ERR_CONFIG, "unknown ansatz kind");
  if (n < 1 || L < 1) return fail(QPINN_ERR_CONFIG, "n_qubits and n_layers must be positive");
  if (kind != QPINN_ANSATZ_NO_ENTANGLEMENT && n < 2)
    return fail(QPINN_ERR_CONFIG, "entangling ansatz requires at least 2 qubits");
  if (n > 16) return fail(QPINN_ERR_CAPACITY, "n_qubits > 16 is not supported");
  auto* c = new qpinn_circuit();
  c->kind = kind;
  c->n = n;
  c->L = L;
  std::vector<Gate> gates = build_gates(kind, n, L, &c->n_params);
  c->dump = dump_gates(gates);
  const int D = 1 << n;
  // fuse the layer gates (ansatz.py:117-156)
  std::ostringstream pd;
  size_t i = n;
  while (i < gates.size()) {
    const Gate& g = gates[i];
    if (g.kind == "CNOT") {
      std::vector<std::pair<int, int>> cn;
      size_t j = i;
      while (j < gates.size() && gates[j].kind == "CNOT") {
        cn.push_back({gates[j].w0, gates[j].w1});
        ++j;
      }
      c->cnot_off.push_back((int)(c->cnot_ct.size() / 2));
      for (auto& ct : cn) c->cnot_ct.insert(c->cnot_ct.end(), {ct.first, ct.second});
      std::vector<uint16_t> p = cnot_perm(cn, n);
      std::vector<uint16_t> ip(D);
      for (int k = 0; k < D; ++k) ip[p[k]] = (uint16_t)k;
      c->steps.insert(c->steps.end(), {STEP_PERM, -1, c->n_perm++});
      c->perm.insert(c->perm.end(), p.begin(), p.end());
      c->iperm.insert(c->iperm.end(), ip.begin(), ip.end());
      pd << "perm ";
      for (int k = 0; k < D; ++k) pd << (k ? "," : "") << p[k];
      pd << "\n";
      i = j;
    } else if (g.kind == "CRZ") {
      size_t j = i;
      c->phase_off.push_back((int)(c->pairs.size() / 3));
      pd << "phases";
      while (j < gates.size() && gates[j].kind == "CRZ") {
        c->pairs.insert(c->pairs.end(), {gates[j].w0, gates[j].w1, gates[j].s[0]});
        pd << " " << gates[j].w0 << ":" << gates[j].w1 << ":" << gates[j].s[0];
        ++j;
      }
      pd << "\n";
      c->steps.insert(c->steps.end(), {STEP_PHASE, -1, c->n_phase++});
      i = j;
    } else if (g.kind == "RX" && i + 1 < gates.size() && gates[i + 1].kind == "RZ" &&
               gates[i + 1].w0 == g.w0) {
      c->steps.insert(c->steps.end(), {STEP_U1, g.w0, c->n_u1++});
      c->u1.insert(c->u1.end(), {U1_RXRZ, g.s[0], gates[i + 1].s[0], 0});
      pd << "u1 rxrz " << g.w0 << " " << g.s[0] << "," << gates[i + 1].s[0] << "\n";
      i += 2;
    } else {
      int k = g.kind == "Rot" ? U1_ROT : g.kind == "RX" ? U1_RX : g.kind == "RY" ? U1_RY : U1_RZ;
      c->steps.insert(c->steps.end(), {STEP_U1, g.w0, c->n_u1++});
      c->u1.insert(c->u1.end(), {k, g.s[0], g.s[1], g.s[2]});
      std::string kn = g.kind == "Rot" ? "rot" : g.kind == "RX" ? "rx" : g.kind == "RY" ? "ry" : "rz";
      pd << "u1 " << kn << " " << g.w0 << " ";
      for (int k2 = 0; k2 < g.ns; ++k2) pd << (k2 ? "," : "") << g.s[k2];
      pd << "\n";
      ++i;
    }
  }
  c->phase_off.push_back((int)(c->pairs.size() / 3));
  c->cnot_off.push_back((int)(c->cnot_ct.size() / 2));
  c->plan_dump = pd.str();
  const int n_steps = (int)c->steps.size() / 3;
  if (n_steps > kMaxSteps) {
    delete c;
    return fail(QPINN_ERR_CAPACITY, "fused plan too long");
  }
  *out = c;
  return QPINN_OK;
}

void qpinn_circuit_destroy(qpinn_circuit* c) {
  if (!c) return;
  if (c->dev_block) cudaFree(c->dev_block);
  delete c;
}

int qpinn_circuit_param_count(const qpinn_circuit* c) { return c ? c->n_params : -1; }
int qpinn_circuit_n_qubits(const qpinn_circuit* c) { return c ? c->n : -1; }

static size_t copy_out(const std::string& s, char* buf, size_t len) {
  if (buf && len) {
    size_t k = s.size() < len - 1 ? s.size() : len - 1;
    memcpy(buf, s.data(), k);
    buf[k] = 0;
  }
  return s.size() + 1;
}

size_t qpinn_circuit_dump(const qpinn_circuit* c, char* buf, size_t len) {
  return c ? copy_out(c->dump, buf, len) : 0;
}
size_t qpinn_circuit_plan_dump(const qpinn_circuit* c, char* buf, size_t len) {
  return c ? copy_out(c->plan_dump, buf, len) : 0;
}

}  // extern "C"
