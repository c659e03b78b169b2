// Dispatch for the large-n cluster kernels; the kernels themselves are
// instantiated per n in pqc_big_n*.cu so the build parallelises.
#include "pqc_big.cuh"

namespace qpinn {

// instantiated in pqc_big_n*.cu; extern here so this TU does not compile every kernel again
#define QPINN_BIG_EXTERN(N)                                                              \
  extern template int big_n<float, N>(bool, int, const qpinn_circuit*, const KArgs<float>*); \
  extern template int big_n<double, N>(bool, int, const qpinn_circuit*, const KArgs<double>*);
QPINN_BIG_EXTERN(9)
QPINN_BIG_EXTERN(10)
QPINN_BIG_EXTERN(11)
QPINN_BIG_EXTERN(12)
QPINN_BIG_EXTERN(13)
QPINN_BIG_EXTERN(14)
QPINN_BIG_EXTERN(15)
extern template int big_n<float, 16>(bool, int, const qpinn_circuit*, const KArgs<float>*);
#undef QPINN_BIG_EXTERN

template <typename T>
int big_dispatch(bool fwd, const qpinn_circuit* c, const KArgs<T>* a) {
  const int ent = layer_entangler(c);
  if (ent < 0) return fail(QPINN_ERR_CAPACITY, "large-n kernels need the standard layer plan");
  switch (c->n) {
    case 9: return big_n<T, 9>(fwd, ent, c, a);
    case 10: return big_n<T, 10>(fwd, ent, c, a);
    case 11: return big_n<T, 11>(fwd, ent, c, a);
    case 12: return big_n<T, 12>(fwd, ent, c, a);
    case 13: return big_n<T, 13>(fwd, ent, c, a);
    case 14: return big_n<T, 14>(fwd, ent, c, a);
    case 15: return big_n<T, 15>(fwd, ent, c, a);
    case 16:
      if constexpr (sizeof(T) == 4) return big_n<float, 16>(fwd, ent, c, (const KArgs<float>*)a);
      return fail(QPINN_ERR_CAPACITY, "float64 large-n kernels cover n <= 15");
    default: return fail(QPINN_ERR_CAPACITY, "n_qubits out of range");
  }
}

template int big_dispatch<float>(bool, const qpinn_circuit*, const KArgs<float>*);
template int big_dispatch<double>(bool, const qpinn_circuit*, const KArgs<double>*);

bool big_bwd_supported(const qpinn_circuit* c, int dtype) {
  auto ok = [&](auto tag) -> bool {
    using T = decltype(tag);
    switch (c->n) {
      case 9: return BigGeo<T, 9, 4, true>::CB <= 4;
      case 10: return BigGeo<T, 10, 4, true>::CB <= 4;
      case 11: return BigGeo<T, 11, 4, true>::CB <= 4;
      case 12: return BigGeo<T, 12, 4, true>::CB <= 4;
      case 13: return BigGeo<T, 13, 4, true>::CB <= 4;
      case 14: return BigGeo<T, 14, 4, true>::CB <= 4;
      case 15: return BigGeo<T, 15, 4, true>::CB <= 4;
      case 16: return sizeof(T) == 4 && BigGeo<T, 16, 4, true>::CB <= 4;
      default: return false;
    }
  };
  return dtype == QPINN_F64 ? ok(double{}) : ok(float{});
}

bool big_fwd_supported(const qpinn_circuit* c, int dtype) {
  return c->n >= 9 && (c->n <= 15 || (c->n == 16 && dtype == QPINN_F32));
}

size_t big_workspace_bytes(const qpinn_circuit* c, int dtype) {
  const size_t D = (size_t)1 << c->n, es = dtype == QPINN_F64 ? 16 : 8;
  const size_t n_acc = 8 * (size_t)c->n_u1 + D * c->n_phase;
  const size_t rows = (size_t)num_sms() * 2;  // clusters never exceed SMs x 2 blocks
  size_t o = 256 + align_up(8 * n_acc * rows, 256) + align_up(8 * n_acc, 256);
  o += align_up(es * 4 * c->n_u1, 256) + 2 * align_up(4 * D * c->n_perm, 256) +
       align_up(es * D * c->n_phase, 256);
  return o;
}

}  // namespace qpinn
