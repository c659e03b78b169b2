// Layer-loop K1 / K2, float64 instantiations (see pqc_layer.cuh).
#include "pqc_layer.cuh"

namespace qpinn {
template int layer_dispatch<double>(bool, const qpinn_circuit*, const KArgs<double>*);
}  // namespace qpinn
