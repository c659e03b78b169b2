// Layer-loop K1 / K2, float32 instantiations (the kernels are in pqc_layer.cuh;
// float64 is compiled in pqc_layer_f64.cu so the two build in parallel).
#define QPINN_LAYER_DEFINE_ENTANGLER
#include "pqc_layer.cuh"

namespace qpinn {
template int layer_dispatch<float>(bool, const qpinn_circuit*, const KArgs<float>*);
}  // namespace qpinn
