// Large-n cluster PQC kernels instantiated for n = 16 (see pqc_big.cuh).
#include "pqc_big.cuh"

namespace qpinn {
template int big_n<float, 16>(bool, int, const qpinn_circuit*, const KArgs<float>*);
}  // namespace qpinn
