// Large-n cluster PQC kernels instantiated for n = 11 (see pqc_big.cuh).
#include "pqc_big.cuh"

namespace qpinn {
template int big_n<float, 11>(bool, int, const qpinn_circuit*, const KArgs<float>*);
template int big_n<double, 11>(bool, int, const qpinn_circuit*, const KArgs<double>*);
}  // namespace qpinn
