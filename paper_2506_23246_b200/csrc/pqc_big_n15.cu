// Large-n cluster PQC kernels instantiated for n = 15 (see pqc_big.cuh).
#include "pqc_big.cuh"

namespace qpinn {
template int big_n<float, 15>(bool, int, const qpinn_circuit*, const KArgs<float>*);
template int big_n<double, 15>(bool, int, const qpinn_circuit*, const KArgs<double>*);
}  // namespace qpinn
