// k_sweep instantiations: double state, heavy mask class K2 = 3.
#include "sweep_impl.cuh"

namespace fq {

int sweep_c128_k3(const SweepKind &k, const SweepParams &S, cudaStream_t st, bool dry) {
    return sweep_dispatch<double, 3>(k, S, st, dry);
}

}  // namespace fq
