// k_sweep instantiations: double state, heavy mask class K2 = 4.
#include "sweep_impl.cuh"

namespace fq {

int sweep_c128_k4(const SweepKind &k, const SweepParams &S, cudaStream_t st, bool dry) {
    return sweep_dispatch<double, 4>(k, S, st, dry);
}

}  // namespace fq
