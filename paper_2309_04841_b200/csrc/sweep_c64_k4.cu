// k_sweep instantiations: float state, heavy mask class K2 = 4.
#include "sweep_impl.cuh"

namespace fq {

int sweep_c64_k4(const SweepKind &k, const SweepParams &S, cudaStream_t st, bool dry) {
    return sweep_dispatch<float, 4>(k, S, st, dry);
}

}  // namespace fq
