// Dispatch of the slab sweeps (sweep.cuh) to the instantiation units.
#include "sweep.cuh"

namespace fq {

int sweep_c128_k3(const SweepKind &k, const SweepParams &S, cudaStream_t st, bool dry);
int sweep_c128_k4(const SweepKind &k, const SweepParams &S, cudaStream_t st, bool dry);
int sweep_c64_k3(const SweepKind &k, const SweepParams &S, cudaStream_t st, bool dry);
int sweep_c64_k4(const SweepKind &k, const SweepParams &S, cudaStream_t st, bool dry);

static int route(int mix, int cost, bool c64, const SweepKind &k, const SweepParams *S, cudaStream_t st, bool dry) {
    if (mix != MIX_RX || cost != FQ_COST_U16) return FQ_ERR_UNSUPPORTED;
    static const SweepParams empty = {};
    const SweepParams &P = S ? *S : empty;
    if (k.k2 == 3) return c64 ? sweep_c64_k3(k, P, st, dry) : sweep_c128_k3(k, P, st, dry);
    if (k.k2 == K_FULL) return c64 ? sweep_c64_k4(k, P, st, dry) : sweep_c128_k4(k, P, st, dry);
    return FQ_ERR_UNSUPPORTED;
}

bool sweep_supported(int mix, int cost, bool c64, const SweepKind &k) {
    return route(mix, cost, c64, k, nullptr, nullptr, true) == FQ_OK;
}

int launch_sweep(int mix, int cost, bool c64, const SweepKind &k, const SweepParams &S, cudaStream_t st) {
    const int s = route(mix, cost, c64, k, &S, st, false);
    if (s == FQ_ERR_UNSUPPORTED) set_error("launch_sweep: no instantiation for this pass pair");
    return s;
}

}  // namespace fq
