// Instantiations of k_pass16 for sharded complex64 states (G = true, R = float):
// X mixer, both cost encodings, every round program (fq_qaoa_evolve_sharded).
#include "pass.cuh"

namespace fq {

template <int COST>
static int global_c64_seq(const PassParams &P, const PassMaps &M, int seq, int ph, int ma, int mb, int k, int grid,
                          cudaStream_t st) {
    switch (seq) {
        case SEQ_840: return select_seq<MIX_RX, COST, SEQ_840, float, true>(P, M, ph, ma, mb, k, grid, st);
        case SEQ_84: return select_seq<MIX_RX, COST, SEQ_84, float, true>(P, M, ph, ma, mb, k, grid, st);
        case SEQ_84048: return select_seq<MIX_RX, COST, SEQ_84048, float, true>(P, M, ph, ma, mb, k, grid, st);
        case SEQ_848: return select_seq<MIX_RX, COST, SEQ_848, float, true>(P, M, ph, ma, mb, k, grid, st);
        default: break;
    }
    set_error("launch_pass_global_c64: bad round program %d", seq);
    return FQ_ERR_UNSUPPORTED;
}

int launch_pass_global_c64(int cost, const PassParams &P, const PassMaps &M, int seq, int ph, int ma, int mb, int k,
                           int grid, cudaStream_t st) {
    return cost == FQ_COST_U16 ? global_c64_seq<FQ_COST_U16>(P, M, seq, ph, ma, mb, k, grid, st)
                               : global_c64_seq<FQ_COST_F64>(P, M, seq, ph, ma, mb, k, grid, st);
}

}  // namespace fq
