// Instantiations of k_pass16 for sharded states (G = true), f64 costs: passes
// whose tile spans the k global qubits, i.e. all K peer-mapped shards
// (fq_qaoa_evolve_sharded).  complex128; X and custom mixers, every round program.
#include "pass.cuh"

namespace fq {

template <int MIX>
static int global_seq(const PassParams &P, const PassMaps &M, int seq, int ph, int ma, int mb, int k, int grid,
                      cudaStream_t st) {
    switch (seq) {
        case SEQ_840: return select_seq<MIX, FQ_COST_F64, SEQ_840, double, true>(P, M, ph, ma, mb, k, grid, st);
        case SEQ_84: return select_seq<MIX, FQ_COST_F64, SEQ_84, double, true>(P, M, ph, ma, mb, k, grid, st);
        case SEQ_84048: return select_seq<MIX, FQ_COST_F64, SEQ_84048, double, true>(P, M, ph, ma, mb, k, grid, st);
        case SEQ_848: return select_seq<MIX, FQ_COST_F64, SEQ_848, double, true>(P, M, ph, ma, mb, k, grid, st);
        default: break;
    }
    set_error("launch_pass_global_f64: bad round program %d", seq);
    return FQ_ERR_UNSUPPORTED;
}

int launch_pass_global_f64(int mix, const PassParams &P, const PassMaps &M, int seq, int ph, int ma, int mb, int k,
                           int grid, cudaStream_t st) {
    return mix == MIX_SU2 ? global_seq<MIX_SU2>(P, M, seq, ph, ma, mb, k, grid, st)
                          : global_seq<MIX_RX>(P, M, seq, ph, ma, mb, k, grid, st);
}

}  // namespace fq
