// Instantiations of k_pass16 for complex64 states (R = float): X mixer, f64 costs,
// every round program.  Amplitudes and butterflies in fp32; phase angles and the
// expectation accumulate in fp64 (see phase16 / the store loop of k_pass16).
#include "pass.cuh"

namespace fq {

int launch_pass_c64_f64(const PassParams &P, const PassMaps &M, int seq, int ph, int ma, int mb, int k, int grid, cudaStream_t st) {
    if (seq == SEQ_840) return select_seq<MIX_RX, FQ_COST_F64, SEQ_840, float>(P, M, ph, ma, mb, k, grid, st);
    if (seq == SEQ_84) return select_seq<MIX_RX, FQ_COST_F64, SEQ_84, float>(P, M, ph, ma, mb, k, grid, st);
    if (seq == SEQ_84048) return select_seq<MIX_RX, FQ_COST_F64, SEQ_84048, float>(P, M, ph, ma, mb, k, grid, st);
    if (seq == SEQ_848) return select_seq<MIX_RX, FQ_COST_F64, SEQ_848, float>(P, M, ph, ma, mb, k, grid, st);
    set_error("launch_pass_c64_f64: bad round program %d", seq);
    return FQ_ERR_UNSUPPORTED;
}

}  // namespace fq
