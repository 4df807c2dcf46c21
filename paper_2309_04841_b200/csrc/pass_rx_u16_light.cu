// Instantiations of k_pass16: X mixer, u16 costs, light round programs (SEQ_840, SEQ_84).
#include "pass.cuh"

namespace fq {

int launch_pass_rx_u16_light(const PassParams &P, const PassMaps &M, int seq, int ph, int ma, int mb, int k, int grid, cudaStream_t st) {
    if (seq == SEQ_840) return select_seq<MIX_RX, FQ_COST_U16, SEQ_840>(P, M, ph, ma, mb, k, grid, st);
    if (seq == SEQ_84) return select_seq<MIX_RX, FQ_COST_U16, SEQ_84>(P, M, ph, ma, mb, k, grid, st);
    set_error("launch_pass_rx_u16_light: bad round program %d", seq);
    return FQ_ERR_UNSUPPORTED;
}

}  // namespace fq
