// Instantiations of k_pass16: X mixer, u16 costs, heavy round programs (SEQ_84048, SEQ_848).
#include "pass.cuh"

namespace fq {

int launch_pass_rx_u16_heavy(const PassParams &P, const PassMaps &M, int seq, int ph, int ma, int mb, int k, int grid, cudaStream_t st) {
    if (seq == SEQ_84048) return select_seq<MIX_RX, FQ_COST_U16, SEQ_84048>(P, M, ph, ma, mb, k, grid, st);
    if (seq == SEQ_848) return select_seq<MIX_RX, FQ_COST_U16, SEQ_848>(P, M, ph, ma, mb, k, grid, st);
    set_error("launch_pass_rx_u16_heavy: bad round program %d", seq);
    return FQ_ERR_UNSUPPORTED;
}

}  // namespace fq
