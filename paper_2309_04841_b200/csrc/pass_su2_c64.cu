// Instantiations of k_pass16 for complex64 states (R = float): custom SU(2)
// mixer, both cost encodings, all round programs.  Coefficients are rounded to
// fp32 per pass; phase angles and the expectation stay fp64.
#include "pass.cuh"

namespace fq {

int launch_pass_su2_c64(const PassParams &P, const PassMaps &M, int cost, int seq, int ph, int mb, int k, int grid,
                        cudaStream_t st) {
#define FQ_S(C, Q) \
    if (cost == C && seq == Q) return select_seq<MIX_SU2, C, Q, float>(P, M, ph, 0, mb, k, grid, st);
    FQ_S(FQ_COST_U16, SEQ_840) FQ_S(FQ_COST_U16, SEQ_84) FQ_S(FQ_COST_U16, SEQ_84048) FQ_S(FQ_COST_U16, SEQ_848)
    FQ_S(FQ_COST_F64, SEQ_840) FQ_S(FQ_COST_F64, SEQ_84) FQ_S(FQ_COST_F64, SEQ_84048) FQ_S(FQ_COST_F64, SEQ_848)
#undef FQ_S
    set_error("launch_pass_su2_c64: bad round program %d", seq);
    return FQ_ERR_UNSUPPORTED;
}

}  // namespace fq
