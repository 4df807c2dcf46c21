// Instantiation helper for k_sweep (included by the sweep_*.cu units, which
// nvcc compiles in parallel): one unit per (state type, heavy mask class).
#pragma once

#include "sweep.cuh"

namespace fq {

template <int MIX, int COST, int SEQ1, int PH1, int MA1, int MB1, int K1, int SEQ2, int PH2, int MA2, int MB2, int K2,
          typename R>
static int launch_sweep_t(const SweepParams &S, cudaStream_t st) {
    static bool configured = false;
    constexpr int CP = table_copies<R>();
    const size_t smem_max = (size_t)(kTilePadded + (kTableLo + kMaxTableHi) * CP) * sizeof(C2<R>);
    auto fn = k_sweep<MIX, COST, SEQ1, PH1, MA1, MB1, K1, SEQ2, PH2, MA2, MB2, K2, R>;
    if (!configured) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
        configured = true;
    }
    const int th = (PH1 == 1 || PH1 == 2) ? S.P1.table_hi : S.P2.table_hi;
    const size_t need = (size_t)(kTilePadded + (kTableLo + th) * CP) * sizeof(C2<R>);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(S.n_teams * S.team_size));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = need;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // every team co-resident: the spinning barrier cannot deadlock
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    FQ_CUDA(cudaLaunchKernelEx(&cfg, fn, S));
    return FQ_OK;
}

// The sweeps of the X-mixer program: sub-pass 1 = a light pass over the low
// 12-target group (SEQ_840, no phase), sub-pass 2 = the fused two-layer pass
// of a high group (SEQ_848, mid phase) or the program's last pass (SEQ_84 +
// expectation).  K2 = mask class of sub-pass 2 (3: 7 high targets, n = 26).
template <typename R, int K2>
static int sweep_dispatch(const SweepKind &k, const SweepParams &S, cudaStream_t st, bool dry) {
#define FQ_SW(MA1, SEQ2, PH2, MA2, MB2)                                                                        \
    if (k.ma1 == MA1 && k.seq2 == SEQ2 && k.ph2 == PH2 && k.ma2 == MA2 && k.mb2 == MB2)                         \
        return dry ? FQ_OK                                                                                      \
                   : launch_sweep_t<MIX_RX, FQ_COST_U16, SEQ_840, 0, MA1, 2, K_FULL, SEQ2, PH2, MA2, MB2, K2, R>(S, st);
    if (k.seq1 != SEQ_840 || k.ph1 != 0 || k.mb1 != 2 || k.k1 != K_FULL || k.k2 != K2) return FQ_ERR_UNSUPPORTED;
    FQ_SW(0, SEQ_848, 2, 0, 0) FQ_SW(0, SEQ_848, 2, 0, 1) FQ_SW(0, SEQ_848, 2, 1, 0) FQ_SW(0, SEQ_848, 2, 1, 1)
    FQ_SW(1, SEQ_848, 2, 0, 0) FQ_SW(1, SEQ_848, 2, 0, 1) FQ_SW(1, SEQ_848, 2, 1, 0) FQ_SW(1, SEQ_848, 2, 1, 1)
    FQ_SW(0, SEQ_84, 3, 0, 2) FQ_SW(0, SEQ_84, 3, 1, 2) FQ_SW(1, SEQ_84, 3, 0, 2) FQ_SW(1, SEQ_84, 3, 1, 2)
#undef FQ_SW
    return FQ_ERR_UNSUPPORTED;
}

}  // namespace fq
