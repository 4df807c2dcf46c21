// EXPERIMENT, NOT BUILT (round 2, measured slower; kept as the record of the
// negative result in DESIGN.md section 3.1 and profiles/r02_v2/pass8_ab.log).  To
// rebuild it, copy it into paper_2309_04841_b200/csrc/, add it to _build.SOURCES
// and dispatch SEQ_848 / K = 3 passes to launch_pass8 from evolve.cu launch_pass.
//
// k_pass8: the fused two-layer pass (mixer_l, phase_{l+1}, mixer_{l+1}) of a
// 7-target high group (tile bits 5..11 targets, 0..4 spectators: the n = 26
// headline's fusion points) with 8 amplitudes per thread and 512 threads per
// 2^12 tile -- twice the warps per SM of k_pass16 (64 registers per thread,
// two CTAs per SM), for the latency-bound fused pass.
//
// Register patterns (3 tile bits in registers):
//   PA: registers = tile bits 9..11; thread bits = tile bits 0..8 (lanes on
//       0..4: every global access is a 512-B run);
//   PB: registers = tile bits 6..8; lane bit 0 = tile bit 5 (its butterflies
//       run across lanes, warp shuffles), lane bits 1..4 = tile bits 0..3,
//       warp bits = tile bits 4, 9, 10, 11.
// Program: PA (layer A on 9..11) | PB (layer A on 6..8 + lane 5, phase,
// layer B on lane 5 + 6..8) | PA (layer B on 9..11) -- two transposes.
// Shared-memory slot of tile index e: e ^ (((e >> 5) & 1) << 2) (16-B
// elements, no padding): a quarter-warp's eight accesses hit eight distinct
// bank groups in both patterns, and since the XOR only moves bits 0..2 by
// bit 5 (a thread bit in both patterns) every access is thread base +
// register immediate.  uint16 costs are staged through a shared cost tile.
#include "tmap.cuh"

namespace fq {

constexpr int kP8Threads = 512;
constexpr int kP8Regs = 8;

__device__ __forceinline__ int p8_slot(int e) { return e ^ (((e >> 5) & 1) << 2); }

// tile index of thread t's register 0 in pattern PB
__device__ __forceinline__ int p8_eb(int t) {
    return ((t & 1) << 5) | ((t >> 1) & 15) | (((t >> 5) & 1) << 4) | (((t >> 6) & 7) << 9);
}

template <int M>
__device__ __forceinline__ void p8_bfly(double2 (&v)[kP8Regs], double r) {
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int i = 0; i < kP8Regs; ++i)
            if (!(i & (1 << k))) {
                if (M == 0) bfly_rx0(v[i], v[i | (1 << k)], r);
                else bfly_rx1(v[i], v[i | (1 << k)], r);
            }
}

// tile bit 5 = lane bit 0 in PB: own' = own - i t partner (M = 0) or u own - i partner (M = 1)
template <int M>
__device__ __forceinline__ void p8_lane(double2 (&v)[kP8Regs], double r) {
#pragma unroll
    for (int i = 0; i < kP8Regs; ++i) {
        const double px = __shfl_xor_sync(0xffffffffu, v[i].x, 1), py = __shfl_xor_sync(0xffffffffu, v[i].y, 1);
        if (M == 0) v[i] = make_double2(fma(r, py, v[i].x), fma(-r, px, v[i].y));
        else v[i] = make_double2(fma(r, v[i].x, py), fma(r, v[i].y, -px));
    }
}

template <int MA, int MB>
__global__ void __launch_bounds__(kP8Threads, 2) k_pass8(const __grid_constant__ PassParams P,
                                                         const __grid_constant__ CUtensorMap tm_state,
                                                         const __grid_constant__ CUtensorMap tm_cost) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2 *tile = reinterpret_cast<double2 *>(smem_raw);
    double2 *tlo = tile + kTile;
    double2 *thi = tlo + kTableLo * 8;
    unsigned short *ctile = reinterpret_cast<unsigned short *>(thi + P.table_hi * 8);
    const int tid = threadIdx.x;
    build_phase_tables<double>(tlo, thi, P.table_hi, P.gamma, P.cost_scale, P.cost_offset);
    __syncthreads();
    // PA thread offset (tile bits 0..8) and the cost-vector offset (tile bits 3..11)
    int thrA = 0, thrc = 0;  // < 2^31 amplitudes (host)
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        if ((tid >> j) & 1) {
            thrA += 1 << P.tile_pos[j];
            thrc += 1 << P.tile_pos[3 + j];
        }
    }
    const int sA = p8_slot(tid), eB = p8_eb(tid), sB = p8_slot(eB);
    const int cp = tid & 7;  // phase-table copy of this lane
    const bool pf = P.pf_dist > 0 && tid == 0;
    long long base = tile_base(P, P.reverse ? P.n_tiles - 1 - blockIdx.x : blockIdx.x);
    for (long long t = blockIdx.x; t < P.n_tiles; t += gridDim.x,
                   base = P.reverse ? prev_base(base, P.tile_mask, P.step_dep) : next_base(base, P.tile_mask, P.step_dep)) {
        if (pf) {
            const long long tp = t + (long long)P.pf_dist * gridDim.x;
            if (tp < P.n_tiles) prefetch_tile(P, &tm_state, &tm_cost, P.reverse ? P.n_tiles - 1 - tp : tp, true);
        }
        const char *ps = reinterpret_cast<const char *>(static_cast<const double2 *>(P.psi) + base + thrA);
        double2 v[kP8Regs];
#pragma unroll
        for (int i = 0; i < kP8Regs; ++i)  // PA register i = tile bits 9..11 = k_pass16's PAT8 register 2 i
            v[i] = ld_stream(reinterpret_cast<const double2 *>(ps + P.roff[PAT8][2 * i]));
        const uint4 *cg = reinterpret_cast<const uint4 *>(static_cast<const char *>(P.costs) + (base + thrc) * 2);
        const uint4 cv = P.cost_l2 ? __ldcg(cg) : __ldcs(cg);
        // ---- layer A, tile bits 9..11 (PA)
        p8_bfly<MA>(v, P.A.r);
        // ---- transpose PA -> PB (the cost tile rides on its first barrier)
        reinterpret_cast<uint4 *>(ctile)[tid] = cv;
#pragma unroll
        for (int i = 0; i < kP8Regs; ++i) tile[sA + 512 * i] = v[i];
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kP8Regs; ++i) v[i] = tile[sB + 64 * i];
        __syncthreads();
        // ---- layer A, tile bits 6..8 and 5 (PB); phase; layer B, tile bits 5 and 6..8
        p8_bfly<MA>(v, P.A.r);
        p8_lane<MA>(v, P.A.r);
        asm volatile("" ::: "memory");
#pragma unroll
        for (int i = 0; i < kP8Regs; ++i) {
            const unsigned raw = ctile[eB + 64 * i];
            v[i] = cmul(v[i], cmul(thi[(raw >> 6) * 8 + cp], tlo[(raw & 63) * 8 + cp]));
        }
        p8_lane<MB>(v, P.B.r);
        p8_bfly<MB>(v, P.B.r);
        // ---- transpose PB -> PA
#pragma unroll
        for (int i = 0; i < kP8Regs; ++i) tile[sB + 64 * i] = v[i];
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kP8Regs; ++i) v[i] = tile[sA + 512 * i];
        __syncthreads();
        // ---- layer B, tile bits 9..11 (PA); store
        p8_bfly<MB>(v, P.B.r);
        char *pw = reinterpret_cast<char *>(static_cast<double2 *>(P.psi) + base + thrA);
#pragma unroll
        for (int i = 0; i < kP8Regs; ++i)
            st_stream(reinterpret_cast<double2 *>(pw + P.roff[PAT8][2 * i]), make_double2(v[i].x * P.final_scale, v[i].y * P.final_scale));
    }
}

// The fused pass of a 7-target high group as k_pass8 (complex128, uint16 costs
// with phase tables and a staged cost tile, X mixer, no expectation).
int launch_pass8(const PassParams &P, const PassMaps &M, int ma, int mb, int grid, cudaStream_t st) {
    static bool configured = false;
    const size_t smax = (size_t)(kTile + (kTableLo + kMaxTableHi) * 8) * sizeof(double2) + kTile * 2;
    if (!configured) {
        cudaFuncSetAttribute(k_pass8<0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax);
        cudaFuncSetAttribute(k_pass8<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax);
        cudaFuncSetAttribute(k_pass8<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax);
        cudaFuncSetAttribute(k_pass8<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax);
        configured = true;
    }
    const size_t need = (size_t)(kTile + (kTableLo + P.table_hi) * 8) * sizeof(double2) + kTile * 2;
    if (ma == 0 && mb == 0) k_pass8<0, 0><<<grid, kP8Threads, need, st>>>(P, M.state, M.cost);
    else if (ma == 0) k_pass8<0, 1><<<grid, kP8Threads, need, st>>>(P, M.state, M.cost);
    else if (mb == 0) k_pass8<1, 0><<<grid, kP8Threads, need, st>>>(P, M.state, M.cost);
    else k_pass8<1, 1><<<grid, kP8Threads, need, st>>>(P, M.state, M.cost);
    FQ_LAUNCHED("k_pass8");
    return FQ_OK;
}

}  // namespace fq
