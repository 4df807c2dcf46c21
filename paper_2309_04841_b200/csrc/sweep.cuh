// L2-resident slab sweeps (sm_100a): two consecutive passes of the fused
// program in ONE HBM round trip.
//
// Passes i and i+1 of a plan touch the tile bits T1 and T2.  Every tile of
// either pass lies inside a "slab": the 2^|T1 u T2| amplitudes that share
// the bits outside T1 u T2 (LABS n = 26: 19 bits, 8 MiB of complex128).  A
// team of CTAs takes one slab at a time: sub-pass 1 streams the slab's tiles
// from HBM and leaves its results in L2 (stores with an L2::evict_last
// policy), a team barrier, then sub-pass 2 re-reads the slab from L2 and
// streams the final result back to HBM.  With ~9 teams the slabs in flight
// (~72 MiB) stay inside the 126 MB L2, so the pair costs one read + one
// write of the state in HBM instead of two of each (microbenchmark,
// scripts/microbench/l2_sweep.cu: two copy-like passes 0.71 ms -> 0.45 ms).
// Each sub-pass runs the same tile body as k_pass16 (pass_tile); the team
// barrier is a counter in global memory (cooperative launch: all teams
// co-resident, so spinning cannot deadlock; a 5 s timeout sets an error word
// that turns the program's objective into NaN instead of hanging).
#pragma once

#include "pass.cuh"

namespace fq {

constexpr int kMaxDep = 40;

struct SweepParams {
    PassParams P1, P2;                 // sub-pass 1 / 2; at most one of them applies a phase
    unsigned char dep1[kMaxDep];       // physical bit of tile-number bit i (slab-inner bits first, then slab index)
    unsigned char dep2[kMaxDep];
    unsigned char cdep[kMaxDep];       // physical bit of slab-cost-run bit i (inner run-index bits, then slab index)
    int n_dep;                         // tile-number bits: n - 12
    int log2_tiles;                    // tiles of one sub-pass per slab = 2^log2_tiles
    int cost_run_log2;                 // slab's cost slice = runs of 2^cost_run_log2 contiguous levels (0: no prefetch)
    int log2_cost_runs;                // runs per slab
    long long n_slabs;
    int team_size, n_teams;
    unsigned *counters;                // one 128-B line per team, zeroed before the launch
    int *err;                          // set by a barrier timeout
    int pf1_bytes;                     // > 0: sub-pass 1's tile is one contiguous run of this many bytes (bulk L2 prefetch)
};

__device__ __forceinline__ unsigned long long sweep_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Team barrier: every CTA of the team publishes its sub-pass-1 stores
// (gpu-scope fence), arrives on the team counter, and waits for all.
__device__ __forceinline__ void team_barrier(unsigned *ctr, unsigned target, int *err) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        const unsigned long long t0 = sweep_ns();
        while (ld_acquire_gpu(ctr) < target) {
            if (sweep_ns() - t0 > 5000000000ULL) {
                atomicExch(err, 1);
                break;
            }
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ long long deposit_bits(long long x, const unsigned char *dep, int nb) {
    long long out = 0;
    for (int i = 0; i < nb; ++i)
        if ((x >> i) & 1) out |= 1LL << dep[i];
    return out;
}

__device__ __forceinline__ void bulk_prefetch_l2(const void *p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <int MIX, int COST, int SEQ1, int PH1, int MA1, int MB1, int K1, int SEQ2, int PH2, int MA2, int MB2, int K2,
          typename R>
__global__ void __launch_bounds__(kThreads, 2) k_sweep(const __grid_constant__ SweepParams S) {
    using T = C2<R>;
    static_assert(!((PH1 == 1 || PH1 == 2) && (PH2 == 1 || PH2 == 2)), "one phase per sweep (one set of tables)");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *tile = reinterpret_cast<T *>(smem_raw);
    T *tlo = tile + kTilePadded;
    T *thi = tlo + kTableLo * table_copies<R>();
    __shared__ double red[kThreads / 32];
    const int tid = threadIdx.x;
    constexpr bool TAB1 = COST == FQ_COST_U16 && (PH1 == 1 || PH1 == 2);
    constexpr bool TAB2 = COST == FQ_COST_U16 && (PH2 == 1 || PH2 == 2);
    if (TAB1 || TAB2) {
        const PassParams &Q = TAB1 ? S.P1 : S.P2;
        if (Q.table_hi > 0) build_phase_tables<R>(tlo, thi, Q.table_hi, Q.gamma, Q.cost_scale, Q.cost_offset);
        __syncthreads();
    }
    const int team = blockIdx.x / S.team_size, tr = blockIdx.x % S.team_size;
    const int G = S.team_size;
    const int tiles = 1 << S.log2_tiles;
    const unsigned long long pol = l2_evict_last_policy();
    double eacc = 0.0;
    unsigned nb = 0;
    for (long long slab = team; team < S.n_teams && slab < S.n_slabs; slab += S.n_teams) {
        const long long sbits = slab << S.log2_tiles;
        // this CTA's share of the slab's cost slice (sub-pass 2 reads it) into L2
        if (S.cost_run_log2 > 0 && tid == 0) {
            const int runs = 1 << S.log2_cost_runs;
            for (int r = tr; r < runs; r += G) {
                const long long c0 = deposit_bits((slab << S.log2_cost_runs) | r, S.cdep, S.n_dep + 12 - S.cost_run_log2);
                bulk_prefetch_l2(static_cast<const unsigned short *>(S.P2.costs) + c0, 2u << S.cost_run_log2);
            }
        }
        {  // sub-pass 1: HBM -> L2
            const long long thr8 = thread_offset<PAT8, false>(S.P1, tid);
            const long long thr4 = thread_offset<PAT4, false>(S.P1, tid);
            for (int j = tr; j < tiles; j += G) {
                if (S.pf1_bytes > 0 && tid == 0) {  // the next tile of this CTA
                    const long long jn = j + G < tiles ? sbits + j + G : ((slab + S.n_teams) << S.log2_tiles) + tr;
                    if (jn < (S.n_slabs << S.log2_tiles))
                        bulk_prefetch_l2(static_cast<const T *>(S.P1.psi) + deposit_bits(jn, S.dep1, S.n_dep),
                                         (unsigned)S.pf1_bytes);
                }
                const long long base = deposit_bits(sbits + j, S.dep1, S.n_dep);
                pass_tile<MIX, COST, SEQ1, PH1, MA1, MB1, K1, R, false, LD_STREAM, ST_L2_KEEP>(S.P1, base, tile, tlo, thi,
                                                                                           thr8, thr4, eacc, pol);
            }
        }
        team_barrier(S.counters + 32 * team, (unsigned)G * ++nb, S.err);
        {  // sub-pass 2: L2 -> HBM
            const long long thr8 = thread_offset<PAT8, false>(S.P2, tid);
            const long long thr4 = thread_offset<PAT4, false>(S.P2, tid);
            for (int j = tr; j < tiles; j += G) {
                const long long base = deposit_bits(sbits + j, S.dep2, S.n_dep);
                pass_tile<MIX, COST, SEQ2, PH2, MA2, MB2, K2, R, false, LD_L2, ST_STREAM>(S.P2, base, tile, tlo, thi,
                                                                                      thr8, thr4, eacc, pol);
            }
        }
    }
    if (S.P2.expect) {
        const double s = block_sum<kThreads>(eacc, red);
        if (tid == 0) S.P2.partials[blockIdx.x] = s;
    }
}

// Instantiated sub-pass pairs (sweep.cu); returns FQ_ERR_UNSUPPORTED when the
// pair has no instantiation (the planner then runs the two passes separately).
struct SweepKind {
    int seq1, ph1, ma1, mb1, k1;
    int seq2, ph2, ma2, mb2, k2;
};
bool sweep_supported(int mix, int cost, bool c64, const SweepKind &k);
int launch_sweep(int mix, int cost, bool c64, const SweepKind &k, const SweepParams &S, cudaStream_t st);

}  // namespace fq
