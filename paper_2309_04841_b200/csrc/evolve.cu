// Fused QAOA evolution for sm_100a — the hot path of the reference's
// QaoaSimulator.simulate_qaoa (qaoa.py:137-149) + get_expectation
// (statevec.py:94-97): p x (phase psi *= exp(-i gamma c), mixer), then
// sum_k c_k |psi_k|^2.
//
// Design:
//  * The state is processed in tiles of 2^12 amplitudes (64 KiB).  A tile is
//    defined by 12 "tile bits" (physical index bits); the remaining index bits
//    select the tile.  One HBM pass streams every tile once, applies every
//    butterfly whose qubit is a tile bit, and writes it back: 12 qubits per
//    HBM round trip instead of one (reference _kernels.py:14-27 is one pass
//    per qubit).
//  * Inside a tile each of the 256 threads holds 16 amplitudes in registers
//    (4 tile bits); three register "rounds" (tile bits 8-11, 0-3, 4-7) cover
//    the 12 bits with two shared-memory transposes in between (XOR-swizzled,
//    conflict-free for 16-B accesses).
//  * The phase is applied inside the pass (never a separate sweep); the
//    first pass of the program generates |+>^n instead of loading it; the
//    last pass accumulates the expectation.  Consecutive layers traverse the
//    qubit groups in alternating order, so the last pass of layer l and the
//    first pass of layer l+1 touch the same tile bits and are fused into one
//    HBM pass (mixer_l on the tile, phase_{l+1}, mixer_{l+1} on the tile):
//    1 + p*(P-1) passes for P groups instead of p*P.
//  * The X mixer uses the scaled form Rx = f (alpha I - i delta X) with
//    (alpha, delta) = (1, tan b) or (cot b, 1) whichever keeps |.| <= 1: one FMA
//    per output component; the product of the f's is applied once per pass.
//  * uint16 level costs (lossless CompactCostVector, terms.py:123-175) make
//    the phase two table lookups + one complex multiply
//    (e^{-i g (s*256h+o)} * e^{-i g s l}), no sincos in the stream.
//  * States of n <= 12 qubits run the entire program in one CTA (smem-resident),
//    which is also the batched multi-parameter path for optimiser loops.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include <type_traits>

#include "common.cuh"

namespace fq {

constexpr int kTileBits = 12;
constexpr int kTile = 1 << kTileBits;
constexpr int kThreads = 256;
constexpr int kRegs = 16;

enum { MIX_RX = 0, MIX_SU2 = 1 };
enum { PAT8 = 0, PAT0 = 1, PAT4 = 2 };  // tile bits held in registers: 8-11 / 0-3 / 4-7

struct CoefSet {
    double r;      // RX: t (mode 0) or u (mode 1)
    int mode;      // RX: 0 -> (1, t), 1 -> (u, 1)
    double2 a[kTileBits], b[kTileBits];  // SU2: per tile bit
};

struct PassParams {
    double2 *psi;
    const void *costs;
    double cost_scale, cost_offset;
    double *partials;
    double init_amp;
    double gamma;
    double final_scale;
    long long n_tiles;
    int tile_pos[kTileBits];  // physical bit of tile bit i (ascending)
    int nrounds;              // 3 or 5
    int phase_round;          // -1: none
    int phase_at;             // 1: before set A, 2: between A and B
    int init;                 // generate |+> instead of loading
    int expect;               // accumulate sum c|x|^2 in the last round
    int table_hi;             // U16 phase: rows of the high table (0 -> sincos of the decoded cost)
    unsigned char maskA[8], maskB[8];  // per round: register bits getting set A / set B butterflies
    CoefSet A, B;
    // TMA staging (k_pass_tma): tensor-map dims in ascending physical order
    int tma_rank;             // state map rank (dim 0 = doubles)
    int tma_outer_shift[5];   // outer dims: coordinate = (tile >> shift) & ((1 << bits) - 1)
    int tma_outer_bits[5];    // 0 for tile dims (coordinate 0)
    int cost_tma;             // costs staged by TMA (same dims) instead of LDG
    int cost_rank;
    int cost_outer_shift[5];
    int cost_outer_bits[5];
    int probe_l2;             // development probe: tiles alias a 64 MiB L2-resident set (compute-bound timing)
};

constexpr int kTableLo = 64;     // low-table rows (6 level bits)
constexpr int kMaxTableHi = 256; // high-table rows -> levels < 16384 use tables
constexpr int kCopies = 8;       // one copy per 16-B bank group: conflict-free random lookups

template <int PAT>
__device__ __forceinline__ int tile_bit_of_reg(int j) {
    return PAT == PAT8 ? 8 + j : (PAT == PAT0 ? j : 4 + j);
}

template <int PAT>
__device__ __forceinline__ int tidx(int tid, int i) {
    if (PAT == PAT8) return tid | (i << 8);
    if (PAT == PAT0) return (tid << 4) | i;
    return (tid & 15) | (i << 4) | ((tid >> 4) << 8);
}

// Transpose scratch layout: tile index e lives at slot e + (e >> 4) (one pad
// entry per 16).  For all three register patterns the thread part and the
// register part of the slot are additive (slot = pat_base(tid) + pat_step(i)),
// so every access is [base register + immediate], and a quarter-warp's eight
// 16-B accesses always fall in eight distinct bank groups.
constexpr int kTilePadded = kTile + kTile / 16;

template <int PAT>
__device__ __forceinline__ int pat_base(int tid) {
    if (PAT == PAT8) return tid + (tid >> 4);
    if (PAT == PAT0) return 17 * tid;
    return (tid & 15) + 272 * (tid >> 4);
}
template <int PAT>
__host__ __device__ constexpr int pat_step(int i) {
    return PAT == PAT8 ? 272 * i : (PAT == PAT0 ? i : 17 * i);
}
// raw (unpadded, TMA box order) index: thread part + register part, additive
template <int PAT>
__device__ __forceinline__ int raw_base(int tid) {
    if (PAT == PAT8) return tid;
    if (PAT == PAT0) return tid << 4;
    return (tid & 15) + ((tid >> 4) << 8);
}
template <int PAT>
__host__ __device__ constexpr int raw_step(int i) {
    return PAT == PAT8 ? (i << 8) : (PAT == PAT0 ? i : (i << 4));
}

// physical offset of this thread's element 0 for pattern PAT
template <int PAT>
__device__ __forceinline__ long long thread_offset(const PassParams &P, int tid) {
    long long off = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        int tb;
        if (PAT == PAT8) tb = j;
        else if (PAT == PAT0) tb = 4 + j;
        else tb = (j < 4) ? j : j + 4;
        if ((tid >> j) & 1) off += 1LL << P.tile_pos[tb];
    }
    return off;
}

template <int PAT>
__device__ __forceinline__ void reg_offsets(const PassParams &P, long long (&o)[kRegs]) {
    long long s[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) s[j] = 1LL << P.tile_pos[tile_bit_of_reg<PAT>(j)];
    o[0] = 0;
#pragma unroll
    for (int i = 1; i < kRegs; ++i) o[i] = o[i & (i - 1)] + s[(i & 1) ? 0 : (i & 2) ? 1 : (i & 4) ? 2 : 3];
}

template <int PAT>
__device__ __forceinline__ void transpose_out(double2 *sm, const double2 (&v)[kRegs], int tid) {
    double2 *p = sm + pat_base<PAT>(tid);
#pragma unroll
    for (int i = 0; i < kRegs; ++i) p[pat_step<PAT>(i)] = v[i];
}
template <int PAT>
__device__ __forceinline__ void transpose_in(const double2 *sm, double2 (&v)[kRegs], int tid) {
    const double2 *p = sm + pat_base<PAT>(tid);
#pragma unroll
    for (int i = 0; i < kRegs; ++i) v[i] = p[pat_step<PAT>(i)];
}

template <int FROM, int TO>
__device__ __forceinline__ void transpose(double2 *sm, double2 (&v)[kRegs], int tid) {
    transpose_out<FROM>(sm, v, tid);
    __syncthreads();
    transpose_in<TO>(sm, v, tid);
    __syncthreads();
}

// ---- butterflies
__device__ __forceinline__ void bfly_rx0(double2 &x0, double2 &x1, double t) {
    // (x0 - i t x1, x1 - i t x0)
    const double2 a = x0, b = x1;
    x0 = make_double2(fma(t, b.y, a.x), fma(-t, b.x, a.y));
    x1 = make_double2(fma(t, a.y, b.x), fma(-t, a.x, b.y));
}
__device__ __forceinline__ void bfly_rx1(double2 &x0, double2 &x1, double u) {
    // (u x0 - i x1, u x1 - i x0)
    const double2 a = x0, b = x1;
    x0 = make_double2(fma(u, a.x, b.y), fma(u, a.y, -b.x));
    x1 = make_double2(fma(u, b.x, a.y), fma(u, b.y, -a.x));
}
__device__ __forceinline__ void bfly_su2(double2 &x0, double2 &x1, double2 a, double2 b) {
    // y0 = a x0 - conj(b) x1 ; y1 = b x0 + conj(a) x1   (reference _kernels.py:26-27)
    const double2 p = x0, q = x1;
    x0 = make_double2(a.x * p.x - a.y * p.y - b.x * q.x - b.y * q.y,
                      a.x * p.y + a.y * p.x - b.x * q.y + b.y * q.x);
    x1 = make_double2(b.x * p.x - b.y * p.y + a.x * q.x + a.y * q.y,
                      b.x * p.y + b.y * p.x + a.x * q.y - a.y * q.x);
}

template <int MIX, int PAT>
__device__ __forceinline__ void butterflies(double2 (&v)[kRegs], const CoefSet &C, int mask) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (!((mask >> j) & 1)) continue;
        if (MIX == MIX_RX) {
            const double r = C.r;
            if (C.mode == 0) {
#pragma unroll
                for (int i = 0; i < kRegs; ++i)
                    if (!(i & (1 << j))) bfly_rx0(v[i], v[i | (1 << j)], r);
            } else {
#pragma unroll
                for (int i = 0; i < kRegs; ++i)
                    if (!(i & (1 << j))) bfly_rx1(v[i], v[i | (1 << j)], r);
            }
        } else {
            const int tb = tile_bit_of_reg<PAT>(j);
            const double2 a = C.a[tb], b = C.b[tb];
#pragma unroll
            for (int i = 0; i < kRegs; ++i)
                if (!(i & (1 << j))) bfly_su2(v[i], v[i | (1 << j)], a, b);
        }
    }
}

// ---- phase
// exp(-i gamma c) for a float64 cost: the reference's angle = gamma * c, then sincos.
__device__ __forceinline__ double2 phase_f64(double c, double gamma) {
    double s, co;
    sincos(gamma * c, &s, &co);
    return make_double2(co, -s);
}

// exp(-i gamma c) for a uint16 level v, c = scale*v + offset:
// T_hi[v >> 6] * T_lo[v & 63], each table replicated once per 16-B bank group
// (copy = lane & 7) so a quarter-warp's random lookups never conflict.
__device__ __forceinline__ double2 phase_u16(unsigned v, const PassParams &P, const double2 *tlo, const double2 *thi) {
    if (P.table_hi == 0) return phase_f64(decode_u16((uint16_t)v, P.cost_scale, P.cost_offset), P.gamma);
    const int cp = threadIdx.x & (kCopies - 1);
    return cmul(thi[(v >> 6) * kCopies + cp], tlo[(v & 63) * kCopies + cp]);
}

template <int COST>
__device__ __forceinline__ double2 phase_factor(const PassParams &P, long long k, const double2 *tlo,
                                                const double2 *thi) {
    if (COST == FQ_COST_F64) return phase_f64(static_cast<const double *>(P.costs)[k], P.gamma);
    return phase_u16(static_cast<const uint16_t *>(P.costs)[k], P, tlo, thi);
}

template <int COST>
__device__ __forceinline__ double cost_value(const void *costs, long long k, double scale, double offset) {
    if (COST == FQ_COST_F64) return static_cast<const double *>(costs)[k];
    return decode_u16(static_cast<const uint16_t *>(costs)[k], scale, offset);
}

// e^{-i gamma c} tables for uint16 levels: c = scale*(64 h + l) + offset
__device__ __forceinline__ void build_phase_tables(double2 *tlo, double2 *thi, int n_hi, double gamma, double scale,
                                                   double offset) {
    for (int i = threadIdx.x; i < kTableLo + n_hi; i += blockDim.x) {
        double s, c;
        if (i < kTableLo) sincos(gamma * (scale * (double)i), &s, &c);
        else sincos(gamma * (scale * (double)(64 * (i - kTableLo)) + offset), &s, &c);
        double2 *row = (i < kTableLo) ? tlo + i * kCopies : thi + (i - kTableLo) * kCopies;
#pragma unroll
        for (int k = 0; k < kCopies; ++k) row[k] = make_double2(c, -s);
    }
}

// One register round: [phase] butterflies(A) [phase] butterflies(B).
// `cost(i)` yields the raw cost entry (double, or uint16 level) of element i.
template <int MIX, int COST, int PAT, typename CostFn>
__device__ __forceinline__ void run_round(const PassParams &P, int r, double2 (&v)[kRegs], CostFn cost,
                                          const double2 *tlo, const double2 *thi) {
    const bool ph = (P.phase_round == r);
    if (ph && P.phase_at == 1) {
#pragma unroll
        for (int i = 0; i < kRegs; ++i)
            v[i] = cmul(v[i], COST == FQ_COST_F64 ? phase_f64(cost(i), P.gamma) : phase_u16((unsigned)cost(i), P, tlo, thi));
    }
    if (P.maskA[r]) butterflies<MIX, PAT>(v, P.A, P.maskA[r]);
    if (ph && P.phase_at == 2) {
#pragma unroll
        for (int i = 0; i < kRegs; ++i)
            v[i] = cmul(v[i], COST == FQ_COST_F64 ? phase_f64(cost(i), P.gamma) : phase_u16((unsigned)cost(i), P, tlo, thi));
    }
    if (P.maskB[r]) butterflies<MIX, PAT>(v, P.B, P.maskB[r]);
}

template <int COST>
__device__ __forceinline__ double global_cost(const PassParams &P, long long k) {
    if (COST == FQ_COST_F64) return static_cast<const double *>(P.costs)[k];
    return (double)static_cast<const uint16_t *>(P.costs)[k];
}

template <int COST>
__device__ __forceinline__ double decode_cost(const PassParams &P, double raw) {
    if (COST == FQ_COST_F64) return raw;
    return decode_u16((uint16_t)raw, P.cost_scale, P.cost_offset);
}

// tile number -> base address: insert a zero at every tile bit position
__device__ __forceinline__ long long tile_base(const PassParams &P, long long t) {
    long long base = P.probe_l2 ? (t & 1023) : t;
#pragma unroll
    for (int j = 0; j < kTileBits; ++j) {
        const int p = P.tile_pos[j];
        base = ((base >> p) << (p + 1)) | (base & ((1LL << p) - 1));
    }
    return base;
}

__device__ __forceinline__ size_t table_doubles2(int n_hi) { return (size_t)(kTableLo + n_hi) * kCopies; }

// ---------------------------------------------------------------- 16-amplitude pass (default)
// Register-load pass, 256 threads x 16 amplitudes per 2^12 tile, 2 CTAs/SM.
// Everything that varies between passes of one program is a template
// parameter, so the tile loop contains no runtime branches on it and the
// kernel body stays I-cache resident:
//   PH: 0 no phase, 1 phase before set A (round 0), 2 phase between set A and
//       set B (round 2, then rounds 3-4 finish set B: a fused layer boundary);
//   MA, MB: RX form of sets A/B (0: (1, tan b), 1: (cot b, 1)); MB = 2: no set
//       B; MB = 3: set B present, form chosen at run time (rare: gamma = 0).
//   PROBE: development memory-pattern probe (load + store only).
template <int MIX, int M, int PAT>
__device__ __forceinline__ void bfly16(double2 (&v)[kRegs], const CoefSet &C, int mask) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (!((mask >> j) & 1)) continue;
        if (MIX == MIX_RX) {
            const double r = C.r;
            if (M == 0) {
#pragma unroll
                for (int i = 0; i < kRegs; ++i)
                    if (!(i & (1 << j))) bfly_rx0(v[i], v[i | (1 << j)], r);
            } else {
#pragma unroll
                for (int i = 0; i < kRegs; ++i)
                    if (!(i & (1 << j))) bfly_rx1(v[i], v[i | (1 << j)], r);
            }
        } else {
            const int tb = tile_bit_of_reg<PAT>(j);
            const double2 a = C.a[tb], b = C.b[tb];
#pragma unroll
            for (int i = 0; i < kRegs; ++i)
                if (!(i & (1 << j))) bfly_su2(v[i], v[i | (1 << j)], a, b);
        }
    }
}

template <int MIX, int M, int PAT>
__device__ __forceinline__ void bfly16_set(double2 (&v)[kRegs], const CoefSet &C, int mask) {
    if (M == 3) {  // run-time form (set B without a separating phase)
        if (C.mode == 0) bfly16<MIX, 0, PAT>(v, C, mask);
        else bfly16<MIX, 1, PAT>(v, C, mask);
    } else {
        bfly16<MIX, M, PAT>(v, C, mask);
    }
}

__device__ __noinline__ double2 phase_sincos_u16(unsigned v, double scale, double offset, double gamma) {
    return phase_f64(decode_u16((uint16_t)v, scale, offset), gamma);
}

template <int COST>
__device__ __forceinline__ double2 phase16(const PassParams &P, double raw, const double2 *tlo, const double2 *thi) {
    if (COST == FQ_COST_F64) return phase_f64(raw, P.gamma);
    const unsigned v = (unsigned)raw;
    if (P.table_hi == 0) return phase_sincos_u16(v, P.cost_scale, P.cost_offset, P.gamma);
    const int cp = threadIdx.x & (kCopies - 1);
    return cmul(thi[(v >> 6) * kCopies + cp], tlo[(v & 63) * kCopies + cp]);
}

template <int MIX, int COST, int PH, int MA, int MB, int PROBE>
__global__ void __launch_bounds__(kThreads, 2) k_pass16(const __grid_constant__ PassParams P) {
    extern __shared__ double2 smem[];
    double2 *tile = smem;
    double2 *tlo = smem + kTilePadded;
    double2 *thi = tlo + kTableLo * kCopies;
    __shared__ double red[kThreads / 32];
    const int tid = threadIdx.x;
    constexpr bool HAS_B = MB != 2;

    if (COST == FQ_COST_U16 && PH != 0 && !PROBE) {
        if (P.table_hi > 0) build_phase_tables(tlo, thi, P.table_hi, P.gamma, P.cost_scale, P.cost_offset);
        __syncthreads();
    }
    const long long thr8 = thread_offset<PAT8>(P, tid);
    const long long thr4 = thread_offset<PAT4>(P, tid);
    double eacc = 0.0;

    for (long long t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
        const long long base = tile_base(P, t);
        double2 v[kRegs];
        double raw[kRegs];  // cost entries of the phase round (loaded with the state)
        {
            long long o[kRegs];
            reg_offsets<PAT8>(P, o);
            if (P.init || PROBE == 2) {
#pragma unroll
                for (int i = 0; i < kRegs; ++i) v[i] = make_double2(P.init_amp + i, (double)t);
            } else {
#pragma unroll
                for (int i = 0; i < kRegs; ++i) v[i] = ld_stream(P.psi + base + thr8 + o[i]);
            }
            if (PH == 1) {
#pragma unroll
                for (int i = 0; i < kRegs; ++i) raw[i] = global_cost<COST>(P, base + thr8 + o[i]);
            }
        }
        if (PH == 2) {
            long long o[kRegs];
            reg_offsets<PAT4>(P, o);
#pragma unroll
            for (int i = 0; i < kRegs; ++i) raw[i] = global_cost<COST>(P, base + thr4 + o[i]);
        }
        if (PROBE != 1) {
            // round 0: tile bits 8-11
            if (PH == 1) {
#pragma unroll
                for (int i = 0; i < kRegs; ++i) v[i] = cmul(v[i], phase16<COST>(P, raw[i], tlo, thi));
            }
            bfly16_set<MIX, MA, PAT8>(v, P.A, P.maskA[0]);
            if (HAS_B && PH != 2) bfly16_set<MIX, MB, PAT8>(v, P.B, P.maskB[0]);
            transpose<PAT8, PAT0>(tile, v, tid);
            // round 1: tile bits 0-3
            bfly16_set<MIX, MA, PAT0>(v, P.A, P.maskA[1]);
            if (HAS_B && PH != 2) bfly16_set<MIX, MB, PAT0>(v, P.B, P.maskB[1]);
            transpose<PAT0, PAT4>(tile, v, tid);
            // round 2: tile bits 4-7
            bfly16_set<MIX, MA, PAT4>(v, P.A, P.maskA[2]);
            if (PH == 2) {
#pragma unroll
                for (int i = 0; i < kRegs; ++i) v[i] = cmul(v[i], phase16<COST>(P, raw[i], tlo, thi));
            }
            if (HAS_B) bfly16_set<MIX, MB, PAT4>(v, P.B, P.maskB[2]);
            if (PH == 2) {
                transpose<PAT4, PAT0>(tile, v, tid);
                bfly16_set<MIX, MB, PAT0>(v, P.B, P.maskB[3]);
                transpose<PAT0, PAT8>(tile, v, tid);
                bfly16_set<MIX, MB, PAT8>(v, P.B, P.maskB[4]);
            }
        }
        constexpr int LAST = (PH == 2 || PROBE == 1) ? PAT8 : PAT4;
        const long long thrL = (PH == 2 || PROBE == 1) ? thr8 : thr4;
        long long o[kRegs];
        reg_offsets<LAST>(P, o);
        const double fs = P.final_scale;
        if (PROBE == 2) {  // on-chip work only: keep the result live, store (almost) nothing
            double acc = 0.0;
#pragma unroll
            for (int i = 0; i < kRegs; ++i) acc += v[i].x * fs + v[i].y;
            if (acc == 1.2345e300) st_stream(P.psi + base + thrL, make_double2(acc, 0.0));
            continue;
        }
#pragma unroll
        for (int i = 0; i < kRegs; ++i) {
            double2 x = v[i];
            if (MIX == MIX_RX && PROBE != 1) x = make_double2(x.x * fs, x.y * fs);
            if (P.expect) eacc += decode_cost<COST>(P, global_cost<COST>(P, base + thrL + o[i])) * (x.x * x.x + x.y * x.y);
            st_stream(P.psi + base + thrL + o[i], x);
        }
    }
    if (P.expect) {
        const double s = block_sum<kThreads>(eacc, red);
        if (tid == 0) P.partials[blockIdx.x] = s;
    }
}

// ---------------------------------------------------------------- TMA-staged pass
// One persistent CTA per SM.  Tiles (and their cost slices) stream into two
// shared-memory stages with cp.async.bulk.tensor; tile i+1 is in flight while
// tile i is transformed in registers (its stage buffer doubling as the
// transpose scratch).  Results go back with streaming 16-B stores.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tma_load(void *dst, const CUtensorMap *map, int rank, const int *c, uint64_t *bar) {
    const uint32_t d = smem_u32(dst), b = smem_u32(bar);
    const uint64_t m = reinterpret_cast<uint64_t>(map);
    switch (rank) {
        case 1:
            asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                         ::"r"(d), "l"(m), "r"(c[0]), "r"(b) : "memory");
            break;
        case 2:
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(b) : "memory");
            break;
        case 3:
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(b) : "memory");
            break;
        case 4:
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                         ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(b) : "memory");
            break;
        default:
            asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                         ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(b) : "memory");
            break;
    }
}

__device__ __forceinline__ void tile_coords(long long t, int rank, const int *shift, const int *bits, int *c) {
#pragma unroll
    for (int d = 0; d < 5; ++d)
        c[d] = (d < rank && bits[d] > 0) ? (int)((t >> shift[d]) & ((1LL << bits[d]) - 1)) : 0;
}

__device__ __forceinline__ void tma_store(const CUtensorMap *map, int rank, const int *c, const void *src) {
    const uint32_t sa = smem_u32(src);
    const uint64_t m = reinterpret_cast<uint64_t>(map);
    switch (rank) {
        case 1:
            asm volatile("cp.async.bulk.tensor.1d.global.shared::cta.bulk_group [%0, {%1}], [%2];"
                         ::"l"(m), "r"(c[0]), "r"(sa) : "memory");
            break;
        case 2:
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                         ::"l"(m), "r"(c[0]), "r"(c[1]), "r"(sa) : "memory");
            break;
        case 3:
            asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                         ::"l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(sa) : "memory");
            break;
        case 4:
            asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];"
                         ::"l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(sa) : "memory");
            break;
        default:
            asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                         ::"l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(sa) : "memory");
            break;
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

constexpr int kStageEntries = kTilePadded;              // double2 per state stage (padded transpose layout)
constexpr int kStateStageBytes = kTilePadded * 16;
constexpr uint32_t kStateTxBytes = kTile * 16;

template <int COST>
__host__ __device__ constexpr int cost_stage_bytes() { return COST == FQ_COST_F64 ? kTile * 8 : kTile * 2; }

template <int COST>
__host__ __device__ constexpr size_t tma_smem_bytes(int n_hi) {
    return 2 * (size_t)kStateStageBytes + 2 * (size_t)cost_stage_bytes<COST>() +
           (COST == FQ_COST_U16 ? (size_t)(kTableLo + n_hi) * kCopies * 16 : 0) + 64;
}

// Persistent CTA per SM, two stages.  Stage b: TMA load (state + costs) ->
// round 0 reads the raw box -> transposes in the padded layout -> last round
// writes the raw box -> TMA store -> (store has read it) next TMA load.
template <int MIX, int COST, int NR>
__global__ void __launch_bounds__(kThreads, 1)
    k_pass_tma(const __grid_constant__ PassParams P, const __grid_constant__ CUtensorMap tm_state,
               const __grid_constant__ CUtensorMap tm_cost) {
    extern __shared__ __align__(128) double2 sm2[];
    double2 *const tlo = sm2 + 2 * kStageEntries + (2 * cost_stage_bytes<COST>()) / 16;
    double2 *const thi = tlo + kTableLo * kCopies;
    uint64_t *const bar = reinterpret_cast<uint64_t *>(
        sm2 + 2 * kStageEntries + (2 * cost_stage_bytes<COST>()) / 16 +
        (COST == FQ_COST_U16 ? (kTableLo + P.table_hi) * kCopies : 0));
    __shared__ double red[kThreads / 32];
    const int tid = threadIdx.x;

    const bool need_cost = (P.phase_round >= 0) || P.expect;
    const bool stage_cost = need_cost && P.cost_tma;
    const bool load_state = !P.init;
    const uint32_t tx = (load_state ? kStateTxBytes : 0) + (stage_cost ? cost_stage_bytes<COST>() : 0);

    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (COST == FQ_COST_U16 && P.phase_round >= 0 && P.table_hi > 0)
        build_phase_tables(tlo, thi, P.table_hi, P.gamma, P.cost_scale, P.cost_offset);
    __syncthreads();

    auto issue = [&](long long t, int b) {
        if (tx == 0) return;
        mbar_expect_tx(&bar[b], tx);
        int c[5];
        if (load_state) {
            tile_coords(P.probe_l2 ? (t & 1023) : t, P.tma_rank, P.tma_outer_shift, P.tma_outer_bits, c);
            tma_load(sm2 + b * kStageEntries, &tm_state, P.tma_rank, c, &bar[b]);
        }
        if (stage_cost) {
            tile_coords(P.probe_l2 ? (t & 1023) : t, P.cost_rank, P.cost_outer_shift, P.cost_outer_bits, c);
            tma_load(sm2 + 2 * kStageEntries + b * (cost_stage_bytes<COST>() / 16), &tm_cost, P.cost_rank, c, &bar[b]);
        }
    };
    if (tid == 0) {
        if (blockIdx.x < P.n_tiles) issue(blockIdx.x, 0);
        if (blockIdx.x + gridDim.x < P.n_tiles) issue(blockIdx.x + gridDim.x, 1);
    }

    double eacc = 0.0;
    int it = 0;
    for (long long t = blockIdx.x; t < P.n_tiles; t += gridDim.x, ++it) {
        const int b = it & 1;
        double2 *const buf = sm2 + b * kStageEntries;
        const void *const cs = sm2 + 2 * kStageEntries + b * (cost_stage_bytes<COST>() / 16);
        if (tx) mbar_wait(&bar[b], (it >> 1) & 1);
        long long base = -1;  // global base, only for the LDG cost fallback
        auto scost = [&](auto pat_tag) {
            constexpr int PAT = decltype(pat_tag)::value;
            return [&](int i) -> double {
                if (P.cost_tma) {
                    const int e = raw_base<PAT>(tid) + raw_step<PAT>(i);
                    if (COST == FQ_COST_F64) return static_cast<const double *>(cs)[e];
                    return (double)static_cast<const uint16_t *>(cs)[e];
                }
                if (base < 0) base = tile_base(P, t);
                long long o[kRegs];
                reg_offsets<PAT>(P, o);
                return global_cost<COST>(P, base + thread_offset<PAT>(P, tid) + o[i]);
            };
        };
        double2 v[kRegs];
        if (P.init) {
#pragma unroll
            for (int i = 0; i < kRegs; ++i) v[i] = make_double2(P.init_amp, 0.0);
        } else {
            const double2 *p = buf + raw_base<PAT8>(tid);
#pragma unroll
            for (int i = 0; i < kRegs; ++i) v[i] = p[raw_step<PAT8>(i)];
        }
        run_round<MIX, COST, PAT8>(P, 0, v, scost(std::integral_constant<int, PAT8>{}), tlo, thi);
        __syncthreads();  // every thread has consumed the raw stage layout
        transpose<PAT8, PAT0>(buf, v, tid);
        run_round<MIX, COST, PAT0>(P, 1, v, scost(std::integral_constant<int, PAT0>{}), tlo, thi);
        transpose<PAT0, PAT4>(buf, v, tid);
        run_round<MIX, COST, PAT4>(P, 2, v, scost(std::integral_constant<int, PAT4>{}), tlo, thi);
        if (NR == 5) {
            transpose<PAT4, PAT0>(buf, v, tid);
            run_round<MIX, COST, PAT0>(P, 3, v, scost(std::integral_constant<int, PAT0>{}), tlo, thi);
            transpose<PAT0, PAT8>(buf, v, tid);
            run_round<MIX, COST, PAT8>(P, 4, v, scost(std::integral_constant<int, PAT8>{}), tlo, thi);
        }
        constexpr int LAST = (NR == 5) ? PAT8 : PAT4;
        auto lastcost = scost(std::integral_constant<int, LAST>{});
        const double fs = P.final_scale;
        double2 *q = buf + raw_base<LAST>(tid);
#pragma unroll
        for (int i = 0; i < kRegs; ++i) {
            double2 x = v[i];
            if (MIX == MIX_RX) x = make_double2(x.x * fs, x.y * fs);
            if (P.expect) eacc += decode_cost<COST>(P, lastcost(i)) * (x.x * x.x + x.y * x.y);
            q[raw_step<LAST>(i)] = x;
        }
        fence_proxy_async();  // make this thread's raw-box writes visible to the TMA engine
        __syncthreads();
        if (tid == 0) {
            int c[5];
            tile_coords(P.probe_l2 ? (t & 1023) : t, P.tma_rank, P.tma_outer_shift, P.tma_outer_bits, c);
            tma_store(&tm_state, P.tma_rank, c, buf);
            if (t + 2 * (long long)gridDim.x < P.n_tiles) {
                tma_store_wait_read();  // the store has read stage b: reload it
                issue(t + 2 * (long long)gridDim.x, b);
            }
        }
    }
    if (tid == 0) tma_store_wait_all();
    if (P.expect) {
        const double s = block_sum<kThreads>(eacc, red);
        if (tid == 0) P.partials[blockIdx.x] = s;
    }
}

// ---------------------------------------------------------------- 8-amplitude pass (default)
// 512 threads x 8 amplitudes per 2^12 tile, two CTAs per SM (32 warps): the
// pass is latency-bound at 16-amplitude / 8-warp occupancy, so it trades one
// more shared-memory transpose for 4x the resident warps.  Register round r
// holds tile bits [f_r, f_r + 3) with f = 9, 0, 3, 6 (round 0 = global load
// pattern: lanes on tile bits 0-4, coalesced; round 3 = store pattern, also
// lanes on bits 0-4).  A fused two-layer pass with a phase between runs the
// rounds 0 1 2 3 | 3 2 1 0.
constexpr int k8Threads = 512;
constexpr int k8Regs = 8;
constexpr int k8Padded = kTile + kTile / 8;  // slot = e + (e >> 3)

__host__ __device__ constexpr int f8(int r) { return r == 0 ? 9 : 3 * (r - 1); }

template <int F>
__device__ __forceinline__ int p8_base(int tid) {
    const int low = tid & ((1 << F) - 1), high = tid >> F;
    return low + (low >> 3) + 9 * (high << F);
}
template <int F>
__host__ __device__ constexpr int p8_step(int i) { return (i << F) + ((i << F) >> 3); }
template <int F>
__device__ __forceinline__ int raw8_base(int tid) {
    const int low = tid & ((1 << F) - 1), high = tid >> F;
    return low | (high << (F + 3));
}
template <int F>
__host__ __device__ constexpr int raw8_step(int i) { return i << F; }

// physical offset of this thread's element 0 when tile bits [F, F+3) are in registers
template <int F>
__device__ __forceinline__ long long thr8_offset(const PassParams &P, int tid) {
    long long off = 0;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        const int tb = j < F ? j : j + 3;
        if ((tid >> j) & 1) off += 1LL << P.tile_pos[tb];
    }
    return off;
}
template <int F>
__device__ __forceinline__ void reg8_offsets(const PassParams &P, long long (&o)[k8Regs]) {
    const long long s0 = 1LL << P.tile_pos[F], s1 = 1LL << P.tile_pos[F + 1], s2 = 1LL << P.tile_pos[F + 2];
    o[0] = 0; o[1] = s0; o[2] = s1; o[3] = s0 + s1;
    o[4] = s2; o[5] = s2 + s0; o[6] = s2 + s1; o[7] = s2 + s1 + s0;
}

template <int F>
__device__ __forceinline__ void t8_out(double2 *sm, const double2 (&v)[k8Regs], int tid) {
    double2 *p = sm + p8_base<F>(tid);
#pragma unroll
    for (int i = 0; i < k8Regs; ++i) p[p8_step<F>(i)] = v[i];
}
template <int F>
__device__ __forceinline__ void t8_in(const double2 *sm, double2 (&v)[k8Regs], int tid) {
    const double2 *p = sm + p8_base<F>(tid);
#pragma unroll
    for (int i = 0; i < k8Regs; ++i) v[i] = p[p8_step<F>(i)];
}
template <int FROM, int TO>
__device__ __forceinline__ void t8(double2 *sm, double2 (&v)[k8Regs], int tid) {
    t8_out<FROM>(sm, v, tid);
    __syncthreads();
    t8_in<TO>(sm, v, tid);
    __syncthreads();
}

template <int MIX, int F>
__device__ __forceinline__ void bfly8(double2 (&v)[k8Regs], const CoefSet &C, int mask) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        if (!((mask >> j) & 1)) continue;
        if (MIX == MIX_RX) {
            const double r = C.r;
            if (C.mode == 0) {
#pragma unroll
                for (int i = 0; i < k8Regs; ++i)
                    if (!(i & (1 << j))) bfly_rx0(v[i], v[i | (1 << j)], r);
            } else {
#pragma unroll
                for (int i = 0; i < k8Regs; ++i)
                    if (!(i & (1 << j))) bfly_rx1(v[i], v[i | (1 << j)], r);
            }
        } else {
            const double2 a = C.a[F + j], b = C.b[F + j];
#pragma unroll
            for (int i = 0; i < k8Regs; ++i)
                if (!(i & (1 << j))) bfly_su2(v[i], v[i | (1 << j)], a, b);
        }
    }
}

// one round: [phase] A [phase] B ; costs read from global at this round's pattern
template <int MIX, int COST, int F>
__device__ __forceinline__ void round8(const PassParams &P, int r, double2 (&v)[k8Regs], long long base, int tid,
                                       const double2 *tlo, const double2 *thi) {
    const bool ph = P.phase_round == r;
    if (ph) {
        const long long thr = thr8_offset<F>(P, tid);
        long long o[k8Regs];
        reg8_offsets<F>(P, o);
        double raw[k8Regs];
#pragma unroll
        for (int i = 0; i < k8Regs; ++i) raw[i] = global_cost<COST>(P, base + thr + o[i]);
        if (P.phase_at == 1) {
#pragma unroll
            for (int i = 0; i < k8Regs; ++i)
                v[i] = cmul(v[i], COST == FQ_COST_F64 ? phase_f64(raw[i], P.gamma)
                                                      : phase_u16((unsigned)raw[i], P, tlo, thi));
        }
        if (P.maskA[r]) bfly8<MIX, F>(v, P.A, P.maskA[r]);
        if (P.phase_at == 2) {
#pragma unroll
            for (int i = 0; i < k8Regs; ++i)
                v[i] = cmul(v[i], COST == FQ_COST_F64 ? phase_f64(raw[i], P.gamma)
                                                      : phase_u16((unsigned)raw[i], P, tlo, thi));
        }
    } else if (P.maskA[r]) {
        bfly8<MIX, F>(v, P.A, P.maskA[r]);
    }
    if (P.maskB[r]) bfly8<MIX, F>(v, P.B, P.maskB[r]);
}

// NR = 4 (rounds f = 9,0,3,6) or 7 (9,0,3,6 | 6,3,0,9 with round 3 shared: 9,0,3,6,3,0,9)
template <int MIX, int COST, int NR>
__global__ void __launch_bounds__(k8Threads, 2) k_pass8(const __grid_constant__ PassParams P) {
    extern __shared__ double2 smem[];
    double2 *tile = smem;
    double2 *tlo = smem + k8Padded;
    double2 *thi = tlo + kTableLo * kCopies;
    __shared__ double red[k8Threads / 32];
    const int tid = threadIdx.x;

    if (COST == FQ_COST_U16 && P.phase_round >= 0 && P.table_hi > 0) {
        build_phase_tables(tlo, thi, P.table_hi, P.gamma, P.cost_scale, P.cost_offset);
        __syncthreads();
    }
    double eacc = 0.0;
    for (long long t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
        const long long base = tile_base(P, t);
        double2 v[k8Regs];
        {
            const long long thr = thr8_offset<9>(P, tid);
            long long o[k8Regs];
            reg8_offsets<9>(P, o);
            if (P.init) {
#pragma unroll
                for (int i = 0; i < k8Regs; ++i) v[i] = make_double2(P.init_amp, 0.0);
            } else {
#pragma unroll
                for (int i = 0; i < k8Regs; ++i) v[i] = ld_stream(P.psi + base + thr + o[i]);
            }
        }
        round8<MIX, COST, 9>(P, 0, v, base, tid, tlo, thi);
        t8<9, 0>(tile, v, tid);
        round8<MIX, COST, 0>(P, 1, v, base, tid, tlo, thi);
        t8<0, 3>(tile, v, tid);
        round8<MIX, COST, 3>(P, 2, v, base, tid, tlo, thi);
        t8<3, 6>(tile, v, tid);
        round8<MIX, COST, 6>(P, 3, v, base, tid, tlo, thi);
        if (NR == 7) {
            t8<6, 3>(tile, v, tid);
            round8<MIX, COST, 3>(P, 4, v, base, tid, tlo, thi);
            t8<3, 0>(tile, v, tid);
            round8<MIX, COST, 0>(P, 5, v, base, tid, tlo, thi);
            t8<0, 9>(tile, v, tid);
            round8<MIX, COST, 9>(P, 6, v, base, tid, tlo, thi);
        }
        constexpr int FL = (NR == 7) ? 9 : 6;
        const long long thr = thr8_offset<FL>(P, tid);
        long long o[k8Regs];
        reg8_offsets<FL>(P, o);
        const double fs = P.final_scale;
#pragma unroll
        for (int i = 0; i < k8Regs; ++i) {
            double2 x = v[i];
            if (MIX == MIX_RX) x = make_double2(x.x * fs, x.y * fs);
            if (P.expect) eacc += decode_cost<COST>(P, global_cost<COST>(P, base + thr + o[i])) * (x.x * x.x + x.y * x.y);
            st_stream(P.psi + base + thr + o[i], x);
        }
    }
    if (P.expect) {
        const double s = block_sum<k8Threads>(eacc, red);
        if (tid == 0) P.partials[blockIdx.x] = s;
    }
}

// ---------------------------------------------------------------- 8-amplitude pass, TMA-staged
// One persistent 512-thread CTA per SM (16 warps, up to 128 registers).
// Tile i+1's raw box (and its cost slice) is in flight (cp.async.bulk.tensor)
// while tile i is transformed; the state stage is re-armed as soon as the last
// transpose has drained it, the cost stage at the end of the iteration.
// Results leave with coalesced streaming stores straight from registers.
template <int COST>
__host__ __device__ constexpr size_t p8t_smem_bytes(int n_hi) {
    return 2 * (size_t)k8Padded * 16 + 2 * (size_t)cost_stage_bytes<COST>() +
           (COST == FQ_COST_U16 ? (size_t)(kTableLo + n_hi) * kCopies * 16 : 0) + 64;
}

template <int MIX, int COST, int NR>
__global__ void __launch_bounds__(k8Threads, 1)
    k_pass8t(const __grid_constant__ PassParams P, const __grid_constant__ CUtensorMap tm_state,
             const __grid_constant__ CUtensorMap tm_cost) {
    extern __shared__ __align__(128) double2 sm2[];
    constexpr int CSTAGE = cost_stage_bytes<COST>() / 16;  // in double2 units
    double2 *const tlo = sm2 + 2 * k8Padded + 2 * CSTAGE;
    double2 *const thi = tlo + kTableLo * kCopies;
    uint64_t *const bar = reinterpret_cast<uint64_t *>(
        sm2 + 2 * k8Padded + 2 * CSTAGE + (COST == FQ_COST_U16 ? (kTableLo + P.table_hi) * kCopies : 0));
    // bar[0..1]: state stages, bar[2..3]: cost stages
    __shared__ double red[k8Threads / 32];
    const int tid = threadIdx.x;

    const bool need_cost = (P.phase_round >= 0) || P.expect;
    const bool stage_cost = need_cost && P.cost_tma;
    const bool load_state = !P.init;

    if (tid == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (COST == FQ_COST_U16 && P.phase_round >= 0 && P.table_hi > 0)
        build_phase_tables(tlo, thi, P.table_hi, P.gamma, P.cost_scale, P.cost_offset);
    __syncthreads();

    auto issue_state = [&](long long t, int b) {
        if (!load_state) return;
        int c[5];
        mbar_expect_tx(&bar[b], kStateTxBytes);
        tile_coords(P.probe_l2 ? (t & 1023) : t, P.tma_rank, P.tma_outer_shift, P.tma_outer_bits, c);
        tma_load(sm2 + b * k8Padded, &tm_state, P.tma_rank, c, &bar[b]);
    };
    auto issue_cost = [&](long long t, int b) {
        if (!stage_cost) return;
        int c[5];
        mbar_expect_tx(&bar[2 + b], cost_stage_bytes<COST>());
        tile_coords(P.probe_l2 ? (t & 1023) : t, P.cost_rank, P.cost_outer_shift, P.cost_outer_bits, c);
        tma_load(sm2 + 2 * k8Padded + b * CSTAGE, &tm_cost, P.cost_rank, c, &bar[2 + b]);
    };
    if (tid == 0) {
        for (int k = 0; k < 2; ++k) {
            const long long t = blockIdx.x + (long long)k * gridDim.x;
            if (t < P.n_tiles) {
                issue_state(t, k);
                issue_cost(t, k);
            }
        }
    }

    double eacc = 0.0;
    int it = 0;
    for (long long t = blockIdx.x; t < P.n_tiles; t += gridDim.x, ++it) {
        const int b = it & 1;
        const uint32_t par = (it >> 1) & 1;
        double2 *const buf = sm2 + b * k8Padded;
        const void *const cs = sm2 + 2 * k8Padded + b * CSTAGE;
        const long long base = tile_base(P, t);
        const long long next = t + 2 * (long long)gridDim.x;
        bool cost_ready = false;
        // costs of element i in the round whose register bits start at F
        auto cost_of = [&](auto ftag, int i) -> double {
            constexpr int F = decltype(ftag)::value;
            if (P.cost_tma) {
                const int e = raw8_base<F>(tid) + raw8_step<F>(i);
                if (COST == FQ_COST_F64) return static_cast<const double *>(cs)[e];
                return (double)static_cast<const uint16_t *>(cs)[e];
            }
            long long o[k8Regs];
            reg8_offsets<F>(P, o);
            return global_cost<COST>(P, base + thr8_offset<F>(P, tid) + o[i]);
        };
        auto round = [&](auto ftag, int r, double2 (&v)[k8Regs]) {
            constexpr int F = decltype(ftag)::value;
            if (P.phase_round == r) {
                if (stage_cost && !cost_ready) {
                    mbar_wait(&bar[2 + b], par);
                    cost_ready = true;
                }
                double raw[k8Regs];
#pragma unroll
                for (int i = 0; i < k8Regs; ++i) raw[i] = cost_of(ftag, i);
                if (P.phase_at == 1) {
#pragma unroll
                    for (int i = 0; i < k8Regs; ++i)
                        v[i] = cmul(v[i], COST == FQ_COST_F64 ? phase_f64(raw[i], P.gamma)
                                                              : phase_u16((unsigned)raw[i], P, tlo, thi));
                }
                if (P.maskA[r]) bfly8<MIX, F>(v, P.A, P.maskA[r]);
                if (P.phase_at == 2) {
#pragma unroll
                    for (int i = 0; i < k8Regs; ++i)
                        v[i] = cmul(v[i], COST == FQ_COST_F64 ? phase_f64(raw[i], P.gamma)
                                                              : phase_u16((unsigned)raw[i], P, tlo, thi));
                }
            } else if (P.maskA[r]) {
                bfly8<MIX, F>(v, P.A, P.maskA[r]);
            }
            if (P.maskB[r]) bfly8<MIX, F>(v, P.B, P.maskB[r]);
        };

        double2 v[k8Regs];
        if (load_state) {
            mbar_wait(&bar[b], par);
            const double2 *p = buf + raw8_base<9>(tid);
#pragma unroll
            for (int i = 0; i < k8Regs; ++i) v[i] = p[raw8_step<9>(i)];
        } else {
#pragma unroll
            for (int i = 0; i < k8Regs; ++i) v[i] = make_double2(P.init_amp, 0.0);
        }
        round(std::integral_constant<int, 9>{}, 0, v);
        __syncthreads();  // raw box consumed by every thread
        t8<9, 0>(buf, v, tid);
        round(std::integral_constant<int, 0>{}, 1, v);
        t8<0, 3>(buf, v, tid);
        round(std::integral_constant<int, 3>{}, 2, v);
        if (NR == 4) {
            t8_out<3>(buf, v, tid);
            __syncthreads();
            t8_in<6>(buf, v, tid);
            fence_proxy_async();  // order this thread's generic accesses before the TMA refill
            __syncthreads();
            if (tid == 0 && next < P.n_tiles) issue_state(next, b);  // state stage drained: re-arm it
        } else {
            t8<3, 6>(buf, v, tid);
        }
        round(std::integral_constant<int, 6>{}, 3, v);
        if (NR == 7) {
            t8<6, 3>(buf, v, tid);
            round(std::integral_constant<int, 3>{}, 4, v);
            t8<3, 0>(buf, v, tid);
            round(std::integral_constant<int, 0>{}, 5, v);
            t8_out<0>(buf, v, tid);
            __syncthreads();
            t8_in<9>(buf, v, tid);
            fence_proxy_async();
            __syncthreads();
            if (tid == 0 && next < P.n_tiles) issue_state(next, b);
            round(std::integral_constant<int, 9>{}, 6, v);
        }
        constexpr int FL = (NR == 7) ? 9 : 6;
        if (P.expect && stage_cost && !cost_ready) {
            mbar_wait(&bar[2 + b], par);
            cost_ready = true;
        }
        const long long thr = thr8_offset<FL>(P, tid);
        long long o[k8Regs];
        reg8_offsets<FL>(P, o);
        const double fs = P.final_scale;
#pragma unroll
        for (int i = 0; i < k8Regs; ++i) {
            double2 x = v[i];
            if (MIX == MIX_RX) x = make_double2(x.x * fs, x.y * fs);
            if (P.expect) eacc += decode_cost<COST>(P, cost_of(std::integral_constant<int, FL>{}, i)) *
                                  (x.x * x.x + x.y * x.y);
            st_stream(P.psi + base + thr + o[i], x);
        }
        if (stage_cost) {
            __syncthreads();  // cost stage b fully read
            if (tid == 0 && next < P.n_tiles) issue_cost(next, b);
        }
    }
    if (P.expect) {
        const double s = block_sum<k8Threads>(eacc, red);
        if (tid == 0) P.partials[blockIdx.x] = s;
    }
}

// ---------------------------------------------------------------- resident (n <= 12)
// One CTA owns a whole 2^n state in shared memory and runs every layer.
// Layer data arrives as kernel parameters (no host->device copies).
constexpr int kResThreads = 512;
constexpr int kResMaxLayers = 512;   // angle slots per launch (longer programs are chunked)
constexpr int kResMaxGates = 256;    // XY gate list (complete n=12: 66)

struct ResParams {
    const double2 *psi_in;  // per-batch initial states (or single shared, stride 0), nullable
    long long in_stride;
    double2 *psi_out;       // nullable
    const void *costs;
    double cost_scale, cost_offset;
    double *exp_out;        // [batch], nullable
    double init_amp;
    int n, p, mixer, init, apply_phase_mask_all;
    int n_gates;
    unsigned char gates[kResMaxGates][2];
    // per (batch row, layer) angles: gam[b*p + l], bet[b*p + l]; row b = blockIdx.x
    double gam[kResMaxLayers], bet[kResMaxLayers];
    unsigned char phase_on[kResMaxLayers];  // indexed by layer (shared by all rows)
    unsigned char qlo[kResMaxLayers], qhi[kResMaxLayers];  // X/custom qubit range per layer
};

template <int COST>
__device__ __forceinline__ double2 res_phase(const void *costs, int k, double gamma, double scale, double offset) {
    double c;
    if (COST == FQ_COST_F64) c = static_cast<const double *>(costs)[k];
    else c = decode_u16(static_cast<const uint16_t *>(costs)[k], scale, offset);
    double s, co;
    sincos(gamma * c, &s, &co);
    return make_double2(co, -s);
}

template <int COST>
__global__ void __launch_bounds__(kResThreads) k_resident(const __grid_constant__ ResParams P,
                                                          const double *__restrict__ su2) {
    extern __shared__ double2 st[];
    __shared__ double red[kResThreads / 32];
    const int n = P.n, N = 1 << n, tid = threadIdx.x;
    const int b = blockIdx.x;
    if (P.init || P.psi_in == nullptr) {
        for (int k = tid; k < N; k += kResThreads) st[k] = make_double2(P.init_amp, 0.0);
    } else {
        const double2 *src = P.psi_in + (long long)b * P.in_stride;
        for (int k = tid; k < N; k += kResThreads) st[k] = src[k];
    }
    __syncthreads();
    for (int l = 0; l < P.p; ++l) {
        const double gamma = P.gam[b * P.p + l];
        const double beta = P.bet[b * P.p + l];
        if (P.phase_on[l] && gamma != 0.0) {
            for (int k = tid; k < N; k += kResThreads)
                st[k] = cmul(st[k], res_phase<COST>(P.costs, k, gamma, P.cost_scale, P.cost_offset));
            __syncthreads();
        }
        if (P.mixer == FQ_MIXER_X || P.mixer == FQ_MIXER_CUSTOM) {
            double2 a, bb;
            if (P.mixer == FQ_MIXER_X) {
                double s, c;
                sincos(beta, &s, &c);
                a = make_double2(c, 0.0);
                bb = make_double2(0.0, -s);
            }
            for (int q = P.qlo[l]; q < P.qhi[l]; ++q) {
                if (P.mixer == FQ_MIXER_CUSTOM) {
                    const double *c4 = su2 + ((long long)l * n + q) * 4;
                    a = make_double2(c4[0], c4[1]);
                    bb = make_double2(c4[2], c4[3]);
                }
                const int bit = 1 << q;
                for (int g = tid; g < (N >> 1); g += kResThreads) {
                    const int l0 = ((g >> q) << (q + 1)) | (g & (bit - 1));
                    double2 x0 = st[l0], x1 = st[l0 | bit];
                    bfly_su2(x0, x1, a, bb);
                    st[l0] = x0;
                    st[l0 | bit] = x1;
                }
                __syncthreads();
            }
        } else {
            double s, c;
            sincos(beta, &s, &c);
            for (int gi = 0; gi < P.n_gates; ++gi) {
                const int plo = P.gates[gi][0], phi = P.gates[gi][1];
                const int blo = 1 << plo, bhi = 1 << phi;
                for (int g = tid; g < (N >> 2); g += kResThreads) {
                    const int t = ((g >> plo) << (plo + 1)) | (g & (blo - 1));
                    const int base = ((t >> phi) << (phi + 1)) | (t & (bhi - 1));
                    const double2 xl = st[base | blo], xh = st[base | bhi];
                    st[base | blo] = make_double2(c * xl.x + s * xh.y, c * xl.y - s * xh.x);
                    st[base | bhi] = make_double2(s * xl.y + c * xh.x, c * xh.y - s * xl.x);
                }
                __syncthreads();
            }
        }
    }
    if (P.exp_out) {
        double acc = 0.0;
        for (int k = tid; k < N; k += kResThreads) {
            const double c = (COST == FQ_COST_F64) ? static_cast<const double *>(P.costs)[k]
                                                   : decode_u16(static_cast<const uint16_t *>(P.costs)[k],
                                                                P.cost_scale, P.cost_offset);
            const double2 x = st[k];
            acc += c * (x.x * x.x + x.y * x.y);
        }
        const double t = block_sum<kResThreads>(acc, red);
        if (tid == 0) P.exp_out[b] = t;
    }
    if (P.psi_out) {
        double2 *dst = P.psi_out + (long long)b * N;
        for (int k = tid; k < N; k += kResThreads) dst[k] = st[k];
    }
}

// ---------------------------------------------------------------- standalone phase (uint16)
__global__ void k_phase_u16(double2 *__restrict__ psi, const uint16_t *__restrict__ lv, long long size, double gamma,
                            double scale, double offset) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < size;
         k += (long long)gridDim.x * blockDim.x)
        psi[k] = cmul(psi[k], phase_f64(decode_u16(lv[k], scale, offset), gamma));
}

__global__ void k_phase_f64(double2 *__restrict__ psi, const double *__restrict__ costs, long long size,
                            double gamma) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < size;
         k += (long long)gridDim.x * blockDim.x) {
        double s, c;
        sincos(gamma * costs[k], &s, &c);
        psi[k] = cmul(psi[k], make_double2(c, -s));
    }
}

// ---------------------------------------------------------------- host planning
struct Group {
    std::vector<int> targets;  // physical qubit positions, ascending
    int tile_pos[kTileBits];
};

static bool same_targets(const std::vector<int> &a, const std::vector<int> &b) { return a == b; }

// Split targets into tile groups: the low group (targets < 12) rides a
// contiguous tile; higher targets are chunked evenly (<= 10 per pass, so at
// least 2 low spectator bits keep every global access >= 64 B contiguous).
static std::vector<Group> make_groups(int n, const std::vector<int> &targets) {
    std::vector<std::vector<int>> chunks;
    std::vector<int> low, high;
    for (int q : targets) (q < kTileBits ? low : high).push_back(q);
    if (!low.empty()) chunks.push_back(low);
    if (!high.empty()) {
        const int m = (int)((high.size() + 9) / 10);
        size_t at = 0;
        for (int c = 0; c < m; ++c) {
            const size_t sz = (high.size() - at) / (m - c);
            chunks.emplace_back(high.begin() + at, high.begin() + at + sz);
            at += sz;
        }
    }
    std::vector<Group> out;
    for (auto &ch : chunks) {
        Group g;
        g.targets = ch;
        std::vector<int> bits = ch;
        for (int q = 0; q < n && (int)bits.size() < kTileBits; ++q)
            if (std::find(ch.begin(), ch.end(), q) == ch.end()) bits.push_back(q);
        std::sort(bits.begin(), bits.end());
        for (int i = 0; i < kTileBits; ++i) g.tile_pos[i] = bits[i];
        out.push_back(g);
    }
    return out;
}

struct PlannedPass {
    int group;           // index into groups
    int layerA;          // layer whose mixer is applied first (-1 none)
    int layerB;          // fused next layer (-1 none)
    int phase_layer;     // layer whose phase is applied (-1 none)
    int phase_at;        // 1: before A, 2: between A and B
};

static bool phase_active(const fq_layer &L) { return L.apply_phase && L.gamma != 0.0; }

static void rx_coef(double beta, CoefSet &C, double &f) {
    const double c = std::cos(beta), s = std::sin(beta);
    if (std::fabs(c) >= std::fabs(s)) {
        C.mode = 0;
        C.r = s / c;
        f = c;
    } else {
        C.mode = 1;
        C.r = c / s;
        f = s;
    }
}

// ---- tensor maps (driver entry point fetched through the runtime; no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// Describe one tile (12 physical index bits) of a 2^n vector as a TMA box:
// runs of tile bits become box dims (full extent), runs of outer bits become
// box-1 dims whose coordinate comes from the tile number.  `per_amp` elements
// of `elem_bytes` per amplitude (state: 2 doubles).  False if the layout
// cannot be expressed (rank > 5, sub-16-B rows or strides).
static bool build_tile_map(CUtensorMap *map, const void *gaddr, int n, const int *tile_pos, CUtensorMapDataType dt,
                           int elem_bytes, int per_amp, int &rank, int *outer_shift, int *outer_bits) {
    auto fn = encode_fn();
    if (!fn) return false;
    bool is_tile[64] = {};
    for (int i = 0; i < kTileBits; ++i) is_tile[tile_pos[i]] = true;
    if (!is_tile[0]) return false;
    struct Dim { bool tile; int start, len; };
    std::vector<Dim> dims;
    const int cap0 = (per_amp == 2) ? 7 : 8;
    for (int b = 0; b < n;) {
        int e = b;
        while (e < n && is_tile[e] == is_tile[b]) ++e;
        if (is_tile[b]) {
            int at = b;
            while (at < e) {
                const int cap = dims.empty() ? cap0 : 8;
                const int len = std::min(cap, e - at);
                dims.push_back({true, at, len});
                at += len;
            }
        } else {
            dims.push_back({false, b, e - b});
        }
        b = e;
    }
    if (dims.size() > 5) return false;
    rank = (int)dims.size();
    cuuint64_t gdim[5], gstride[5];
    cuuint32_t box[5], estr[5];
    int shift = 0;
    for (int d = 0; d < rank; ++d) {
        gdim[d] = (cuuint64_t)(d == 0 ? per_amp : 1) << dims[d].len;
        box[d] = dims[d].tile ? (cuuint32_t)gdim[d] : 1u;
        estr[d] = 1;
        if (d > 0) {
            gstride[d - 1] = ((cuuint64_t)1 << dims[d].start) * per_amp * elem_bytes;
            if (gstride[d - 1] % 16) return false;
        }
        outer_shift[d] = dims[d].tile ? 0 : shift;
        outer_bits[d] = dims[d].tile ? 0 : dims[d].len;
        if (!dims[d].tile) shift += dims[d].len;
    }
    if ((box[0] * (cuuint32_t)elem_bytes) % 16) return false;
    for (int d = rank; d < 5; ++d) outer_shift[d] = outer_bits[d] = 0;
    CUresult r = fn(map, dt, (cuuint32_t)rank, const_cast<void *>(gaddr), gdim, gstride, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

static int max_blocks_per_sm = 2;

template <int MIX, int COST, int PH, int MA, int MB, int PROBE>
static int launch_pass16(const PassParams &P, int grid, cudaStream_t st) {
    static bool configured = false;
    const size_t smem = (size_t)(kTilePadded + (kTableLo + kMaxTableHi) * kCopies) * sizeof(double2);
    if (!configured) {
        cudaFuncSetAttribute(k_pass16<MIX, COST, PH, MA, MB, PROBE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        configured = true;
    }
    const size_t need = (size_t)(kTilePadded + (kTableLo + P.table_hi) * kCopies) * sizeof(double2);
    k_pass16<MIX, COST, PH, MA, MB, PROBE><<<grid, kThreads, need, st>>>(P);
    FQ_LAUNCHED("k_pass16");
    return FQ_OK;
}

template <int MIX, int COST>
static int select_pass16(const PassParams &P, int ph, int ma, int mb, int grid, cudaStream_t st) {
    if (MIX == MIX_SU2) {
        ma = 0;
        if (mb != 2) mb = 3;
    }
    if (ph != 2 && mb != 2) mb = 3;
#define FQ_S(PHV, MAV, MBV) \
    if (ph == PHV && ma == MAV && mb == MBV) return launch_pass16<MIX, COST, PHV, MAV, MBV, 0>(P, grid, st)
    FQ_S(0, 0, 2); FQ_S(0, 1, 2); FQ_S(0, 0, 3); FQ_S(0, 1, 3);
    FQ_S(1, 0, 2); FQ_S(1, 1, 2); FQ_S(1, 0, 3); FQ_S(1, 1, 3);
    if (MIX == MIX_RX) {
        FQ_S(2, 0, 0); FQ_S(2, 0, 1); FQ_S(2, 1, 0); FQ_S(2, 1, 1);
    } else {
        FQ_S(2, 0, 3);
    }
#undef FQ_S
    set_error("select_pass16: unsupported combination ph=%d ma=%d mb=%d", ph, ma, mb);
    return FQ_ERR_UNSUPPORTED;
}

template <int MIX, int COST, int NR>
static int launch_tma(const PassParams &P, const CUtensorMap &ms, const CUtensorMap &mc, int grid, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_pass_tma<MIX, COST, NR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)tma_smem_bytes<COST>(kMaxTableHi));
        configured = true;
    }
    k_pass_tma<MIX, COST, NR><<<grid, kThreads, tma_smem_bytes<COST>(P.table_hi), st>>>(P, ms, mc);
    FQ_LAUNCHED("k_pass_tma");
    return FQ_OK;
}

template <int MIX, int COST, int NR>
static int launch_pass8(const PassParams &P, int grid, cudaStream_t st) {
    static bool configured = false;
    const size_t smem = (size_t)(k8Padded + (kTableLo + kMaxTableHi) * kCopies) * sizeof(double2);
    if (!configured) {
        cudaFuncSetAttribute(k_pass8<MIX, COST, NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    const size_t need = (size_t)(k8Padded + (kTableLo + P.table_hi) * kCopies) * sizeof(double2);
    k_pass8<MIX, COST, NR><<<grid, k8Threads, need, st>>>(P);
    FQ_LAUNCHED("k_pass8");
    return FQ_OK;
}

template <int MIX, int COST, int NR>
static int launch_pass8t(const PassParams &P, const CUtensorMap &ms, const CUtensorMap &mc, int grid,
                         cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_pass8t<MIX, COST, NR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)p8t_smem_bytes<COST>(kMaxTableHi));
        configured = true;
    }
    k_pass8t<MIX, COST, NR><<<grid, k8Threads, p8t_smem_bytes<COST>(P.table_hi), st>>>(P, ms, mc);
    FQ_LAUNCHED("k_pass8t");
    return FQ_OK;
}

// 0: 16-amplitude register-load pass, 1: 16-amplitude TMA-staged pass,
// 2: 8-amplitude register-load pass, 3: 8-amplitude TMA-staged pass
static int g_kernel = 0;
static bool g_phase_tables = true;
static bool g_fuse = true;
static int g_probe = 0;  // development: time the tile access pattern alone (kernel 0)

// Launches one planned pass with the selected kernel family.  Returns the grid
// actually used (the expectation partial count) through *grid_out.
static int dispatch_pass(int mix, int cost, int nr, PassParams &P, long long n_tiles, int n, cudaStream_t st,
                         int *grid_out) {
    const int sms = sm_count() > 0 ? sm_count() : 148;
    alignas(64) CUtensorMap ms, mc;
    std::memset(&ms, 0, sizeof ms);
    std::memset(&mc, 0, sizeof mc);
    P.probe_l2 = g_probe == 2;
    bool tma = g_kernel == 1 || g_kernel == 3;
    if (tma)
        tma = build_tile_map(&ms, P.psi, n, P.tile_pos, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, 2, P.tma_rank,
                             P.tma_outer_shift, P.tma_outer_bits);
    P.cost_tma = 0;
    if (tma && P.costs && (P.phase_round >= 0 || P.expect)) {
        const bool ok = (cost == FQ_COST_F64)
                            ? build_tile_map(&mc, P.costs, n, P.tile_pos, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, 1,
                                             P.cost_rank, P.cost_outer_shift, P.cost_outer_bits)
                            : build_tile_map(&mc, P.costs, n, P.tile_pos, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, 1,
                                             P.cost_rank, P.cost_outer_shift, P.cost_outer_bits);
        P.cost_tma = ok ? 1 : 0;
    }
    if (g_kernel == 3 && tma) {
        const int grid = (int)std::min<long long>(n_tiles, sms);
        *grid_out = grid;
#define FQ_8T(M, C, R) if (mix == M && cost == C && nr == R) return launch_pass8t<M, C, R>(P, ms, mc, grid, st)
        FQ_8T(MIX_RX, FQ_COST_F64, 4); FQ_8T(MIX_RX, FQ_COST_F64, 7);
        FQ_8T(MIX_RX, FQ_COST_U16, 4); FQ_8T(MIX_RX, FQ_COST_U16, 7);
        FQ_8T(MIX_SU2, FQ_COST_F64, 4); FQ_8T(MIX_SU2, FQ_COST_F64, 7);
        FQ_8T(MIX_SU2, FQ_COST_U16, 4); FQ_8T(MIX_SU2, FQ_COST_U16, 7);
#undef FQ_8T
    } else if (g_kernel >= 2) {
        const int grid = (int)std::min<long long>(n_tiles, (long long)sms * 2);
        *grid_out = grid;
#define FQ_8(M, C, R) if (mix == M && cost == C && nr == R) return launch_pass8<M, C, R>(P, grid, st)
        FQ_8(MIX_RX, FQ_COST_F64, 4); FQ_8(MIX_RX, FQ_COST_F64, 7);
        FQ_8(MIX_RX, FQ_COST_U16, 4); FQ_8(MIX_RX, FQ_COST_U16, 7);
        FQ_8(MIX_SU2, FQ_COST_F64, 4); FQ_8(MIX_SU2, FQ_COST_F64, 7);
        FQ_8(MIX_SU2, FQ_COST_U16, 4); FQ_8(MIX_SU2, FQ_COST_U16, 7);
#undef FQ_8
    } else if (tma) {
        const int grid = (int)std::min<long long>(n_tiles, sms);
        *grid_out = grid;
#define FQ_T(M, C, R) if (mix == M && cost == C && nr == R) return launch_tma<M, C, R>(P, ms, mc, grid, st)
        FQ_T(MIX_RX, FQ_COST_F64, 3); FQ_T(MIX_RX, FQ_COST_F64, 5);
        FQ_T(MIX_RX, FQ_COST_U16, 3); FQ_T(MIX_RX, FQ_COST_U16, 5);
        FQ_T(MIX_SU2, FQ_COST_F64, 3); FQ_T(MIX_SU2, FQ_COST_F64, 5);
        FQ_T(MIX_SU2, FQ_COST_U16, 3); FQ_T(MIX_SU2, FQ_COST_U16, 5);
#undef FQ_T
    } else {
        const int grid = (int)std::min<long long>(n_tiles, (long long)sms * max_blocks_per_sm);
        *grid_out = grid;
        if (g_probe == 1) {  // memory-pattern ceiling: same tiles, no math, no transposes
            P.phase_round = -1;
            P.expect = 0;
            return launch_pass16<MIX_RX, FQ_COST_U16, 0, 0, 2, 1>(P, grid, st);
        }
        if (g_probe == 3 && mix == MIX_RX && cost == FQ_COST_U16 && P.phase_round < 0 &&
            !(nr == 5 || P.maskB[0] || P.maskB[1] || P.maskB[2])) {  // on-chip compute only
            P.expect = 0;
            return P.A.mode ? launch_pass16<MIX_RX, FQ_COST_U16, 0, 1, 2, 2>(P, grid, st)
                            : launch_pass16<MIX_RX, FQ_COST_U16, 0, 0, 2, 2>(P, grid, st);
        }
        const int ph = P.phase_round < 0 ? 0 : (P.phase_at == 1 ? 1 : 2);
        const bool has_b = nr == 5 || P.maskB[0] || P.maskB[1] || P.maskB[2];
        const int ma = P.A.mode, mb = has_b ? P.B.mode : 2;
        if (mix == MIX_RX && cost == FQ_COST_F64) return select_pass16<MIX_RX, FQ_COST_F64>(P, ph, ma, mb, grid, st);
        if (mix == MIX_RX && cost == FQ_COST_U16) return select_pass16<MIX_RX, FQ_COST_U16>(P, ph, ma, mb, grid, st);
        if (mix == MIX_SU2 && cost == FQ_COST_F64) return select_pass16<MIX_SU2, FQ_COST_F64>(P, ph, ma, mb, grid, st);
        if (mix == MIX_SU2 && cost == FQ_COST_U16) return select_pass16<MIX_SU2, FQ_COST_U16>(P, ph, ma, mb, grid, st);
    }
    set_error("dispatch_pass: unsupported combination");
    return FQ_ERR_UNSUPPORTED;
}

static std::vector<PlannedPass> plan_x(int n, int nl, const fq_layer *layers, std::vector<Group> &groups,
                                       std::vector<int> &layer_group_base, bool fuse) {
    groups.clear();
    layer_group_base.assign(nl, 0);
    std::vector<PlannedPass> seq;
    std::vector<int> prev_targets;
    int prev_base = -1, dir = 0;
    for (int l = 0; l < nl; ++l) {
        std::vector<int> targets;
        for (int q = std::max(0, layers[l].q_lo); q < std::min(n, layers[l].q_hi); ++q) targets.push_back(q);
        int gbase;
        if (prev_base >= 0 && same_targets(targets, prev_targets)) {
            gbase = prev_base;
        } else {
            gbase = (int)groups.size();
            auto g = make_groups(n, targets);
            groups.insert(groups.end(), g.begin(), g.end());
            dir = 0;
        }
        const int ng = (int)(targets.empty() ? 0 : make_groups(n, targets).size());
        layer_group_base[l] = gbase;
        if (ng == 0) {  // phase-only layer
            if (phase_active(layers[l])) seq.push_back({-1, -1, -1, l, 1});
            prev_targets = targets;
            prev_base = gbase;
            continue;
        }
        for (int i = 0; i < ng; ++i) {
            const int gi = gbase + (dir ? ng - 1 - i : i);
            if (i == 0 && fuse && !seq.empty() && seq.back().group == gi && seq.back().layerB < 0 &&
                seq.back().layerA == l - 1 && (seq.back().phase_layer < 0 || !phase_active(layers[l]))) {
                // fuse: mixer_{l-1} on tile, phase_l, mixer_l on tile
                seq.back().layerB = l;
                if (phase_active(layers[l])) {
                    seq.back().phase_layer = l;
                    seq.back().phase_at = 2;
                }
                continue;
            }
            PlannedPass pp{gi, l, -1, (i == 0 && phase_active(layers[l])) ? l : -1, 1};
            seq.push_back(pp);
        }
        dir ^= 1;
        prev_targets = targets;
        prev_base = gbase;
    }
    return seq;
}

static int run_x_program(const fq_evolve_desc *d, cudaStream_t st) {
    const int n = d->n;
    std::vector<Group> groups;
    std::vector<int> gbase;
    auto seq = plan_x(n, d->n_layers, d->layers, groups, gbase, g_fuse);
    const int mix = (d->mixer == FQ_MIXER_X) ? MIX_RX : MIX_SU2;
    const long long n_tiles = 1LL << (n - kTileBits);
    int table_hi = 0;
    if (d->cost_kind == FQ_COST_U16 && d->cost_levels > 0 && g_phase_tables) {
        const int rows = ((d->cost_levels - 1) >> 6) + 1;
        table_hi = rows <= kMaxTableHi ? rows : 0;
    }
    bool init_pending = d->init != 0;
    double2 *psi = static_cast<double2 *>(d->psi);
    const long long size = 1LL << n;

    if (seq.empty()) {
        if (init_pending) {
            int s = fq_init_state(psi, size, -1, d->init_amp, 0, st);
            if (s) return s;
        }
        if (d->expectation_dev)
            return fq_expectation(psi, d->costs, d->cost_kind, d->cost_scale, d->cost_offset, size,
                                  d->expectation_dev, d->scratch, st);
        return FQ_OK;
    }
    for (size_t si = 0; si < seq.size(); ++si) {
        const PlannedPass &pp = seq[si];
        const bool last = (si + 1 == seq.size());
        if (pp.group < 0) {  // standalone phase
            if (init_pending) {
                int s = fq_init_state(psi, size, -1, d->init_amp, 0, st);
                if (s) return s;
                init_pending = false;
            }
            const fq_layer &L = d->layers[pp.phase_layer];
            if (d->cost_kind == FQ_COST_U16)
                k_phase_u16<<<grid_for(size, 256, 8), 256, 0, st>>>(psi, static_cast<const uint16_t *>(d->costs), size,
                                                                    L.gamma, d->cost_scale, d->cost_offset);
            else
                k_phase_f64<<<grid_for(size, 256, 8), 256, 0, st>>>(psi, static_cast<const double *>(d->costs), size,
                                                                    L.gamma);
            FQ_LAUNCHED("k_phase");
            if (last && d->expectation_dev)
                return fq_expectation(psi, d->costs, d->cost_kind, d->cost_scale, d->cost_offset, size,
                                      d->expectation_dev, d->scratch, st);
            continue;
        }
        const Group &g = groups[pp.group];
        PassParams P;
        std::memset(&P, 0, sizeof P);
        P.psi = psi;
        P.costs = d->costs;
        P.cost_scale = d->cost_scale;
        P.cost_offset = d->cost_offset;
        P.partials = d->scratch;
        P.init_amp = d->init_amp;
        P.n_tiles = n_tiles;
        P.table_hi = table_hi;
        for (int i = 0; i < kTileBits; ++i) P.tile_pos[i] = g.tile_pos[i];
        P.init = init_pending ? 1 : 0;
        init_pending = false;
        P.expect = (last && d->expectation_dev) ? 1 : 0;
        // target mask over tile bits
        int tmask = 0;
        for (int i = 0; i < kTileBits; ++i)
            if (std::find(g.targets.begin(), g.targets.end(), g.tile_pos[i]) != g.targets.end()) tmask |= 1 << i;
        const bool two = pp.layerB >= 0;
        const bool mid_phase = two && pp.phase_layer >= 0 && pp.phase_at == 2;
        // Round programs.  16-amplitude kernels: register tile bits start at
        // 8,0,4 (| 0,8); 8-amplitude kernel: 9,0,3,6 (| 3,0,9).  Without a phase
        // between the two layers both sets run back to back in every round.
        const bool k8 = g_kernel >= 2;
        const int rb16[5] = {8, 0, 4, 0, 8}, rb8[7] = {9, 0, 3, 6, 3, 0, 9};
        const int base_rounds = k8 ? 4 : 3;
        P.nrounds = mid_phase ? 2 * base_rounds - 1 : base_rounds;
        for (int r = 0; r < 8; ++r) {
            P.maskA[r] = P.maskB[r] = 0;
            if (r >= P.nrounds) continue;
            const int m = k8 ? (tmask >> rb8[r]) & 7 : (tmask >> rb16[r]) & 15;
            if (!mid_phase) {
                P.maskA[r] = m;
                P.maskB[r] = two ? m : 0;
            } else {
                P.maskA[r] = r < base_rounds ? m : 0;
                P.maskB[r] = r >= base_rounds - 1 ? m : 0;
            }
        }
        P.phase_round = -1;
        if (pp.phase_layer >= 0) {
            P.gamma = d->layers[pp.phase_layer].gamma;
            if (pp.phase_at == 1) {
                P.phase_round = 0;
                P.phase_at = 1;
            } else {
                P.phase_round = base_rounds - 1;
                P.phase_at = 2;
            }
        }
        // coefficients
        double fscale = 1.0;
        const int ntarget = (int)g.targets.size();
        auto fill = [&](int layer, CoefSet &C) {
            if (mix == MIX_RX) {
                double f;
                rx_coef(d->layers[layer].beta, C, f);
                fscale *= std::pow(f, ntarget);
            } else {
                for (int i = 0; i < kTileBits; ++i) {
                    const double *c4 = d->su2 + ((size_t)layer * n + g.tile_pos[i]) * 4;
                    C.a[i] = make_double2(c4[0], c4[1]);
                    C.b[i] = make_double2(c4[2], c4[3]);
                }
            }
        };
        fill(pp.layerA, P.A);
        if (two) fill(pp.layerB, P.B);
        P.final_scale = fscale;
        int grid = 0;
        int s = dispatch_pass(mix, d->cost_kind, P.nrounds, P, n_tiles, n, st, &grid);
        if (s) return s;
        if (P.expect) {
            k_sum_partials<<<1, 32, 0, st>>>(d->scratch, grid, d->expectation_dev);
            FQ_LAUNCHED("k_sum_partials");
        }
    }
    return FQ_OK;
}

// XY mixers above the resident size: phase sweep + one pair kernel per gate in
// the documented order (reference mixers.py:109-137).
static void xy_gates(int n, int kind, std::vector<std::pair<int, int>> &g) {
    g.clear();
    if (kind == FQ_MIXER_XY_RING) {
        if (n == 2) { g.push_back({0, 1}); return; }
        for (int q = 0; q < n - 1; q += 2) g.push_back({q, q + 1});
        for (int q = 1; q < n - 1; q += 2) g.push_back({q, q + 1});
        g.push_back({n - 1, 0});
    } else {
        for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j) g.push_back({i, j});
    }
}

static int run_xy_program(const fq_evolve_desc *d, cudaStream_t st) {
    const int n = d->n;
    const long long size = 1LL << n;
    double2 *psi = static_cast<double2 *>(d->psi);
    if (d->init) {
        int s = fq_init_state(psi, size, -1, d->init_amp, 0, st);
        if (s) return s;
    }
    std::vector<std::pair<int, int>> gates;
    xy_gates(n, d->mixer, gates);
    for (int l = 0; l < d->n_layers; ++l) {
        const fq_layer &L = d->layers[l];
        if (phase_active(L)) {
            if (d->cost_kind == FQ_COST_U16)
                k_phase_u16<<<grid_for(size, 256, 8), 256, 0, st>>>(psi, static_cast<const uint16_t *>(d->costs), size,
                                                                    L.gamma, d->cost_scale, d->cost_offset);
            else
                k_phase_f64<<<grid_for(size, 256, 8), 256, 0, st>>>(psi, static_cast<const double *>(d->costs), size,
                                                                    L.gamma);
            FQ_LAUNCHED("k_phase");
        }
        const double c = std::cos(L.beta), s = std::sin(L.beta);
        for (auto &gp : gates) {
            int r = fq_xy_on_pairs(psi, size, c, s, std::min(gp.first, gp.second), std::max(gp.first, gp.second), st);
            if (r) return r;
        }
    }
    if (d->expectation_dev)
        return fq_expectation(psi, d->costs, d->cost_kind, d->cost_scale, d->cost_offset, size, d->expectation_dev,
                              d->scratch, st);
    return FQ_OK;
}

template <int COST>
static int launch_resident(const ResParams &P, int batch, const double *su2_dev, cudaStream_t st) {
    const size_t smem = (size_t)(1 << P.n) * sizeof(double2);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_resident<COST>, cudaFuncAttributeMaxDynamicSharedMemorySize, 1 << 16);
        configured = true;
    }
    k_resident<COST><<<batch, kResThreads, smem, st>>>(P, su2_dev);
    FQ_LAUNCHED("k_resident");
    return FQ_OK;
}

static void fill_gates(ResParams &P, int n, int mixer) {
    P.n_gates = 0;
    if (mixer == FQ_MIXER_XY_RING || mixer == FQ_MIXER_XY_COMPLETE) {
        std::vector<std::pair<int, int>> g;
        xy_gates(n, mixer, g);
        for (auto &e : g) {
            P.gates[P.n_gates][0] = (unsigned char)std::min(e.first, e.second);
            P.gates[P.n_gates][1] = (unsigned char)std::max(e.first, e.second);
            ++P.n_gates;
        }
    }
}

static int run_resident_program(const fq_evolve_desc *d, cudaStream_t st) {
    // chunk the layers into launches of kResMaxLayers; custom-mixer
    // coefficients travel through the caller's scratch buffer.
    const int n = d->n;
    for (int l0 = 0; l0 < std::max(1, d->n_layers); l0 += kResMaxLayers) {
        const int cnt = std::min(kResMaxLayers, d->n_layers - l0);
        ResParams *P = new ResParams;
        std::memset(P, 0, sizeof *P);
        P->n = n;
        P->p = std::max(cnt, 0);
        P->mixer = d->mixer;
        P->costs = d->costs;
        P->cost_scale = d->cost_scale;
        P->cost_offset = d->cost_offset;
        P->init = (l0 == 0 && d->init) ? 1 : 0;
        P->init_amp = d->init_amp;
        P->psi_in = static_cast<const double2 *>(d->psi);
        P->in_stride = 0;
        P->psi_out = static_cast<double2 *>(d->psi);
        const bool last = (l0 + kResMaxLayers >= d->n_layers);
        P->exp_out = last ? d->expectation_dev : nullptr;
        for (int i = 0; i < cnt; ++i) {
            P->gam[i] = d->layers[l0 + i].gamma;
            P->bet[i] = d->layers[l0 + i].beta;
            P->phase_on[i] = (unsigned char)(d->layers[l0 + i].apply_phase != 0);
            P->qlo[i] = (unsigned char)std::max(0, std::min(n, d->layers[l0 + i].q_lo));
            P->qhi[i] = (unsigned char)std::max((int)P->qlo[i], std::min(n, d->layers[l0 + i].q_hi));
        }
        fill_gates(*P, n, d->mixer);
        const double *su2_dev = nullptr;
        if (d->mixer == FQ_MIXER_CUSTOM && cnt > 0) {
            const size_t bytes = (size_t)cnt * n * 4 * sizeof(double);
            if (bytes > FQ_SCRATCH_DOUBLES * sizeof(double)) {
                delete P;
                set_error("custom mixer program too large for scratch (%d layers x %d qubits)", cnt, n);
                return FQ_ERR_UNSUPPORTED;
            }
            cudaError_t e = cudaMemcpyAsync(d->scratch, d->su2 + (size_t)l0 * n * 4, bytes, cudaMemcpyHostToDevice, st);
            if (e != cudaSuccess) { delete P; return cuda_status(e, "cudaMemcpyAsync(su2)"); }
            su2_dev = d->scratch;
        }
        int s = (d->cost_kind == FQ_COST_U16) ? launch_resident<FQ_COST_U16>(*P, 1, su2_dev, st)
                                              : launch_resident<FQ_COST_F64>(*P, 1, su2_dev, st);
        delete P;
        if (s) return s;
        if (d->mixer == FQ_MIXER_CUSTOM && cnt > 0) {
            // the scratch buffer is reused by the next chunk: order it behind this launch
            cudaError_t e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) return cuda_status(e, "cudaStreamSynchronize");
        }
        if (d->n_layers <= 0) break;
    }
    return FQ_OK;
}

}  // namespace fq

using namespace fq;

extern "C" {

int fq_qaoa_evolve(const fq_evolve_desc *d, void *stream) {
    FQ_CHECK_ARG(d && d->psi && d->n >= 1 && d->n <= 40, "fq_qaoa_evolve: bad descriptor");
    FQ_CHECK_ARG(d->n_layers >= 0 && (d->n_layers == 0 || d->layers), "fq_qaoa_evolve: bad layers");
    bool need_costs = d->expectation_dev != nullptr;
    for (int l = 0; l < d->n_layers; ++l) need_costs |= d->layers[l].apply_phase != 0;
    FQ_CHECK_ARG(d->costs || !need_costs, "fq_qaoa_evolve: null costs");
    FQ_CHECK_ARG(d->cost_kind == FQ_COST_F64 || d->cost_kind == FQ_COST_U16, "fq_qaoa_evolve: bad cost kind");
    FQ_CHECK_ARG(d->mixer >= FQ_MIXER_X && d->mixer <= FQ_MIXER_CUSTOM, "fq_qaoa_evolve: bad mixer");
    FQ_CHECK_ARG(d->mixer != FQ_MIXER_CUSTOM || d->su2, "fq_qaoa_evolve: custom mixer needs su2 table");
    FQ_CHECK_ARG(!d->expectation_dev || d->scratch, "fq_qaoa_evolve: expectation needs scratch");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (d->n <= kTileBits) {
        FQ_CHECK_ARG(d->mixer != FQ_MIXER_CUSTOM || d->scratch, "fq_qaoa_evolve: custom mixer needs scratch");
        return run_resident_program(d, st);
    }
    if (d->mixer == FQ_MIXER_XY_RING || d->mixer == FQ_MIXER_XY_COMPLETE) return run_xy_program(d, st);
    return run_x_program(d, st);
}

int fq_set_option(const char *name, int value) {
    if (!name) return FQ_ERR_ARG;
    if (std::strcmp(name, "kernel") == 0) {
        if (value < 0 || value > 3) return FQ_ERR_ARG;
        g_kernel = value;
        return FQ_OK;
    }
    if (std::strcmp(name, "probe") == 0) {
        g_probe = value;
        return FQ_OK;
    }
    if (std::strcmp(name, "fuse") == 0) {
        g_fuse = value != 0;
        return FQ_OK;
    }
    if (std::strcmp(name, "phase_tables") == 0) {
        g_phase_tables = value != 0;
        return FQ_OK;
    }
    set_error("fq_set_option: unknown option %s", name);
    return FQ_ERR_ARG;
}

int fq_plan_x_passes(int n, int n_layers, const fq_layer *layers) {
    if (n <= kTileBits) return n_layers > 0 ? 1 : 0;
    std::vector<Group> groups;
    std::vector<int> gbase;
    return (int)plan_x(n, n_layers, layers, groups, gbase, g_fuse).size();
}

int fq_qaoa_evolve_batched(int n, int mixer, const void *costs, int cost_kind, double scale, double offset, int p,
                           int batch, const double *gammas, const double *betas, const void *psi_init, void *psi_out,
                           double *out_dev, void *stream) {
    FQ_CHECK_ARG(n >= 1 && n <= kTileBits, "fq_qaoa_evolve_batched: n=%d must be in [1, %d]", n, kTileBits);
    FQ_CHECK_ARG(costs && out_dev && batch >= 1 && p >= 0 && gammas && betas, "fq_qaoa_evolve_batched: bad args");
    FQ_CHECK_ARG(mixer != FQ_MIXER_CUSTOM, "fq_qaoa_evolve_batched: custom mixers are not batched");
    FQ_CHECK_ARG((long long)batch * p <= kResMaxLayers, "fq_qaoa_evolve_batched: batch*p must be <= %d",
                 kResMaxLayers);
    ResParams *P = new ResParams;
    std::memset(P, 0, sizeof *P);
    P->n = n;
    P->p = p;
    P->mixer = mixer;
    P->costs = costs;
    P->cost_scale = scale;
    P->cost_offset = offset;
    P->init = psi_init ? 0 : 1;
    P->init_amp = 1.0 / std::sqrt((double)(1LL << n));
    P->psi_in = static_cast<const double2 *>(psi_init);
    P->in_stride = 0;
    P->psi_out = static_cast<double2 *>(psi_out);
    P->exp_out = out_dev;
    fill_gates(*P, n, mixer);
    for (int l = 0; l < p; ++l) {
        P->phase_on[l] = 1;
        P->qlo[l] = 0;
        P->qhi[l] = (unsigned char)n;
    }
    for (long long i = 0; i < (long long)batch * p; ++i) {
        P->gam[i] = gammas[i];
        P->bet[i] = betas[i];
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int s = (cost_kind == FQ_COST_U16) ? launch_resident<FQ_COST_U16>(*P, batch, nullptr, st)
                                             : launch_resident<FQ_COST_F64>(*P, batch, nullptr, st);
    delete P;
    return s;
}

}  // extern "C"
