// Tiled pass kernel of the fused QAOA evolution (sm_100a), shared by the
// evolve.cu planner and the per-(mixer, cost) instantiation units
// pass_*.cu, which are compiled in parallel.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstring>
#include <type_traits>
#include <vector>

#include <cuda.h>

#include "common.cuh"

namespace fq {


constexpr int kTileBits = 12;
constexpr int kTile = 1 << kTileBits;
constexpr int kThreads = 256;
constexpr int kRegs = 16;

enum { MIX_RX = 0, MIX_SU2 = 1 };

// State precision: R = double (complex128, the reference's) or float
// (complex64, optional).  C2<R> is the interleaved complex element.
template <typename R> struct Cx;
template <> struct Cx<double> {
    using T = double2;
    static __host__ __device__ __forceinline__ double2 make(double x, double y) { return make_double2(x, y); }
};
template <> struct Cx<float> {
    using T = float2;
    static __host__ __device__ __forceinline__ float2 make(float x, float y) { return make_float2(x, y); }
};
template <typename R> using C2 = typename Cx<R>::T;
// phase-table copies: one per bank group of the access width (16 B: 8 per 128 B, 8 B: 16)
template <typename R> constexpr int table_copies() { return 128 / (int)sizeof(C2<R>); }
enum { PAT8 = 0, PAT0 = 1, PAT4 = 2 };  // tile bits held in registers: 8-11 / 0-3 / 4-7

// Round programs (register patterns visited by one pass):
//   SEQ_840   8 | 0 | 4        one layer (or two with no phase between) on a 12-bit group
//   SEQ_84    8 | 4            same, targets only in tile bits 4-11
//   SEQ_84048 8 | 0 | 4 ph 4 | 0 | 8   two layers with the phase between, 12-bit group
//   SEQ_848   8 | 4 ph 4 | 8            two layers with the phase between, targets in bits 4-11
enum { SEQ_840 = 0, SEQ_84 = 1, SEQ_84048 = 2, SEQ_848 = 3 };

__host__ __device__ constexpr int seq_rounds(int seq) {
    return seq == SEQ_840 ? 3 : seq == SEQ_84 ? 2 : seq == SEQ_84048 ? 5 : 3;
}
__host__ __device__ constexpr int seq_pat(int seq, int r) {
    return seq == SEQ_840   ? (r == 0 ? PAT8 : r == 1 ? PAT0 : PAT4)
         : seq == SEQ_84    ? (r == 0 ? PAT8 : PAT4)
         : seq == SEQ_84048 ? (r == 0 || r == 4 ? PAT8 : (r == 1 || r == 3) ? PAT0 : PAT4)
                            : (r == 1 ? PAT4 : PAT8);
}
__host__ __device__ constexpr int pat_first_bit(int pat) { return pat == PAT8 ? 8 : pat == PAT0 ? 0 : 4; }
__host__ __device__ constexpr bool seq_heavy(int seq) { return seq == SEQ_84048 || seq == SEQ_848; }

struct CoefSet {
    double r;      // RX: t (mode 0) or u (mode 1)
    int mode;      // RX: 0 -> (1, t), 1 -> (u, 1)
    double2 a[kTileBits], b[kTileBits];  // SU2: per tile bit
};

struct PassParams {
    void *psi;                // C2<R>[2^n]
    const void *costs;
    double cost_scale, cost_offset;
    double *partials;
    double init_amp;
    double gamma;
    double final_scale;
    long long n_tiles;
    int tile_pos[kTileBits];  // physical bit of tile bit i (ascending)
    int init;                 // generate |+> instead of loading
    int expect;               // accumulate sum c|x|^2 in the last round
    int table_hi;             // U16 phase: rows of the high table (0 -> sincos of the decoded cost)
    unsigned char maskA[8], maskB[8];  // per round: register bits getting set A / set B butterflies
    int pf_dist;              // L2 prefetch distance in grid strides (0: off)
    int run_bits;             // tile bits 0..run_bits-1 sit at physical bits 0..run_bits-1 (contiguous runs)
    int pf_cost;              // also prefetch the cost slice of the tile
    int cost_l2;              // cost loads at normal L2 priority (short cost runs), else evict-first
    int cost_stage;           // uint16 costs consumed after a transpose: two 16-B loads per thread into a
                              // shared cost tile instead of 16 scattered 2-B loads (needs run_bits >= 3)
    long long c11;            // byte offset of tile bit 11 in the uint16 cost vector
    int lane;                 // K_LANE3 programs: tile bits 0..3 (here only bit 3) that are targets, applied as
                              // lane butterflies (warp shuffles) in the PAT4 rounds
    int sm_rank, sm_shift[5], sm_bits[5];  // state tensor map: rank, outer-dim coordinate = (t >> shift) & (2^bits - 1)
    int cm_rank, cm_shift[5], cm_bits[5];  // cost tensor map (cm_rank = 0: no cost prefetch)
    int probe;                // development: 1 no cost loads, 2 fixed table row, 4 no phase multiply
    long long roff[3][kRegs]; // per pattern: BYTE offset of register i in the state (read from the constant
                              // bank, so no register holds the 16 offsets across the rounds)
    long long coff[3][kRegs]; // the same in the cost vector (bytes)
    long long tile_mask;      // bits at the tile positions
    long long step_dep;       // pdep(gridDim.x) into the non-tile positions: base(t + grid) = next_base(base(t))
    int reverse;              // walk the tiles from the top (alternate passes: L2 reuse)
    CoefSet A, B;
    // sharded state (G = true passes): the tile's top k tile bits are the k global
    // qubits, i.e. the shard index.  psi / costs point at shard 0's mapping in
    // this process and sdelta[s] / cdelta[s] are shard s's byte offsets from it
    // (peer allocations: not additive over the global bits, so they enter as
    // whole per-shard offsets: register offsets of PAT8, thread offsets of PAT4).
    long long tile0;          // first tile of this launch (rank r: its 1/K of the tiles)
    int gbits;                // k: tile bits 12-k..11 are the global qubits (their tile_pos is unused)
    int gshift;               // PAT4: shard index = (tid >> gshift) & gmask
    int gmask;
    long long sdelta[8], cdelta[8];
};

constexpr int kTableLo = 64;     // low-table rows (6 level bits)
constexpr int kMaxTableHi = 256; // high-table rows -> levels < 16384 use tables
constexpr int kCopies = 8;       // one copy per 16-B bank group: conflict-free random lookups

template <int PAT>
__device__ __forceinline__ int tile_bit_of_reg(int j) {
    return PAT == PAT8 ? 8 + j : (PAT == PAT0 ? j : 4 + j);
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

// physical offset of this thread's element 0 for pattern PAT (G: the global
// tile bits contribute through the shard offsets instead)
template <int PAT, bool G = false>
__device__ __forceinline__ long long thread_offset(const PassParams &P, int tid) {
    long long off = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        int tb;
        if (PAT == PAT8) tb = j;
        else if (PAT == PAT0) tb = 4 + j;
        else tb = (j < 4) ? j : j + 4;
        if (G && tb >= kTileBits - P.gbits) continue;
        if ((tid >> j) & 1) off += 1LL << P.tile_pos[tb];
    }
    return off;
}

struct NoOp {
    __device__ __forceinline__ void operator()() const {}
};

// `mid` runs between the two barriers (shared data written before the first is
// visible, and every thread is done with it before anyone passes the second).
template <int FROM, int TO, typename T, typename F = NoOp>
__device__ __forceinline__ void transpose(T *sm, T (&v)[kRegs], int tid, F mid = F()) {
    T *p = sm + pat_base<FROM>(tid);
#pragma unroll
    for (int i = 0; i < kRegs; ++i) p[pat_step<FROM>(i)] = v[i];
    __syncthreads();
    mid();
    const T *q = sm + pat_base<TO>(tid);
#pragma unroll
    for (int i = 0; i < kRegs; ++i) v[i] = q[pat_step<TO>(i)];
    __syncthreads();
}

// ---- butterflies
template <typename T, typename R>
__device__ __forceinline__ void bfly_rx0(T &x0, T &x1, R t) {
    // (x0 - i t x1, x1 - i t x0)
    const T a = x0, b = x1;
    x0 = Cx<R>::make(fma(t, b.y, a.x), fma(-t, b.x, a.y));
    x1 = Cx<R>::make(fma(t, a.y, b.x), fma(-t, a.x, b.y));
}
template <typename T, typename R>
__device__ __forceinline__ void bfly_rx1(T &x0, T &x1, R u) {
    // (u x0 - i x1, u x1 - i x0)
    const T a = x0, b = x1;
    x0 = Cx<R>::make(fma(u, a.x, b.y), fma(u, a.y, -b.x));
    x1 = Cx<R>::make(fma(u, b.x, a.y), fma(u, b.y, -a.x));
}
template <typename T>
__device__ __forceinline__ void bfly_su2(T &x0, T &x1, T a, T b) {
    // y0 = a x0 - conj(b) x1 ; y1 = b x0 + conj(a) x1   (reference _kernels.py:26-27)
    const T p = x0, q = x1;
    x0.x = a.x * p.x - a.y * p.y - b.x * q.x - b.y * q.y;
    x0.y = a.x * p.y + a.y * p.x - b.x * q.y + b.y * q.x;
    x1.x = b.x * p.x - b.y * p.y + a.x * q.x + a.y * q.y;
    x1.y = b.x * p.y + b.y * p.x + a.x * q.y - a.y * q.x;
}

// Butterflies of one coefficient set on the register bits in `mask`.
// M: RX form 0 -> (1, t), 1 -> (u, 1), 3 -> chosen at run time.
template <int MIX, int M, int PAT, typename R>
__device__ __forceinline__ void bfly16(C2<R> (&v)[kRegs], const CoefSet &C, int mask) {
    if (MIX == MIX_RX && M == 3) {
        if (C.mode == 0) bfly16<MIX, 0, PAT, R>(v, C, mask);
        else bfly16<MIX, 1, PAT, R>(v, C, mask);
        return;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (!((mask >> j) & 1)) continue;
        if (MIX == MIX_RX) {
            const R r = (R)C.r;
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
            const C2<R> a = Cx<R>::make((R)C.a[tb].x, (R)C.a[tb].y), b = Cx<R>::make((R)C.b[tb].x, (R)C.b[tb].y);
#pragma unroll
            for (int i = 0; i < kRegs; ++i)
                if (!(i & (1 << j))) bfly_su2(v[i], v[i | (1 << j)], a, b);
        }
    }
}

// RX butterflies on a lane bit: the partner amplitude sits in lane ^ LM; both
// halves of the pair take the same form, own' = own - i t partner (M = 0) or
// u own - i partner (M = 1), with the register butterflies' FMA order (bit-identical).
template <int M, int LM, typename R>
__device__ __forceinline__ void lane_bfly16(C2<R> (&v)[kRegs], const CoefSet &C) {
    if constexpr (M == 3) {
        if (C.mode == 0) lane_bfly16<0, LM, R>(v, C);
        else lane_bfly16<1, LM, R>(v, C);
        return;
    } else {
        const R r = (R)C.r;
#pragma unroll
        for (int i = 0; i < kRegs; ++i) {
            const R px = __shfl_xor_sync(0xffffffffu, v[i].x, LM), py = __shfl_xor_sync(0xffffffffu, v[i].y, LM);
            if (M == 0) v[i] = Cx<R>::make(fma(r, py, v[i].x), fma(-r, px, v[i].y));
            else v[i] = Cx<R>::make(fma(r, v[i].x, py), fma(r, v[i].y, -px));
        }
    }
}

// ---- phase
// exp(-i gamma c) for a float64 cost: the reference's angle = gamma * c, then sincos.
__device__ __forceinline__ double2 phase_f64(double c, double gamma) {
    double s, co;
    fq_sincos(gamma * c, &s, &co);
    return make_double2(co, -s);
}

static __device__ __noinline__ double2 phase_sincos_u16(unsigned v, double scale, double offset, double gamma) {
    return phase_f64(decode_u16((uint16_t)v, scale, offset), gamma);
}

// raw cost entry as held in registers: the double itself, or the uint16 level
template <int COST>
using CostRaw = typename std::conditional<COST == FQ_COST_F64, double, unsigned>::type;

template <int COST>
__device__ __forceinline__ CostRaw<COST> load_cost(const PassParams &P, long long k) {
    if constexpr (COST == FQ_COST_F64) return __ldcs(static_cast<const double *>(P.costs) + k);
    else return (unsigned)__ldcs(static_cast<const unsigned short *>(P.costs) + k);
}

// l2: keep the line in L2 at normal priority instead of evict-first.  With
// short cost runs (< 32 B: 3 low spectators x uint16) a sector holds entries of
// the neighbouring tile, which another CTA reads moments later.
template <int COST>
__device__ __forceinline__ CostRaw<COST> load_cost_at(const char *p, int l2 = 0) {
    if constexpr (COST == FQ_COST_F64) {
        const double *q = reinterpret_cast<const double *>(p);
        return l2 ? __ldcg(q) : __ldcs(q);
    } else {
        const unsigned short *q = reinterpret_cast<const unsigned short *>(p);
        return (unsigned)(l2 ? __ldcg(q) : __ldcs(q));
    }
}

template <int COST>
__device__ __forceinline__ double decode_cost(const PassParams &P, CostRaw<COST> raw) {
    if constexpr (COST == FQ_COST_F64) return raw;
    else return decode_u16((uint16_t)raw, P.cost_scale, P.cost_offset);
}

// exp(-i gamma c): float64 -> sincos; uint16 level v -> T_hi[v >> 6] * T_lo[v & 63],
// each table replicated once per bank group of the access width (copy = lane
// mod copies) so a (quarter- or half-) warp's random lookups never conflict.
// Angles are reduced in double even for complex64 states (gamma * c reaches 1e3).
template <int COST, typename R>
__device__ __forceinline__ C2<R> phase16(const PassParams &P, CostRaw<COST> raw, const C2<R> *tlo,
                                         const C2<R> *thi) {
    if constexpr (COST == FQ_COST_F64) {
        const double2 f = phase_f64(raw, P.gamma);
        return Cx<R>::make((R)f.x, (R)f.y);
    } else {
        if (P.table_hi == 0) {
            const double2 f = phase_sincos_u16(raw, P.cost_scale, P.cost_offset, P.gamma);
            return Cx<R>::make((R)f.x, (R)f.y);
        }
        constexpr int CP = table_copies<R>();
        const int cp = threadIdx.x & (CP - 1);
        return cmul(thi[(raw >> 6) * CP + cp], tlo[(raw & 63) * CP + cp]);
    }
}

// e^{-i gamma c} tables for uint16 levels: c = scale*(64 h + l) + offset
template <typename R>
__device__ __forceinline__ void build_phase_tables(C2<R> *tlo, C2<R> *thi, int n_hi, double gamma, double scale,
                                                   double offset) {
    constexpr int CP = table_copies<R>();
    for (int i = threadIdx.x; i < kTableLo + n_hi; i += blockDim.x) {
        double s, c;
        if (i < kTableLo) sincos(gamma * (scale * (double)i), &s, &c);
        else sincos(gamma * (scale * (double)(64 * (i - kTableLo)) + offset), &s, &c);
        C2<R> *row = (i < kTableLo) ? tlo + i * CP : thi + (i - kTableLo) * CP;
#pragma unroll
        for (int k = 0; k < CP; ++k) row[k] = Cx<R>::make((R)c, (R)-s);
    }
}

// tile number -> base address: insert a zero at every tile bit position
__device__ __forceinline__ long long tile_base(const PassParams &P, long long t) {
    long long base = t;
#pragma unroll
    for (int j = 0; j < kTileBits; ++j) {
        const int p = P.tile_pos[j];
        base = ((base >> p) << (p + 1)) | (base & ((1LL << p) - 1));
    }
    return base;
}

// Tile bases advance in "deposited" space: adding Y = pdep(stride) with the
// tile-bit positions pre-filled with ones lets carries hop over them.
__device__ __forceinline__ long long next_base(long long base, long long mask, long long y) {
    return ((base | mask) + y) & ~mask;
}

__device__ __forceinline__ long long prev_base(long long base, long long mask, long long y) {
    return (base - y) & ~mask;  // borrows pass through the (zero) tile positions
}

// L2 prefetch of a future tile with ONE instruction: the tile is described
// by a tensor map (runs of tile bits = full box dims, runs of outer bits =
// box-1 dims whose coordinates come from the tile number), and
// cp.async.bulk.prefetch.tensor (SASS UTMAPF) fetches the whole strided box
// into L2 while the CTA is busy with the current tile.
__device__ __forceinline__ void tile_coords(long long t, int rank, const int *shift, const int *bits, int *c) {
#pragma unroll
    for (int d = 0; d < 5; ++d)
        c[d] = (d < rank && bits[d] > 0) ? (int)((t >> shift[d]) & ((1LL << bits[d]) - 1)) : 0;
}

__device__ __forceinline__ void tensor_prefetch_l2(const CUtensorMap *map, int rank, const int *c) {
    const uint64_t m = reinterpret_cast<uint64_t>(map);
    switch (rank) {
        case 1:
            asm volatile("cp.async.bulk.prefetch.tensor.1d.L2.global.tile [%0, {%1}];" ::"l"(m), "r"(c[0]) : "memory");
            break;
        case 2:
            asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(m), "r"(c[0]), "r"(c[1])
                         : "memory");
            break;
        case 3:
            asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(m), "r"(c[0]),
                         "r"(c[1]), "r"(c[2]) : "memory");
            break;
        case 4:
            asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(m), "r"(c[0]),
                         "r"(c[1]), "r"(c[2]), "r"(c[3]) : "memory");
            break;
        default:
            asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(m),
                         "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]) : "memory");
            break;
    }
}

__device__ __forceinline__ void prefetch_tile(const PassParams &P, const CUtensorMap *ms, const CUtensorMap *mc,
                                              long long t, bool state) {
    int c[5];
    if (state && P.sm_rank > 0) {
        tile_coords(t, P.sm_rank, P.sm_shift, P.sm_bits, c);
        tensor_prefetch_l2(ms, P.sm_rank, c);
    }
    if (P.pf_cost && P.cm_rank > 0) {
        tile_coords(t, P.cm_rank, P.cm_shift, P.cm_bits, c);
        tensor_prefetch_l2(mc, P.cm_rank, c);
    }
}

// Target mask of round r.  K = 0: the run-time masks of PassParams; K = 4: every
// visited quad is all targets; K = 1..3 (SEQ_84 / SEQ_848 only): the PAT8 quad is
// all targets and the PAT4 quad has its top K bits as targets (a high group of
// 4 + K targets above 8 - K spectators).
// K = K_LANE3 (SEQ_84 / SEQ_848, X mixer): both quads all targets, and tile bit 3
// too — in PAT4 it is lane bit 3, so its butterflies run across lanes (warp
// shuffles) inside the PAT4 rounds: a 9-target high group (3 low spectators,
// n >= 30) runs the two-pattern programs instead of 8|0|4 (one transpose less,
// two less in the fused two-layer pass).
enum { K_RUNTIME = 0, K_FULL = 4, K_LANE3 = 5 };
template <int K, int SEQ>
__device__ __forceinline__ int round_mask(const unsigned char *rt, int r) {
    if constexpr (K == K_RUNTIME) return rt[r];
    else if constexpr (K == K_FULL || K == K_LANE3) return 0xF;
    else return seq_pat(SEQ, r) == PAT4 ? ((0xF << (4 - K)) & 0xF) : 0xF;
}

// Global-memory access modes of a tile: LD_STREAM / ST_STREAM evict-first
// streaming (one HBM round trip per pass); LD_L2 reads through L2 only (data a
// previous sub-pass of a slab sweep left there); ST_L2_KEEP stores with an
// L2::evict_last policy (the next sub-pass re-reads it from L2).
enum { LD_STREAM = 0, LD_L2 = 1 };
enum { ST_STREAM = 0, ST_L2_KEEP = 1 };

template <int LD, typename T>
__device__ __forceinline__ T tile_load(const T *p) {
    if constexpr (LD == LD_L2) return __ldcg(p);
    else return ld_stream(p);
}

__device__ __forceinline__ void st_keep(double2 *p, double2 v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep(float2 *p, float2 v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y), "l"(pol) : "memory");
}

template <int ST, typename T>
__device__ __forceinline__ void tile_store(T *p, T v, unsigned long long pol) {
    if constexpr (ST == ST_L2_KEEP) st_keep(p, v, pol);
    else st_stream(p, v);
}

__device__ __forceinline__ unsigned long long l2_evict_last_policy() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// Shared cost tile (uint16 costs, cost_stage): tile index e at slot
// e + 16 (e >> 8): the 16-B vector writes are conflict-free and so are the
// 2-B reads of every register pattern (PAT4's lane bit 4 lands 8 banks over).
template <int PAT>
__device__ __forceinline__ int cslot_base(int tid) {
    if (PAT == PAT8) return tid + 16 * (tid >> 8);
    if (PAT == PAT4) return (tid & 15) + 272 * (tid >> 4);
    return 16 * tid + 16 * (tid >> 4);  // PAT0: e = 16 tid + i
}
template <int PAT>
__host__ __device__ constexpr int cslot_step(int i) {
    return PAT == PAT8 ? 272 * i : (PAT == PAT4 ? 16 * i : i);
}
constexpr int kCostTileSlots = kTile + kTile / 16;

// One tile of a pass: load (or generate |+>), the round program SEQ with its
// phase / expectation, store.  `base`: the tile's physical base index.
// Shared by k_pass16 (one tile after another, streaming) and k_sweep (two
// sub-passes per L2-resident slab).
template <int MIX, int COST, int SEQ, int PH, int MA, int MB, int K, typename R, bool G, int LD, int ST>
__device__ __forceinline__ void pass_tile(const PassParams &P, long long base, C2<R> *tile, const C2<R> *tlo,
                                          const C2<R> *thi, long long thr8, long long thr4, double &eacc,
                                          unsigned long long pol, unsigned short *ctile = nullptr,
                                          long long thrc = 0) {
    using T = C2<R>;
    const int tid = threadIdx.x;
    // staged costs: the phase (PH 2) or expectation (PH 3) reads them after the first
    // transpose, whose barrier orders the cost tile's writes before its reads
    constexpr bool CST_OK = COST == FQ_COST_U16 && !G && (PH == 2 || PH == 3);
    const bool cst = CST_OK && ctile != nullptr;
    uint4 cv0 = make_uint4(0, 0, 0, 0), cv1 = cv0;
    constexpr bool HAS_B = MB != 2;
    constexpr int NR = seq_rounds(SEQ);
    constexpr int LAST = seq_pat(SEQ, NR - 1);
    constexpr int CB = COST == FQ_COST_F64 ? 8 : 2;
    const long long thrL = LAST == PAT8 ? thr8 : thr4;
    auto g4s = [&]() -> long long {
        if constexpr (G) return P.sdelta[(tid >> P.gshift) & P.gmask];
        else return 0;
    };
    auto g4c = [&]() -> long long {
        if constexpr (G) return P.cdelta[(tid >> P.gshift) & P.gmask];
        else return 0;
    };
            // per-tile base pointers; the registers' offsets are constant-bank byte offsets
            const char *ps8 = reinterpret_cast<const char *>(static_cast<T *>(P.psi) + base + thr8);
            const char *cs = static_cast<const char *>(P.costs) + base * CB;
            T v[kRegs];
            CostRaw<COST> raw[kRegs];  // cost entries of the phase round, loaded with the state
            if (P.init) {
    #pragma unroll
                for (int i = 0; i < kRegs; ++i) v[i] = Cx<R>::make((R)P.init_amp, (R)0);
            } else {
    #pragma unroll
                for (int i = 0; i < kRegs; ++i) v[i] = tile_load<LD>(reinterpret_cast<const T *>(ps8 + P.roff[PAT8][i]));
            }
            if constexpr (CST_OK) {
                if (cst) {  // tile indices 8 tid .. 8 tid + 7 and the same + 2048 (tile bit 11)
                    const uint4 *c0 = reinterpret_cast<const uint4 *>(cs + thrc * CB);
                    const uint4 *c1 = reinterpret_cast<const uint4 *>(cs + thrc * CB + P.c11);
                    cv0 = P.cost_l2 ? __ldcg(c0) : __ldcs(c0);
                    cv1 = P.cost_l2 ? __ldcg(c1) : __ldcs(c1);
                }
            }
            auto stage_costs = [&]() {  // before the first transpose (its barrier publishes them)
                if constexpr (CST_OK) {
                    if (cst) {
                        uint4 *ct = reinterpret_cast<uint4 *>(ctile);
                        ct[tid + 2 * (tid >> 5)] = cv0;
                        ct[tid + 256 + 2 * ((tid + 256) >> 5)] = cv1;
                    }
                }
            };
            auto read_costs = [&](auto pat) {  // cost entries of pattern PAT from the shared cost tile
                constexpr int PT = decltype(pat)::value;
                const unsigned short *c = ctile + cslot_base<PT>(tid);
    #pragma unroll
                for (int i = 0; i < kRegs; ++i) raw[i] = (CostRaw<COST>)c[cslot_step<PT>(i)];
            };
            // the expectation's costs (store pattern) are read inside the program's LAST
            // transpose: after it no barrier precedes the next tile's stage_costs
            auto exp_mid = [&]() {
                if constexpr (CST_OK) {
                    if (cst && (PH == 3 || P.expect)) read_costs(std::integral_constant<int, LAST>());
                }
            };
            if (PH == 1) {
                const char *c8 = cs + thr8 * CB;
    #pragma unroll
                for (int i = 0; i < kRegs; ++i) raw[i] = load_cost_at<COST>(c8 + P.coff[PAT8][i], P.cost_l2);
            }
            if (PH == 3 && !cst) {  // the program's last pass: its expectation costs, in the store pattern
                const char *cl = cs + thrL * CB + (LAST == PAT8 ? 0 : g4c());
    #pragma unroll
                for (int i = 0; i < kRegs; ++i) raw[i] = load_cost_at<COST>(cl + P.coff[LAST][i], P.cost_l2);
            }
            if (PH == 2 && !cst) {
                if (P.probe & 1) {
    #pragma unroll
                    for (int i = 0; i < kRegs; ++i) raw[i] = (CostRaw<COST>)((tid * 7 + i * 131) & 1023);
                } else {
                    const char *c4 = cs + thr4 * CB + g4c();
    #pragma unroll
                    for (int i = 0; i < kRegs; ++i) raw[i] = load_cost_at<COST>(c4 + P.coff[PAT4][i], P.cost_l2);
                }
            }
            auto phase_all = [&]() {
                // keep the table lookups behind the preceding butterflies: hoisted
                // early they would hold 64 registers of phase factors and spill
                asm volatile("" ::: "memory");
                if constexpr (CST_OK && PH == 2) {
                    if (cst) read_costs(std::integral_constant<int, PAT4>());
                }
                if (P.probe & 4) return;
                if (P.probe & 2) {
    #pragma unroll
                    for (int i = 0; i < kRegs; ++i) v[i] = cmul(v[i], phase16<COST, R>(P, (CostRaw<COST>)0, tlo, thi));
                    return;
                }
    #pragma unroll
                for (int i = 0; i < kRegs; ++i) v[i] = cmul(v[i], phase16<COST, R>(P, raw[i], tlo, thi));
            };
            // ---- round 0 (PAT8)
            if (PH == 1) phase_all();
            bfly16<MIX, MA, PAT8, R>(v, P.A, round_mask<K, SEQ>(P.maskA, 0));
            if constexpr (SEQ == SEQ_840) {
                if (HAS_B) bfly16<MIX, MB, PAT8, R>(v, P.B, round_mask<K, SEQ>(P.maskB, 0));
                stage_costs();
                transpose<PAT8, PAT0>(tile, v, tid);
                bfly16<MIX, MA, PAT0, R>(v, P.A, round_mask<K, SEQ>(P.maskA, 1));
                if (HAS_B) bfly16<MIX, MB, PAT0, R>(v, P.B, round_mask<K, SEQ>(P.maskB, 1));
                transpose<PAT0, PAT4>(tile, v, tid, exp_mid);
                bfly16<MIX, MA, PAT4, R>(v, P.A, round_mask<K, SEQ>(P.maskA, 2));
                if (HAS_B) bfly16<MIX, MB, PAT4, R>(v, P.B, round_mask<K, SEQ>(P.maskB, 2));
            } else if constexpr (SEQ == SEQ_84) {
                if (HAS_B) bfly16<MIX, MB, PAT8, R>(v, P.B, round_mask<K, SEQ>(P.maskB, 0));
                stage_costs();
                transpose<PAT8, PAT4>(tile, v, tid, exp_mid);
                bfly16<MIX, MA, PAT4, R>(v, P.A, round_mask<K, SEQ>(P.maskA, 1));
                if constexpr (K == K_LANE3) lane_bfly16<MA, 8, R>(v, P.A);
                if (HAS_B) bfly16<MIX, MB, PAT4, R>(v, P.B, round_mask<K, SEQ>(P.maskB, 1));
                if constexpr (K == K_LANE3 && HAS_B) lane_bfly16<MB, 8, R>(v, P.B);
            } else if constexpr (SEQ == SEQ_84048) {
                stage_costs();
                transpose<PAT8, PAT0>(tile, v, tid);
                bfly16<MIX, MA, PAT0, R>(v, P.A, round_mask<K, SEQ>(P.maskA, 1));
                transpose<PAT0, PAT4>(tile, v, tid);
                bfly16<MIX, MA, PAT4, R>(v, P.A, round_mask<K, SEQ>(P.maskA, 2));
                phase_all();
                bfly16<MIX, MB, PAT4, R>(v, P.B, round_mask<K, SEQ>(P.maskB, 2));
                transpose<PAT4, PAT0>(tile, v, tid);
                bfly16<MIX, MB, PAT0, R>(v, P.B, round_mask<K, SEQ>(P.maskB, 3));
                transpose<PAT0, PAT8>(tile, v, tid, exp_mid);
                bfly16<MIX, MB, PAT8, R>(v, P.B, round_mask<K, SEQ>(P.maskB, 4));
            } else {  // SEQ_848
                stage_costs();
                transpose<PAT8, PAT4>(tile, v, tid);
                bfly16<MIX, MA, PAT4, R>(v, P.A, round_mask<K, SEQ>(P.maskA, 1));
                if constexpr (K == K_LANE3) lane_bfly16<MA, 8, R>(v, P.A);
                phase_all();
                if constexpr (K == K_LANE3) lane_bfly16<MB, 8, R>(v, P.B);
                bfly16<MIX, MB, PAT4, R>(v, P.B, round_mask<K, SEQ>(P.maskB, 1));
                transpose<PAT4, PAT8>(tile, v, tid, exp_mid);
                bfly16<MIX, MB, PAT8, R>(v, P.B, round_mask<K, SEQ>(P.maskB, 2));
            }
            // ---- store (+ expectation) in the last round's pattern
            const R fs = (R)P.final_scale;
            if (PH != 3 && P.expect && !cst) {  // cost entries of the last pattern (final pass with a phase)
                const char *cl = cs + thrL * CB + (LAST == PAT8 ? 0 : g4c());
    #pragma unroll
                for (int i = 0; i < kRegs; ++i) raw[i] = load_cost_at<COST>(cl + P.coff[LAST][i], P.cost_l2);
            }
            char *psl = reinterpret_cast<char *>(static_cast<T *>(P.psi) + base + thrL) + (LAST == PAT8 ? 0 : g4s());
    #pragma unroll
            for (int i = 0; i < kRegs; ++i) {
                T x = v[i];
                if (MIX == MIX_RX) x = Cx<R>::make(x.x * fs, x.y * fs);
                if (P.expect) eacc += decode_cost<COST>(P, raw[i]) * ((double)x.x * x.x + (double)x.y * x.y);
                tile_store<ST>(reinterpret_cast<T *>(psl + P.roff[LAST][i]), x, pol);
            }
}

// ---------------------------------------------------------------- the pass kernel
// Register-load pass, 256 threads x 16 amplitudes per 2^12 tile, 2 CTAs/SM
// (grid-stride over tiles).  Everything that varies between passes of one
// program is a template parameter, so the tile loop has no runtime branches
// on it:
//   SEQ: round program (see SEQ_*);
//   PH: 0 no phase, 1 phase before set A in round 0, 2 phase between set A and
//       set B in the middle (PAT4) round of a heavy SEQ, 3 no phase and the
//       expectation's costs loaded with the state (the program's last pass);
//   MA, MB: RX form of sets A/B (0: (1, tan b), 1: (cot b, 1), 3: chosen at run
//       time); MB = 2: no set B;
//   K: target-mask class of the rounds (see round_mask): compile-time masks keep
//       the butterfly code branch-free (run-time masks force register moves at
//       every merge point).
template <int MIX, int COST, int SEQ, int PH, int MA, int MB, int K, typename R = double, bool G = false>
__global__ void __launch_bounds__(kThreads, 2) k_pass16(const __grid_constant__ PassParams P,
                                                        const __grid_constant__ CUtensorMap tm_state,
                                                        const __grid_constant__ CUtensorMap tm_cost) {
    using T = C2<R>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *tile = reinterpret_cast<T *>(smem_raw);
    T *tlo = tile + kTilePadded;
    T *thi = tlo + kTableLo * table_copies<R>();
    __shared__ double red[kThreads / 32];
    const int tid = threadIdx.x;
    constexpr bool HAS_B = MB != 2;
    constexpr bool HEAVY = seq_heavy(SEQ);
    static_assert(!HEAVY || (PH == 2 && HAS_B), "heavy round programs carry the mid-layer phase");
    static_assert(HEAVY || PH != 2, "the mid-layer phase needs a heavy round program");
    static_assert(!HEAVY || PH != 3, "PH = 3 (expectation preload) is a light-pass mode");

    if (COST == FQ_COST_U16 && (PH == 1 || PH == 2)) {
        if (P.table_hi > 0) build_phase_tables<R>(tlo, thi, P.table_hi, P.gamma, P.cost_scale, P.cost_offset);
        __syncthreads();
    }
    // G: PAT4's thread bits include the shard index (PAT8's never do); the
    // shard byte offsets are re-read from the parameter bank at each use
    const long long thr8 = thread_offset<PAT8, G>(P, tid);
    const long long thr4 = thread_offset<PAT4, G>(P, tid);
    double eacc = 0.0;
    // staged costs: thread tid loads tile indices 8 tid .. 8 tid + 7 (tile bits 3..10 = tid bits)
    unsigned short *ctile = nullptr;
    long long thrc = 0;
    if (!G && COST == FQ_COST_U16 && P.cost_stage) {
        ctile = reinterpret_cast<unsigned short *>(thi + P.table_hi * table_copies<R>());
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if ((tid >> j) & 1) thrc += 1LL << P.tile_pos[3 + j];
    }

    const bool pf = P.pf_dist > 0 && tid == 0;
    if (pf) {  // prologue: tiles 1 .. pf_dist-1 of this CTA
        for (int d = 1; d < P.pf_dist; ++d) {
            const long long tp = blockIdx.x + (long long)d * gridDim.x;
            if (tp < P.n_tiles) prefetch_tile(P, &tm_state, &tm_cost, P.reverse ? P.n_tiles - 1 - tp : tp, !P.init);
        }
    }
    // reverse passes walk the tiles from the top: the previous pass ended there,
    // so the first tiles read are still in L2 (written moments ago)
    long long base = tile_base(P, P.tile0 + (P.reverse ? P.n_tiles - 1 - blockIdx.x : blockIdx.x));
    for (long long t = blockIdx.x; t < P.n_tiles; t += gridDim.x,
                   base = P.reverse ? prev_base(base, P.tile_mask, P.step_dep) : next_base(base, P.tile_mask, P.step_dep)) {
        if (pf) {
            const long long tp = t + (long long)P.pf_dist * gridDim.x;
            if (tp < P.n_tiles) prefetch_tile(P, &tm_state, &tm_cost, P.reverse ? P.n_tiles - 1 - tp : tp, !P.init);
        }
        pass_tile<MIX, COST, SEQ, PH, MA, MB, K, R, G, LD_STREAM, ST_STREAM>(P, base, tile, tlo, thi, thr8, thr4, eacc, 0ull,
                                                                             ctile, thrc);
    }
    if (P.expect) {
        const double s = block_sum<kThreads>(eacc, red);
        if (tid == 0) P.partials[blockIdx.x] = s;
    }
}

// Sharded execution context (fq_qaoa_evolve_sharded); null for one state.
struct ShardCtx {
    int k = 0, K = 1;
    int rank = 0;                          // -1: every shard belongs to this process (one stream)
    void *const *shards = nullptr;         // [K] state shards as mapped in this process
    const void *const *costs = nullptr;    // [K] cost shards
    void *const *flags = nullptr;          // [K] peer barrier flag arrays (rank >= 0)
    unsigned *epoch = nullptr;
    int *err = nullptr;
};

// ---------------------------------------------------------------- launch
struct PassMaps {
    alignas(64) CUtensorMap state;
    alignas(64) CUtensorMap cost;
};

template <int MIX, int COST, int SEQ, int PH, int MA, int MB, int K, typename R = double, bool G = false>
static int launch_pass16(const PassParams &P, const PassMaps &M, int grid, cudaStream_t st) {
    static bool configured = false;
    constexpr int CP = table_copies<R>();
    const size_t smem = (size_t)(kTilePadded + (kTableLo + kMaxTableHi) * CP) * sizeof(C2<R>) +
                        kCostTileSlots * sizeof(unsigned short);
    if (!configured) {
        cudaFuncSetAttribute(k_pass16<MIX, COST, SEQ, PH, MA, MB, K, R, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        configured = true;
    }
    const size_t need = (size_t)(kTilePadded + (kTableLo + P.table_hi) * CP) * sizeof(C2<R>) +
                        (P.cost_stage ? kCostTileSlots * sizeof(unsigned short) : 0);
    k_pass16<MIX, COST, SEQ, PH, MA, MB, K, R, G><<<grid, kThreads, need, st>>>(P, M.state, M.cost);
    FQ_LAUNCHED("k_pass16");
    return FQ_OK;
}

// Template dispatch for one round program SEQ of one (mixer, cost) pair.
// ph/ma/mb/k as the k_pass16 parameters (ma/mb already normalised by the
// caller); a mask class k without an instantiation runs with the run-time
// masks (K_RUNTIME), which PassParams always carries.
template <int MIX, int COST, int SEQ, typename R = double, bool G = false>
static int select_seq(const PassParams &P, const PassMaps &M, int ph, int ma, int mb, int k, int grid, cudaStream_t st) {
    constexpr bool kHigh = SEQ == SEQ_84 || SEQ == SEQ_848;
#define FQ_K(PHV, MAV, MBV)                                                                                  \
    if (ph == PHV && ma == MAV && mb == MBV) {                                                               \
        if (k == K_FULL) return launch_pass16<MIX, COST, SEQ, PHV, MAV, MBV, K_FULL, R, G>(P, M, grid, st);   \
        if constexpr (kHigh && MIX == MIX_RX && !G) {                                                        \
            if (k == K_LANE3) return launch_pass16<MIX, COST, SEQ, PHV, MAV, MBV, K_LANE3, R, G>(P, M, grid, st); \
        }                                                                                                    \
        if constexpr (kHigh && MIX == MIX_RX) {                                                              \
            if (k == 1) return launch_pass16<MIX, COST, SEQ, PHV, MAV, MBV, 1, R, G>(P, M, grid, st);         \
            if (k == 2) return launch_pass16<MIX, COST, SEQ, PHV, MAV, MBV, 2, R, G>(P, M, grid, st);         \
            if (k == 3) return launch_pass16<MIX, COST, SEQ, PHV, MAV, MBV, 3, R, G>(P, M, grid, st);         \
        }                                                                                                    \
        if (k == K_LANE3) break; /* lane butterflies have no run-time-mask form */                            \
        return launch_pass16<MIX, COST, SEQ, PHV, MAV, MBV, K_RUNTIME, R, G>(P, M, grid, st);                 \
    }
    do {
        if constexpr (seq_heavy(SEQ)) {
            if constexpr (MIX == MIX_RX) {
                FQ_K(2, 0, 0) FQ_K(2, 0, 1) FQ_K(2, 1, 0) FQ_K(2, 1, 1)
            } else {
                FQ_K(2, 0, 3)
            }
        } else {
            FQ_K(0, 0, 2) FQ_K(0, 0, 3) FQ_K(1, 0, 2) FQ_K(1, 0, 3) FQ_K(3, 0, 2)
            if constexpr (MIX == MIX_RX) { FQ_K(0, 1, 2) FQ_K(0, 1, 3) FQ_K(1, 1, 2) FQ_K(1, 1, 3) FQ_K(3, 1, 2) }
        }
    } while (0);
#undef FQ_K
    set_error("k_pass16: no instantiation for seq=%d ph=%d ma=%d mb=%d k=%d", SEQ, ph, ma, mb, k);
    return FQ_ERR_UNSUPPORTED;
}

// Instantiation units (pass_*.cu), compiled in parallel.
int launch_pass_rx_u16_light(const PassParams &P, const PassMaps &M, int seq, int ph, int ma, int mb, int k, int grid, cudaStream_t st);
int launch_pass_rx_u16_heavy(const PassParams &P, const PassMaps &M, int seq, int ph, int ma, int mb, int k, int grid, cudaStream_t st);
int launch_pass_rx_f64_light(const PassParams &P, const PassMaps &M, int seq, int ph, int ma, int mb, int k, int grid, cudaStream_t st);
int launch_pass_rx_f64_heavy(const PassParams &P, const PassMaps &M, int seq, int ph, int ma, int mb, int k, int grid, cudaStream_t st);
int launch_pass_su2(const PassParams &P, const PassMaps &M, int cost, int seq, int ph, int mb, int k, int grid, cudaStream_t st);
int launch_pass_su2_c64(const PassParams &P, const PassMaps &M, int cost, int seq, int ph, int mb, int k, int grid,
                        cudaStream_t st);
// sharded states (G = true, complex128): passes whose tile spans the global
// qubits; every mixer and round program, one unit per cost encoding (pass_global_*.cu)
int launch_pass_global_u16(int mix, const PassParams &P, const PassMaps &M, int seq, int ph, int ma, int mb, int k,
                           int grid, cudaStream_t st);
int launch_pass_global_f64(int mix, const PassParams &P, const PassMaps &M, int seq, int ph, int ma, int mb, int k,
                           int grid, cudaStream_t st);
// sharded complex64 states (G = true, R = float): X mixer (pass_global_c64.cu)
int launch_pass_global_c64(int cost, const PassParams &P, const PassMaps &M, int seq, int ph, int ma, int mb, int k,
                           int grid, cudaStream_t st);
// complex64 states (R = float): X mixer, all round programs, one unit per cost encoding
int launch_pass_c64_u16(const PassParams &P, const PassMaps &M, int seq, int ph, int ma, int mb, int k, int grid, cudaStream_t st);
int launch_pass_c64_f64(const PassParams &P, const PassMaps &M, int seq, int ph, int ma, int mb, int k, int grid, cudaStream_t st);

}  // namespace fq
