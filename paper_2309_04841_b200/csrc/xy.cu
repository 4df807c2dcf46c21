// Tiled XY mixers (reference mixers.py:94-137, _kernels.py:30-48): the
// documented gate sequence of a layer (ring: even pairs, odd pairs, wrap;
// complete: lexicographic, mixers.py:5-15) is cut into HBM passes.  A pass
// owns a set of <= 12 tile bits (the gates' qubits plus low spectator bits
// for coalescing) and applies, tile by tile, every gate of a dependency-closed
// subsequence whose qubits are tile bits — order preserved wherever two
// gates share a qubit (gates on disjoint pairs commute).  Inside a pass the
// gates run in register "rounds": 16 amplitudes per thread = 4 tile bits in
// registers, each gate's two bits in the same round, XOR-swizzled
// shared-memory transposes between rounds.  The layer's phase rides in the
// first pass, the expectation in the program's last pass.
//
// Reference cost: one full state sweep per gate (26 per ring layer, 325 per
// complete layer at n = 26); here a handful of passes per layer.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tmap.cuh"

namespace fq {

constexpr int kXyMaxRounds = 24;
int g_xy_prefetch = 1;  // option xy_prefetch: L2 tensor prefetch of XY tiles (-1: runs >= 256 B only; measured: always on is best)
int g_xy_pad = 1;      // option xy_pad: gate-free first / last rounds keep loads and stores on tile bits 0..4
int g_xy_min_run = 0;  // minimum contiguous run (log2 amplitudes) of an XY pass tile; 0 = chosen by the cost model
constexpr int kXyMaxGates = 6;  // C(4, 2): distinct pairs of one 4-bit register set

struct XyRound {
    unsigned char reg[4];         // tile bits held in registers (register index bit j <- tile bit reg[j])
    unsigned char tb[8];          // thread bit k <- tile bit tb[k]
    unsigned char ngates;
    unsigned char gate[kXyMaxGates];  // code = 4 * a + b: lo qubit at register bit a, hi qubit at b
    unsigned short sreg[kRegs];   // swizzled smem BYTE offset of register i's tile-index part
    unsigned short tnib[32];      // swizzled smem byte offset of the thread part: [tid & 15] ^ [16 + (tid >> 4)]
};

struct XyParams {
    void *psi;                // C2<R>[2^n] (complex128 or complex64)
    const void *costs;
    double cost_scale, cost_offset;
    double *partials;
    double init_amp;
    double gamma;
    double c, s;  // cos(beta), sin(beta)
    long long n_tiles;
    int tile_pos[kTileBits];
    long long roff_first[kRegs], roff_last[kRegs];  // physical offsets of the registers, first / last round
    int init, expect, table_hi;
    int pf;                                   // L2 tile prefetch (one tensor-map instruction per tile)
    int sm_rank, sm_shift[5], sm_bits[5];     // state map
    int cm_rank, cm_shift[5], cm_bits[5];     // cost map (cm_rank = 0: not needed)
    int nrounds;
    XyRound rounds[kXyMaxRounds];
    // sharded state (G = true): amplitude indices are global; index k lives in
    // shard k >> nl at local offset k & (2^nl - 1) (peer-mapped shard pointers)
    long long tile0;  // first tile of this launch
    int nl;
    void *shard[8];
    const void *cshard[8];
};

template <bool G, typename T>
__device__ __forceinline__ T *xy_amp(const XyParams &P, long long k) {
    if constexpr (G) return static_cast<T *>(P.shard[k >> P.nl]) + (k & ((1LL << P.nl) - 1));
    else return static_cast<T *>(P.psi) + k;
}

template <bool G, typename C>
__device__ __forceinline__ const C *xy_cost(const XyParams &P, long long k) {
    if constexpr (G) return static_cast<const C *>(P.cshard[k >> P.nl]) + (k & ((1LL << P.nl) - 1));
    else return static_cast<const C *>(P.costs) + k;
}

// XOR swizzle of a 12-bit tile index (bijective; GF(2)-linear, so the slot of
// thread part | register part is the XOR of the parts' slots).  16-B elements
// (complex128): the bank group of slot e is fold3(e), and a quarter-warp whose
// three lane bits sit on tile bits of distinct residues mod 3 is conflict-free.
// 8-B elements (complex64): a half-warp is one 128-B wavefront, the bank pair
// is fold4(e), and the four lane bits need distinct residues mod 4.
__host__ __device__ __forceinline__ int xy_slot(int e) { return e ^ (((e >> 3) ^ (e >> 6) ^ (e >> 9)) & 7); }
__host__ __device__ __forceinline__ int xy_slot8(int e) { return e ^ (((e >> 4) ^ (e >> 8)) & 15); }
__host__ __device__ __forceinline__ int xy_slot_of(int e, int elem) { return elem == 8 ? xy_slot8(e) : xy_slot(e); }

// x_lo' = c x_lo - i s x_hi ; x_hi' = -i s x_lo + c x_hi   (reference _kernels.py:44-47)
template <int A, int B, typename T, typename R>
__device__ __forceinline__ void xy_gate(T (&v)[kRegs], R c, R s) {
#pragma unroll
    for (int i = 0; i < kRegs; ++i) {
        if (((i >> A) & 1) && !((i >> B) & 1)) {
            const int j = i ^ (1 << A) ^ (1 << B);
            const T xl = v[i], xh = v[j];
            v[i] = Cx<R>::make(fma(c, xl.x, s * xh.y), fma(c, xl.y, -s * xh.x));
            v[j] = Cx<R>::make(fma(s, xl.y, c * xh.x), fma(c, xh.y, -s * xl.x));
        }
    }
}

template <typename T, typename R>
__device__ __forceinline__ void xy_apply(T (&v)[kRegs], int code, R c, R s) {
    switch (code) {
        case 1: xy_gate<0, 1>(v, c, s); break;
        case 2: xy_gate<0, 2>(v, c, s); break;
        case 3: xy_gate<0, 3>(v, c, s); break;
        case 4: xy_gate<1, 0>(v, c, s); break;
        case 6: xy_gate<1, 2>(v, c, s); break;
        case 7: xy_gate<1, 3>(v, c, s); break;
        case 8: xy_gate<2, 0>(v, c, s); break;
        case 9: xy_gate<2, 1>(v, c, s); break;
        case 11: xy_gate<2, 3>(v, c, s); break;
        case 12: xy_gate<3, 0>(v, c, s); break;
        case 13: xy_gate<3, 1>(v, c, s); break;
        case 14: xy_gate<3, 2>(v, c, s); break;
        default: break;
    }
}

__device__ __forceinline__ long long xy_tphys(const XyParams &P, const XyRound &R, int tid) {
    long long o = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if ((tid >> k) & 1) o += 1LL << P.tile_pos[R.tb[k]];
    return o;
}

__device__ __forceinline__ long long xy_tile_base(const int *tile_pos, long long t) {
    long long base = t;
#pragma unroll
    for (int j = 0; j < kTileBits; ++j) {
        const int p = tile_pos[j];
        base = ((base >> p) << (p + 1)) | (base & ((1LL << p) - 1));
    }
    return base;
}

template <int COST, typename R>
__device__ __forceinline__ C2<R> xy_phase(const XyParams &P, CostRaw<COST> raw, const C2<R> *tlo,
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

template <int COST, int PH, bool G = false, typename RT = double>
__global__ void __launch_bounds__(kThreads, 2) k_xy_pass(const __grid_constant__ XyParams P,
                                                         const __grid_constant__ CUtensorMap tm_state,
                                                         const __grid_constant__ CUtensorMap tm_cost) {
    using T = C2<RT>;
    extern __shared__ __align__(16) unsigned char xy_smem_raw[];
    T *tile = reinterpret_cast<T *>(xy_smem_raw);
    T *tlo = tile + kTile;
    T *thi = tlo + kTableLo * table_copies<RT>();
    __shared__ double red[kThreads / 32];
    // per round, the thread part of the swizzled slot (byte offsets) by tid nibble:
    // two shared loads per transpose instead of rebuilding it from the round's bit map
    // and the register parts (same for every thread: broadcast reads)
    __shared__ int tnib[kXyMaxRounds][32];
    __shared__ __align__(16) int sreg[kXyMaxRounds][kRegs];
    const int tid = threadIdx.x;
    for (int i = tid; i < P.nrounds * 32; i += kThreads) tnib[i >> 5][i & 31] = P.rounds[i >> 5].tnib[i & 31];
    for (int i = tid; i < P.nrounds * kRegs; i += kThreads) sreg[i / kRegs][i % kRegs] = P.rounds[i / kRegs].sreg[i % kRegs];
    if (COST == FQ_COST_U16 && PH) {
        if (P.table_hi > 0) build_phase_tables<RT>(tlo, thi, P.table_hi, P.gamma, P.cost_scale, P.cost_offset);
    }
    __syncthreads();
    char *const tb = reinterpret_cast<char *>(tile);
    const int lo_n = tid & 15, hi_n = 16 + (tid >> 4);
    const long long thr_first = xy_tphys(P, P.rounds[0], tid);
    const long long thr_last = xy_tphys(P, P.rounds[P.nrounds - 1], tid);
    double eacc = 0.0;
    for (long long t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
        const long long base = xy_tile_base(P.tile_pos, P.tile0 + t);
        if (!G && P.pf && tid == 0 && t + gridDim.x < P.n_tiles) {  // next tile of this CTA into L2
            int c[5];
            if (!P.init && P.sm_rank) {
                tile_coords(t + gridDim.x, P.sm_rank, P.sm_shift, P.sm_bits, c);
                tensor_prefetch_l2(&tm_state, P.sm_rank, c);
            }
            if (P.cm_rank) {
                tile_coords(t + gridDim.x, P.cm_rank, P.cm_shift, P.cm_bits, c);
                tensor_prefetch_l2(&tm_cost, P.cm_rank, c);
            }
        }
        T v[kRegs];
        if (P.init) {
#pragma unroll
            for (int i = 0; i < kRegs; ++i) v[i] = Cx<RT>::make((RT)P.init_amp, (RT)0);
        } else {
#pragma unroll
            for (int i = 0; i < kRegs; ++i) v[i] = ld_stream(xy_amp<G, T>(P, base + thr_first + P.roff_first[i]));
        }
        if (PH) {
            CostRaw<COST> raw[kRegs];
#pragma unroll
            for (int i = 0; i < kRegs; ++i) {
                const long long k = base + thr_first + P.roff_first[i];
                if constexpr (COST == FQ_COST_F64) raw[i] = *xy_cost<G, double>(P, k);
                else raw[i] = *xy_cost<G, unsigned short>(P, k);
            }
#pragma unroll
            for (int i = 0; i < kRegs; ++i)
                v[i] = cmul(v[i], xy_phase<COST, RT>(P, raw[i], tlo, thi));
        }
        int sq = tnib[0][lo_n] ^ tnib[0][hi_n];
        for (int r = 0; r < P.nrounds; ++r) {
            const XyRound &R = P.rounds[r];
            if (r > 0) {  // transpose from round r-1's pattern to round r's
                const int sr = tnib[r][lo_n] ^ tnib[r][hi_n];
                int so[kRegs];
#pragma unroll
                for (int i = 0; i < kRegs; i += 4) {
                    const int4 q = *reinterpret_cast<const int4 *>(&sreg[r - 1][i]);
                    so[i] = q.x; so[i + 1] = q.y; so[i + 2] = q.z; so[i + 3] = q.w;
                }
                __syncthreads();
#pragma unroll
                for (int i = 0; i < kRegs; ++i) *reinterpret_cast<T *>(tb + (sq ^ so[i])) = v[i];
#pragma unroll
                for (int i = 0; i < kRegs; i += 4) {
                    const int4 q = *reinterpret_cast<const int4 *>(&sreg[r][i]);
                    so[i] = q.x; so[i + 1] = q.y; so[i + 2] = q.z; so[i + 3] = q.w;
                }
                __syncthreads();
#pragma unroll
                for (int i = 0; i < kRegs; ++i) v[i] = *reinterpret_cast<const T *>(tb + (sr ^ so[i]));
                sq = sr;
            }
            for (int g = 0; g < R.ngates; ++g) xy_apply(v, R.gate[g], (decltype(v[0].x))P.c, (decltype(v[0].x))P.s);
        }
#pragma unroll
        for (int i = 0; i < kRegs; ++i) {
            const long long k = base + thr_last + P.roff_last[i];
            if (P.expect) {
                double cv;
                if constexpr (COST == FQ_COST_F64) cv = *xy_cost<G, double>(P, k);
                else cv = decode_u16(*xy_cost<G, unsigned short>(P, k), P.cost_scale, P.cost_offset);
                eacc += cv * ((double)v[i].x * v[i].x + (double)v[i].y * v[i].y);
            }
            st_stream(xy_amp<G, T>(P, k), v[i]);
        }
    }
    if (P.expect) {
        const double sum = block_sum<kThreads>(eacc, red);
        if (tid == 0) P.partials[blockIdx.x] = sum;
    }
}

// ---------------------------------------------------------------- host scheduler
struct XyPassPlan {
    std::vector<int> tile;                          // 12 physical bits, ascending
    std::vector<std::vector<int>> round_bits;       // tile-bit indices in registers, per round
    std::vector<std::vector<std::pair<int, int>>> round_gates;  // (lo qubit, hi qubit), per round
};

static int run_bits_of(const std::vector<int> &tile) {
    int r = 0;
    while (r < (int)tile.size() && tile[r] == r) ++r;
    return r;
}

static std::vector<int> tile_for(int n, const std::vector<int> &targets) {
    std::vector<int> bits = targets;
    for (int q = 0; q < n && (int)bits.size() < kTileBits; ++q)
        if (std::find(targets.begin(), targets.end(), q) == targets.end()) bits.push_back(q);
    std::sort(bits.begin(), bits.end());
    return bits;
}

// Greedy dependency-respecting cut of an ordered gate list: scan the remaining
// gates in order; a gate joins the current group if none of its qubits was
// touched by a gate left behind (it would have to wait for it) and its qubits
// fit the capacity test; a gate left behind blocks its qubits.
// row_cap: a gate's leading (first) qubit may bring at most row_cap new other
// qubits into a group — so a pass over the complete graph's lexicographic
// order takes a block of rows x columns instead of one long row.
template <typename Fits>
static std::vector<std::vector<int>> cut_groups(const std::vector<std::pair<int, int>> &gates, std::vector<int> idx,
                                                Fits fits, int row_cap = 64) {
    std::vector<std::vector<int>> groups;
    while (!idx.empty()) {
        std::vector<int> taken, rest, qubits;
        std::vector<char> blocked(64, 0);
        std::vector<int> row_new(64, 0);
        for (int gi : idx) {
            const int a = gates[gi].first, b = gates[gi].second;
            bool ok = !blocked[a] && !blocked[b];
            if (ok) {
                std::vector<int> q2 = qubits;
                const bool new_b = std::find(q2.begin(), q2.end(), b) == q2.end();
                if (std::find(q2.begin(), q2.end(), a) == q2.end()) q2.push_back(a);
                if (new_b) q2.push_back(b);
                ok = fits(q2) && (!new_b || row_new[a] < row_cap);
                if (ok) {
                    qubits = q2;
                    row_new[a] += new_b ? 1 : 0;
                }
            }
            if (ok) {
                taken.push_back(gi);
            } else {
                rest.push_back(gi);
                blocked[a] = blocked[b] = 1;
            }
        }
        groups.push_back(taken);
        idx = rest;
    }
    return groups;
}

// One dependency-respecting scan with a fixed register set R: takes every
// remaining gate inside R whose qubits no skipped gate has touched.
static void scan_round(const std::vector<std::pair<int, int>> &gates, const std::vector<int> &idx, const int *R,
                       std::vector<int> &taken, std::vector<int> &rest) {
    taken.clear();
    rest.clear();
    std::vector<char> blocked(64, 0);
    auto in_r = [&](int q) { return q == R[0] || q == R[1] || q == R[2] || q == R[3]; };
    for (int gi : idx) {
        const int a = gates[gi].first, b = gates[gi].second;
        if (!blocked[a] && !blocked[b] && in_r(a) && in_r(b)) {
            taken.push_back(gi);
        } else {
            rest.push_back(gi);
            blocked[a] = blocked[b] = 1;
        }
    }
}

// Register rounds of one pass: each round holds 4 qubits; the first remaining
// gate's two qubits are always in it and the other two are chosen (exhaustively
// over the pass's qubits) to maximise the gates the round can take — e.g. a
// 2 x 2 block (r1, r2) x (c1, c2) of the complete graph's lexicographic order
// (4 gates) where a plain in-order cut takes 3.
static std::vector<std::vector<int>> round_cut(const std::vector<std::pair<int, int>> &gates, std::vector<int> idx) {
    std::vector<std::vector<int>> rounds;
    std::vector<int> qs;
    for (int gi : idx)
        for (int x : {gates[gi].first, gates[gi].second})
            if (std::find(qs.begin(), qs.end(), x) == qs.end()) qs.push_back(x);
    std::vector<int> taken, rest, best_taken, best_rest;
    while (!idx.empty()) {
        const int a = gates[idx[0]].first, b = gates[idx[0]].second;
        std::vector<int> others;
        for (int q : qs)
            if (q != a && q != b) others.push_back(q);
        best_taken.clear();
        if (others.size() < 2) {
            int R[4] = {a, b, others.empty() ? a : others[0], a};
            scan_round(gates, idx, R, best_taken, best_rest);
        } else {
            for (size_t i = 0; i < others.size(); ++i)
                for (size_t j = i + 1; j < others.size(); ++j) {
                    int R[4] = {a, b, others[i], others[j]};
                    scan_round(gates, idx, R, taken, rest);
                    if (taken.size() > best_taken.size()) {
                        best_taken = taken;
                        best_rest = rest;
                    }
                }
        }
        rounds.push_back(best_taken);
        idx = best_rest;
    }
    return rounds;
}

static std::vector<XyPassPlan> plan_xy_with(int n, const std::vector<std::pair<int, int>> &gates, int min_run,
                                            int row_cap) {
    std::vector<int> all(gates.size());
    for (size_t i = 0; i < gates.size(); ++i) all[i] = (int)i;
    // passes: the tile (targets + spectators) must keep runs of >= 16 amplitudes
    auto pass_fits = [&](const std::vector<int> &q) {
        return (int)q.size() <= kTileBits && run_bits_of(tile_for(n, q)) >= min_run;
    };
    std::vector<XyPassPlan> plans;
    // consecutive groups over the same tile become one pass (the row cap can
    // end a group early while the next one still fits the same 12 bits)
    auto qubits_of = [&](const std::vector<int> &g) {
        std::vector<int> q;
        for (int gi : g)
            for (int x : {gates[gi].first, gates[gi].second})
                if (std::find(q.begin(), q.end(), x) == q.end()) q.push_back(x);
        return q;
    };
    std::vector<std::vector<int>> groups;
    for (auto &pg : cut_groups(gates, all, pass_fits, row_cap)) {
        if (!groups.empty()) {
            std::vector<int> q = qubits_of(groups.back()), q2 = qubits_of(pg);
            std::vector<int> u = q;
            for (int x : q2)
                if (std::find(u.begin(), u.end(), x) == u.end()) u.push_back(x);
            if (pass_fits(u) && tile_for(n, u) == tile_for(n, q)) {
                groups.back().insert(groups.back().end(), pg.begin(), pg.end());
                continue;
            }
        }
        groups.push_back(pg);
    }
    for (auto &pg : groups) {
        XyPassPlan pl;
        std::vector<int> q;
        for (int gi : pg) {
            for (int x : {gates[gi].first, gates[gi].second})
                if (std::find(q.begin(), q.end(), x) == q.end()) q.push_back(x);
        }
        pl.tile = tile_for(n, q);
        auto tbit = [&](int qubit) { return (int)(std::find(pl.tile.begin(), pl.tile.end(), qubit) - pl.tile.begin()); };
        // rounds: 4 register bits
        for (auto &rg : round_cut(gates, pg)) {
            std::vector<int> bits;
            std::vector<std::pair<int, int>> gl;
            for (int gi : rg) {
                for (int x : {gates[gi].first, gates[gi].second})
                    if (std::find(bits.begin(), bits.end(), tbit(x)) == bits.end()) bits.push_back(tbit(x));
                gl.push_back(gates[gi]);
            }
            // pad with spectator-most (highest unused) tile bits so loads/stores keep lanes on the low bits
            for (int b = kTileBits - 1; (int)bits.size() < 4 && b >= 0; --b)
                if (std::find(bits.begin(), bits.end(), b) == bits.end()) bits.push_back(b);
            pl.round_bits.push_back(bits);
            pl.round_gates.push_back(gl);
        }
        // load / store rounds keep the warp's lanes on tile bits 0..4 (coalesced): if the
        // first (last) round holds one of them in registers, add a gate-free round before (after)
        auto low_ok = [](const std::vector<int> &bits) {
            for (int b : bits)
                if (b < 5) return false;
            return true;
        };
        const std::vector<int> top = {8, 9, 10, 11};
        if (g_xy_pad && !low_ok(pl.round_bits.front())) {
            pl.round_bits.insert(pl.round_bits.begin(), top);
            pl.round_gates.insert(pl.round_gates.begin(), std::vector<std::pair<int, int>>());
        }
        if (g_xy_pad && !low_ok(pl.round_bits.back())) {
            pl.round_bits.push_back(top);
            pl.round_gates.push_back({});
        }
        // more rounds than one launch carries: consecutive chunks over the same tile
        constexpr int kChunk = kXyMaxRounds - 2;
        if ((int)pl.round_bits.size() <= kXyMaxRounds) {
            plans.push_back(pl);
            continue;
        }
        for (size_t r0 = 0; r0 < pl.round_bits.size(); r0 += kChunk) {
            XyPassPlan part;
            part.tile = pl.tile;
            const size_t r1 = std::min(pl.round_bits.size(), r0 + kChunk);
            part.round_bits.assign(pl.round_bits.begin() + r0, pl.round_bits.begin() + r1);
            part.round_gates.assign(pl.round_gates.begin() + r0, pl.round_gates.begin() + r1);
            if (g_xy_pad && !low_ok(part.round_bits.front())) {
                part.round_bits.insert(part.round_bits.begin(), top);
                part.round_gates.insert(part.round_gates.begin(), std::vector<std::pair<int, int>>());
            }
            if (g_xy_pad && !low_ok(part.round_bits.back())) {
                part.round_bits.push_back(top);
                part.round_gates.push_back({});
            }
            plans.push_back(part);
        }
    }
    return plans;
}

int g_xy_row_cap = 0;  // option xy_row_cap: 0 = chosen by the cost model

// Relative cost of one register round (a shared-memory transpose of the whole
// state plus its gates) against one HBM pass of the tile kernel (B200).
// Fitted on B200 (portfolio n = 26, XY complete, 7 plans): 0.30 ms per pass,
// 0.056 ms per round.
constexpr double kXyRoundCost = 0.19;

// Plans for every (minimum run, row cap) and the cheapest by
// passes + kXyRoundCost * rounds; memoised per (n, gate list, options).
static std::vector<XyPassPlan> plan_xy(int n, const std::vector<std::pair<int, int>> &gates, int mixer) {
    static std::mutex mu;
    static std::vector<std::pair<std::vector<int>, std::vector<XyPassPlan>>> memo;
    std::vector<int> key = {n, mixer, g_xy_min_run, g_xy_row_cap, g_xy_pad, (int)gates.size()};
    for (auto &gp : gates) {
        key.push_back(gp.first);
        key.push_back(gp.second);
    }
    {
        std::lock_guard<std::mutex> lock(mu);
        for (auto &m : memo)
            if (m.first == key) return m.second;
    }
    std::vector<int> runs = g_xy_min_run > 0 ? std::vector<int>{g_xy_min_run} : std::vector<int>{3, 4, 5};
    std::vector<int> caps = g_xy_row_cap > 0 ? std::vector<int>{g_xy_row_cap} : std::vector<int>{1, 2, 3, 4, 6, 64};
    std::vector<XyPassPlan> best;
    double best_cost = 1e300;
    for (int mr : runs)
        for (int cap : caps) {
            auto plans = plan_xy_with(n, gates, mr, cap);
            size_t rounds = 0;
            for (auto &pl : plans) rounds += pl.round_bits.size();
            // shorter runs cost DRAM efficiency (as the X passes, evolve.cu run_factor)
            const double run_pen = mr >= 5 ? 1.0 : mr == 4 ? 1.04 : 1.18;
            const double c = run_pen * (double)plans.size() + kXyRoundCost * (double)rounds;
            if (c < best_cost - 1e-9) {
                best_cost = c;
                best = std::move(plans);
            }
        }
    std::lock_guard<std::mutex> lock(mu);
    if (memo.size() >= 16) memo.erase(memo.begin());
    memo.emplace_back(key, best);
    return best;
}

static void fill_round(XyRound &R, const std::vector<int> &bits, const std::vector<std::pair<int, int>> &gl,
                       const std::vector<int> &tile, int elem) {
    std::memset(&R, 0, sizeof R);
    for (int j = 0; j < 4; ++j) R.reg[j] = (unsigned char)bits[j];
    // thread bits: the other 8 tile bits; the three lane bits of a quarter-warp get
    // distinct residues mod 3 when possible (conflict-free swizzled smem), the rest ascending
    std::vector<int> rest;
    for (int b = 0; b < kTileBits; ++b)
        if (std::find(bits.begin(), bits.end(), b) == bits.end()) rest.push_back(b);
    std::vector<int> order;
    bool low_lanes = true;  // keep lanes 0..4 on tile bits 0..4 when they are all thread bits (global access)
    for (int b = 0; b < 5; ++b) low_lanes &= std::find(rest.begin(), rest.end(), b) != rest.end();
    if (low_lanes) {
        order = rest;
    } else {
        std::vector<int> pool = rest;
        const int mod = elem == 8 ? 4 : 3;  // lanes of one wavefront on distinct residues (see xy_slot)
        for (int res = 0; res < mod; ++res) {
            auto it = std::find_if(pool.begin(), pool.end(), [&](int b) { return b % mod == res; });
            if (it != pool.end()) {
                order.push_back(*it);
                pool.erase(it);
            }
        }
        for (int b : pool) order.push_back(b);
    }
    for (int k = 0; k < 8; ++k) R.tb[k] = (unsigned char)order[k];
    for (int i = 0; i < kRegs; ++i) {
        int e = 0;
        for (int j = 0; j < 4; ++j)
            if ((i >> j) & 1) e |= 1 << bits[j];
        R.sreg[i] = (unsigned short)(xy_slot_of(e, elem) * elem);
    }
    // thread part by nibble of tid (the swizzle is GF(2)-linear: slot(a | b) = slot(a) ^ slot(b))
    for (int h = 0; h < 2; ++h)
        for (int v = 0; v < 16; ++v) {
            int e = 0;
            for (int k = 0; k < 4; ++k)
                if ((v >> k) & 1) e |= 1 << R.tb[4 * h + k];
            R.tnib[16 * h + v] = (unsigned short)(xy_slot_of(e, elem) * elem);
        }
    R.ngates = (unsigned char)gl.size();
    for (size_t g = 0; g < gl.size(); ++g) {
        const int lo = std::min(gl[g].first, gl[g].second), hi = std::max(gl[g].first, gl[g].second);
        const int tlo_bit = (int)(std::find(tile.begin(), tile.end(), lo) - tile.begin());
        const int thi_bit = (int)(std::find(tile.begin(), tile.end(), hi) - tile.begin());
        const int a = (int)(std::find(bits.begin(), bits.end(), tlo_bit) - bits.begin());
        const int b = (int)(std::find(bits.begin(), bits.end(), thi_bit) - bits.begin());
        R.gate[g] = (unsigned char)(4 * a + b);
    }
}

struct XyMaps {
    alignas(64) CUtensorMap state;
    alignas(64) CUtensorMap cost;
};

template <int COST, int PH, bool G = false, typename R = double>
static int launch_xy(const XyParams &P, const XyMaps &M, int grid, cudaStream_t st) {
    static bool configured = false;
    constexpr int CP = table_copies<R>();
    const size_t smem = (size_t)(kTile + (kTableLo + kMaxTableHi) * CP) * sizeof(C2<R>);
    if (!configured) {
        cudaFuncSetAttribute(k_xy_pass<COST, PH, G, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    const size_t need = (size_t)(kTile + (PH && COST == FQ_COST_U16 ? (kTableLo + P.table_hi) * CP : 0)) *
                        sizeof(C2<R>);
    k_xy_pass<COST, PH, G, R><<<grid, kThreads, need, st>>>(P, M.state, M.cost);
    FQ_LAUNCHED("k_xy_pass");
    return FQ_OK;
}

// every (cost, phase, spanning) combination for one real type
template <typename R>
static int launch_xy_any(int cost, bool ph, bool g, const XyParams &P, const XyMaps &M, int grid, cudaStream_t st) {
    if (cost == FQ_COST_U16) {
        if (g) return ph ? launch_xy<FQ_COST_U16, 1, true, R>(P, M, grid, st) : launch_xy<FQ_COST_U16, 0, true, R>(P, M, grid, st);
        return ph ? launch_xy<FQ_COST_U16, 1, false, R>(P, M, grid, st) : launch_xy<FQ_COST_U16, 0, false, R>(P, M, grid, st);
    }
    if (g) return ph ? launch_xy<FQ_COST_F64, 1, true, R>(P, M, grid, st) : launch_xy<FQ_COST_F64, 0, true, R>(P, M, grid, st);
    return ph ? launch_xy<FQ_COST_F64, 1, false, R>(P, M, grid, st) : launch_xy<FQ_COST_F64, 0, false, R>(P, M, grid, st);
}

// Whole XY program (n >= 13): p x (phase, gate sequence), expectation.
// Sharded (sh != null, fq_qaoa_evolve_sharded): the plan covers all n = nl + k
// qubits; a pass whose tile holds global qubits spans the shards it covers
// (G kernel, shard pointer per amplitude index), each rank taking the tiles of
// its own shard set, with device barriers around it; other passes run on the
// rank's own shard(s).
int run_xy_tiled(const fq_evolve_desc *d, const std::vector<std::pair<int, int>> &gates, cudaStream_t st,
                 int *passes_out, const ShardCtx *sh) {
    const int nl = d->n;
    const int kq = sh ? sh->k : 0;
    const int nv = nl + kq, K = 1 << kq;
    const long long size = 1LL << nl;
    const auto plans = plan_xy(nv, gates, d->mixer);
    for (auto &pl : plans)
        if ((int)pl.round_bits.size() > kXyMaxRounds) {
            set_error("run_xy_tiled: a pass needs %d register rounds (max %d)", (int)pl.round_bits.size(),
                      kXyMaxRounds);
            return FQ_ERR_UNSUPPORTED;
        }
    if (passes_out) *passes_out = (int)plans.size() * d->n_layers;
    int table_hi = 0;
    if (d->cost_kind == FQ_COST_U16 && d->cost_levels > 0) {
        const int rows = ((d->cost_levels - 1) >> 6) + 1;
        table_hi = rows <= kMaxTableHi ? rows : 0;
    }
    std::vector<int> mine;
    if (!sh) mine.push_back(0);
    else if (sh->rank >= 0) mine.push_back(sh->rank);
    else for (int r = 0; r < K; ++r) mine.push_back(r);
    const bool c64 = d->state_kind == FQ_STATE_C64;
    auto shard_psi = [&](int r) { return sh ? sh->shards[r] : d->psi; };
    auto launch = [&](bool ph, bool g, const XyParams &Q, const XyMaps &M, int gr) {
        return c64 ? launch_xy_any<float>(d->cost_kind, ph, g, Q, M, gr, st)
                   : launch_xy_any<double>(d->cost_kind, ph, g, Q, M, gr, st);
    };
    auto shard_costs = [&](int r) { return sh ? sh->costs[r] : d->costs; };
    auto barrier = [&]() -> int {
        if (!sh || sh->rank < 0) return FQ_OK;
        return fq_peer_barrier(sh->flags, K, sh->rank, ++*sh->epoch, sh->err, st);
    };
    const int sms = sm_count() > 0 ? sm_count() : 148;
    const long long n_tiles = 1LL << (nl - kTileBits);
    const int grid = (int)std::min<long long>(n_tiles, (long long)sms * 2);
    bool init_pending = d->init != 0;
    double *const shard_sums = d->scratch ? d->scratch + FQ_SCRATCH_DOUBLES - 16 : nullptr;
    XyParams *P = new XyParams;
    auto fail = [&](int s) {
        delete P;
        return s;
    };
    for (int l = 0; l < d->n_layers; ++l) {
        const fq_layer &L = d->layers[l];
        for (size_t pi = 0; pi < plans.size(); ++pi) {
            const XyPassPlan &pl = plans[pi];
            int gmask = 0;  // global qubits among the tile bits
            for (int i = 0; i < kTileBits; ++i)
                if (pl.tile[i] >= nl) gmask |= 1 << (pl.tile[i] - nl);
            std::memset(P, 0, sizeof *P);
            P->cost_scale = d->cost_scale;
            P->cost_offset = d->cost_offset;
            P->partials = d->scratch;
            P->init_amp = d->init_amp;
            P->gamma = L.gamma;
            P->c = std::cos(L.beta);
            P->s = std::sin(L.beta);
            for (int i = 0; i < kTileBits; ++i) P->tile_pos[i] = pl.tile[i];
            P->init = init_pending ? 1 : 0;
            init_pending = false;
            P->expect = (l + 1 == d->n_layers && pi + 1 == plans.size() && d->expectation_dev) ? 1 : 0;
            P->table_hi = table_hi;
            P->nrounds = (int)pl.round_bits.size();
            for (int r = 0; r < P->nrounds; ++r)
                fill_round(P->rounds[r], pl.round_bits[r], pl.round_gates[r], pl.tile, c64 ? 8 : 16);
            for (int i = 0; i < kRegs; ++i) {
                long long a = 0, b = 0;
                for (int j = 0; j < 4; ++j)
                    if ((i >> j) & 1) {
                        a += 1LL << pl.tile[P->rounds[0].reg[j]];
                        b += 1LL << pl.tile[P->rounds[P->nrounds - 1].reg[j]];
                    }
                P->roff_first[i] = a;
                P->roff_last[i] = b;
            }
            const bool ph = pi == 0 && L.apply_phase && L.gamma != 0.0;
            int launches = 0;
            if (gmask) {
                // spanning pass: tile index = [non-tile global bits | local non-tile bits]; the
                // 2^(k - kt) shard sets are contiguous tile ranges, split among their members
                if (int s = barrier()) return fail(s);
                const long long T = 1LL << (nv - kTileBits);
                P->nl = nl;
                for (int r = 0; r < K; ++r) {
                    P->shard[r] = sh->shards[r];
                    P->cshard[r] = sh->costs[r];
                }
                P->psi = P->shard[0];
                P->costs = P->cshard[0];
                P->pf = 0;
                if (sh->rank < 0) {
                    P->tile0 = 0;
                    P->n_tiles = T;
                } else {
                    int g_nt = 0, g_t = 0, cnt_nt = 0, cnt_t = 0;
                    for (int b = 0; b < kq; ++b) {
                        const int bit = (sh->rank >> b) & 1;
                        if ((gmask >> b) & 1) g_t |= bit << cnt_t++;
                        else g_nt |= bit << cnt_nt++;
                    }
                    const long long Tset = T >> cnt_nt;  // tiles of one shard set
                    P->n_tiles = Tset >> cnt_t;
                    P->tile0 = (long long)g_nt * Tset + (long long)g_t * P->n_tiles;
                }
                XyMaps M;
                std::memset(&M, 0, sizeof M);
                const int ggrid = (int)std::min<long long>(P->n_tiles, (long long)sms * 2);
                if (int s = launch(ph, true, *P, M, ggrid)) return fail(s);
                launches = ggrid;
                if (int s2 = barrier()) return fail(s2);
            } else {
                P->n_tiles = n_tiles;
                for (int r : mine) {
                    P->psi = shard_psi(r);
                    P->costs = shard_costs(r);
                    P->partials = d->scratch + launches;
                    XyMaps M;
                    std::memset(&M, 0, sizeof M);
                    // tensor prefetch of the next tile (XY passes, unlike the X passes, gain from it at
                    // 128-B runs too: 2.22 vs 2.32 ms per ring layer at n = 26)
                    P->pf = g_xy_prefetch >= 0 ? g_xy_prefetch : ((16 << run_bits_of(pl.tile)) >= 256 ? 1 : 0);
                    P->sm_rank = c64 ? cached_tile_map(&M.state, P->psi, nl, P->tile_pos, CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                                       4, 2, P->sm_shift, P->sm_bits)
                                     : cached_tile_map(&M.state, P->psi, nl, P->tile_pos, CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                                                       8, 2, P->sm_shift, P->sm_bits);
                    P->cm_rank = 0;
                    if (ph || P->expect)
                        P->cm_rank = d->cost_kind == FQ_COST_F64
                                         ? cached_tile_map(&M.cost, P->costs, nl, P->tile_pos,
                                                          CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, 1, P->cm_shift, P->cm_bits)
                                         : cached_tile_map(&M.cost, P->costs, nl, P->tile_pos,
                                                          CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, 1, P->cm_shift, P->cm_bits);
                    if (int s = launch(ph, false, *P, M, grid)) return fail(s);
                    launches += grid;
                }
            }
            if (P->expect) {
                k_sum_partials<<<1, 32, 0, st>>>(d->scratch, launches, d->expectation_dev);
                FQ_LAUNCHED("k_sum_partials");
            }
        }
    }
    delete P;
    if (init_pending) {  // zero layers
        for (int r : mine)
            if (int s = c64 ? fq_init_state_c64(shard_psi(r), size, -1, d->init_amp, 0, st)
                            : fq_init_state(shard_psi(r), size, -1, d->init_amp, 0, st))
                return s;
    }
    if (d->n_layers == 0 && d->expectation_dev) {
        auto expect = c64 ? fq_expectation_c64 : fq_expectation;
        if (mine.size() == 1)
            return expect(shard_psi(mine[0]), shard_costs(mine[0]), d->cost_kind, d->cost_scale, d->cost_offset, size,
                          d->expectation_dev, d->scratch, st);
        for (size_t i = 0; i < mine.size(); ++i)
            if (int s = expect(shard_psi(mine[i]), shard_costs(mine[i]), d->cost_kind, d->cost_scale, d->cost_offset,
                               size, shard_sums + i, d->scratch, st))
                return s;
        k_sum_partials<<<1, 32, 0, st>>>(shard_sums, (int)mine.size(), d->expectation_dev);
        FQ_LAUNCHED("k_sum_partials");
    }
    return FQ_OK;
}

int plan_xy_passes(int n, int mixer, const std::vector<std::pair<int, int>> &gates, int *rounds) {
    const auto plans = plan_xy(n, gates, mixer);
    if (std::getenv("FQ_XY_DUMP")) {  // development: the plan on stderr (tile qubits; per round: register tile bits / gates)
        for (auto &pl : plans) {
            std::fprintf(stderr, "pass tile=");
            for (int q : pl.tile) std::fprintf(stderr, "%d,", q);
            std::fprintf(stderr, "\n");
            for (size_t r = 0; r < pl.round_bits.size(); ++r) {
                std::fprintf(stderr, "  R");
                for (int b : pl.round_bits[r]) std::fprintf(stderr, " %d", b);
                std::fprintf(stderr, " :");
                for (auto &g : pl.round_gates[r]) std::fprintf(stderr, " (%d,%d)", g.first, g.second);
                std::fprintf(stderr, "\n");
            }
        }
    }
    if (rounds) {
        *rounds = 0;
        for (auto &pl : plans) *rounds += (int)pl.round_bits.size();
    }
    return (int)plans.size();
}

}  // namespace fq
