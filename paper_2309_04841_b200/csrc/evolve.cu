// Fused QAOA evolution for sm_100a — the hot path of the reference's
// QaoaSimulator.simulate_qaoa (qaoa.py:137-149) + get_expectation
// (statevec.py:94-97): p x (phase psi *= exp(-i gamma c), mixer), then
// sum_k c_k |psi_k|^2.
//
// Design:
//  * The state is processed in tiles of 2^12 amplitudes (64 KiB).  A tile is
//    defined by 12 "tile bits" (physical index bits); the remaining index bits
//    select the tile.  One HBM pass streams every tile once, applies every
//    butterfly whose qubit is a tile bit, and writes it back: up to 12 qubits
//    per HBM round trip instead of one (reference _kernels.py:14-27 is one
//    pass per qubit).
//  * Inside a tile each of the 256 threads holds 16 amplitudes in registers
//    (4 tile bits).  A pass is a short "round program": register rounds on the
//    tile-bit quads 8-11 / 0-3 / 4-7 with XOR-padded shared-memory transposes
//    in between (conflict-free 16-B accesses).  Quads without a target are
//    never visited, so a group whose targets all sit in tile bits >= 4 costs
//    one transpose per layer instead of two.
//  * The phase is applied inside a pass (never a separate sweep); the first
//    pass of the program generates |+>^n instead of loading it; the last pass
//    accumulates the expectation.  Consecutive layers traverse the qubit
//    groups in alternating order, so the last pass of layer l and the first
//    pass of layer l+1 touch the same tile and are fused (mixer_l, phase_{l+1},
//    mixer_{l+1}): 1 + p*(G-1) passes for G groups instead of p*G.  The host
//    planner puts small (<= 8-target) groups at the fusion points, so a fused
//    pass is three rounds / two transposes like an ordinary one.
//  * The X mixer uses the scaled form Rx = f (alpha I - i delta X) with
//    (alpha, delta) = (1, tan b) or (cot b, 1) whichever keeps |.| <= 1: one FMA
//    per output component; the product of the f's is applied once per pass.
//  * uint16 level costs (lossless CompactCostVector, terms.py:123-175) make
//    the phase two table lookups + one complex multiply
//    (e^{-i g (s*64h+o)} * e^{-i g s l}), no sincos in the stream.
//  * Each CTA keeps the tile it will process next in flight with an L2 bulk
//    prefetch (cp.async.bulk.prefetch.L2), so HBM stays busy while the CTA is
//    in its shared-memory / FP64 rounds.
//  * States of n <= 12 qubits run the entire program in one CTA (smem-resident),
//    which is also the batched multi-parameter path for optimiser loops.
#include <chrono>
#include <string>

#include "sweep.cuh"
#include "tmap.cuh"

namespace fq {

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
    int table_hi;           // k_resident16, uint16 costs: rows of the high phase table (0: sincos)
    int n_gates;
    unsigned char gates[kResMaxGates][2];
    // per (batch row, layer) angles: gam[b*p + l], bet[b*p + l]; row b = blockIdx.x
    double gam[kResMaxLayers], bet[kResMaxLayers];
    int all_tables;         // k_resident8 with ang: uint16 phase tables of every layer built at once
    const double *ang;      // non-null (one parameter set): device [2p] = gamma_l, beta_l, read instead of
                            // gam / bet -- a captured CUDA graph replays with new angles (fq_objective_graph_*)
    unsigned char phase_on[kResMaxLayers];  // indexed by layer (shared by all rows)
    unsigned char qlo[kResMaxLayers], qhi[kResMaxLayers];  // X/custom qubit range per layer
};

// Graph-replayed objective (ResParams::ang set): the angles live in pinned host
// memory the device reads directly; staged once per CTA in shared memory.
constexpr int kResGraphMaxLayers = 64;

__device__ __forceinline__ void res_stage_angles(const ResParams &P, double *s_ang) {
    if (P.ang) {
        for (int i = threadIdx.x; i < 2 * P.p; i += blockDim.x) s_ang[i] = P.ang[i];
        __syncthreads();
    }
}

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
    __shared__ double s_ang[2 * kResGraphMaxLayers];
    res_stage_angles(P, s_ang);
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
        const double gamma = P.ang ? s_ang[2 * l] : P.gam[b * P.p + l];
        const double beta = P.ang ? s_ang[2 * l + 1] : P.bet[b * P.p + l];
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

// ---------------------------------------------------------------- resident, register rounds (n <= 12, X / custom)
// The whole state is ONE 2^12 tile of k_pass16 (qubit q = tile bit q; for
// n < 12 the tile bits >= n carry zero amplitudes that are never stored):
// 256 threads x 16 amplitudes in registers, a layer = phase + three radix-16
// rounds over the register quads (8-11 | 0-3 | 4-7, walked forward on even
// layers and backward on odd ones, so consecutive layers share a pattern and
// a layer costs two shared-memory transposes), instead of k_resident's one
// shared-memory sweep + barrier per qubit.  One CTA runs a whole program, so
// the kernel is latency- and instruction-fetch-bound: the code is kept small
// (one mixer per instantiation, one loop body for every register pattern,
// the sincos phase out of line).
constexpr int kRes16Smem = (kTilePadded + (kTableLo + kMaxTableHi) * 8) * (int)sizeof(double2);

// Register pattern at run time (the layer loop is one small body for every
// pattern): element index of register i = ibase + i * istep, padded
// transpose slot = sbase + i * sstep, register bit j = qubit first + j.
struct Res16Pat {
    int ibase, istep, sbase, sstep, first;
};
__device__ __forceinline__ Res16Pat res16_pat(int pat, int tid) {
    Res16Pat r;
    if (pat == PAT8) {
        r.ibase = tid; r.istep = 256; r.sbase = pat_base<PAT8>(tid); r.sstep = pat_step<PAT8>(1); r.first = 8;
    } else if (pat == PAT0) {
        r.ibase = tid << 4; r.istep = 1; r.sbase = pat_base<PAT0>(tid); r.sstep = pat_step<PAT0>(1); r.first = 0;
    } else {
        r.ibase = (tid & 15) | ((tid >> 4) << 8); r.istep = 16; r.sbase = pat_base<PAT4>(tid);
        r.sstep = pat_step<PAT4>(1); r.first = 4;
    }
    return r;
}

// e^{-i gamma c_e}, float64 cost or a uint16 level without tables (out of line)
template <int COST>
static __device__ __noinline__ double2 res16_phase_sincos(const ResParams &P, int e, double gamma) {
    double c;
    if (COST == FQ_COST_F64) c = static_cast<const double *>(P.costs)[e];
    else c = decode_u16(static_cast<const uint16_t *>(P.costs)[e], P.cost_scale, P.cost_offset);
    return phase_f64(c, gamma);
}

template <int COST, int MIX>
__global__ void __launch_bounds__(kThreads, 2) k_resident16(const __grid_constant__ ResParams P,
                                                            const double *__restrict__ su2) {
    extern __shared__ __align__(16) unsigned char res_smem[];
    double2 *tile = reinterpret_cast<double2 *>(res_smem);
    double2 *tlo = tile + kTilePadded;
    double2 *thi = tlo + kTableLo * 8;
    __shared__ double red[kThreads / 32];
    __shared__ double s_ang[2 * kResGraphMaxLayers];
    res_stage_angles(P, s_ang);
    const int tid = threadIdx.x, N = 1 << P.n, b = blockIdx.x;
    const int table_hi = COST == FQ_COST_U16 ? P.table_hi : 0;
    double2 v[kRegs];
    Res16Pat cur = res16_pat(PAT8, tid);
    const double2 *src = (P.init || P.psi_in == nullptr) ? nullptr : P.psi_in + (long long)b * P.in_stride;
#pragma unroll
    for (int i = 0; i < kRegs; ++i) {
        const int e = cur.ibase + i * cur.istep;
        v[i] = e >= N ? make_double2(0.0, 0.0) : src ? src[e] : make_double2(P.init_amp, 0.0);
    }
    int pat = PAT8;
#pragma unroll 1
    for (int l = 0; l < P.p; ++l) {
        const double gamma = P.ang ? s_ang[2 * l] : P.gam[b * P.p + l];
        if (P.phase_on[l] && gamma != 0.0) {
            if (COST == FQ_COST_U16 && table_hi > 0) {
                // the previous layer's lookups are behind its transposes' barriers
                build_phase_tables<double>(tlo, thi, table_hi, gamma, P.cost_scale, P.cost_offset);
                __syncthreads();
            }
#pragma unroll
            for (int i = 0; i < kRegs; ++i) {
                const int e = cur.ibase + i * cur.istep;
                if (e >= N) continue;
                double2 f;
                if (COST == FQ_COST_U16 && table_hi > 0) {
                    const unsigned raw = static_cast<const uint16_t *>(P.costs)[e];
                    f = cmul(thi[(raw >> 6) * 8 + (tid & 7)], tlo[(raw & 63) * 8 + (tid & 7)]);
                } else {
                    f = res16_phase_sincos<COST>(P, e, gamma);
                }
                v[i] = cmul(v[i], f);
            }
        }
        const int qlo = P.qlo[l], qhi = P.qhi[l];
        // RX in the tiled passes' form: f (1, tan b) or f (cot b, 1), two DFMA per
        // amplitude and qubit, the layer's f^targets applied once at its end
        double rc = 0.0, f = 1.0;
        int mode = 0;
        if (MIX == MIX_RX) {
            double s, c;
            sincos(P.ang ? s_ang[2 * l + 1] : P.bet[b * P.p + l], &s, &c);
            if (fabs(c) >= fabs(s)) { rc = s / c; f = c; }
            else { mode = 1; rc = c / s; f = s; }
        }
        // three rounds: 8 -> 0 -> 4 from PAT8, 4 -> 0 -> 8 from PAT4
#pragma unroll 1
        for (int r = 0; r < 3; ++r) {
            if (r > 0) {
                const int next = r == 1 ? PAT0 : (pat == PAT0 ? (l & 1 ? PAT8 : PAT4) : pat);
                const Res16Pat nx = res16_pat(next, tid);
#pragma unroll
                for (int i = 0; i < kRegs; ++i) tile[cur.sbase + i * cur.sstep] = v[i];
                __syncthreads();
#pragma unroll
                for (int i = 0; i < kRegs; ++i) v[i] = tile[nx.sbase + i * nx.sstep];
                __syncthreads();
                cur = nx;
                pat = next;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int q = cur.first + j;
                if (q < qlo || q >= qhi) continue;
                if constexpr (MIX == MIX_RX) {
                    if (mode == 0) {
#pragma unroll
                        for (int i = 0; i < kRegs; ++i)
                            if (!(i & (1 << j))) bfly_rx0(v[i], v[i | (1 << j)], rc);
                    } else {
#pragma unroll
                        for (int i = 0; i < kRegs; ++i)
                            if (!(i & (1 << j))) bfly_rx1(v[i], v[i | (1 << j)], rc);
                    }
                } else {
                    const double *c4 = su2 + ((long long)l * P.n + q) * 4;
                    const double2 a = make_double2(c4[0], c4[1]), bb = make_double2(c4[2], c4[3]);
#pragma unroll
                    for (int i = 0; i < kRegs; ++i)
                        if (!(i & (1 << j))) bfly_su2(v[i], v[i | (1 << j)], a, bb);
                }
            }
        }
        if (MIX == MIX_RX) {
            double fs = 1.0;
            for (int q = max(qlo, 0); q < min(qhi, P.n); ++q) fs *= f;
#pragma unroll
            for (int i = 0; i < kRegs; ++i) v[i] = make_double2(v[i].x * fs, v[i].y * fs);
        }
    }
    // objective and state in the final pattern
    double acc = 0.0;
    double2 *dst = P.psi_out ? P.psi_out + (long long)b * N : nullptr;
#pragma unroll
    for (int i = 0; i < kRegs; ++i) {
        const int e = cur.ibase + i * cur.istep;
        if (e >= N) continue;
        if (P.exp_out) {
            const double cv = (COST == FQ_COST_F64) ? static_cast<const double *>(P.costs)[e]
                                                    : decode_u16(static_cast<const uint16_t *>(P.costs)[e],
                                                                 P.cost_scale, P.cost_offset);
            acc += cv * (v[i].x * v[i].x + v[i].y * v[i].y);
        }
        if (dst) dst[e] = v[i];
    }
    if (P.exp_out) {
        const double t = block_sum<kThreads>(acc, red);
        if (tid == 0) P.exp_out[b] = t;
    }
}

// 512 threads x 8 amplitudes: twice the warps of k_resident16 (a single CTA
// is latency-bound), rounds over register triples (bits 9-11 | 0-2 | 3-5 |
// 6-8, forward on even layers, backward on odd ones: three transposes per
// layer).  Transpose slot e + (e >> 3): a quarter-warp's eight 16-B accesses
// hit eight distinct bank groups in all four patterns.
constexpr int kRes8Threads = 512;
constexpr int kRes8Regs = 8;
constexpr int kRes8Padded = kTile + kTile / 8;
constexpr int kRes8Smem = 224 * 1024;  // max dynamic smem (all_tables: every layer's phase tables)

// register pattern k (k = 0..3): registers hold tile bits 3k..3k+2
__device__ __forceinline__ Res16Pat res8_pat(int k, int tid) {
    Res16Pat r;
    const int lowm = (1 << (3 * k)) - 1;
    r.ibase = (tid & lowm) | ((tid >> (3 * k)) << (3 * k + 3));
    r.istep = 1 << (3 * k);
    r.sbase = r.ibase + (r.ibase >> 3);
    r.sstep = r.istep + (r.istep >> 3);
    r.first = 3 * k;
    return r;
}

template <int COST, int MIX>
__global__ void __launch_bounds__(kRes8Threads, 1) k_resident8(const __grid_constant__ ResParams P,
                                                               const double *__restrict__ su2) {
    extern __shared__ __align__(16) unsigned char res_smem[];
    double2 *tile = reinterpret_cast<double2 *>(res_smem);
    double2 *tlo = tile + kRes8Padded;
    double2 *thi = tlo + kTableLo * 8;
    __shared__ double red[kRes8Threads / 32];
    __shared__ double s_ang[2 * kResGraphMaxLayers];
    res_stage_angles(P, s_ang);
    const int tid = threadIdx.x, N = 1 << P.n, b = blockIdx.x;
    const int table_hi = COST == FQ_COST_U16 ? P.table_hi : 0;
    const int rows = kTableLo + table_hi;
    if (COST == FQ_COST_U16 && P.all_tables) {
        // graph-replayed evaluation: the tables of all layers in one parallel sweep and one
        // barrier (instead of one sincos round + barrier per layer on the critical path)
        for (int i = tid; i < P.p * rows; i += kRes8Threads) {
            const int l = i / rows, r = i - l * rows;
            double sn, cn;
            if (r < kTableLo) sincos(s_ang[2 * l] * (P.cost_scale * (double)r), &sn, &cn);
            else sincos(s_ang[2 * l] * (P.cost_scale * (double)(64 * (r - kTableLo)) + P.cost_offset), &sn, &cn);
            double2 *row = tlo + ((size_t)l * rows + r) * 8;
#pragma unroll
            for (int k = 0; k < 8; ++k) row[k] = make_double2(cn, -sn);
        }
        __syncthreads();
    }
    double2 v[kRes8Regs];
    int pat = 3;
    Res16Pat cur = res8_pat(pat, tid);
    const double2 *src = (P.init || P.psi_in == nullptr) ? nullptr : P.psi_in + (long long)b * P.in_stride;
#pragma unroll
    for (int i = 0; i < kRes8Regs; ++i) {
        const int e = cur.ibase + i * cur.istep;
        v[i] = e >= N ? make_double2(0.0, 0.0) : src ? src[e] : make_double2(P.init_amp, 0.0);
    }
#pragma unroll 1
    for (int l = 0; l < P.p; ++l) {
        const double gamma = P.ang ? s_ang[2 * l] : P.gam[b * P.p + l];
        if (P.phase_on[l] && gamma != 0.0) {
            const double2 *tl = tlo, *th = thi;
            if (COST == FQ_COST_U16 && P.all_tables) {
                tl = tlo + (size_t)l * rows * 8;
                th = tl + kTableLo * 8;
            } else if (COST == FQ_COST_U16 && table_hi > 0) {
                build_phase_tables<double>(tlo, thi, table_hi, gamma, P.cost_scale, P.cost_offset);
                __syncthreads();
            }
#pragma unroll
            for (int i = 0; i < kRes8Regs; ++i) {
                const int e = cur.ibase + i * cur.istep;
                if (e >= N) continue;
                double2 f;
                if (COST == FQ_COST_U16 && table_hi > 0) {
                    const unsigned raw = static_cast<const uint16_t *>(P.costs)[e];
                    f = cmul(th[(raw >> 6) * 8 + (tid & 7)], tl[(raw & 63) * 8 + (tid & 7)]);
                } else {
                    f = res16_phase_sincos<COST>(P, e, gamma);
                }
                v[i] = cmul(v[i], f);
            }
        }
        const int qlo = P.qlo[l], qhi = P.qhi[l];
        double rc = 0.0, f = 1.0;
        int mode = 0;
        if (MIX == MIX_RX) {
            double sn, cs;
            sincos(P.ang ? s_ang[2 * l + 1] : P.bet[b * P.p + l], &sn, &cs);
            if (fabs(cs) >= fabs(sn)) { rc = sn / cs; f = cs; }
            else { mode = 1; rc = cs / sn; f = sn; }
        }
        const int dir = l & 1;  // even layers 3 -> 0 -> 1 -> 2, odd layers 2 -> 1 -> 0 -> 3
#pragma unroll 1
        for (int r = 0; r < 4; ++r) {
            if (r > 0) {
                const int next = dir ? (r == 3 ? 3 : 2 - r) : r - 1;
                const Res16Pat nx = res8_pat(next, tid);
#pragma unroll
                for (int i = 0; i < kRes8Regs; ++i) tile[cur.sbase + i * cur.sstep] = v[i];
                __syncthreads();
#pragma unroll
                for (int i = 0; i < kRes8Regs; ++i) v[i] = tile[nx.sbase + i * nx.sstep];
                __syncthreads();
                cur = nx;
                pat = next;
            }
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const int q = cur.first + j;
                if (q < qlo || q >= qhi) continue;
                if constexpr (MIX == MIX_RX) {
                    if (mode == 0) {
#pragma unroll
                        for (int i = 0; i < kRes8Regs; ++i)
                            if (!(i & (1 << j))) bfly_rx0(v[i], v[i | (1 << j)], rc);
                    } else {
#pragma unroll
                        for (int i = 0; i < kRes8Regs; ++i)
                            if (!(i & (1 << j))) bfly_rx1(v[i], v[i | (1 << j)], rc);
                    }
                } else {
                    const double *c4 = su2 + ((long long)l * P.n + q) * 4;
                    const double2 a = make_double2(c4[0], c4[1]), bb = make_double2(c4[2], c4[3]);
#pragma unroll
                    for (int i = 0; i < kRes8Regs; ++i)
                        if (!(i & (1 << j))) bfly_su2(v[i], v[i | (1 << j)], a, bb);
                }
            }
        }
        if (MIX == MIX_RX) {
            double fs = 1.0;
            for (int q = max(qlo, 0); q < min(qhi, P.n); ++q) fs *= f;
#pragma unroll
            for (int i = 0; i < kRes8Regs; ++i) v[i] = make_double2(v[i].x * fs, v[i].y * fs);
        }
    }
    double acc = 0.0;
    double2 *dst = P.psi_out ? P.psi_out + (long long)b * N : nullptr;
#pragma unroll
    for (int i = 0; i < kRes8Regs; ++i) {
        const int e = cur.ibase + i * cur.istep;
        if (e >= N) continue;
        if (P.exp_out) {
            const double cv = (COST == FQ_COST_F64) ? static_cast<const double *>(P.costs)[e]
                                                    : decode_u16(static_cast<const uint16_t *>(P.costs)[e],
                                                                 P.cost_scale, P.cost_offset);
            acc += cv * (v[i].x * v[i].x + v[i].y * v[i].y);
        }
        if (dst) dst[e] = v[i];
    }
    if (P.exp_out) {
        const double t = block_sum<kRes8Threads>(acc, red);
        if (tid == 0) P.exp_out[b] = t;
    }
    (void)pat;
}

// ---------------------------------------------------------------- standalone phase (uint16)
// T = double2 (complex128 states) or float2 (complex64); the angle is always fp64
template <typename T>
__global__ void k_phase_u16(T *__restrict__ psi, const uint16_t *__restrict__ lv, long long size, double gamma,
                            double scale, double offset) {
    using R = decltype(T::x);
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < size;
         k += (long long)gridDim.x * blockDim.x) {
        const double2 f = phase_f64(decode_u16(lv[k], scale, offset), gamma);
        psi[k] = cmul(psi[k], T{(R)f.x, (R)f.y});
    }
}

template <typename T>
__global__ void k_phase_f64(T *__restrict__ psi, const double *__restrict__ costs, long long size, double gamma) {
    using R = decltype(T::x);
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < size;
         k += (long long)gridDim.x * blockDim.x) {
        double s, c;
        sincos(gamma * costs[k], &s, &c);
        psi[k] = cmul(psi[k], T{(R)c, (R)-s});
    }
}

// standalone phase / state init / expectation on either state type
template <typename T>
static void launch_phase(T *psi, const fq_evolve_desc *d, long long size, double gamma, cudaStream_t st) {
    if (d->cost_kind == FQ_COST_U16)
        k_phase_u16<<<grid_for(size, 256, 8), 256, 0, st>>>(psi, static_cast<const uint16_t *>(d->costs), size, gamma,
                                                            d->cost_scale, d->cost_offset);
    else
        k_phase_f64<<<grid_for(size, 256, 8), 256, 0, st>>>(psi, static_cast<const double *>(d->costs), size, gamma);
}

static int state_init(const fq_evolve_desc *d, void *psi, long long size, cudaStream_t st) {
    return d->state_kind == FQ_STATE_C64 ? fq_init_state_c64(psi, size, -1, d->init_amp, 0, st)
                                         : fq_init_state(psi, size, -1, d->init_amp, 0, st);
}

static int state_expectation(const fq_evolve_desc *d, const void *psi, long long size, cudaStream_t st) {
    return d->state_kind == FQ_STATE_C64
               ? fq_expectation_c64(psi, d->costs, d->cost_kind, d->cost_scale, d->cost_offset, size,
                                    d->expectation_dev, d->scratch, st)
               : fq_expectation(psi, d->costs, d->cost_kind, d->cost_scale, d->cost_offset, size, d->expectation_dev,
                                d->scratch, st);
}

// ---------------------------------------------------------------- host planning
struct Group {
    std::vector<int> targets;  // physical qubit positions, ascending
    int tile_pos[kTileBits];
};

// Tile of a target group: the targets plus the lowest non-target physical
// bits as spectators (so every global access is a run of >= 2^spectators
// amplitudes), sorted ascending.
static Group make_group(int n, const std::vector<int> &targets) {
    Group g;
    g.targets = targets;
    std::vector<int> bits = targets;
    for (int q = 0; q < n && (int)bits.size() < kTileBits; ++q)
        if (std::find(targets.begin(), targets.end(), q) == targets.end()) bits.push_back(q);
    std::sort(bits.begin(), bits.end());
    for (int i = 0; i < kTileBits; ++i) g.tile_pos[i] = bits[i];
    return g;
}

static std::vector<std::vector<int>> split_even(const std::vector<int> &v, int parts) {
    std::vector<std::vector<int>> out;
    size_t at = 0;
    for (int c = 0; c < parts; ++c) {
        const size_t sz = (v.size() - at) / (parts - c);
        out.emplace_back(v.begin() + at, v.begin() + at + sz);
        at += sz;
    }
    return out;
}

// Candidate orderings of the target groups of one layer (the first and last
// group of a layer are the fusion points with the neighbouring layers), high
// targets in even chunks of <= tmax:
//   style 0: [low, high chunks]                 (all-qubit passes, legacy)
//   style 1: [high_0, low, high_1 .. high_m-1], so both fusion points are
//      small groups (3-round fused passes)
// A chunk of t high targets leaves 12 - t low spectators: the tile's global
// accesses are runs of 2^(12-t) amplitudes, which sets the pass's bandwidth
// (run_factor), so fewer targets per pass can win at large n.
static std::vector<std::vector<int>> candidate_groups(const std::vector<int> &targets, int style, int tmax) {
    std::vector<int> low, high;
    for (int q : targets) (q < kTileBits ? low : high).push_back(q);
    std::vector<std::vector<int>> out;
    const int chunks = (int)((high.size() + tmax - 1) / tmax);
    if (style == 0 || high.empty() || low.empty()) {
        if (!low.empty()) out.push_back(low);
        if (!high.empty())
            for (auto &c : split_even(high, chunks)) out.push_back(c);
        return out;
    }
    auto hs = split_even(high, chunks);
    out.push_back(hs[0]);
    out.push_back(low);
    for (size_t i = 1; i < hs.size(); ++i) out.push_back(hs[i]);
    return out;
}

struct PlannedPass {
    int group;           // index into groups (-1: standalone phase)
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

static int g_fuse = 1;
static int g_prefetch = -1;  // L2 prefetch distance (grid strides); -1: 1 for runs >= 256 B, else 0
static int g_phase_tables = 1;
static int g_plan = -1;      // -1: choose by cost model, else force style (0 / 1, legacy chunk sizes)
static int g_plan_tmax = 0;  // > 0: force the high-group chunk size (4..12) of the X plan (parity tests of every shape)
static int g_sweep = 0;          // run eligible pass pairs as L2-resident slab sweeps (sweep.cuh); off: measured slower
static int g_sweep_team = 32;    // CTAs per sweep team
static int g_sweep_slab_log2 = 23;  // largest slab (bytes, log2): 8 MiB x ~9 teams in flight stay in L2
static long long g_sweeps_launched = 0;
// scratch layout of the sweeps: team counters (16 x 128 B) and the barrier error word
constexpr int kSweepCtrOffset = 2048;  // doubles
constexpr int kSweepErrOffset = 2048 + 16 * 16;
static int *S_err_ptr(const fq_evolve_desc *d) { return reinterpret_cast<int *>(d->scratch + kSweepErrOffset); }

// sum of partials, NaN when a sweep's team barrier timed out (never a silent wrong objective)
__global__ void k_sum_partials_checked(const double *partials, int count, const int *err, double *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < count; ++i) t += partials[i];
        *out = (*err) ? __longlong_as_double(0x7ff8000000000000LL) : t;
    }
}
static int g_time_passes = 0;
static int g_probe = 0;      // development probe bits (PassParams::probe)
static int g_zigzag = 1;     // alternate the tile walk direction pass to pass (L2 reuse across passes)

// Per-pass record of the last X program (fq_last_passes): kind + event timing.
struct PassRecord {
    int seq, ph, targets, init, expect;
};
static std::vector<PassRecord> g_last_plan;
static std::vector<cudaEvent_t> g_events;  // g_last_plan.size() + 1 when timing is on

static std::vector<PlannedPass> plan_with(int n, int nl, const fq_layer *layers, std::vector<Group> &groups, int style,
                                          int tmax, bool fuse) {
    groups.clear();
    std::vector<PlannedPass> seq;
    std::vector<int> prev_targets;
    int prev_base = -1, prev_ng = 0, dir = 0;
    for (int l = 0; l < nl; ++l) {
        std::vector<int> targets;
        for (int q = std::max(0, layers[l].q_lo); q < std::min(n, layers[l].q_hi); ++q) targets.push_back(q);
        int gbase, ng;
        if (prev_base >= 0 && targets == prev_targets) {
            gbase = prev_base;
            ng = prev_ng;
        } else {
            gbase = (int)groups.size();
            auto chunks = candidate_groups(targets, style, tmax);
            for (auto &c : chunks) groups.push_back(make_group(n, c));
            ng = (int)chunks.size();
            dir = 0;
        }
        prev_targets = targets;
        prev_base = gbase;
        prev_ng = ng;
        if (ng == 0) {  // phase-only layer
            if (phase_active(layers[l])) seq.push_back({-1, -1, -1, l, 1});
            continue;
        }
        for (int i = 0; i < ng; ++i) {
            const int gi = gbase + (dir ? ng - 1 - i : i);
            if (i == 0 && fuse && !seq.empty() && seq.back().group == gi && seq.back().layerB < 0 &&
                seq.back().layerA == l - 1 && (seq.back().phase_layer < 0 || !phase_active(layers[l]))) {
                // fuse: mixer_{l-1} on the tile, phase_l, mixer_l on the tile
                seq.back().layerB = l;
                if (phase_active(layers[l])) {
                    seq.back().phase_layer = l;
                    seq.back().phase_at = 2;
                }
                continue;
            }
            seq.push_back({gi, l, -1, (i == 0 && phase_active(layers[l])) ? l : -1, 1});
        }
        dir ^= 1;
    }
    return seq;
}

static int target_mask(const Group &g) {
    int m = 0;
    for (int i = 0; i < kTileBits; ++i)
        if (std::find(g.targets.begin(), g.targets.end(), g.tile_pos[i]) != g.targets.end()) m |= 1 << i;
    return m;
}

// lane_ok (X mixer, shard-local group, option lane3): a group whose only target
// among tile bits 0..3 is bit 3 runs the two-pattern programs with bit 3 as a
// lane butterfly (K_LANE3)
static int g_lane3 = 1;
static int g_cost_stage = 1;  // shared cost tile for the phase / expectation read after a transpose
static int g_cost_l2 = -1;  // cost loads at normal L2 priority: -1 when cost runs < 32 B, 0 never, 1 always
static int lane_bits(const Group &g, bool lane_ok) {
    return lane_ok && g_lane3 && (target_mask(g) & 0xF) == 0x8 ? 0x8 : 0;
}

static int pass_seq(const Group &g, const PlannedPass &pp, bool lane_ok = false) {
    const bool heavy = pp.layerB >= 0 && pp.phase_layer >= 0 && pp.phase_at == 2;
    const bool low_quad = (target_mask(g) & 0xF) != 0 && !lane_bits(g, lane_ok);
    if (heavy) return low_quad ? SEQ_84048 : SEQ_848;
    return low_quad ? SEQ_840 : SEQ_84;
}

// Relative pass cost (measured on B200, LABS n=26: an HBM-bound 3-round pass = 1).
static double pass_cost(int seq) {
    switch (seq) {
        case SEQ_840: return 1.0;
        case SEQ_84: return 0.97;
        case SEQ_84048: return 1.7;
        default: return 1.08;
    }
}

// contiguous low tile bits: every global access of the tile is a run of
// 2^run_bits amplitudes
static int run_bits_of(const Group &g) {
    int r = 0;
    while (r < kTileBits && g.tile_pos[r] == r) ++r;
    return r;
}

// Pass time vs the contiguous run length of its accesses, relative to runs
// >= 512 B (measured on B200, LABS n = 26..34, c128 and c64):
// heavy (latency-bound, fused) passes lose bandwidth to short runs much faster.
static double run_factor(long long run_bytes, bool heavy) {
    if (run_bytes >= 512) return 1.0;
    if (run_bytes >= 256) return heavy ? 1.13 : 1.04;
    if (run_bytes >= 128) return heavy ? 1.25 : 1.15;
    if (run_bytes >= 64) return heavy ? 3.9 : 2.33;
    return heavy ? 8.0 : 4.7;
}

// Sharded states (fq_qaoa_evolve_sharded): the top kq of the n positions are
// global qubits (the shard index).  A group holds all of them or none: its
// tile then spans every shard (a peer-memory pass, G = true).
static int global_count(const Group &g, int n, int kq) {
    int c = 0;
    for (int q : g.targets) c += q >= n - kq;
    return c;
}

// extra cost of the lane-shuffle butterflies of a K_LANE3 pass (light, heavy)
static const double kLanePassCost[2] = {0.08, 0.16};

// A peer-memory pass moves (K-1)/K of its bytes over NVLink (~0.9 TB/s per
// direction vs ~6.5 TB/s of HBM).
constexpr double kGlobalPassCost = 5.0;

static double plan_cost(const std::vector<PlannedPass> &seq, const std::vector<Group> &gs, int n, int elem,
                        int kq = 0, bool rx = true) {
    for (auto &g : gs) {
        const int c = global_count(g, n, kq);
        if (c != 0 && c != kq) return 1e300;
    }
    // a state that stays in L2 (126 MB) between passes does not see DRAM run lengths
    const bool l2_resident = ((long long)elem << (n - kq)) <= (64LL << 20);
    double c = 0.0;
    for (auto &pp : seq) {
        if (pp.group < 0) {
            c += 1.0;
            continue;
        }
        const bool lane_ok = rx && global_count(gs[pp.group], n, kq) == 0;
        const int sq = pass_seq(gs[pp.group], pp, lane_ok);
        double pc = pass_cost(sq) * (l2_resident ? 1.0 : run_factor((long long)elem << run_bits_of(gs[pp.group]), seq_heavy(sq)));
        if (lane_bits(gs[pp.group], lane_ok)) pc += seq_heavy(sq) ? kLanePassCost[1] : kLanePassCost[0];
        // a spanning pass is NVLink-bound: its DRAM run lengths hide behind the link
        // (and its round program too: the link time is the same for every program)
        if (kq > 0 && global_count(gs[pp.group], n, kq) > 0) pc = std::max(pc, kGlobalPassCost);
        c += pc;
    }
    return c;
}

// elem: bytes per amplitude (16 complex128, 8 complex64); kq: global qubits of a sharded state
static std::vector<PlannedPass> plan_x_search(int n, int nl, const fq_layer *layers, std::vector<Group> &groups,
                                              bool fuse, int elem, int kq, bool rx) {
    std::vector<PlannedPass> best;
    double best_cost = 1e300;
    if (g_plan >= 0 || g_plan_tmax > 0) {  // forced shape (style and / or chunk size); invalid -> search
        for (int style = 0; style < 2; ++style) {
            if (g_plan >= 0 && style != g_plan) continue;
            const int tmax = g_plan_tmax > 0 ? g_plan_tmax : (style == 0 ? 10 : 8);
            std::vector<Group> gs;
            auto seq = plan_with(n, nl, layers, gs, style, tmax, fuse);
            const double c = plan_cost(seq, gs, n, elem, kq, rx);
            if (c < best_cost - 1e-9 && c < 1e299) {
                best_cost = c;
                best = seq;
                groups = gs;
            }
        }
        if (best_cost < 1e299) return best;
    }
    for (int style = 0; style < 2; ++style) {
        for (int tmax = 12; tmax >= 4; --tmax) {
            std::vector<Group> gs;
            auto seq = plan_with(n, nl, layers, gs, style, tmax, fuse);
            const double c = plan_cost(seq, gs, n, elem, kq, rx);
            if (c < best_cost - 1e-9) {
                best_cost = c;
                best = seq;
                groups = gs;
            }
        }
    }
    return best;
}

// The search prices 18 candidate plans (~0.1 ms of host time), on the path of
// every simulate_qaoa call, before the first launch: plans are memoised by
// everything they depend on (sizes, options, and per layer the qubit range and
// whether a phase is applied — not the angles).
struct PlanMemo {
    std::vector<long long> key;
    std::vector<PlannedPass> seq;
    std::vector<Group> groups;
};

static std::vector<PlannedPass> plan_x(int n, int nl, const fq_layer *layers, std::vector<Group> &groups, bool fuse,
                                       int elem, int kq = 0, bool rx = true) {
    static std::mutex mu;
    static std::vector<PlanMemo> memo;
    static size_t next = 0;
    std::vector<long long> key = {n, nl, elem, kq, fuse ? 1 : 0, g_plan, g_plan_tmax, rx ? 1 : 0, g_lane3};
    key.reserve(key.size() + 3 * (size_t)nl);
    for (int l = 0; l < nl; ++l) {
        key.push_back(layers[l].q_lo);
        key.push_back(layers[l].q_hi);
        key.push_back(phase_active(layers[l]) ? 1 : 0);
    }
    {
        std::lock_guard<std::mutex> lock(mu);
        for (auto &m : memo)
            if (m.key == key) {
                groups = m.groups;
                return m.seq;
            }
    }
    auto seq = plan_x_search(n, nl, layers, groups, fuse, elem, kq, rx);
    std::lock_guard<std::mutex> lock(mu);
    PlanMemo m{std::move(key), seq, groups};
    if (memo.size() < 32) memo.push_back(std::move(m));
    else memo[next++ % 32] = std::move(m);
    return seq;
}

// pdep: the bits of x into the positions NOT set in mask (ascending)
static long long deposit(long long x, long long mask) {
    long long out = 0;
    for (int b = 0; b < 63 && x; ++b) {
        if ((mask >> b) & 1) continue;
        if (x & 1) out |= 1LL << b;
        x >>= 1;
    }
    return out;
}

// Mask class of a pass (template K of k_pass16) from its per-round masks.
static int mask_class(int seq, const unsigned char *maskA, int lane = 0) {
    const int nr = seq_rounds(seq);
    bool full = true;
    for (int r = 0; r < nr; ++r) full &= maskA[r] == 0xF;
    if (lane) return full && lane == 0x8 && (seq == SEQ_84 || seq == SEQ_848) ? K_LANE3 : -1;
    if (full) return K_FULL;
    if (seq == SEQ_84 || seq == SEQ_848) {
        for (int k = 1; k <= 3; ++k) {
            bool ok = true;
            for (int r = 0; r < nr; ++r)
                ok &= maskA[r] == (seq_pat(seq, r) == PAT4 ? ((0xF << (4 - k)) & 0xF) : 0xF);
            if (ok) return k;
        }
    }
    return K_RUNTIME;
}

// RX forms are compile-time for set A and for set B of heavy passes (set B of
// a light pass runs in the run-time form: it only occurs for gamma = 0 layers).
static int launch_pass(int mix, int cost, bool c64, const PassParams &P, const PassMaps &M, int seq, int ph, int ma,
                       int mb, int grid, cudaStream_t st) {
    const int k = mask_class(seq, P.maskA, P.lane);
    if (k < 0) {
        set_error("launch_pass: lane butterflies on tile bits 0x%x are not supported", P.lane);
        return FQ_ERR_UNSUPPORTED;
    }
    if (mix == MIX_SU2)
        return c64 ? launch_pass_su2_c64(P, M, cost, seq, ph, mb == 2 ? 2 : 3, k, grid, st)
                   : launch_pass_su2(P, M, cost, seq, ph, mb == 2 ? 2 : 3, k, grid, st);
    if (!seq_heavy(seq) && mb != 2) mb = 3;
    if (c64)
        return cost == FQ_COST_U16 ? launch_pass_c64_u16(P, M, seq, ph, ma, mb, k, grid, st)
                                   : launch_pass_c64_f64(P, M, seq, ph, ma, mb, k, grid, st);
    if (cost == FQ_COST_U16)
        return seq_heavy(seq) ? launch_pass_rx_u16_heavy(P, M, seq, ph, ma, mb, k, grid, st)
                              : launch_pass_rx_u16_light(P, M, seq, ph, ma, mb, k, grid, st);
    return seq_heavy(seq) ? launch_pass_rx_f64_heavy(P, M, seq, ph, ma, mb, k, grid, st)
                          : launch_pass_rx_f64_light(P, M, seq, ph, ma, mb, k, grid, st);
}

static int run_x_program(const fq_evolve_desc *d, cudaStream_t st, const ShardCtx *sh = nullptr) {
    const int nl = d->n;                      // qubits per shard (= n for one state)
    const int kq = sh ? sh->k : 0;
    const int nv = nl + kq;                   // qubits of the whole register
    const int K = 1 << kq;
    std::vector<Group> groups;
    const bool c64 = d->state_kind == FQ_STATE_C64;
    const long long elem = c64 ? (long long)sizeof(float2) : (long long)sizeof(double2);
    const int CB = d->cost_kind == FQ_COST_F64 ? 8 : 2;
    const int mix = (d->mixer == FQ_MIXER_X) ? MIX_RX : MIX_SU2;
    auto seq = plan_x(nv, d->n_layers, d->layers, groups, g_fuse != 0, (int)elem, kq, mix == MIX_RX);
    const long long n_tiles = 1LL << (nl - kTileBits);  // per shard
    int table_hi = 0;
    if (d->cost_kind == FQ_COST_U16 && d->cost_levels > 0 && g_phase_tables) {
        const int rows = ((d->cost_levels - 1) >> 6) + 1;
        table_hi = rows <= kMaxTableHi ? rows : 0;
    }
    bool init_pending = d->init != 0;
    // the shards this process works on: its own (rank), or all of them (in-process)
    std::vector<int> mine;
    if (!sh) mine.push_back(0);
    else if (sh->rank >= 0) mine.push_back(sh->rank);
    else for (int r = 0; r < K; ++r) mine.push_back(r);
    auto shard_psi = [&](int r) -> void * { return sh ? sh->shards[r] : d->psi; };
    auto shard_costs = [&](int r) -> const void * { return sh ? sh->costs[r] : d->costs; };
    auto shard_desc = [&](int r) {
        fq_evolve_desc e = *d;
        e.psi = shard_psi(r);
        e.costs = shard_costs(r);
        return e;
    };
    const long long size = 1LL << nl;
    const int sms = sm_count() > 0 ? sm_count() : 148;
    const int grid = (int)std::min<long long>(n_tiles, (long long)sms * 2);
    // expectation of several shards: per-shard sums in the top of the scratch, then one sum
    double *const shard_sums = d->scratch ? d->scratch + FQ_SCRATCH_DOUBLES - 16 : nullptr;
    auto expect_shards = [&]() -> int {
        if (mine.size() == 1) {
            fq_evolve_desc e = shard_desc(mine[0]);
            return state_expectation(&e, e.psi, size, st);
        }
        for (size_t i = 0; i < mine.size(); ++i) {
            fq_evolve_desc e = shard_desc(mine[i]);
            e.expectation_dev = shard_sums + i;
            if (int s = state_expectation(&e, e.psi, size, st)) return s;
        }
        k_sum_partials<<<1, 32, 0, st>>>(shard_sums, (int)mine.size(), d->expectation_dev);
        FQ_LAUNCHED("k_sum_partials");
        return FQ_OK;
    };
    auto init_shards = [&]() -> int {
        for (int r : mine) {
            fq_evolve_desc e = shard_desc(r);
            if (int s = state_init(&e, e.psi, size, st)) return s;
        }
        return FQ_OK;
    };
    auto barrier = [&]() -> int {
        if (!sh || sh->rank < 0) return FQ_OK;  // one stream orders everything
        return fq_peer_barrier(sh->flags, K, sh->rank, ++*sh->epoch, sh->err, st);
    };

    if (seq.empty()) {
        if (d->n_layers > 0 && kq > 0) {
            for (int l = 0; l < d->n_layers; ++l)
                if (d->layers[l].q_hi > d->layers[l].q_lo) {
                    set_error("fq_qaoa_evolve_sharded: no valid plan (the global qubits must share one group)");
                    return FQ_ERR_UNSUPPORTED;
                }
        }
        if (init_pending)
            if (int s = init_shards()) return s;
        if (d->expectation_dev) return expect_shards();
        return FQ_OK;
    }
    g_last_plan.clear();
    auto mark = [&](size_t k) -> int {  // event k: after pass k-1 (0 = program start)
        if (!g_time_passes) return FQ_OK;
        while (g_events.size() <= k) {
            cudaEvent_t e;
            FQ_CUDA(cudaEventCreate(&e));
            g_events.push_back(e);
        }
        FQ_CUDA(cudaEventRecord(g_events[k], st));
        return FQ_OK;
    };
    if (int s0 = mark(0)) return s0;
    // PassParams of pass si_ of the plan (everything but the per-launch buffer /
    // tile-range fields), its round program, phase mode and RX forms
    auto build = [&](size_t si_, bool init_, bool expect_, PassParams &P, int &sq, int &ph, int &ma, int &mb,
                     bool &two) {
        const PlannedPass &pp = seq[si_];
        const Group &g = groups[pp.group];
        const bool global = global_count(g, nv, kq) > 0;
        std::memset(&P, 0, sizeof P);
        P.cost_scale = d->cost_scale;
        P.cost_offset = d->cost_offset;
        P.init_amp = d->init_amp;
        P.table_hi = table_hi;
        // global tile bits (the top kq) carry no address: their tile_pos only
        // inserts zeros above every local bit (tile_base)
        for (int i = 0; i < kTileBits; ++i) P.tile_pos[i] = g.tile_pos[i] < nl ? g.tile_pos[i] : 62;
        P.gbits = global ? kq : 0;
        P.gshift = 8 - kq;
        P.gmask = K - 1;
        if (global)
            for (int r = 0; r < K; ++r) {
                P.sdelta[r] = static_cast<const char *>(sh->shards[r]) - static_cast<const char *>(sh->shards[0]);
                P.cdelta[r] = static_cast<const char *>(sh->costs[r]) - static_cast<const char *>(sh->costs[0]);
            }
        for (int pat = 0; pat < 3; ++pat) {
            const int f = pat_first_bit(pat);
            for (int i = 0; i < kRegs; ++i) {
                long long o = 0;
                int shard = 0;
                for (int j = 0; j < 4; ++j) {
                    if (!((i >> j) & 1)) continue;
                    const int q = g.tile_pos[f + j];
                    if (q < nl) o += 1LL << q;
                    else shard |= 1 << (q - nl);  // global bit (PAT8 registers only)
                }
                P.roff[pat][i] = o * elem + (global ? P.sdelta[shard] : 0);
                P.coff[pat][i] = o * CB + (global ? P.cdelta[shard] : 0);
            }
        }
        P.init = init_ ? 1 : 0;
        P.expect = expect_ ? 1 : 0;
        const int tmask = target_mask(g);
        two = pp.layerB >= 0;
        const bool lane_ok = mix == MIX_RX && !global;
        sq = pass_seq(g, pp, lane_ok);
        P.lane = lane_bits(g, lane_ok);
        for (int r = 0; r < seq_rounds(sq); ++r)
            P.maskA[r] = P.maskB[r] = (unsigned char)((tmask >> pat_first_bit(seq_pat(sq, r))) & 15);
        ph = 0;
        if (pp.phase_layer >= 0) {
            P.gamma = d->layers[pp.phase_layer].gamma;
            ph = pp.phase_at == 1 ? 1 : 2;
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
                    const double *c4 = d->su2 + ((size_t)layer * nv + g.tile_pos[i]) * 4;
                    C.a[i] = make_double2(c4[0], c4[1]);
                    C.b[i] = make_double2(c4[2], c4[3]);
                }
            }
        };
        fill(pp.layerA, P.A);
        if (two) fill(pp.layerB, P.B);
        P.final_scale = fscale;
        P.tile_mask = 0;
        for (int i = 0; i < kTileBits; ++i)
            if (g.tile_pos[i] < nl) P.tile_mask |= 1LL << g.tile_pos[i];
        P.step_dep = deposit(grid, P.tile_mask);
        P.reverse = g_zigzag ? (int)(si_ & 1) : 0;
        P.probe = g_probe;
        P.run_bits = 0;
        while (P.run_bits < kTileBits && g.tile_pos[P.run_bits] == P.run_bits) ++P.run_bits;
        P.pf_cost = (ph != 0 || P.expect) ? 1 : 0;
        // cost runs shorter than a 32-B sector: the rest of the sector is the neighbouring
        // tile's, read by another CTA moments later -- keep it in L2 (option cost_l2: -1 auto)
        P.cost_l2 = g_cost_l2 >= 0 ? g_cost_l2 : ((CB << P.run_bits) < 32 ? 1 : 0);
        ma = P.A.mode;
        mb = two ? P.B.mode : 2;
        if (P.expect && ph == 0 && !two && !seq_heavy(sq)) ph = 3;  // preload the expectation's costs
        // uint16 costs read after the first transpose (mid-layer phase, expectation): staged
        // through a shared cost tile with two 16-B loads per thread, if the tile's runs hold
        // >= 8 entries and the extra 8.5 KB keeps two CTAs per SM
        P.cost_stage = 0;
        if (g_cost_stage && d->cost_kind == FQ_COST_U16 && !global && P.run_bits >= 3 && (ph == 2 || ph == 3)) {
            const size_t need = (size_t)elem * kTilePadded + (size_t)(kTableLo + table_hi) * 128 +
                                kCostTileSlots * sizeof(unsigned short);
            if (need <= 113 * 1024) {
                P.cost_stage = 1;
                P.c11 = 2LL << g.tile_pos[kTileBits - 1];
            }
        }
    };
    // Passes si and si+1 as one L2-resident slab sweep (sweep.cuh) when the
    // pair has an instantiation and its slab fits the L2 budget; `swept` tells.
    bool sweep_err_reset = false;
    auto sweep_pair = [&](size_t si, bool /*last*/, bool &swept) -> int {
        swept = false;
        const bool last2 = si + 2 == seq.size();
        const Group &g1 = groups[seq[si].group], &g2 = groups[seq[si + 1].group];
        if (global_count(g1, nv, kq) || global_count(g2, nv, kq)) return FQ_OK;
        long long U = 0;  // slab bits
        for (int i = 0; i < kTileBits; ++i) U |= (1LL << g1.tile_pos[i]) | (1LL << g2.tile_pos[i]);
        const int ub = __builtin_popcountll(U);
        const int log2_tiles = ub - kTileBits;
        const int team = std::max(1, g_sweep_team);
        if ((1 << log2_tiles) < team || (elem << ub) > (1LL << g_sweep_slab_log2)) return FQ_OK;
        const long long n_slabs = 1LL << (nl - ub);
        const int n_teams = (int)std::min<long long>({(long long)(2 * sms) / team, n_slabs, 16LL});
        if (n_teams < 1) return FQ_OK;
        PassParams P1, P2;
        int sq1, ph1, ma1, mb1, sq2, ph2, ma2, mb2;
        bool two1, two2;
        build(si, init_pending, false, P1, sq1, ph1, ma1, mb1, two1);
        build(si + 1, false, last2 && d->expectation_dev, P2, sq2, ph2, ma2, mb2, two2);
        if ((ph1 == 1 || ph1 == 2) && (ph2 == 1 || ph2 == 2)) return FQ_OK;
        if (P1.lane || P2.lane) return FQ_OK;  // no sweep instantiation with lane butterflies
        SweepKind kind{sq1, ph1, ma1, mb1, mask_class(sq1, P1.maskA), sq2, ph2, ma2, mb2, mask_class(sq2, P2.maskA)};
        if (!sweep_supported(mix, d->cost_kind, c64, kind)) return FQ_OK;
        SweepParams *S = new SweepParams;
        std::memset(S, 0, sizeof *S);
        S->P1 = P1;
        S->P2 = P2;
        for (PassParams *Q : {&S->P1, &S->P2}) {
            Q->psi = d->psi;
            Q->costs = d->costs;
            Q->partials = d->scratch;
            Q->pf_dist = 0;
        }
        // tile-number bits of each sub-pass: slab-inner bits (U minus its tile bits), then the slab index
        auto fill_dep = [&](const Group &g, unsigned char *dep) {
            long long tb = 0;
            for (int i = 0; i < kTileBits; ++i) tb |= 1LL << g.tile_pos[i];
            int c = 0;
            for (int b = 0; b < nl; ++b)
                if (((U >> b) & 1) && !((tb >> b) & 1)) dep[c++] = (unsigned char)b;
            for (int b = 0; b < nl; ++b)
                if (!((U >> b) & 1)) dep[c++] = (unsigned char)b;
        };
        fill_dep(g1, S->dep1);
        fill_dep(g2, S->dep2);
        S->n_dep = nl - kTileBits;
        S->log2_tiles = log2_tiles;
        S->n_slabs = n_slabs;
        S->team_size = team;
        S->n_teams = n_teams;
        // sub-pass 2's cost slice, per slab: runs of the slab's low contiguous bits (<= 2^14 levels)
        const bool costs2 = ph2 != 0 || S->P2.expect;
        int rb = 0;
        while (rb < nl && ((U >> rb) & 1)) ++rb;
        rb = std::min(rb, 14);
        if (costs2 && d->cost_kind == FQ_COST_U16 && rb >= 3) {
            S->cost_run_log2 = rb;
            S->log2_cost_runs = ub - rb;
            int c = 0;
            for (int b = rb; b < nl; ++b)
                if ((U >> b) & 1) S->cdep[c++] = (unsigned char)b;
            for (int b = 0; b < nl; ++b)
                if (!((U >> b) & 1)) S->cdep[c++] = (unsigned char)b;
        }
        S->pf1_bytes = (run_bits_of(g1) == kTileBits && !P1.init) ? (int)(elem << kTileBits) : 0;
        unsigned *ctr = reinterpret_cast<unsigned *>(d->scratch + kSweepCtrOffset);
        S->counters = ctr;
        S->err = reinterpret_cast<int *>(d->scratch + kSweepErrOffset);
        if (!sweep_err_reset) {
            cudaError_t e = cudaMemsetAsync(S->err, 0, sizeof(int), st);
            if (e != cudaSuccess) { delete S; return cuda_status(e, "cudaMemsetAsync(sweep err)"); }
            sweep_err_reset = true;
        }
        cudaError_t e = cudaMemsetAsync(ctr, 0, 16 * 32 * sizeof(unsigned), st);
        if (e != cudaSuccess) { delete S; return cuda_status(e, "cudaMemsetAsync(sweep counters)"); }
        const int s = launch_sweep(mix, d->cost_kind, c64, kind, *S, st);
        delete S;
        if (s) return s;
        init_pending = false;
        swept = true;
        g_last_plan.push_back({100 + 10 * sq1 + sq2, ph1 ? ph1 : ph2, (int)g2.targets.size(), P1.init, P2.expect});
        if (P2.expect) {
            k_sum_partials_checked<<<1, 32, 0, st>>>(d->scratch, n_teams * team, S_err_ptr(d), d->expectation_dev);
            FQ_LAUNCHED("k_sum_partials_checked");
        }
        ++g_sweeps_launched;
        return FQ_OK;
    };
    for (size_t si = 0; si < seq.size(); ++si) {
        const PlannedPass &pp = seq[si];
        const bool last = (si + 1 == seq.size());
        if (pp.group < 0) {  // standalone phase, shard-local
            g_last_plan.push_back({-1, 1, 0, init_pending ? 1 : 0, (last && d->expectation_dev) ? 1 : 0});
            if (init_pending) {
                if (int s = init_shards()) return s;
                init_pending = false;
            }
            const fq_layer &L = d->layers[pp.phase_layer];
            for (int r : mine) {
                fq_evolve_desc e = shard_desc(r);
                if (c64) launch_phase(static_cast<float2 *>(e.psi), &e, size, L.gamma, st);
                else launch_phase(static_cast<double2 *>(e.psi), &e, size, L.gamma, st);
                FQ_LAUNCHED("k_phase");
            }
            if (last && d->expectation_dev)
                if (int s = expect_shards()) return s;
            if (int s = mark(g_last_plan.size())) return s;
            continue;
        }
        if (g_sweep && !sh && si + 1 < seq.size() && seq[si + 1].group >= 0) {
            bool swept = false;
            if (int s = sweep_pair(si, last, swept)) return s;
            if (swept) {
                ++si;  // the pair ran as one sweep
                if (int s2 = mark(g_last_plan.size())) return s2;
                continue;
            }
        }
        const Group &g = groups[pp.group];
        const int gq = global_count(g, nv, kq);
        if (gq != 0 && gq != kq) {
            set_error("fq_qaoa_evolve_sharded: a group holds %d of the %d global qubits", gq, kq);
            return FQ_ERR_UNSUPPORTED;
        }
        const bool global = gq > 0;
        PassParams P;
        int sq, ph, ma, mb;
        bool two;
        build(si, init_pending, last && d->expectation_dev, P, sq, ph, ma, mb, two);
        init_pending = false;
        int launches = 0;
        if (global) {
            // one pass over every shard: rank r takes its 1/K of the tiles (in-process: all)
            if (int s = barrier()) return s;
            const long long T = 1LL << (nv - kTileBits);
            const bool all = sh->rank < 0;
            P.psi = sh->shards[0];
            P.costs = sh->costs[0];
            P.tile0 = all ? 0 : (T / K) * sh->rank;
            P.n_tiles = all ? T : T / K;
            P.partials = d->scratch;
            P.pf_dist = 0;  // the tile spans several allocations: no single tensor map
            PassMaps M;
            std::memset(&M, 0, sizeof M);
            const int ggrid = (int)std::min<long long>(P.n_tiles, (long long)sms * 2);
            P.step_dep = deposit(ggrid, P.tile_mask);
            int k = mask_class(sq, P.maskA, P.lane);
            int mbv = (mix == MIX_RX && !seq_heavy(sq) && mb != 2) ? 3 : mb;
            if (mix == MIX_SU2) mbv = mb == 2 ? 2 : 3;
            const int s = c64 ? launch_pass_global_c64(d->cost_kind, P, M, sq, ph, ma, mbv, k, ggrid, st)
                          : d->cost_kind == FQ_COST_U16
                              ? launch_pass_global_u16(mix, P, M, sq, ph, mix == MIX_SU2 ? 0 : ma, mbv, k, ggrid, st)
                              : launch_pass_global_f64(mix, P, M, sq, ph, mix == MIX_SU2 ? 0 : ma, mbv, k, ggrid, st);
            if (s) return s;
            launches = ggrid;
            if (int s2 = barrier()) return s2;
        } else {
            P.n_tiles = n_tiles;
            P.tile0 = 0;
            // the tensor prefetch pays for long runs only: with short runs its many
            // small requests compete with the demand loads (measured, n = 28..34)
            const int pf = g_prefetch >= 0 ? g_prefetch : ((elem << run_bits_of(g)) >= 256 ? 1 : 0);
            for (size_t mi = 0; mi < mine.size(); ++mi) {
                const int r = mine[mi];
                P.psi = shard_psi(r);
                P.costs = shard_costs(r);
                P.partials = d->scratch + launches;
                P.pf_dist = pf;
                P.sm_rank = P.cm_rank = 0;
                PassMaps M;
                std::memset(&M, 0, sizeof M);
                if (P.pf_dist > 0) {
                    P.sm_rank = c64 ? cached_tile_map(&M.state, P.psi, nl, g.tile_pos, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                                                      2, P.sm_shift, P.sm_bits)
                                    : cached_tile_map(&M.state, P.psi, nl, g.tile_pos, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8,
                                                      2, P.sm_shift, P.sm_bits);
                    if (P.pf_cost)
                        P.cm_rank = d->cost_kind == FQ_COST_F64
                                        ? cached_tile_map(&M.cost, P.costs, nl, g.tile_pos,
                                                         CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, 1, P.cm_shift, P.cm_bits)
                                        : cached_tile_map(&M.cost, P.costs, nl, g.tile_pos,
                                                         CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, 1, P.cm_shift, P.cm_bits);
                    if (P.sm_rank == 0 && P.cm_rank == 0) P.pf_dist = 0;
                }
                const int s = launch_pass(mix, d->cost_kind, c64, P, M, sq, ph, ma, mb, grid, st);
                if (s) return s;
                launches += grid;
            }
        }
        g_last_plan.push_back({sq, ph, (int)g.targets.size(), P.init, P.expect});
        if (P.expect) {
            k_sum_partials<<<1, 32, 0, st>>>(d->scratch, launches, d->expectation_dev);
            FQ_LAUNCHED("k_sum_partials");
        }
        if (int s2 = mark(g_last_plan.size())) return s2;
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

int run_xy_tiled(const fq_evolve_desc *d, const std::vector<std::pair<int, int>> &gates, cudaStream_t st,
                 int *passes_out, const ShardCtx *sh = nullptr);
int plan_xy_passes(int n, int mixer, const std::vector<std::pair<int, int>> &gates, int *rounds);
static int g_xy_tiled = 1;   // tiled XY passes (0: one pair kernel per gate, the reference's structure)
extern int g_xy_min_run;     // xy.cu
extern int g_xy_row_cap;     // xy.cu
extern int g_xy_pad;         // xy.cu
extern int g_xy_prefetch;    // xy.cu

static int run_xy_program(const fq_evolve_desc *d, cudaStream_t st) {
    const int n = d->n;
    const long long size = 1LL << n;
    double2 *psi = static_cast<double2 *>(d->psi);
    if (g_xy_tiled) {
        std::vector<std::pair<int, int>> gates;
        xy_gates(n, d->mixer, gates);
        return run_xy_tiled(d, gates, st, nullptr);
    }
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

static int g_res16 = 2;  // n <= 12, X / custom mixers: 0 one sweep per qubit (k_resident), 1 register rounds
                         // of 16 amplitudes (k_resident16), 2 of 8 amplitudes x 512 threads (k_resident8)

// uint16 levels -> rows of the high phase table (0: too many levels, sincos per amplitude)
static int table_rows(int cost_levels) {
    if (cost_levels <= 0) return 0;
    const int rows = ((cost_levels - 1) >> 6) + 1;
    return rows <= kMaxTableHi ? rows : 0;
}

template <int COST>
static int launch_resident(const ResParams &P, int batch, const double *su2_dev, cudaStream_t st) {
    if (g_res16 == 2 && (P.mixer == FQ_MIXER_X || P.mixer == FQ_MIXER_CUSTOM)) {
        static bool configured8 = false;
        if (!configured8) {
            cudaFuncSetAttribute(k_resident8<COST, MIX_RX>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRes8Smem);
            cudaFuncSetAttribute(k_resident8<COST, MIX_SU2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRes8Smem);
            configured8 = true;
        }
        const int th = COST == FQ_COST_U16 ? P.table_hi : 0;
        const size_t smem8 = (size_t)(kRes8Padded + (P.all_tables ? P.p : 1) * (kTableLo + th) * 8) * sizeof(double2);
        if (P.mixer == FQ_MIXER_X) k_resident8<COST, MIX_RX><<<batch, kRes8Threads, smem8, st>>>(P, su2_dev);
        else k_resident8<COST, MIX_SU2><<<batch, kRes8Threads, smem8, st>>>(P, su2_dev);
        FQ_LAUNCHED("k_resident8");
        return FQ_OK;
    }
    if (g_res16 == 1 && (P.mixer == FQ_MIXER_X || P.mixer == FQ_MIXER_CUSTOM)) {
        static bool configured16 = false;
        if (!configured16) {
            cudaFuncSetAttribute(k_resident16<COST, MIX_RX>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRes16Smem);
            cudaFuncSetAttribute(k_resident16<COST, MIX_SU2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRes16Smem);
            configured16 = true;
        }
        const int th = COST == FQ_COST_U16 ? P.table_hi : 0;
        const size_t smem16 = (size_t)(kTilePadded + (kTableLo + th) * 8) * sizeof(double2);
        if (P.mixer == FQ_MIXER_X) k_resident16<COST, MIX_RX><<<batch, kThreads, smem16, st>>>(P, su2_dev);
        else k_resident16<COST, MIX_SU2><<<batch, kThreads, smem16, st>>>(P, su2_dev);
        FQ_LAUNCHED("k_resident16");
        return FQ_OK;
    }
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
    // custom-mixer coefficients (4 doubles per layer and qubit) travel through the
    // scratch buffer: a chunk carries at most FQ_SCRATCH_DOUBLES / (4 n) layers
    const int chunk = d->mixer == FQ_MIXER_CUSTOM ? std::min(kResMaxLayers, FQ_SCRATCH_DOUBLES / (4 * n))
                                                  : kResMaxLayers;
    for (int l0 = 0; l0 < std::max(1, d->n_layers); l0 += chunk) {
        const int cnt = std::min(chunk, d->n_layers - l0);
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
        const bool last = (l0 + chunk >= d->n_layers);
        P->exp_out = last ? d->expectation_dev : nullptr;
        P->table_hi = d->cost_kind == FQ_COST_U16 && g_phase_tables ? table_rows(d->cost_levels) : 0;
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

// One objective evaluation of a small state (n <= 12, X mixer, from |+>) as a
// captured CUDA graph: H2D copy of the angles from a pinned host array into a
// device buffer the resident kernel reads (ResParams::ang), the kernel, D2H
// copy of the objective into a pinned host double.  Replaying it needs one
// graph launch per evaluation instead of building and launching the program.
struct ObjGraph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaStream_t st = nullptr;
    cudaEvent_t ev = nullptr;
    volatile unsigned long long *out = nullptr;  // the pinned objective slot (bit pattern)
};

// Written into the objective slot before each replay; the kernel's 8-byte store of
// the objective replaces it (a NaN payload no arithmetic produces).
constexpr unsigned long long kObjPending = 0x7ff4dead00c0ffeeULL;

static void obj_graph_free(ObjGraph *g) {
    if (!g) return;
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    if (g->ev) cudaEventDestroy(g->ev);
    if (g->st) cudaStreamDestroy(g->st);
    delete g;
}

}  // namespace fq

using namespace fq;

extern "C" {

int fq_objective_graph_create(const fq_evolve_desc *d, const double *ang_host, double *out_host, void **handle) {
    FQ_CHECK_ARG(d && ang_host && out_host && handle, "fq_objective_graph_create: null argument");
    FQ_CHECK_ARG(d->n >= 1 && d->n <= kTileBits && d->mixer == FQ_MIXER_X && d->init && d->expectation_dev &&
                     d->state_kind == FQ_STATE_C128 && d->n_layers >= 1 && d->n_layers <= kResGraphMaxLayers &&
                     d->layers && d->psi && d->costs,
                 "fq_objective_graph_create: n <= %d complex128, X mixer from |+>, 1..%d layers, with an expectation",
                 kTileBits, kResGraphMaxLayers);
    FQ_CHECK_ARG(d->cost_kind == FQ_COST_F64 || d->cost_kind == FQ_COST_U16, "fq_objective_graph_create: bad cost kind");
    *handle = nullptr;
    ObjGraph *g = new ObjGraph;
    const int p = d->n_layers;
    auto fail = [&](cudaError_t e, const char *what) {
        const int s = cuda_status(e, what);
        obj_graph_free(g);
        return s;
    };
    // the kernel reads the angles from, and writes the objective to, the pinned host
    // buffers themselves (their device-side aliases): the graph is the kernel alone
    double *ang_dev = nullptr, *out_dev = nullptr;
    cudaError_t e = cudaHostGetDevicePointer(reinterpret_cast<void **>(&ang_dev), const_cast<double *>(ang_host), 0);
    if (e != cudaSuccess) return fail(e, "cudaHostGetDevicePointer(angles): ang_host must be pinned");
    if ((e = cudaHostGetDevicePointer(reinterpret_cast<void **>(&out_dev), out_host, 0)) != cudaSuccess)
        return fail(e, "cudaHostGetDevicePointer(objective): out_host must be pinned");
    if ((e = cudaStreamCreateWithFlags(&g->st, cudaStreamNonBlocking)) != cudaSuccess) return fail(e, "cudaStreamCreate");
    if ((e = cudaEventCreateWithFlags(&g->ev, cudaEventDisableTiming)) != cudaSuccess) return fail(e, "cudaEventCreate");
    g->out = reinterpret_cast<volatile unsigned long long *>(out_host);
    ResParams *P = new ResParams;
    std::memset(P, 0, sizeof *P);
    P->n = d->n;
    P->p = p;
    P->mixer = d->mixer;
    P->costs = d->costs;
    P->cost_scale = d->cost_scale;
    P->cost_offset = d->cost_offset;
    P->init = 1;
    P->init_amp = d->init_amp;
    P->psi_out = nullptr;  // the objective only: the final state is not written back
    P->exp_out = out_dev;
    P->table_hi = d->cost_kind == FQ_COST_U16 && g_phase_tables ? table_rows(d->cost_levels) : 0;
    P->ang = ang_dev;
    // every layer's uint16 phase tables at kernel start, when they fit the shared memory
    P->all_tables = (d->cost_kind == FQ_COST_U16 && P->table_hi > 0 && g_res16 == 2 &&
                     (size_t)(kRes8Padded + (size_t)p * (kTableLo + P->table_hi) * 8) * sizeof(double2) <=
                         (size_t)kRes8Smem) ? 1 : 0;
    for (int i = 0; i < p; ++i) {
        P->phase_on[i] = (unsigned char)(d->layers[i].apply_phase != 0);
        P->qlo[i] = (unsigned char)std::max(0, std::min(d->n, d->layers[i].q_lo));
        P->qhi[i] = (unsigned char)std::max((int)P->qlo[i], std::min(d->n, d->layers[i].q_hi));
    }
    auto enqueue = [&]() -> int {
        return d->cost_kind == FQ_COST_U16 ? launch_resident<FQ_COST_U16>(*P, 1, nullptr, g->st)
                                           : launch_resident<FQ_COST_F64>(*P, 1, nullptr, g->st);
    };
    // once eagerly (kernel attributes, module loading; after the device's pending work,
    // e.g. the diagonal's precompute on the caller's stream), then captured
    int s = FQ_OK;
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) s = cuda_status(e, "cudaDeviceSynchronize");
    if (!s) s = enqueue();
    if (!s && (e = cudaStreamSynchronize(g->st)) != cudaSuccess) s = cuda_status(e, "cudaStreamSynchronize");
    if (!s && (e = cudaStreamBeginCapture(g->st, cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
        s = cuda_status(e, "cudaStreamBeginCapture");
    if (!s) {
        const int s2 = enqueue();
        e = cudaStreamEndCapture(g->st, &g->graph);
        s = s2 ? s2 : (e != cudaSuccess ? cuda_status(e, "cudaStreamEndCapture") : FQ_OK);
    }
    if (!s && (e = cudaGraphInstantiate(&g->exec, g->graph, 0)) != cudaSuccess) s = cuda_status(e, "cudaGraphInstantiate");
    delete P;
    if (s) {
        obj_graph_free(g);
        return s;
    }
    *handle = g;
    return FQ_OK;
}

int fq_objective_graph_run(void *handle, void *stream) {
    FQ_CHECK_ARG(handle, "fq_objective_graph_run: null handle");
    ObjGraph *g = static_cast<ObjGraph *>(handle);
    // on the caller's stream (ordered behind its work); completion is detected by
    // spinning on the pinned objective slot until the kernel's 8-byte store replaces
    // the pending pattern (a stream synchronisation's wake-up costs several
    // microseconds); after 2 s of spinning, the stream is synchronised to surface
    // an error instead
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    *g->out = kObjPending;
    FQ_CUDA(cudaGraphLaunch(g->exec, st));
    const auto t0 = std::chrono::steady_clock::now();
    for (unsigned spins = 0; *g->out == kObjPending; ++spins) {
        if ((spins & 1023) == 1023 && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(2)) {
            FQ_CUDA(cudaStreamSynchronize(st));
            if (*g->out == kObjPending) {
                set_error("fq_objective_graph_run: the evaluation did not write its objective");
                return FQ_ERR_UNSUPPORTED;
            }
            break;
        }
    }
    return FQ_OK;
}

int fq_objective_graph_destroy(void *handle) {
    obj_graph_free(static_cast<ObjGraph *>(handle));
    return FQ_OK;
}

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
    FQ_CHECK_ARG(d->state_kind == FQ_STATE_C128 || d->state_kind == FQ_STATE_C64, "fq_qaoa_evolve: bad state kind");
    const bool is_xy = d->mixer == FQ_MIXER_XY_RING || d->mixer == FQ_MIXER_XY_COMPLETE;
    if (d->state_kind == FQ_STATE_C64 && (d->n <= kTileBits || (is_xy && !g_xy_tiled))) {
        set_error("fq_qaoa_evolve: complex64 states run the tiled passes, n > %d qubits (got n=%d, mixer=%d)",
                  kTileBits, d->n, d->mixer);
        return FQ_ERR_UNSUPPORTED;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (d->n <= kTileBits) {
        FQ_CHECK_ARG(d->mixer != FQ_MIXER_CUSTOM || d->scratch, "fq_qaoa_evolve: custom mixer needs scratch");
        return run_resident_program(d, st);
    }
    if (d->mixer == FQ_MIXER_XY_RING || d->mixer == FQ_MIXER_XY_COMPLETE) return run_xy_program(d, st);
    return run_x_program(d, st);
}

int fq_qaoa_objective(const fq_evolve_desc *d, double *out_host, void *stream) {
    FQ_CHECK_ARG(d && out_host && d->expectation_dev, "fq_qaoa_objective: needs expectation_dev and out_host");
    if (int s = fq_qaoa_evolve(d, stream)) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    FQ_CUDA(cudaMemcpyAsync(out_host, d->expectation_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
    FQ_CUDA(cudaStreamSynchronize(st));
    return FQ_OK;
}

int fq_qaoa_evolve_sharded(const fq_evolve_desc *d, const fq_shard_desc *s, void *stream) {
    FQ_CHECK_ARG(d && s, "fq_qaoa_evolve_sharded: null descriptor");
    FQ_CHECK_ARG(s->k >= 1 && s->k <= 3, "fq_qaoa_evolve_sharded: k=%d must be in [1, 3]", s->k);
    const int K = 1 << s->k;
    FQ_CHECK_ARG(s->rank >= -1 && s->rank < K, "fq_qaoa_evolve_sharded: bad rank %d", s->rank);
    FQ_CHECK_ARG(d->n >= kTileBits && d->n + s->k <= 40, "fq_qaoa_evolve_sharded: n_local=%d must be >= %d", d->n,
                 kTileBits);
    FQ_CHECK_ARG(d->state_kind == FQ_STATE_C128 || (d->state_kind == FQ_STATE_C64 && d->mixer != FQ_MIXER_CUSTOM),
                 "fq_qaoa_evolve_sharded: complex128 states, or complex64 under the X / XY mixers");
    FQ_CHECK_ARG(d->mixer >= FQ_MIXER_X && d->mixer <= FQ_MIXER_CUSTOM, "fq_qaoa_evolve_sharded: bad mixer");
    FQ_CHECK_ARG(d->mixer != FQ_MIXER_CUSTOM || d->su2, "fq_qaoa_evolve_sharded: custom mixer needs su2 table");
    FQ_CHECK_ARG(d->n_layers >= 0 && (d->n_layers == 0 || d->layers), "fq_qaoa_evolve_sharded: bad layers");
    FQ_CHECK_ARG(d->cost_kind == FQ_COST_F64 || d->cost_kind == FQ_COST_U16, "fq_qaoa_evolve_sharded: bad cost kind");
    FQ_CHECK_ARG(d->scratch, "fq_qaoa_evolve_sharded: needs scratch");
    FQ_CHECK_ARG(s->shards && s->costs, "fq_qaoa_evolve_sharded: null shard tables");
    for (int r = 0; r < K; ++r)
        FQ_CHECK_ARG(s->shards[r] && s->costs[r], "fq_qaoa_evolve_sharded: null shard %d", r);
    FQ_CHECK_ARG(s->rank < 0 || (s->flags && s->epoch && s->barrier_err),
                 "fq_qaoa_evolve_sharded: a rank needs the peer barrier (flags, epoch, error word)");
    ShardCtx ctx;
    ctx.k = s->k;
    ctx.K = K;
    ctx.rank = s->rank;
    ctx.shards = s->shards;
    ctx.costs = s->costs;
    ctx.flags = s->flags;
    ctx.epoch = s->epoch;
    ctx.err = s->barrier_err;
    if (d->mixer == FQ_MIXER_XY_RING || d->mixer == FQ_MIXER_XY_COMPLETE) {
        std::vector<std::pair<int, int>> gates;
        xy_gates(d->n + s->k, d->mixer, gates);
        return run_xy_tiled(d, gates, static_cast<cudaStream_t>(stream), nullptr, &ctx);
    }
    return run_x_program(d, static_cast<cudaStream_t>(stream), &ctx);
}

int fq_plan_sharded_passes(int n_local, int k, int n_layers, const fq_layer *layers, int *global_passes) {
    if (global_passes) *global_passes = 0;
    if (n_local < kTileBits || k < 1 || k > 3) return -1;
    std::vector<Group> groups;
    const int nv = n_local + k;
    auto seq = plan_x(nv, n_layers, layers, groups, g_fuse != 0, 16, k);
    int gp = 0;
    for (auto &pp : seq)
        if (pp.group >= 0 && global_count(groups[pp.group], nv, k) > 0) ++gp;
    if (global_passes) *global_passes = gp;
    return (int)seq.size();
}

int fq_set_option(const char *name, int value) {
    if (!name) return FQ_ERR_ARG;
    struct { const char *name; int *slot; int lo, hi; } opts[] = {
        {"prefetch", &g_prefetch, -1, 8},    // L2 prefetch distance of the pass kernel (grid strides)
        {"fuse", &g_fuse, 0, 1},            // fuse the passes at layer boundaries
        {"phase_tables", &g_phase_tables, 0, 1},  // uint16 phase via smem tables (else sincos)
        {"plan", &g_plan, -1, 1},           // group plan: -1 cost model, 0 legacy, 1 small fusion groups
        {"plan_tmax", &g_plan_tmax, 0, 12},  // force the high-group chunk size (0: cost model)
        {"cost_l2", &g_cost_l2, -1, 1},
        {"cost_stage", &g_cost_stage, 0, 1},  // uint16 costs through a shared cost tile (16-B loads)     // cost loads at normal L2 priority (-1: runs < 32 B)
        {"lane3", &g_lane3, 0, 1},          // 9-target high groups: tile bit 3 as lane butterflies (K_LANE3)
        {"res16", &g_res16, 0, 2},          // n <= 12 X / custom: resident kernel variant (2: k_resident8)
        {"sweep", &g_sweep, 0, 1},          // L2-resident slab sweeps of pass pairs
        {"sweep_team", &g_sweep_team, 1, 256},  // CTAs per sweep team
        {"sweep_slab_log2", &g_sweep_slab_log2, 16, 30},  // largest sweep slab, log2 bytes
        {"time_passes", &g_time_passes, 0, 1},  // CUDA events around every pass (fq_last_passes)
        {"xy_tiled", &g_xy_tiled, 0, 1},    // tiled XY passes (0: one kernel per gate)
        {"zigzag", &g_zigzag, 0, 1},        // alternate tile walk direction pass to pass
        {"xy_min_run", &g_xy_min_run, 0, 8},  // XY pass tiles: min contiguous run, log2 amplitudes (0 = auto)
        {"xy_row_cap", &g_xy_row_cap, 0, 64},  // XY pass cut: new qubits per leading qubit (0 = auto)
        {"xy_pad", &g_xy_pad, 0, 1},        // XY passes: gate-free load / store rounds for coalescing
        {"xy_prefetch", &g_xy_prefetch, -1, 1},  // XY passes: L2 tensor prefetch (-1: runs >= 256 B)
        {"probe", &g_probe, 0, 7},          // development: isolate phase costs (results invalid when != 0)
    };
    for (auto &o : opts) {
        if (std::strcmp(name, o.name) == 0) {
            if (value < o.lo || value > o.hi) {
                set_error("fq_set_option: %s=%d out of range [%d, %d]", name, value, o.lo, o.hi);
                return FQ_ERR_ARG;
            }
            *o.slot = value;
            return FQ_OK;
        }
    }
    set_error("fq_set_option: unknown option %s", name);
    return FQ_ERR_ARG;
}

int fq_plan_x_passes(int n, int n_layers, const fq_layer *layers, int state_kind) {
    if (n <= kTileBits) return n_layers > 0 ? 1 : 0;
    std::vector<Group> groups;
    return (int)plan_x(n, n_layers, layers, groups, g_fuse != 0, state_kind == FQ_STATE_C64 ? 8 : 16).size();
}

int fq_plan_x_describe(int n, int n_layers, const fq_layer *layers, int state_kind, int k, char *buf, int len) {
    if (!buf || len <= 0) return -1;
    buf[0] = 0;
    if (n <= kTileBits + k || k < 0 || k > 3) return -1;
    std::vector<Group> groups;
    const auto seq = plan_x(n, n_layers, layers, groups, g_fuse != 0, state_kind == FQ_STATE_C64 ? 8 : 16, k);
    std::string out;
    char tmp[64];
    for (size_t gi = 0; gi < groups.size(); ++gi) {
        out += gi ? ";" : "groups=";
        for (size_t i = 0; i < groups[gi].targets.size(); ++i) {
            std::snprintf(tmp, sizeof tmp, "%s%d", i ? "," : "", groups[gi].targets[i]);
            out += tmp;
        }
        std::snprintf(tmp, sizeof tmp, "/run%d", run_bits_of(groups[gi]));
        out += tmp;
    }
    out += " passes=";
    for (size_t i = 0; i < seq.size(); ++i) {
        const PlannedPass &pp = seq[i];
        if (pp.group < 0) std::snprintf(tmp, sizeof tmp, "%sP", i ? "," : "");
        else std::snprintf(tmp, sizeof tmp, "%s%d%s", i ? "," : "", pp.group,
                           pp.layerB >= 0 ? (pp.phase_at == 2 ? "f" : "d") : "");
        out += tmp;
    }
    std::snprintf(buf, (size_t)len, "%s", out.c_str());
    return (int)seq.size();
}

int fq_plan_xy_passes(int n, int mixer, int *rounds) {
    if (rounds) *rounds = 0;
    if (n <= kTileBits) return 1;
    if (mixer != FQ_MIXER_XY_RING && mixer != FQ_MIXER_XY_COMPLETE) return -1;
    std::vector<std::pair<int, int>> gates;
    xy_gates(n, mixer, gates);
    return plan_xy_passes(n, mixer, gates, rounds);
}

int fq_last_passes(int *info, float *ms, int max) {
    const int n = (int)g_last_plan.size();
    const bool timed = g_time_passes && g_events.size() > (size_t)n && n > 0;
    if (timed) {
        cudaError_t e = cudaEventSynchronize(g_events[n]);
        if (e != cudaSuccess) return -cuda_status(e, "cudaEventSynchronize");
    }
    for (int i = 0; i < n && i < max; ++i) {
        const PassRecord &r = g_last_plan[i];
        if (info) {
            int *o = info + 5 * i;
            o[0] = r.seq; o[1] = r.ph; o[2] = r.targets; o[3] = r.init; o[4] = r.expect;
        }
        if (ms) {
            ms[i] = -1.0f;
            if (timed) cudaEventElapsedTime(&ms[i], g_events[i], g_events[i + 1]);
        }
    }
    return n;
}

int fq_qaoa_evolve_batched(int n, int mixer, const void *costs, int cost_kind, double scale, double offset, int p,
                           int batch, const double *gammas, const double *betas, const void *psi_init, void *psi_out,
                           double *out_dev, void *stream) {
    return fq_qaoa_evolve_batched_levels(n, mixer, costs, cost_kind, scale, offset, 0, p, batch, gammas, betas,
                                         psi_init, psi_out, out_dev, stream);
}

int fq_qaoa_evolve_batched_levels(int n, int mixer, const void *costs, int cost_kind, double scale, double offset,
                                  int cost_levels, int p, int batch, const double *gammas, const double *betas,
                                  const void *psi_init, void *psi_out, double *out_dev, void *stream) {
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
    P->table_hi = cost_kind == FQ_COST_U16 && g_phase_tables ? table_rows(cost_levels) : 0;
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
