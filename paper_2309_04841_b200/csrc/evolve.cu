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
    unsigned char maskA[5], maskB[5];
    CoefSet A, B;
};

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

__device__ __forceinline__ int swz(int e) { return e ^ (((e >> 3) ^ (e >> 6) ^ (e >> 9)) & 7); }

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
#pragma unroll
    for (int i = 0; i < kRegs; ++i) sm[swz(tidx<PAT>(tid, i))] = v[i];
}
template <int PAT>
__device__ __forceinline__ void transpose_in(const double2 *sm, double2 (&v)[kRegs], int tid) {
#pragma unroll
    for (int i = 0; i < kRegs; ++i) v[i] = sm[swz(tidx<PAT>(tid, i))];
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
template <int COST>
__device__ __forceinline__ double2 phase_factor(const void *costs, long long k, double gamma, const double2 *tlo,
                                                const double2 *thi) {
    if (COST == FQ_COST_F64) {
        double s, c;
        sincos(gamma * static_cast<const double *>(costs)[k], &s, &c);
        return make_double2(c, -s);
    } else {
        const unsigned v = static_cast<const uint16_t *>(costs)[k];
        return cmul(thi[v >> 8], tlo[v & 255]);
    }
}

template <int COST>
__device__ __forceinline__ double cost_value(const void *costs, long long k, double scale, double offset) {
    if (COST == FQ_COST_F64) return static_cast<const double *>(costs)[k];
    return decode_u16(static_cast<const uint16_t *>(costs)[k], scale, offset);
}

// e^{-i gamma c} tables for uint16 levels: c = scale*(256 h + l) + offset
__device__ __forceinline__ void build_phase_tables(double2 *tlo, double2 *thi, double gamma, double scale,
                                                   double offset) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        double s, c;
        sincos(gamma * (scale * (double)i), &s, &c);
        tlo[i] = make_double2(c, -s);
        sincos(gamma * (scale * (double)(256 * i) + offset), &s, &c);
        thi[i] = make_double2(c, -s);
    }
}

template <int MIX, int COST, int PAT>
__device__ __forceinline__ void run_round(const PassParams &P, int r, double2 (&v)[kRegs], long long base,
                                          long long thr, const double2 *tlo, const double2 *thi) {
    const bool ph = (P.phase_round == r);
    if (ph && P.phase_at == 1) {
        long long o[kRegs];
        reg_offsets<PAT>(P, o);
#pragma unroll
        for (int i = 0; i < kRegs; ++i) v[i] = cmul(v[i], phase_factor<COST>(P.costs, base + thr + o[i], P.gamma, tlo, thi));
    }
    if (P.maskA[r]) butterflies<MIX, PAT>(v, P.A, P.maskA[r]);
    if (ph && P.phase_at == 2) {
        long long o[kRegs];
        reg_offsets<PAT>(P, o);
#pragma unroll
        for (int i = 0; i < kRegs; ++i) v[i] = cmul(v[i], phase_factor<COST>(P.costs, base + thr + o[i], P.gamma, tlo, thi));
    }
    if (P.maskB[r]) butterflies<MIX, PAT>(v, P.B, P.maskB[r]);
}

template <int MIX, int COST, int NR>
__global__ void __launch_bounds__(kThreads, 2) k_tile_pass(const __grid_constant__ PassParams P) {
    extern __shared__ double2 smem[];
    double2 *tile = smem;
    double2 *tlo = smem + kTile;
    double2 *thi = tlo + 256;
    __shared__ double red[kThreads / 32];
    const int tid = threadIdx.x;

    if (COST == FQ_COST_U16 && P.phase_round >= 0) {
        build_phase_tables(tlo, thi, P.gamma, P.cost_scale, P.cost_offset);
        __syncthreads();
    }
    const long long thr8 = thread_offset<PAT8>(P, tid);
    const long long thr0 = thread_offset<PAT0>(P, tid);
    const long long thr4 = thread_offset<PAT4>(P, tid);
    double eacc = 0.0;

    for (long long t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
        // tile number -> base address: insert a zero at every tile bit position
        long long base = t;
#pragma unroll
        for (int j = 0; j < kTileBits; ++j) {
            const int p = P.tile_pos[j];
            base = ((base >> p) << (p + 1)) | (base & ((1LL << p) - 1));
        }
        double2 v[kRegs];
        {
            long long o[kRegs];
            reg_offsets<PAT8>(P, o);
            if (P.init) {
#pragma unroll
                for (int i = 0; i < kRegs; ++i) v[i] = make_double2(P.init_amp, 0.0);
            } else {
#pragma unroll
                for (int i = 0; i < kRegs; ++i) v[i] = ld_stream(P.psi + base + thr8 + o[i]);
            }
        }
        run_round<MIX, COST, PAT8>(P, 0, v, base, thr8, tlo, thi);
        transpose<PAT8, PAT0>(tile, v, tid);
        run_round<MIX, COST, PAT0>(P, 1, v, base, thr0, tlo, thi);
        transpose<PAT0, PAT4>(tile, v, tid);
        run_round<MIX, COST, PAT4>(P, 2, v, base, thr4, tlo, thi);
        if (NR == 5) {
            transpose<PAT4, PAT0>(tile, v, tid);
            run_round<MIX, COST, PAT0>(P, 3, v, base, thr0, tlo, thi);
            transpose<PAT0, PAT8>(tile, v, tid);
            run_round<MIX, COST, PAT8>(P, 4, v, base, thr8, tlo, thi);
        }
        constexpr int LAST = (NR == 5) ? PAT8 : PAT4;
        const long long thrL = (NR == 5) ? thr8 : thr4;
        long long o[kRegs];
        reg_offsets<LAST>(P, o);
        const double fs = P.final_scale;
#pragma unroll
        for (int i = 0; i < kRegs; ++i) {
            double2 x = v[i];
            if (MIX == MIX_RX) x = make_double2(x.x * fs, x.y * fs);
            if (P.expect) eacc += cost_value<COST>(P.costs, base + thrL + o[i], P.cost_scale, P.cost_offset) *
                                  (x.x * x.x + x.y * x.y);
            st_stream(P.psi + base + thrL + o[i], x);
        }
    }
    if (P.expect) {
        const double s = block_sum<kThreads>(eacc, red);
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
    __shared__ double2 tlo[256], thi[256];
    build_phase_tables(tlo, thi, gamma, scale, offset);
    __syncthreads();
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < size;
         k += (long long)gridDim.x * blockDim.x) {
        const unsigned v = lv[k];
        psi[k] = cmul(psi[k], cmul(thi[v >> 8], tlo[v & 255]));
    }
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

static int max_blocks_per_sm = 2;

template <int MIX, int COST, int NR>
static int launch_pass(const PassParams &P, int grid, size_t smem, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_tile_pass<MIX, COST, NR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kTile + 512) * (int)sizeof(double2));
        configured = true;
    }
    k_tile_pass<MIX, COST, NR><<<grid, kThreads, smem, st>>>(P);
    FQ_LAUNCHED("k_tile_pass");
    return FQ_OK;
}

static int dispatch_pass(int mix, int cost, int nr, const PassParams &P, int grid, cudaStream_t st) {
    const size_t smem = (size_t)(kTile + 512) * sizeof(double2);
#define FQ_D(M, C, R) if (mix == M && cost == C && nr == R) return launch_pass<M, C, R>(P, grid, smem, st)
    FQ_D(MIX_RX, FQ_COST_F64, 3); FQ_D(MIX_RX, FQ_COST_F64, 5);
    FQ_D(MIX_RX, FQ_COST_U16, 3); FQ_D(MIX_RX, FQ_COST_U16, 5);
    FQ_D(MIX_SU2, FQ_COST_F64, 3); FQ_D(MIX_SU2, FQ_COST_F64, 5);
    FQ_D(MIX_SU2, FQ_COST_U16, 3); FQ_D(MIX_SU2, FQ_COST_U16, 5);
#undef FQ_D
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
    auto seq = plan_x(n, d->n_layers, d->layers, groups, gbase, true);
    const int mix = (d->mixer == FQ_MIXER_X) ? MIX_RX : MIX_SU2;
    const int sms = sm_count() > 0 ? sm_count() : 148;
    const long long n_tiles = 1LL << (n - kTileBits);
    const int grid = (int)std::min<long long>(n_tiles, (long long)sms * max_blocks_per_sm);
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
        P.nrounds = mid_phase ? 5 : 3;
        const int rb[5] = {8, 0, 4, 0, 8};  // first tile bit held in registers per round
        for (int r = 0; r < 5; ++r) {
            const int m = (tmask >> rb[r]) & 15;
            if (P.nrounds == 3) {
                P.maskA[r] = r < 3 ? m : 0;
                P.maskB[r] = (r < 3 && two) ? m : 0;
            } else {
                P.maskA[r] = r < 3 ? m : 0;
                P.maskB[r] = r >= 2 ? m : 0;
            }
        }
        P.phase_round = -1;
        if (pp.phase_layer >= 0) {
            P.gamma = d->layers[pp.phase_layer].gamma;
            if (pp.phase_at == 1) {
                P.phase_round = 0;
                P.phase_at = 1;
            } else {
                P.phase_round = 2;
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
        int s = dispatch_pass(mix, d->cost_kind, P.nrounds, P, grid, st);
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

int fq_plan_x_passes(int n, int n_layers, const fq_layer *layers) {
    if (n <= kTileBits) return n_layers > 0 ? 1 : 0;
    std::vector<Group> groups;
    std::vector<int> gbase;
    return (int)plan_x(n, n_layers, layers, groups, gbase, true).size();
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
