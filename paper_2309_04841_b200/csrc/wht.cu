// Cost diagonal of an integer / dyadic-weight polynomial as a Walsh-Hadamard
// transform (replaces accumulate_terms, reference _kernels.py:76-94, for the
// weights it can reproduce exactly).
//
//   c(k) = sum_t w_t (-1)^popcount(k & m_t) = WHT(a)(k),  a[m] = sum_{t: m_t = m} w_t
//
// so the diagonal costs n * 2^n additions (in HBM passes of 12 qubits) instead
// of T * 2^n parity evaluations (LABS n = 26: 1.7e9 instead of 9.2e10).  The
// weights are the integers iw_t = w_t * 2^shift with sum |iw| < 2^53 (checked
// on the host), so every partial sum is an exactly representable integer and
// the result is bit-identical to the reference's sequential double sum in any
// order; 2^-shift is applied once at the end (exact).  A shard of the global
// index space [r 2^nl, (r+1) 2^nl) transforms a_r[m_lo] = sum_{m_hi} a[m_hi,
// m_lo] (-1)^popcount(m_hi & r) over its nl local bits.
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace fq {

constexpr int kWhtBits = 12;
constexpr int kWhtTile = 1 << kWhtBits;
constexpr int kWhtThreads = 256;

__global__ void k_wht_scatter(double *__restrict__ a, int n_local, const int64_t *__restrict__ iw,
                              const int64_t *__restrict__ masks, int64_t T, int64_t shard) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t m = (uint64_t)masks[t];
        const uint64_t lo = m & ((1ULL << n_local) - 1), hi = m >> n_local;
        const double w = (double)iw[t];  // |iw| < 2^53: exact
        atomicAdd(&a[lo], (__popcll(hi & (uint64_t)shard) & 1) ? -w : w);  // exact integer sums: order-free
    }
}

struct WhtParams {
    double *a;
    long long n_tiles;
    int tile_pos[kWhtBits];
    int targets;   // mask over tile bits
    double scale;  // applied on store (2^-shift in the last pass, else 1)
};

// One HBM pass: every tile (12 index bits: targets + low spectators) is loaded
// into shared memory, butterflied (x, y) -> (x + y, x - y) on its target bits,
// scaled and stored.
__global__ void __launch_bounds__(kWhtThreads) k_wht_pass(const __grid_constant__ WhtParams P) {
    __shared__ double s[kWhtTile];
    const int tid = threadIdx.x;
    long long thr = 0;  // thread bits 0..7 <-> tile bits 0..7 (coalesced runs)
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if ((tid >> j) & 1) thr += 1LL << P.tile_pos[j];
    long long roff[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        long long o = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if ((i >> j) & 1) o += 1LL << P.tile_pos[8 + j];
        roff[i] = o;
    }
    for (long long t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
        long long base = t;
#pragma unroll
        for (int j = 0; j < kWhtBits; ++j) {
            const int p = P.tile_pos[j];
            base = ((base >> p) << (p + 1)) | (base & ((1LL << p) - 1));
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 16; ++i) s[tid | (i << 8)] = P.a[base + thr + roff[i]];
        __syncthreads();
        for (int j = 0; j < kWhtBits; ++j) {
            if (!((P.targets >> j) & 1)) continue;
#pragma unroll
            for (int q = tid; q < kWhtTile / 2; q += kWhtThreads) {
                const int e = ((q >> j) << (j + 1)) | (q & ((1 << j) - 1));
                const double x = s[e], y = s[e | (1 << j)];
                s[e] = x + y;
                s[e | (1 << j)] = x - y;
            }
            __syncthreads();
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) P.a[base + thr + roff[i]] = s[tid | (i << 8)] * P.scale;
    }
}

}  // namespace fq

using namespace fq;

extern "C" {

int fq_precompute_wht(double *out, int64_t size, const int64_t *iweights, const int64_t *masks, int64_t n_terms,
                      int shift, int64_t index_base, void *stream) {
    FQ_CHECK_ARG(out && is_pow2(size) && n_terms >= 0 && (n_terms == 0 || (iweights && masks)),
                 "fq_precompute_wht: bad arguments");
    FQ_CHECK_ARG(shift >= 0 && shift < 64, "fq_precompute_wht: bad shift %d", shift);
    const int nl = log2i(size);
    FQ_CHECK_ARG(nl >= kWhtBits, "fq_precompute_wht: needs >= %d local bits (got %d)", kWhtBits, nl);
    FQ_CHECK_ARG(index_base % size == 0, "fq_precompute_wht: shard base must be a multiple of the shard size");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    FQ_CUDA(cudaMemsetAsync(out, 0, size * sizeof(double), st));
    if (n_terms > 0) {
        k_wht_scatter<<<(int)std::min<int64_t>((n_terms + 255) / 256, 1024), 256, 0, st>>>(
            out, nl, iweights, masks, n_terms, index_base / size);
        FQ_LAUNCHED("k_wht_scatter");
    }
    // groups of <= 12 target bits; a high group takes the lowest bits as spectators
    std::vector<std::vector<int>> groups;
    for (int q0 = 0; q0 < nl; q0 += kWhtBits) {
        std::vector<int> g;
        for (int q = q0; q < std::min(nl, q0 + kWhtBits); ++q) g.push_back(q);
        groups.push_back(g);
    }
    const int sms = sm_count() > 0 ? sm_count() : 148;
    for (size_t gi = 0; gi < groups.size(); ++gi) {
        WhtParams P;
        P.a = out;
        P.n_tiles = size >> kWhtBits;
        std::vector<int> bits = groups[gi];
        for (int q = 0; q < nl && (int)bits.size() < kWhtBits; ++q)
            if (std::find(groups[gi].begin(), groups[gi].end(), q) == groups[gi].end()) bits.push_back(q);
        std::sort(bits.begin(), bits.end());
        P.targets = 0;
        for (int j = 0; j < kWhtBits; ++j) {
            P.tile_pos[j] = bits[j];
            if (std::find(groups[gi].begin(), groups[gi].end(), bits[j]) != groups[gi].end()) P.targets |= 1 << j;
        }
        P.scale = (gi + 1 == groups.size()) ? std::ldexp(1.0, -shift) : 1.0;
        const int grid = (int)std::min<long long>(P.n_tiles, (long long)sms * 4);
        k_wht_pass<<<grid, kWhtThreads, 0, st>>>(P);
        FQ_LAUNCHED("k_wht_pass");
    }
    return FQ_OK;
}

}  // extern "C"
