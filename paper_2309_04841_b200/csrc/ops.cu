// Operator layer of libfqaoa: one sm_100a kernel per reference numba kernel
// (fastqaoa/_kernels.py) plus the state/observable kernels of statevec.py.
//
// These are the building blocks for the reference-compatible per-operator API
// (apply_su2, apply_xy, apply_phase, ...).  The fused evolution that the
// simulator actually runs lives in evolve.cu.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "common.cuh"

namespace fq {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

int cuda_status(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return FQ_OK;
    set_error("%s: %s", what, cudaGetErrorString(e));
    return FQ_ERR_CUDA;
}

int sm_count() {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    return sms;
}

int grid_for(int64_t work, int per_block, int blocks_per_sm) {
    int64_t need = (work + per_block - 1) / per_block;
    int sms = sm_count();
    int64_t cap = (int64_t)(sms > 0 ? sms : 148) * blocks_per_sm;
    if (need < 1) need = 1;
    return (int)(need < cap ? need : cap);
}

__global__ void k_sum_partials(const double *partials, int count, double *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < count; ++i) t += partials[i];
        *out = t;
    }
}

// ------------------------------------------------------------ pair kernels
// su2_on_pairs — reference _kernels.py:14-27
__global__ void k_su2_on_pairs(double2 *__restrict__ psi, int64_t half, double2 a, double2 b, int q) {
    const int64_t bit = int64_t(1) << q, low = bit - 1;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < half;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t l0 = ((g >> q) << (q + 1)) | (g & low), l1 = l0 | bit;
        const double2 x0 = psi[l0], x1 = psi[l1];
        // y0 = a x0 - conj(b) x1 ; y1 = b x0 + conj(a) x1
        double2 y0, y1;
        y0.x = a.x * x0.x - a.y * x0.y - (b.x * x1.x + b.y * x1.y);
        y0.y = a.x * x0.y + a.y * x0.x - (b.x * x1.y - b.y * x1.x);
        y1.x = b.x * x0.x - b.y * x0.y + (a.x * x1.x + a.y * x1.y);
        y1.y = b.x * x0.y + b.y * x0.x + (a.x * x1.y - a.y * x1.x);
        psi[l0] = y0;
        psi[l1] = y1;
    }
}

// xy_on_pairs — reference _kernels.py:30-48
__global__ void k_xy_on_pairs(double2 *__restrict__ psi, int64_t quarter, double c, double s, int p_lo,
                              int p_hi) {
    const int64_t bit_lo = int64_t(1) << p_lo, bit_hi = int64_t(1) << p_hi;
    const int64_t m_lo = bit_lo - 1, m_hi = bit_hi - 1;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < quarter;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = ((g >> p_lo) << (p_lo + 1)) | (g & m_lo);
        const int64_t base = ((t >> p_hi) << (p_hi + 1)) | (t & m_hi);
        const double2 xl = psi[base | bit_lo], xh = psi[base | bit_hi];
        psi[base | bit_lo] = make_double2(c * xl.x + s * xh.y, c * xl.y - s * xh.x);
        psi[base | bit_hi] = make_double2(s * xl.y + c * xh.x, c * xh.y - s * xl.x);
    }
}

// swap_bits — reference _kernels.py:51-65
__global__ void k_swap_bits(double2 *__restrict__ psi, int64_t quarter, int p_lo, int p_hi) {
    const int64_t bit_lo = int64_t(1) << p_lo, bit_hi = int64_t(1) << p_hi;
    const int64_t m_lo = bit_lo - 1, m_hi = bit_hi - 1;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < quarter;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = ((g >> p_lo) << (p_lo + 1)) | (g & m_lo);
        const int64_t base = ((t >> p_hi) << (p_hi + 1)) | (t & m_hi);
        const double2 xl = psi[base | bit_lo], xh = psi[base | bit_hi];
        psi[base | bit_lo] = xh;
        psi[base | bit_hi] = xl;
    }
}

// phase_multiply — reference _kernels.py:68-73
__global__ void k_phase(double2 *__restrict__ psi, const double *__restrict__ costs, int64_t size,
                        double gamma) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < size;
         k += (int64_t)gridDim.x * blockDim.x) {
        double s, c;
        sincos(gamma * costs[k], &s, &c);
        const double2 x = psi[k];
        // x * (c - i s)
        psi[k] = make_double2(x.x * c + x.y * s, x.y * c - x.x * s);
    }
}

// abs2_inplace — reference _kernels.py:97-102
__global__ void k_abs2(double2 *__restrict__ psi, int64_t size) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < size;
         k += (int64_t)gridDim.x * blockDim.x) {
        const double2 x = psi[k];
        // re*re + im*im with the reference's two roundings (no FMA contraction)
        psi[k] = make_double2(__dadd_rn(__dmul_rn(x.x, x.x), __dmul_rn(x.y, x.y)), 0.0);
    }
}

// complex64 states: same two roundings in single precision
__global__ void k_abs2_c64(float2 *__restrict__ psi, int64_t size) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < size;
         k += (int64_t)gridDim.x * blockDim.x) {
        const float2 x = psi[k];
        psi[k] = make_float2(__fadd_rn(__fmul_rn(x.x, x.x), __fmul_rn(x.y, x.y)), 0.0f);
    }
}

// ------------------------------------------------------------ precompute
// Terms are staged through shared memory in chunks; every thread walks the
// chunk in term order for its own elements (reference _kernels.py:81-94:
// one accumulator per element, terms left to right).
constexpr int kTermChunk = 1024;
constexpr int kPreThreads = 256;
constexpr int kPreElems = 4;  // elements per thread (independent accumulators -> ILP)

template <typename Mask>
__device__ __forceinline__ int parity(Mask x);
template <>
__device__ __forceinline__ int parity<uint32_t>(uint32_t x) { return __popc(x) & 1; }
template <>
__device__ __forceinline__ int parity<uint64_t>(uint64_t x) { return __popcll(x) & 1; }

// float64 weights, sequential double accumulation (bit-exact vs the reference
// for ANY weights: same per-element operation sequence).
template <typename Mask>
__global__ void __launch_bounds__(kPreThreads) k_accumulate_f64(double *__restrict__ out, int64_t size,
                                                                const double *__restrict__ w,
                                                                const int64_t *__restrict__ m,
                                                                int64_t T, int64_t base) {
    __shared__ double sw[kTermChunk];
    __shared__ Mask sm[kTermChunk];
    const int64_t per_block = (int64_t)kPreThreads * kPreElems;
    for (int64_t blk = blockIdx.x * per_block; blk < size; blk += (int64_t)gridDim.x * per_block) {
        double acc[kPreElems];
        Mask idx[kPreElems];
#pragma unroll
        for (int e = 0; e < kPreElems; ++e) {
            acc[e] = 0.0;
            idx[e] = (Mask)(base + blk + e * kPreThreads + threadIdx.x);
        }
        for (int64_t t0 = 0; t0 < T; t0 += kTermChunk) {
            const int cnt = (int)((T - t0) < kTermChunk ? (T - t0) : kTermChunk);
            __syncthreads();
            for (int i = threadIdx.x; i < cnt; i += kPreThreads) {
                sw[i] = w[t0 + i];
                sm[i] = (Mask)m[t0 + i];
            }
            __syncthreads();
            for (int t = 0; t < cnt; ++t) {
                const double wt = sw[t];
                const Mask mt = sm[t];
#pragma unroll
                for (int e = 0; e < kPreElems; ++e) {
                    if (parity<Mask>(idx[e] & mt)) acc[e] -= wt;
                    else acc[e] += wt;
                }
            }
        }
#pragma unroll
        for (int e = 0; e < kPreElems; ++e) {
            const int64_t k = blk + e * kPreThreads + threadIdx.x;
            if (k < size) out[k] += acc[e];
        }
    }
}

// Integer accumulation of dyadic weights (exact).  MODE 0: out[k] += S*2^-shift
// (float64 diagonal).  MODE 1: uint16 level (S - level_offset) >> shift.
template <typename Mask, typename Acc, int MODE>
__global__ void __launch_bounds__(kPreThreads) k_accumulate_int(void *__restrict__ out_, int64_t size,
                                                                const int64_t *__restrict__ w,
                                                                const int64_t *__restrict__ m,
                                                                int64_t T, int shift, int64_t base,
                                                                int64_t level_offset, int *bad) {
    __shared__ Acc sw[kTermChunk];
    __shared__ Mask sm[kTermChunk];
    const int64_t per_block = (int64_t)kPreThreads * kPreElems;
    const double inv = ldexp(1.0, -shift);
    for (int64_t blk = blockIdx.x * per_block; blk < size; blk += (int64_t)gridDim.x * per_block) {
        Acc acc[kPreElems];
        Mask idx[kPreElems];
#pragma unroll
        for (int e = 0; e < kPreElems; ++e) {
            acc[e] = 0;
            idx[e] = (Mask)(base + blk + e * kPreThreads + threadIdx.x);
        }
        for (int64_t t0 = 0; t0 < T; t0 += kTermChunk) {
            const int cnt = (int)((T - t0) < kTermChunk ? (T - t0) : kTermChunk);
            __syncthreads();
            for (int i = threadIdx.x; i < cnt; i += kPreThreads) {
                sw[i] = (Acc)w[t0 + i];
                sm[i] = (Mask)m[t0 + i];
            }
            __syncthreads();
#pragma unroll 4
            for (int t = 0; t < cnt; ++t) {
                const Acc wt = sw[t];
                const Mask mt = sm[t];
#pragma unroll
                for (int e = 0; e < kPreElems; ++e) {
                    const Acc sgn = -(Acc)parity<Mask>(idx[e] & mt);  // 0 or -1
                    acc[e] += (wt ^ sgn) - sgn;                       // +w or -w
                }
            }
        }
#pragma unroll
        for (int e = 0; e < kPreElems; ++e) {
            const int64_t k = blk + e * kPreThreads + threadIdx.x;
            if (k >= size) continue;
            if (MODE == 0) {
                double *out = static_cast<double *>(out_);
                out[k] += (double)acc[e] * inv;
            } else {
                uint16_t *out = static_cast<uint16_t *>(out_);
                const int64_t d = (int64_t)acc[e] - level_offset;
                const int64_t v = d >> shift;
                if (d < 0 || (v << shift) != d || v > 65535) atomicOr(bad, 1);
                out[k] = (uint16_t)v;
            }
        }
    }
}

// ------------------------------------------------------------ states
template <typename T>
__global__ void k_init_state(T *__restrict__ psi, int64_t size, int weight, double amp, int64_t base) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < size;
         k += (int64_t)gridDim.x * blockDim.x) {
        const bool on = weight < 0 || __popcll((unsigned long long)(base + k)) == weight;
        psi[k] = {on ? (decltype(T::x))amp : (decltype(T::x))0, (decltype(T::x))0};
    }
}

// ------------------------------------------------------------ reductions
template <int KIND>
__device__ __forceinline__ double load_cost(const void *costs, int64_t k, double scale, double offset) {
    if (KIND == FQ_COST_F64) return static_cast<const double *>(costs)[k];
    return decode_u16(static_cast<const uint16_t *>(costs)[k], scale, offset);
}

constexpr int kRedThreads = 256;

// OP 0: sum c|x|^2 ; OP 1: sum_{c <= cutoff} |x|^2 ; OP 2: min c ; OP 3: max c
// T: double2 (complex128 states) or float2 (complex64 states; accumulated in fp64)
template <int KIND, int OP, typename T>
__global__ void __launch_bounds__(kRedThreads) k_reduce(const T *__restrict__ psi, const void *costs,
                                                        double scale, double offset, int64_t size,
                                                        double cutoff, double *partials) {
    __shared__ double red[kRedThreads / 32];
    double acc = (OP == 2) ? INFINITY : (OP == 3 ? -INFINITY : 0.0);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < size;
         k += (int64_t)gridDim.x * blockDim.x) {
        const double c = load_cost<KIND>(costs, k, scale, offset);
        if (OP == 0) {
            const T x = psi[k];
            acc += c * ((double)x.x * x.x + (double)x.y * x.y);
        } else if (OP == 1) {
            if (c <= cutoff) {
                const T x = psi[k];
                acc += (double)x.x * x.x + (double)x.y * x.y;
            }
        } else if (OP == 2) {
            acc = fmin(acc, c);
        } else {
            acc = fmax(acc, c);
        }
    }
    if (OP <= 1) {
        const double t = block_sum<kRedThreads>(acc, red);
        if (threadIdx.x == 0) partials[blockIdx.x] = t;
    } else {
        for (int o = 16; o > 0; o >>= 1) {
            const double y = __shfl_xor_sync(0xffffffffu, acc, o);
            acc = (OP == 2) ? fmin(acc, y) : fmax(acc, y);
        }
        const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
        if (l == 0) red[w] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = red[0];
            for (int i = 1; i < kRedThreads / 32; ++i) t = (OP == 2) ? fmin(t, red[i]) : fmax(t, red[i]);
            partials[blockIdx.x] = t;
        }
    }
}

__global__ void k_minmax_final(const double *pmin, const double *pmax, int count, double *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double a = INFINITY, b = -INFINITY;
        for (int i = 0; i < count; ++i) {
            a = fmin(a, pmin[i]);
            b = fmax(b, pmax[i]);
        }
        out[0] = a;
        out[1] = b;
    }
}

__global__ void k_compact_u16(uint16_t *__restrict__ out, const double *__restrict__ costs, int64_t size,
                              double scale, double offset, int *bad) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < size;
         k += (int64_t)gridDim.x * blockDim.x) {
        const double c = costs[k];
        const double q = rint((c - offset) / scale);
        const bool ok = q >= 0.0 && q <= 65535.0 && decode_u16((uint16_t)q, scale, offset) == c;
        if (!ok) atomicOr(bad, 1);
        out[k] = ok ? (uint16_t)q : (uint16_t)0;
    }
}

// levels[k] -= delta (delta < 0: += -delta), 8 levels per thread-iteration
// (16-B loads/stores).  Lane-wise 16-bit arithmetic in 32-bit words: the caller
// guarantees no level leaves [0, 65535], so no borrow / carry crosses a lane.
__global__ void k_rebase_u16(uint16_t *__restrict__ lv, int64_t size, int delta) {
    const int64_t n8 = size >> 3;
    uint4 *v = reinterpret_cast<uint4 *>(lv);
    const unsigned a = (unsigned)(delta < 0 ? -delta : delta), d2 = a | (a << 16);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n8; k += (int64_t)gridDim.x * blockDim.x) {
        uint4 x = v[k];
        if (delta >= 0) x.x -= d2, x.y -= d2, x.z -= d2, x.w -= d2;
        else x.x += d2, x.y += d2, x.z += d2, x.w += d2;
        v[k] = x;
    }
    for (int64_t k = (n8 << 3) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < size;
         k += (int64_t)gridDim.x * blockDim.x)
        lv[k] = (uint16_t)((int)lv[k] - delta);
}

}  // namespace fq

using namespace fq;

static inline cudaStream_t S(void *s) { return static_cast<cudaStream_t>(s); }

template <int OP>
static int launch_reduce(const void *psi, const void *costs, int kind, double scale, double offset,
                         int64_t size, double cutoff, double *partials, int grid, cudaStream_t st, bool c64 = false) {
    if (c64) {
        const float2 *p = static_cast<const float2 *>(psi);
        if (kind == FQ_COST_F64)
            k_reduce<FQ_COST_F64, OP><<<grid, kRedThreads, 0, st>>>(p, costs, scale, offset, size, cutoff, partials);
        else
            k_reduce<FQ_COST_U16, OP><<<grid, kRedThreads, 0, st>>>(p, costs, scale, offset, size, cutoff, partials);
        FQ_LAUNCHED("k_reduce");
        return FQ_OK;
    }
    const double2 *p = static_cast<const double2 *>(psi);
    if (kind == FQ_COST_F64)
        k_reduce<FQ_COST_F64, OP><<<grid, kRedThreads, 0, st>>>(p, costs, scale, offset, size, cutoff, partials);
    else
        k_reduce<FQ_COST_U16, OP><<<grid, kRedThreads, 0, st>>>(p, costs, scale, offset, size, cutoff, partials);
    FQ_LAUNCHED("k_reduce");
    return FQ_OK;
}

extern "C" {

int fq_version(void) { return 1; }
const char *fq_last_error(void) { return g_err; }
int fq_sm_count(void) { return sm_count(); }

int fq_su2_on_pairs(void *psi, int64_t size, double a_re, double a_im, double b_re, double b_im, int q,
                    void *stream) {
    FQ_CHECK_ARG(psi && is_pow2(size), "fq_su2_on_pairs: bad buffer (size %lld)", (long long)size);
    FQ_CHECK_ARG(q >= 0 && (int64_t(1) << q) < size, "fq_su2_on_pairs: qubit %d out of range", q);
    const int64_t half = size >> 1;
    k_su2_on_pairs<<<grid_for(half, 256, 8), 256, 0, S(stream)>>>(
        static_cast<double2 *>(psi), half, make_double2(a_re, a_im), make_double2(b_re, b_im), q);
    FQ_LAUNCHED("k_su2_on_pairs");
    return FQ_OK;
}

int fq_xy_on_pairs(void *psi, int64_t size, double c, double s, int p_lo, int p_hi, void *stream) {
    FQ_CHECK_ARG(psi && is_pow2(size) && size >= 4, "fq_xy_on_pairs: bad buffer");
    FQ_CHECK_ARG(0 <= p_lo && p_lo < p_hi && (int64_t(1) << p_hi) < size,
                 "fq_xy_on_pairs: need 0 <= p_lo < p_hi < n (got %d, %d)", p_lo, p_hi);
    const int64_t quarter = size >> 2;
    k_xy_on_pairs<<<grid_for(quarter, 256, 8), 256, 0, S(stream)>>>(static_cast<double2 *>(psi), quarter,
                                                                     c, s, p_lo, p_hi);
    FQ_LAUNCHED("k_xy_on_pairs");
    return FQ_OK;
}

int fq_swap_bits(void *psi, int64_t size, int p_lo, int p_hi, void *stream) {
    FQ_CHECK_ARG(psi && is_pow2(size) && size >= 4, "fq_swap_bits: bad buffer");
    FQ_CHECK_ARG(0 <= p_lo && p_lo < p_hi && (int64_t(1) << p_hi) < size,
                 "fq_swap_bits: need 0 <= p_lo < p_hi < n (got %d, %d)", p_lo, p_hi);
    const int64_t quarter = size >> 2;
    k_swap_bits<<<grid_for(quarter, 256, 8), 256, 0, S(stream)>>>(static_cast<double2 *>(psi), quarter, p_lo,
                                                                   p_hi);
    FQ_LAUNCHED("k_swap_bits");
    return FQ_OK;
}

int fq_phase_multiply(void *psi, const double *costs, int64_t size, double gamma, void *stream) {
    FQ_CHECK_ARG(psi && costs && size > 0, "fq_phase_multiply: bad buffer");
    k_phase<<<grid_for(size, 256, 8), 256, 0, S(stream)>>>(static_cast<double2 *>(psi), costs, size, gamma);
    FQ_LAUNCHED("k_phase");
    return FQ_OK;
}

int fq_abs2_inplace(void *psi, int64_t size, void *stream) {
    FQ_CHECK_ARG(psi && size > 0, "fq_abs2_inplace: bad buffer");
    k_abs2<<<grid_for(size, 256, 8), 256, 0, S(stream)>>>(static_cast<double2 *>(psi), size);
    FQ_LAUNCHED("k_abs2");
    return FQ_OK;
}

static bool fits32(int64_t size, int64_t base, const int64_t *) {
    return base >= 0 && base + size <= (int64_t(1) << 32);
}

int fq_accumulate_terms(double *out, int64_t size, const double *weights, const int64_t *masks,
                        int64_t n_terms, int64_t index_base, void *stream) {
    FQ_CHECK_ARG(out && size > 0 && n_terms >= 0 && index_base >= 0, "fq_accumulate_terms: bad args");
    if (n_terms == 0) return FQ_OK;
    FQ_CHECK_ARG(weights && masks, "fq_accumulate_terms: null terms");
    const int g = grid_for(size, kPreThreads * kPreElems, 8);
    if (fits32(size, index_base, masks))
        k_accumulate_f64<uint32_t><<<g, kPreThreads, 0, S(stream)>>>(out, size, weights, masks, n_terms,
                                                                      index_base);
    else
        k_accumulate_f64<uint64_t><<<g, kPreThreads, 0, S(stream)>>>(out, size, weights, masks, n_terms,
                                                                      index_base);
    FQ_LAUNCHED("k_accumulate_f64");
    return FQ_OK;
}

// `wide` = int64 accumulator required (sum |w| >= 2^31)
static int launch_int(void *out, int mode, int64_t size, const int64_t *w, const int64_t *m, int64_t T,
                      int shift, int64_t base, int64_t level_offset, int *bad, bool wide, cudaStream_t st) {
    const int g = grid_for(size, kPreThreads * kPreElems, 8);
    const bool m32 = fits32(size, base, m);
#define FQ_LAUNCH_INT(MASK, ACC, MODE)                                                                   \
    k_accumulate_int<MASK, ACC, MODE><<<g, kPreThreads, 0, st>>>(out, size, w, m, T, shift, base,       \
                                                                 level_offset, bad)
    if (mode == 0) {
        if (m32 && !wide) FQ_LAUNCH_INT(uint32_t, int32_t, 0);
        else if (m32) FQ_LAUNCH_INT(uint32_t, long long, 0);
        else if (!wide) FQ_LAUNCH_INT(uint64_t, int32_t, 0);
        else FQ_LAUNCH_INT(uint64_t, long long, 0);
    } else {
        if (m32 && !wide) FQ_LAUNCH_INT(uint32_t, int32_t, 1);
        else if (m32) FQ_LAUNCH_INT(uint32_t, long long, 1);
        else if (!wide) FQ_LAUNCH_INT(uint64_t, int32_t, 1);
        else FQ_LAUNCH_INT(uint64_t, long long, 1);
    }
#undef FQ_LAUNCH_INT
    FQ_LAUNCHED("k_accumulate_int");
    return FQ_OK;
}

int fq_accumulate_terms_dyadic(double *out, int64_t size, const int64_t *iweights, const int64_t *masks,
                               int64_t n_terms, int shift, int acc_bits, int64_t index_base, void *stream) {
    FQ_CHECK_ARG(out && size > 0 && n_terms >= 0 && index_base >= 0, "fq_accumulate_terms_dyadic: bad args");
    FQ_CHECK_ARG(acc_bits == 32 || acc_bits == 64, "fq_accumulate_terms_dyadic: acc_bits must be 32 or 64");
    FQ_CHECK_ARG(shift >= 0 && shift <= 62, "fq_accumulate_terms_dyadic: shift %d out of range", shift);
    if (n_terms == 0) return FQ_OK;
    return launch_int(out, 0, size, iweights, masks, n_terms, shift, index_base, 0, nullptr, acc_bits == 64,
                      S(stream));
}

int fq_precompute_levels_u16(uint16_t *out, int64_t size, const int64_t *iweights, const int64_t *masks,
                             int64_t n_terms, int acc_bits, int64_t index_base, int64_t level_offset,
                             int level_shift, int *bad_dev, void *stream) {
    FQ_CHECK_ARG(out && size > 0 && n_terms >= 0 && bad_dev, "fq_precompute_levels_u16: bad args");
    FQ_CHECK_ARG(acc_bits == 32 || acc_bits == 64, "fq_precompute_levels_u16: acc_bits must be 32 or 64");
    FQ_CHECK_ARG(level_shift >= 0 && level_shift <= 62, "fq_precompute_levels_u16: bad shift");
    return launch_int(out, 1, size, iweights, masks, n_terms, level_shift, index_base, level_offset, bad_dev,
                      acc_bits == 64, S(stream));
}

int fq_init_state(void *psi, int64_t size, int weight, double amp, int64_t index_base, void *stream) {
    FQ_CHECK_ARG(psi && size > 0, "fq_init_state: bad buffer");
    k_init_state<<<grid_for(size, 256, 8), 256, 0, S(stream)>>>(static_cast<double2 *>(psi), size, weight, amp,
                                                                 index_base);
    FQ_LAUNCHED("k_init_state");
    return FQ_OK;
}

static int reduce_grid(int64_t size) {
    int g = grid_for(size, kRedThreads * 4, 4);
    return g > FQ_SCRATCH_DOUBLES / 2 ? FQ_SCRATCH_DOUBLES / 2 : g;
}

int fq_expectation(const void *psi, const void *costs, int cost_kind, double scale, double offset, int64_t size,
                   double *out_dev, double *scratch, void *stream) {
    FQ_CHECK_ARG(psi && costs && out_dev && scratch && size > 0, "fq_expectation: bad args");
    FQ_CHECK_ARG(cost_kind == FQ_COST_F64 || cost_kind == FQ_COST_U16, "fq_expectation: bad cost kind");
    const int g = reduce_grid(size);
    int s = launch_reduce<0>(psi, costs, cost_kind, scale, offset, size, 0.0, scratch, g, S(stream));
    if (s) return s;
    k_sum_partials<<<1, 32, 0, S(stream)>>>(scratch, g, out_dev);
    FQ_LAUNCHED("k_sum_partials");
    return FQ_OK;
}

int fq_masked_probability(const void *psi, const void *costs, int cost_kind, double scale, double offset,
                          int64_t size, double cutoff, double *out_dev, double *scratch, void *stream) {
    FQ_CHECK_ARG(psi && costs && out_dev && scratch && size > 0, "fq_masked_probability: bad args");
    const int g = reduce_grid(size);
    int s = launch_reduce<1>(psi, costs, cost_kind, scale, offset, size, cutoff, scratch, g, S(stream));
    if (s) return s;
    k_sum_partials<<<1, 32, 0, S(stream)>>>(scratch, g, out_dev);
    FQ_LAUNCHED("k_sum_partials");
    return FQ_OK;
}

// ---- complex64 states (optional single-precision path; observables accumulate in fp64)
int fq_init_state_c64(void *psi, int64_t size, int weight, double amp, int64_t index_base, void *stream) {
    FQ_CHECK_ARG(psi && size > 0, "fq_init_state_c64: bad buffer");
    k_init_state<<<grid_for(size, 256, 8), 256, 0, S(stream)>>>(static_cast<float2 *>(psi), size, weight, amp,
                                                                 index_base);
    FQ_LAUNCHED("k_init_state");
    return FQ_OK;
}

int fq_abs2_inplace_c64(void *psi, int64_t size, void *stream) {
    FQ_CHECK_ARG(psi && size > 0, "fq_abs2_inplace_c64: bad buffer");
    k_abs2_c64<<<grid_for(size, 256, 8), 256, 0, S(stream)>>>(static_cast<float2 *>(psi), size);
    FQ_LAUNCHED("k_abs2");
    return FQ_OK;
}

int fq_expectation_c64(const void *psi, const void *costs, int cost_kind, double scale, double offset,
                       int64_t size, double *out_dev, double *scratch, void *stream) {
    FQ_CHECK_ARG(psi && costs && out_dev && scratch && size > 0, "fq_expectation_c64: bad args");
    FQ_CHECK_ARG(cost_kind == FQ_COST_F64 || cost_kind == FQ_COST_U16, "fq_expectation_c64: bad cost kind");
    const int g = reduce_grid(size);
    int s = launch_reduce<0>(psi, costs, cost_kind, scale, offset, size, 0.0, scratch, g, S(stream), true);
    if (s) return s;
    k_sum_partials<<<1, 32, 0, S(stream)>>>(scratch, g, out_dev);
    FQ_LAUNCHED("k_sum_partials");
    return FQ_OK;
}

int fq_masked_probability_c64(const void *psi, const void *costs, int cost_kind, double scale, double offset,
                              int64_t size, double cutoff, double *out_dev, double *scratch, void *stream) {
    FQ_CHECK_ARG(psi && costs && out_dev && scratch && size > 0, "fq_masked_probability_c64: bad args");
    const int g = reduce_grid(size);
    int s = launch_reduce<1>(psi, costs, cost_kind, scale, offset, size, cutoff, scratch, g, S(stream), true);
    if (s) return s;
    k_sum_partials<<<1, 32, 0, S(stream)>>>(scratch, g, out_dev);
    FQ_LAUNCHED("k_sum_partials");
    return FQ_OK;
}

int fq_cost_minmax(const void *costs, int cost_kind, double scale, double offset, int64_t size, double *out_dev,
                   double *scratch, void *stream) {
    FQ_CHECK_ARG(costs && out_dev && scratch && size > 0, "fq_cost_minmax: bad args");
    const int g = reduce_grid(size);
    int s = launch_reduce<2>(nullptr, costs, cost_kind, scale, offset, size, 0.0, scratch, g, S(stream));
    if (s) return s;
    s = launch_reduce<3>(nullptr, costs, cost_kind, scale, offset, size, 0.0, scratch + g, g, S(stream));
    if (s) return s;
    k_minmax_final<<<1, 32, 0, S(stream)>>>(scratch, scratch + g, g, out_dev);
    FQ_LAUNCHED("k_minmax_final");
    return FQ_OK;
}

int fq_rebase_u16(uint16_t *levels, int64_t size, int delta, void *stream) {
    FQ_CHECK_ARG(levels && size > 0 && delta >= -65535 && delta <= 65535 &&
                     (reinterpret_cast<uintptr_t>(levels) & 15) == 0,
                 "fq_rebase_u16: bad args");
    if (delta == 0) return FQ_OK;
    k_rebase_u16<<<grid_for(size / 8 + 1, 256, 8), 256, 0, S(stream)>>>(levels, size, delta);
    FQ_LAUNCHED("k_rebase_u16");
    return FQ_OK;
}

int fq_compact_u16(uint16_t *out, const double *costs, int64_t size, double scale, double offset, int *bad_dev,
                   void *stream) {
    FQ_CHECK_ARG(out && costs && bad_dev && size > 0 && scale > 0.0, "fq_compact_u16: bad args");
    k_compact_u16<<<grid_for(size, 256, 8), 256, 0, S(stream)>>>(out, costs, size, scale, offset, bad_dev);
    FQ_LAUNCHED("k_compact_u16");
    return FQ_OK;
}

}  // extern "C"
