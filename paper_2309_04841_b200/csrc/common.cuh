// Shared helpers for the libfqaoa kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fqaoa.h"

namespace fq {

// thread-local error text for fq_last_error()
void set_error(const char *fmt, ...);

#define FQ_CHECK_ARG(cond, ...)          \
    do {                                 \
        if (!(cond)) {                   \
            ::fq::set_error(__VA_ARGS__); \
            return FQ_ERR_ARG;           \
        }                                \
    } while (0)

int cuda_status(cudaError_t e, const char *what);
#define FQ_CUDA(call) \
    do { int _s = ::fq::cuda_status((call), #call); if (_s) return _s; } while (0)
#define FQ_LAUNCHED(what) \
    do { int _s = ::fq::cuda_status(cudaGetLastError(), what); if (_s) return _s; } while (0)

int sm_count();
// grid size for a grid-stride kernel over `work` items of `per_block` each
int grid_for(int64_t work, int per_block, int blocks_per_sm);

inline bool is_pow2(int64_t x) { return x >= 2 && (x & (x - 1)) == 0; }
inline int log2i(int64_t x) { int r = 0; while ((int64_t(1) << r) < x) ++r; return r; }

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// Decode of a uint16 level exactly as the reference's CompactCostVector.decode
// (terms.py:133-135: scale * v + offset, two roundings, never contracted to FMA).
__device__ __forceinline__ double decode_u16(uint16_t v, double scale, double offset) {
    return __dadd_rn(__dmul_rn(scale, (double)v), offset);
}

// sin and cos of a double in ~25 FP64 instructions, no branch on the common
// path: Cody-Waite reduction by pi/2 with a three-part constant (FMA, exact
// for |x| < 2^20 pi/2) and the fdlibm minimax kernels on [-pi/4, pi/4]
// (__kernel_sin / __kernel_cos coefficients); |error| ~1e-16, against the
// 1e-10 state tolerance of the reference's np.exp(-1j * gamma * c).  Larger
// arguments take the library sincos.
// coefficients in the constant bank: the FP64 instructions take them as c[][]
// operands (double immediates would be rebuilt with uniform moves every use)
__constant__ double kSinCosCoef[15] = {
    0.63661977236758134308, 1.5707963267948966192, 6.1232339957367658e-17, -1.4973849048591698e-33,
    1.58969099521155010221e-10, -2.50507602534068634195e-08, 2.75573137070700676789e-06,
    -1.98412698298579493134e-04, 8.33333333332248946124e-03, -1.66666666666666324348e-01,
    -1.13596475577881948265e-11, 2.08757232129817482790e-09, -2.75573143513906633035e-07,
    2.48015872894767294178e-05, -1.38888888888741095749e-03};
__constant__ double kCosC1 = 4.16666666666666019037e-02;

__device__ __forceinline__ void fq_sincos(double x, double *sp, double *cp) {
    if (!(fabs(x) < 1.6e6)) {
        sincos(x, sp, cp);
        return;
    }
    const double *K = kSinCosCoef;
    const double k = rint(x * K[0]);  // 2 / pi
    double r = fma(-k, K[1], x);
    r = fma(-k, K[2], r);
    r = fma(-k, K[3], r);
    const double z = r * r;
    double ps = fma(z, K[4], K[5]);
    ps = fma(z, ps, K[6]);
    ps = fma(z, ps, K[7]);
    ps = fma(z, ps, K[8]);
    ps = fma(z, ps, K[9]);
    const double sn = fma(r * z, ps, r);
    double pc = fma(z, K[10], K[11]);
    pc = fma(z, pc, K[12]);
    pc = fma(z, pc, K[13]);
    pc = fma(z, pc, K[14]);
    pc = fma(z, pc, kCosC1);
    const double cs = fma(z * z, pc, fma(-0.5, z, 1.0));
    const int q = (int)(long long)k & 3;
    const double s0 = (q & 1) ? cs : sn, c0 = (q & 1) ? sn : cs;
    *sp = (q & 2) ? -s0 : s0;
    *cp = ((q + 1) & 2) ? -c0 : c0;
}

// streaming (evict-first) 16-B global accesses: each amplitude is touched once per pass
__device__ __forceinline__ double2 ld_stream(const double2 *p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(double2 *p, double2 v) { __stcs(p, v); }
__device__ __forceinline__ float2 ld_stream(const float2 *p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(float2 *p, float2 v) { __stcs(p, v); }

// Deterministic block reduction (fixed shuffle tree + fixed smem order).
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NT / 32; ++i) t += red[i];
    }
    return t;  // valid in thread 0
}

// Sums `count` partials in index order (one thread; count <= FQ_SCRATCH_DOUBLES).
__global__ void k_sum_partials(const double *partials, int count, double *out);

}  // namespace fq
