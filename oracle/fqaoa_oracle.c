/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the QAOA hot path.
 *
 * Plain-C restatement of the six numba kernels of the reference
 * (fastqaoa/_kernels.py).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library, and
 * only as the checker or the timed CPU baseline.  The product path
 * (paper_2309_04841_b200/) never links or calls it.
 *
 * Every loop mirrors the reference's iteration order per output element:
 * the per-element arithmetic (operand order, no FMA contraction — build with
 * -ffp-contract=off) is the reference's, so integer / dyadic diagonals are
 * bit-identical and float-weight diagonals follow the same left-to-right
 * accumulation.  Parallelism is OpenMP over disjoint output indices, the
 * same decomposition as numba's prange.
 *
 * Parity pin: tests/test_oracle_golden.py checks this library against
 * vectors produced by the reference itself (scripts/gen_golden.py).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>

typedef double _Complex c128;

/* su2_on_pairs — reference pkg/src/fastqaoa/_kernels.py:14-27 */
void or_su2_on_pairs(c128 *psi, int64_t size, double a_re, double a_im,
                     double b_re, double b_im, int q) {
    const int64_t bit = (int64_t)1 << q;
    const int64_t low = bit - 1;
    const int64_t half = size >> 1;
#pragma omp parallel for schedule(static)
    for (int64_t g = 0; g < half; ++g) {
        int64_t l0 = ((g >> q) << (q + 1)) | (g & low);
        int64_t l1 = l0 | bit;
        double x0r = creal(psi[l0]), x0i = cimag(psi[l0]);
        double x1r = creal(psi[l1]), x1i = cimag(psi[l1]);
        /* y0 = a*x0 - conj(b)*x1 ; y1 = b*x0 + conj(a)*x1 (line 26-27) */
        double ax0r = a_re * x0r - a_im * x0i, ax0i = a_re * x0i + a_im * x0r;
        double bcx1r = b_re * x1r + b_im * x1i, bcx1i = b_re * x1i - b_im * x1r;
        double bx0r = b_re * x0r - b_im * x0i, bx0i = b_re * x0i + b_im * x0r;
        double acx1r = a_re * x1r + a_im * x1i, acx1i = a_re * x1i - a_im * x1r;
        psi[l0] = CMPLX(ax0r - bcx1r, ax0i - bcx1i);
        psi[l1] = CMPLX(bx0r + acx1r, bx0i + acx1i);
    }
}

/* xy_on_pairs — reference _kernels.py:30-48 (requires p_lo < p_hi) */
void or_xy_on_pairs(c128 *psi, int64_t size, double cos_b, double sin_b,
                    int p_lo, int p_hi) {
    const int64_t bit_lo = (int64_t)1 << p_lo, bit_hi = (int64_t)1 << p_hi;
    const int64_t m_lo = bit_lo - 1, m_hi = bit_hi - 1;
    const int64_t quarter = size >> 2;
#pragma omp parallel for schedule(static)
    for (int64_t g = 0; g < quarter; ++g) {
        int64_t t = ((g >> p_lo) << (p_lo + 1)) | (g & m_lo);
        int64_t base = ((t >> p_hi) << (p_hi + 1)) | (t & m_hi);
        int64_t l_lo = base | bit_lo, l_hi = base | bit_hi;
        double xlr = creal(psi[l_lo]), xli = cimag(psi[l_lo]);
        double xhr = creal(psi[l_hi]), xhi = cimag(psi[l_hi]);
        /* c*x_lo + (-i s)*x_hi ; (-i s)*x_lo + c*x_hi (lines 47-48) */
        psi[l_lo] = CMPLX(cos_b * xlr + sin_b * xhi, cos_b * xli - sin_b * xhr);
        psi[l_hi] = CMPLX(sin_b * xli + cos_b * xhr, -sin_b * xlr + cos_b * xhi);
    }
}

/* swap_bits — reference _kernels.py:51-65 */
void or_swap_bits(c128 *psi, int64_t size, int p_lo, int p_hi) {
    const int64_t bit_lo = (int64_t)1 << p_lo, bit_hi = (int64_t)1 << p_hi;
    const int64_t m_lo = bit_lo - 1, m_hi = bit_hi - 1;
    const int64_t quarter = size >> 2;
#pragma omp parallel for schedule(static)
    for (int64_t g = 0; g < quarter; ++g) {
        int64_t t = ((g >> p_lo) << (p_lo + 1)) | (g & m_lo);
        int64_t base = ((t >> p_hi) << (p_hi + 1)) | (t & m_hi);
        c128 tmp = psi[base | bit_lo];
        psi[base | bit_lo] = psi[base | bit_hi];
        psi[base | bit_hi] = tmp;
    }
}

/* phase_multiply — reference _kernels.py:68-73 */
void or_phase_multiply(c128 *psi, const double *costs, int64_t size, double gamma) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < size; ++k) {
        double angle = gamma * costs[k];
        double c = cos(angle), s = -sin(angle);
        double xr = creal(psi[k]), xi = cimag(psi[k]);
        psi[k] = CMPLX(xr * c - xi * s, xr * s + xi * c);
    }
}

/* accumulate_terms — reference _kernels.py:76-94.  `base` offsets the
 * index (a shard of a larger vector: element k has global index base+k). */
void or_accumulate_terms(double *out, int64_t size, const double *weights,
                         const int64_t *masks, int64_t n_terms, int64_t base) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < size; ++k) {
        double acc = 0.0;
        int64_t idx = base + k;
        for (int64_t t = 0; t < n_terms; ++t) {
            uint64_t x = (uint64_t)(idx & masks[t]);
            x ^= x >> 32; x ^= x >> 16; x ^= x >> 8;
            x ^= x >> 4;  x ^= x >> 2;  x ^= x >> 1;
            if (x & 1) acc -= weights[t];
            else acc += weights[t];
        }
        out[k] += acc;
    }
}

/* abs2_inplace — reference _kernels.py:97-102 */
void or_abs2_inplace(c128 *psi, int64_t size) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < size; ++k) {
        double xr = creal(psi[k]), xi = cimag(psi[k]);
        psi[k] = CMPLX(xr * xr + xi * xi, 0.0);
    }
}

/* expectation — reference statevec.py:94-97 (np.dot(costs, |psi|^2)).
 * Sequential fp64 sum per thread chunk, chunks combined in order. */
double or_expectation(const c128 *psi, const double *costs, int64_t size) {
    double total = 0.0;
#pragma omp parallel for reduction(+ : total) schedule(static)
    for (int64_t k = 0; k < size; ++k) {
        double xr = creal(psi[k]), xi = cimag(psi[k]);
        total += costs[k] * (xr * xr + xi * xi);
    }
    return total;
}

int or_num_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
