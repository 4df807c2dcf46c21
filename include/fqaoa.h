/*
 * fqaoa.h — C ABI of the B200-native QAOA hot path (libfqaoa.so, sm_100a).
 *
 * This is the drop-in seam for the reference's operator layer,
 * fastqaoa/_kernels.py (the numba kernels every higher layer calls), plus
 * fused entry points the per-qubit seam cannot express.
 *
 * Conventions (all functions):
 *   - every pointer is a caller-owned DEVICE buffer unless noted "host";
 *   - states are interleaved complex128 (re, im doubles), index bit q = qubit q
 *     (reference statevec.py:3-4); cost vectors are float64 or uint16 levels;
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); work is
 *     enqueued asynchronously and nothing here synchronises the host except
 *     where stated;
 *   - return 0 on success, otherwise an FQ_ERR_* code; fq_last_error() gives a
 *     thread-local message.  No exception ever crosses the ABI;
 *   - nothing allocates memory proportional to 2^n (in-place contract of
 *     reference _kernels.py:1-6).  Reductions take `scratch`, a device buffer
 *     of at least FQ_SCRATCH_DOUBLES doubles.
 */
#ifndef FQAOA_H
#define FQAOA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FQ_OK 0
#define FQ_ERR_ARG 1
#define FQ_ERR_CUDA 2
#define FQ_ERR_UNSUPPORTED 3

#define FQ_SCRATCH_DOUBLES 4096

/* mixer kinds (reference mixers.py:140-199, Mixer.KINDS) */
#define FQ_MIXER_X 0
#define FQ_MIXER_XY_RING 1
#define FQ_MIXER_XY_COMPLETE 2
#define FQ_MIXER_CUSTOM 3

/* cost-vector encodings */
#define FQ_COST_F64 0 /* double per amplitude (terms.py:102-120 output)       */
#define FQ_COST_U16 1 /* uint16 level v, cost = scale*v + offset (terms.py:123-175) */

/* state element types (fq_evolve_desc.state_kind) */
#define FQ_STATE_C128 0 /* complex128: the reference's state (default)        */
#define FQ_STATE_C64 1  /* complex64: optional single-precision state         */

int fq_version(void);
const char *fq_last_error(void);
/* Number of SMs of the current device (grid sizing), or -1. */
int fq_sm_count(void);

/* ------------------------------------------------------------------ *
 * Operator layer — one entry per reference kernel.                     *
 * ------------------------------------------------------------------ */

/* replaces su2_on_pairs — reference _kernels.py:14-27 (callers mixers.py:71,84,91,
 * distributed.py:147,152).  Pairs (l, l|2^q): y0 = a x0 - conj(b) x1,
 * y1 = b x0 + conj(a) x1. */
int fq_su2_on_pairs(void *psi, int64_t size, double a_re, double a_im, double b_re,
                    double b_im, int q, void *stream);

/* replaces xy_on_pairs — reference _kernels.py:30-48 (callers mixers.py:106,
 * distributed.py:181,202).  Requires p_lo < p_hi. */
int fq_xy_on_pairs(void *psi, int64_t size, double cos_b, double sin_b, int p_lo, int p_hi,
                   void *stream);

/* replaces swap_bits — reference _kernels.py:51-65 (callers distributed.py:194,207). */
int fq_swap_bits(void *psi, int64_t size, int p_lo, int p_hi, void *stream);

/* replaces phase_multiply — reference _kernels.py:68-73 (callers statevec.py:78,
 * distributed.py:134).  psi[k] *= exp(-i gamma costs[k]). */
int fq_phase_multiply(void *psi, const double *costs, int64_t size, double gamma, void *stream);

/* replaces accumulate_terms — reference _kernels.py:76-94 (caller terms.py:118).
 * out[k] += sum_t w_t (-1)^popcount((index_base+k) & masks[t]), accumulated per
 * element left-to-right in term order exactly like the reference (bit-exact for
 * any float weights).  index_base lets a shard evaluate its global slice. */
int fq_accumulate_terms(double *out, int64_t size, const double *weights, const int64_t *masks,
                        int64_t n_terms, int64_t index_base, void *stream);

/* Exact-integer variant of fq_accumulate_terms for dyadic weights:
 * w_t = iweights[t] * 2^-shift.  Accumulates in int64 and converts once, which
 * equals the reference's sequential double sum bit-for-bit whenever
 * sum_t |iweights[t]| < 2^53 (the host checks this before choosing it).
 * acc_bits = 32 selects an int32 accumulator (valid when sum_t |iweights[t]| < 2^31),
 * 64 an int64 one. */
int fq_accumulate_terms_dyadic(double *out, int64_t size, const int64_t *iweights,
                               const int64_t *masks, int64_t n_terms, int shift, int acc_bits,
                               int64_t index_base, void *stream);

/* The same diagonal (dyadic weights w_t = iweights[t] * 2^-shift, sum |iweights| < 2^53)
 * as a Walsh-Hadamard transform of the term weights: out = WHT(a), a[m] = sum of the
 * weights with mask m — n * 2^n exact additions instead of T * 2^n parities, bit-identical
 * to the reference's sequential sum.  size = 2^n_local >= 4096; a shard's index_base is a
 * multiple of size (global bits fold into term signs).  Overwrites out. */
int fq_precompute_wht(double *out, int64_t size, const int64_t *iweights, const int64_t *masks, int64_t n_terms,
                      int shift, int64_t index_base, void *stream);

/* Same exact-integer accumulation, emitted directly as uint16 levels
 * v = (S(k) - level_offset) >> level_shift where S(k) = sum_t iweights[t]*sign.
 * Used when the float64 diagonal does not fit (n=34, K=2).  *bad_dev (device
 * int) is set nonzero if any value falls outside [0, 65535] or off the grid. */
int fq_precompute_levels_u16(uint16_t *out, int64_t size, const int64_t *iweights,
                             const int64_t *masks, int64_t n_terms, int acc_bits, int64_t index_base,
                             int64_t level_offset, int level_shift, int *bad_dev, void *stream);

/* replaces abs2_inplace — reference _kernels.py:97-102 (caller statevec.py:90). */
int fq_abs2_inplace(void *psi, int64_t size, void *stream);

/* ------------------------------------------------------------------ *
 * States and observables (reference statevec.py)                      *
 * ------------------------------------------------------------------ */

/* uniform_state (statevec.py:22-29) when weight < 0, else
 * hamming_weight_state (statevec.py:41-54) restricted to the slice
 * [index_base, index_base+size).  amp = amplitude value of the support. */
int fq_init_state(void *psi, int64_t size, int weight, double amp, int64_t index_base,
                  void *stream);

/* expectation (statevec.py:94-97): *out_dev = sum_k c_k |psi_k|^2.  Deterministic
 * two-stage fp64 reduction.  cost_kind FQ_COST_F64 (costs = double*) or FQ_COST_U16
 * (costs = uint16_t*, c = scale*v + offset). */
int fq_expectation(const void *psi, const void *costs, int cost_kind, double scale,
                   double offset, int64_t size, double *out_dev, double *scratch, void *stream);

/* min / max of the decoded cost vector: out_dev[0] = min, out_dev[1] = max. */
int fq_cost_minmax(const void *costs, int cost_kind, double scale, double offset, int64_t size,
                   double *out_dev, double *scratch, void *stream);

/* overlap numerator (statevec.py:100-111): *out_dev = sum_{c_k <= cutoff} |psi_k|^2
 * (cutoff = min + tol, computed by the caller — globally for sharded runs). */
int fq_masked_probability(const void *psi, const void *costs, int cost_kind, double scale,
                          double offset, int64_t size, double cutoff, double *out_dev,
                          double *scratch, void *stream);

/* complex64 states (an optional single-precision path the reference does not
 * have; north star: "complex128, with complex64 optional", 1e-4 tolerance):
 * the same operations on interleaved float re/im.  Observables accumulate
 * in fp64. */
int fq_init_state_c64(void *psi, int64_t size, int weight, double amp, int64_t index_base,
                      void *stream);
int fq_abs2_inplace_c64(void *psi, int64_t size, void *stream);
int fq_expectation_c64(const void *psi, const void *costs, int cost_kind, double scale,
                       double offset, int64_t size, double *out_dev, double *scratch, void *stream);
int fq_masked_probability_c64(const void *psi, const void *costs, int cost_kind, double scale,
                              double offset, int64_t size, double cutoff, double *out_dev,
                              double *scratch, void *stream);

/* levels[k] -= delta for every k (delta may be negative; the caller keeps
 * every level in [0, 65535]): moves the level origin — to the diagonal's
 * minimum after packing from a bound, or to a common origin across shards —
 * with the decode offset moving by delta*scale, exactly.  levels 16-B aligned. */
int fq_rebase_u16(uint16_t *levels, int64_t size, int delta, void *stream);

/* Lossless uint16 packing of a float64 diagonal (terms.py:155-175):
 * out[k] = rint((c_k - offset)/scale); *bad_dev set nonzero if any level > 65535 or
 * scale*v + offset != c_k bit-for-bit. */
int fq_compact_u16(uint16_t *out, const double *costs, int64_t size, double scale, double offset,
                   int *bad_dev, void *stream);

/* ------------------------------------------------------------------ *
 * Fused evolution (the B200 hot path)                                 *
 * ------------------------------------------------------------------ */

/* One layer of a fused program.  Layer l applies, in order,
 * exp(-i gamma costs) (if apply_phase && gamma != 0) and then the mixer with
 * angle beta restricted to qubit positions [q_lo, q_hi) (X / custom kinds).
 * XY kinds always act on the full gate list of the local register. */
typedef struct fq_layer {
    double gamma;
    double beta;
    int apply_phase;
    int q_lo, q_hi;
} fq_layer;

typedef struct fq_evolve_desc {
    void *psi;            /* complex128[2^n] device, in/out                          */
    int n;                /* local qubit count (log2 of the buffer length)           */
    int cost_kind;        /* FQ_COST_F64 / FQ_COST_U16                               */
    const void *costs;    /* device, same slicing as psi                             */
    double cost_scale;    /* U16 decode: c = scale*v + offset                        */
    double cost_offset;
    int cost_levels;      /* U16: 1 + largest level present (0 = unknown); sizes the
                             phase tables (< 16384 -> table lookups, else sincos)    */
    int mixer;            /* FQ_MIXER_*                                              */
    int n_layers;
    const fq_layer *layers;   /* host array [n_layers]                               */
    const double *su2;    /* host, FQ_MIXER_CUSTOM only: [n_layers][n][4] = a_re,a_im,b_re,b_im */
    int init;             /* 0: psi holds the initial state; 1: start from |+>^n     */
    double init_amp;      /* amplitude used when init == 1 (reference: 1/sqrt(2^n_global)) */
    double *expectation_dev;  /* if non-NULL: sum_k c_k |psi_k|^2 of the final state  */
    double *scratch;      /* device, >= FQ_SCRATCH_DOUBLES doubles                   */
    int state_kind;       /* FQ_STATE_C128 (default, zero) / FQ_STATE_C64: psi is
                             complex64[2^n]; X / custom mixers, n > 12               */
} fq_evolve_desc;

/* Runs the whole p-layer program: phase fused into the first mixer pass of
 * each layer, X/custom mixers applied 12 qubits per HBM pass in registers +
 * shared memory, consecutive layers' passes fused across the layer boundary,
 * expectation fused into the last pass.  States of n <= 12 qubits run the
 * whole program inside one CTA. */
int fq_qaoa_evolve(const fq_evolve_desc *desc, void *stream);

/* One objective evaluation, synchronous (the optimiser-loop call, reference
 * qaoa_objective / QaoaSimulator.get_expectation(simulate_qaoa(...)),
 * qaoa.py:137-149,185-194): fq_qaoa_evolve with desc->expectation_dev set,
 * then the objective copied to *out_host and the stream synchronised — one
 * ABI crossing per evaluation. */
int fq_qaoa_objective(const fq_evolve_desc *desc, double *out_host, void *stream);

/* The same evaluation for small states (n <= 12, X mixer from |+>, complex128,
 * p <= 64) as a captured CUDA graph replayed per call (the optimiser loop of
 * BASELINE config 1): create() captures the one-CTA resident program once per
 * descriptor, reading the angles ang_host[2p] = (gamma_l, beta_l) from and
 * writing the objective to *out_host -- both PINNED host buffers, accessed by
 * the kernel directly (no copies); run() launches the graph on `stream` (after
 * the caller wrote new angles into ang_host) and returns once the kernel has
 * published the objective (it spins on a pinned completion flag; the stream
 * may still be retiring the kernel).  desc's device buffers (state, costs)
 * must outlive the handle; the final state is not written back. */
int fq_objective_graph_create(const fq_evolve_desc *desc, const double *ang_host, double *out_host, void **handle);
int fq_objective_graph_run(void *handle, void *stream);
int fq_objective_graph_destroy(void *handle);

/* Batched small-n evolution: `batch` independent parameter sets (gammas/betas
 * host arrays [batch][p]) for the same cost vector, each evolved from |+>^n
 * (or from psi_init if non-NULL, complex128[2^n] device) entirely on chip;
 * writes expectations to out_dev[batch] and, if psi_out is non-NULL, final
 * states to psi_out[batch][2^n].  n <= 12, X or custom-free kinds. */
int fq_qaoa_evolve_batched(int n, int mixer, const void *costs, int cost_kind, double scale,
                           double offset, int p, int batch, const double *gammas,
                           const double *betas, const void *psi_init, void *psi_out,
                           double *out_dev, void *stream);
/* The same with the number of uint16 cost levels (cost_kind = FQ_COST_U16:
 * the phase then comes from two e^{-i gamma c} tables per layer instead of a
 * sincos per amplitude; 0 = unknown).  Parameter sets run one per CTA. */
int fq_qaoa_evolve_batched_levels(int n, int mixer, const void *costs, int cost_kind, double scale,
                                  double offset, int cost_levels, int p, int batch,
                                  const double *gammas, const double *betas, const void *psi_init,
                                  void *psi_out, double *out_dev, void *stream);

/* A state sharded over K = 2^k ranks by its top k ("global") qubits
 * (reference distributed.py:51-54): shard r holds global indices
 * [r 2^n_local, (r+1) 2^n_local). */
typedef struct fq_shard_desc {
    int k;                          /* global qubits, 1..3 (K = 2..8 shards)                 */
    int rank;                       /* this process's shard; -1: all K shards are this
                                       process's (one device, one stream: the reference's
                                       in-process worker model)                            */
    void *const *shards;            /* [K] state shards (desc->state_kind) as mapped in this
                                       process (peers via fq_ipc_open)                       */
    const void *const *costs;       /* [K] cost shards, one encoding / scale / offset        */
    void *const *flags;             /* [K] peer flag arrays of fq_peer_barrier (rank >= 0)   */
    unsigned *epoch;                /* host: last barrier epoch used; advanced by the call   */
    int *barrier_err;               /* device error word of the barrier                      */
} fq_shard_desc;

/* The fused program on a sharded state (replaces the reference's per-layer
 * Alg. 4 — local sweeps, all_to_all_exchange, k-position sweep, exchange —
 * distributed.py:137-157): ONE plan over all n = n_local + k qubits.  Groups
 * of local qubits run as ordinary passes on the rank's own shard; the group
 * holding the k global qubits runs as one pass whose 2^12-amplitude tiles span
 * all K shards over peer memory (NVLink), rank r taking 1/K of the tiles, with
 * stream-ordered device barriers (fq_peer_barrier) before and after it.  Layer
 * fusion works across the global group like any other, so global passes are
 * about one per two layers, each moving (K-1)/K of its bytes over NVLink once.
 * desc->n = n_local; desc->psi / desc->costs are ignored (shards / costs
 * below); layer qubit ranges and the custom su2 table use global positions
 * [0, n); desc->init_amp = 2^(-n/2); desc->expectation_dev receives this
 * rank's partial sum (rank >= 0: all-reduce it) or the total (rank = -1).
 * XY mixers: the tiled XY plan over all n qubits; a pass whose tile holds
 * global qubits spans the shards it covers, each rank taking the tiles of its
 * own shard set (replaces the reference's park-and-exchange per global pair,
 * distributed.py:160-207).  complex128 (any mixer) or complex64 (X / XY),
 * n_local >= 12. */
int fq_qaoa_evolve_sharded(const fq_evolve_desc *desc, const fq_shard_desc *shards, void *stream);

/* Pass count of fq_qaoa_evolve_sharded's plan and, in *global_passes, how many
 * of them span the shards (peer-memory passes). */
int fq_plan_sharded_passes(int n_local, int k, int n_layers, const fq_layer *layers, int *global_passes);

/* Number of HBM passes fq_qaoa_evolve will run for an X-mixer program on a
 * state of state_kind (FQ_STATE_*; the plan depends on the bytes per
 * amplitude), for the byte model in bench.py / DESIGN.md. */
int fq_plan_x_passes(int n, int n_layers, const fq_layer *layers, int state_kind);

/* ------------------------------------------------------------------ *
 * Sharded state over peer memory                                       *
 * ------------------------------------------------------------------ */

/* Fused global-qubit mixer (replaces the exchange -> k-position pass ->
 * exchange of reference distributed.py:137-153 / Alg. 4): shards[r] (host
 * array of 2^k device pointers, all shard_size amplitudes, peer-mapped) hold
 * the state slice of global index r; applies su2[j] = (a_re, a_im, b_re, b_im)
 * to global qubit j (bit j of r) for the local indices of part `part` of
 * `parts` (each rank / worker passes its own part), in place.  The caller
 * orders it against the other parts' work. */
int fq_global_su2_pass(void *const *shards, int k, int64_t shard_size, int part, int parts, const double *su2,
                       void *stream);

/* CUDA IPC of a device buffer (any pointer inside a cudaMalloc allocation):
 * 64-byte handle + offset; open maps it into this process (same or peer GPU). */
int fq_ipc_handle(const void *dev_ptr, void *handle_out, int64_t *offset_out);
int fq_ipc_open(const void *handle, int64_t offset, void **dev_ptr_out);
int fq_ipc_close(void *dev_ptr, int64_t offset);

/* Stream-ordered barrier over peer memory (no host synchronisation):
 * flag_arrays[q] = rank q's uint32[K] flag array (peer-mapped, zero-initialised);
 * rank `rank` stores `epoch` into slot `rank` of every array, then waits until
 * all K slots of its own array reach `epoch` (epochs increase by one per
 * barrier, identically on every rank).  On a 10 s timeout (device
 * %globaltimer) *err_dev is set and the kernel returns.  K <= 16. */
int fq_peer_barrier(void *const *flag_arrays, int K, int rank, unsigned epoch, int *err_dev, void *stream);

/* Host-only description of the tiled X/custom plan (no device needed): the
 * qubit groups ("groups=t,t,../runR;..": target qubits, contiguous-run bits of
 * the tile) and the pass sequence ("passes=g[f|d],..": group index, f = fused
 * two layers with the phase between, d = two layers without phase, P = a
 * standalone phase sweep) of an n-qubit register whose top k qubits are
 * global (k = 0: one state).  Honours fq_set_option("plan"/"plan_tmax").
 * Returns the pass count (or -1); writes at most len bytes to buf. */
int fq_plan_x_describe(int n, int n_layers, const fq_layer *layers, int state_kind, int k, char *buf, int len);

/* HBM passes per layer of the tiled XY program (ring / complete gate order of
 * reference mixers.py:109-125) at n qubits; 1 for n <= 12 (on chip), -1 for other
 * kinds.  *rounds (if non-NULL): register rounds summed over the passes. */
int fq_plan_xy_passes(int n, int mixer, int *rounds);

/* Passes of the last tiled X/custom program run on this host thread's
 * process: returns the pass count; for i < max fills info[5*i..5*i+4] =
 * (round program: 0 = 8|0|4, 1 = 8|4, 2 = 8|0|4|0|8, 3 = 8|4|8, -1 = standalone
 * phase; phase mode; target count; generates |+>; accumulates the expectation)
 * and, with option "time_passes" on, ms[i] = CUDA-event time of pass i on the
 * launching stream (synchronises with the program's last event).  NULL
 * arrays are skipped. */
int fq_last_passes(int *info, float *ms, int max);

/* Runtime switches (testing / A-B measurement; Python: FQ_OPTIONS="name=value,..."
 * applies them when the library is loaded).  The main ones:
 *   "prefetch"     L2 tensor-prefetch distance of the pass kernel in grid strides
 *                  (default -1: 1 for runs >= 256 B, else 0)
 *   "fuse"         fuse the passes at layer boundaries (default 1)
 *   "phase_tables" uint16 phase through shared-memory tables (default 1, 0 = sincos)
 *   "plan"         group plan: -1 cost model (default), 0 legacy, 1 small fusion groups
 *   "plan_tmax"    force the high-group chunk size (0 = cost model; plan-shape tests)
 *   "lane3"        9-target high groups as two-pattern programs with tile bit 3 as
 *                  warp-shuffle butterflies (default 1)
 *   "cost_l2"      cost loads at normal L2 priority (-1 = when cost runs < 32 B, default)
 *   "cost_stage"   uint16 costs of the mid-layer phase / expectation through a shared
 *                  cost tile (default 1)
 *   "time_passes"  record a CUDA event after every pass (read with fq_last_passes)
 *   "xy_tiled"     tiled XY passes (default 1; 0 = one pair kernel per gate)
 * The full list (with ranges) is the table in evolve.cu:fq_set_option. */
int fq_set_option(const char *name, int value);

#ifdef __cplusplus
}
#endif
#endif /* FQAOA_H */
