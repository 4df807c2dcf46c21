// Fused global-qubit mixer over peer memory (SURVEY.md §5 option 3).
//
// The reference's Alg. 4 (distributed.py:137-153) mixes the
// k = log2 K global qubits with exchange -> local pass -> exchange: every
// amplitude crosses the interconnect twice and HBM four more times.  Here the
// K shards are mapped into every rank's address space (CUDA IPC handles, or
// plain pointers for the in-process K-worker mode) and ONE kernel applies the
// k single-qubit gates directly: for a local index c, the K amplitudes
// psi_r[c] (r = 0..K-1; global qubit j = bit j of r) form a 2^k-dimensional
// vector transformed in registers.  Rank `part` of `parts` owns the local
// indices [part * size / parts, (part + 1) * size / parts), so every amplitude
// is read once and written once over NVLink by exactly one rank, in place.
// The caller orders the kernel against the other ranks' work (barriers).
#include <cmath>
#include <cstring>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace fq {

constexpr int kMaxGlobal = 4;  // k <= 4 (K <= 16 shards)

struct GlobalParams {
    double2 *shard[1 << kMaxGlobal];
    double2 a[kMaxGlobal], b[kMaxGlobal];  // SU(2) of global qubit j: [[a, -conj b], [b, conj a]]
    long long begin, end;                  // local index range of this rank
    int k;
};

template <int K>
__global__ void __launch_bounds__(256) k_global_su2(const __grid_constant__ GlobalParams P) {
    constexpr int NS = 1 << K;
    for (long long c = P.begin + blockIdx.x * (long long)blockDim.x + threadIdx.x; c < P.end;
         c += (long long)gridDim.x * blockDim.x) {
        double2 v[NS];
#pragma unroll
        for (int r = 0; r < NS; ++r) v[r] = __ldcg(P.shard[r] + c);
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const double2 a = P.a[j], b = P.b[j];
#pragma unroll
            for (int r = 0; r < NS; ++r) {
                if (r & (1 << j)) continue;
                const double2 x0 = v[r], x1 = v[r | (1 << j)];
                // y0 = a x0 - conj(b) x1 ; y1 = b x0 + conj(a) x1   (reference _kernels.py:26-27)
                v[r] = make_double2(a.x * x0.x - a.y * x0.y - b.x * x1.x - b.y * x1.y,
                                    a.x * x0.y + a.y * x0.x - b.x * x1.y + b.y * x1.x);
                v[r | (1 << j)] = make_double2(b.x * x0.x - b.y * x0.y + a.x * x1.x + a.y * x1.y,
                                               b.x * x0.y + b.y * x0.x + a.x * x1.y - a.y * x1.x);
            }
        }
#pragma unroll
        for (int r = 0; r < NS; ++r) __stcg(P.shard[r] + c, v[r]);
    }
}

// Device-side barrier over peer memory: rank r stores `epoch` into slot r of
// every rank's flag array (remote stores over NVLink), then spins until all K
// slots of its own array reach `epoch`.  Stream-ordered: the work enqueued
// before it on every rank is complete (and, after the system fence, visible
// to the peers) when any rank passes it — no host synchronisation.  A rank
// that never arrives trips the timeout (10 s of %globaltimer, a nanosecond
// clock independent of the SM clock and of which device runs it): *err is set
// and the kernel returns instead of hanging the device; the host side
// (ShardedQaoaSimulator.check_barrier) reports it after every program.
struct BarrierParams {
    unsigned *flags[1 << kMaxGlobal];  // rank q's flag array (K slots), peer-mapped
    int K, rank;
    unsigned epoch;
    int *err;
    unsigned long long timeout_ns;
};

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_peer_barrier(const __grid_constant__ BarrierParams P) {
    const int t = threadIdx.x;
    __threadfence_system();
    __syncthreads();
    if (t < P.K) {
        volatile unsigned *remote = P.flags[t];
        remote[P.rank] = P.epoch;
    }
    __threadfence_system();
    if (t < P.K) {
        volatile unsigned *mine = P.flags[P.rank];
        const unsigned long long t0 = global_ns();
        while ((int)(mine[t] - P.epoch) < 0) {
            if (global_ns() - t0 > P.timeout_ns) {
                atomicExch(P.err, 1);
                break;
            }
            __nanosleep(64);
        }
    }
    __syncthreads();
    __threadfence_system();
}

}  // namespace fq

using namespace fq;

extern "C" {

int fq_global_su2_pass(void *const *shards, int k, int64_t shard_size, int part, int parts, const double *su2,
                       void *stream) {
    FQ_CHECK_ARG(shards && su2 && k >= 1 && k <= kMaxGlobal, "fq_global_su2_pass: k=%d must be in [1, %d]", k,
                 kMaxGlobal);
    FQ_CHECK_ARG(shard_size >= 1 && parts >= 1 && part >= 0 && part < parts, "fq_global_su2_pass: bad partition");
    GlobalParams P;
    for (int r = 0; r < (1 << k); ++r) {
        FQ_CHECK_ARG(shards[r] != nullptr, "fq_global_su2_pass: null shard %d", r);
        P.shard[r] = static_cast<double2 *>(shards[r]);
    }
    for (int j = 0; j < k; ++j) {
        P.a[j] = make_double2(su2[4 * j + 0], su2[4 * j + 1]);
        P.b[j] = make_double2(su2[4 * j + 2], su2[4 * j + 3]);
    }
    P.begin = shard_size * part / parts;
    P.end = shard_size * (part + 1) / parts;
    P.k = k;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int grid = grid_for(P.end - P.begin, 256, 4);
    switch (k) {
        case 1: k_global_su2<1><<<grid, 256, 0, st>>>(P); break;
        case 2: k_global_su2<2><<<grid, 256, 0, st>>>(P); break;
        case 3: k_global_su2<3><<<grid, 256, 0, st>>>(P); break;
        default: k_global_su2<4><<<grid, 256, 0, st>>>(P); break;
    }
    FQ_LAUNCHED("k_global_su2");
    return FQ_OK;
}

// IPC handles name a whole cudaMalloc allocation; a tensor from a caching
// allocator may sit at an offset inside it, so the offset travels with the handle.
static CUresult alloc_base(const void *ptr, CUdeviceptr *base) {
    static PFN_cuMemGetAddressRange_v3020 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return CUDA_ERROR_NOT_FOUND;
        fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(p);
    }
    size_t size = 0;
    return fn(base, &size, reinterpret_cast<CUdeviceptr>(ptr));
}

int fq_ipc_handle(const void *dev_ptr, void *handle_out, int64_t *offset_out) {
    FQ_CHECK_ARG(dev_ptr && handle_out && offset_out, "fq_ipc_handle: null argument");
    CUdeviceptr base = 0;
    if (alloc_base(dev_ptr, &base) != CUDA_SUCCESS) {
        set_error("fq_ipc_handle: cuMemGetAddressRange failed");
        return FQ_ERR_CUDA;
    }
    cudaIpcMemHandle_t h;
    FQ_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base)));
    std::memcpy(handle_out, &h, sizeof h);
    *offset_out = (int64_t)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
    return FQ_OK;
}

int fq_ipc_open(const void *handle, int64_t offset, void **dev_ptr_out) {
    FQ_CHECK_ARG(handle && dev_ptr_out, "fq_ipc_open: null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    void *base = nullptr;
    FQ_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *dev_ptr_out = static_cast<char *>(base) + offset;
    return FQ_OK;
}

int fq_peer_barrier(void *const *flag_arrays, int K, int rank, unsigned epoch, int *err_dev, void *stream) {
    FQ_CHECK_ARG(flag_arrays && err_dev && K >= 1 && K <= (1 << kMaxGlobal) && rank >= 0 && rank < K,
                 "fq_peer_barrier: bad arguments (K <= %d)", 1 << kMaxGlobal);
    BarrierParams P;
    for (int q = 0; q < K; ++q) P.flags[q] = static_cast<unsigned *>(flag_arrays[q]);
    P.K = K;
    P.rank = rank;
    P.epoch = epoch;
    P.err = err_dev;
    P.timeout_ns = 10ULL * 1000 * 1000 * 1000;  // 10 s
    k_peer_barrier<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(P);
    FQ_LAUNCHED("k_peer_barrier");
    return FQ_OK;
}

int fq_ipc_close(void *dev_ptr, int64_t offset) {
    FQ_CHECK_ARG(dev_ptr, "fq_ipc_close: null pointer");
    FQ_CUDA(cudaIpcCloseMemHandle(static_cast<char *>(dev_ptr) - offset));
    return FQ_OK;
}

}  // extern "C"
