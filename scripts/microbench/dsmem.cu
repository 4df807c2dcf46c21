// Feasibility microbenchmark (development only): what does
// moving a tile's data between the CTAs of a thread-block cluster through
// distributed shared memory (DSMEM) cost, against a local shared-memory
// transpose and against the HBM pass it would replace?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem dsmem.cu
//   ./dsmem        (one line per variant: ns per tile step, bytes per clock per SM)
//
// Every CTA owns a 64 KiB complex128 tile (4096 x 16 B, 256 threads x 16
// registers, like k_pass16).  Variants, each iterated `iters` times per CTA:
//   local   : the pass kernel's transpose (16 STS.128 + 16 LDS.128 per thread,
//             two __syncthreads) -- the on-chip cost of one register round;
//   dsmem_w : cluster of C CTAs, every thread stores (C-1)/C of its 16 registers
//             into the peer CTAs' tiles (st.shared::cluster), cluster barrier,
//             reads its own tile back -- the exchange a 2^(12+log2 C)-amplitude
//             cluster tile needs for each round over a cluster bit;
//   dsmem_r : the same with remote loads (ld.shared::cluster) instead of stores.
// Grid: one CTA per SM (148; clusters of C), the pass kernel's 2 CTAs per SM
// are emulated by `ctas_per_sm`.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int kThreads = 256;
constexpr int kRegs = 16;
constexpr int kTile = 4096;
constexpr int kPadded = kTile + kTile / 16;

__device__ __forceinline__ int slot(int e) { return e + (e >> 4); }

__global__ void __launch_bounds__(kThreads, 2) k_local(int iters, double *sink) {
    extern __shared__ double2 sm[];
    const int tid = threadIdx.x;
    double2 v[kRegs];
#pragma unroll
    for (int i = 0; i < kRegs; ++i) v[i] = make_double2(tid + i, blockIdx.x);
    for (int it = 0; it < iters; ++it) {
        // PAT8 -> PAT4 of the pass kernel (additive padded slots)
        double2 *p = sm + tid + (tid >> 4);
#pragma unroll
        for (int i = 0; i < kRegs; ++i) p[272 * i] = v[i];
        __syncthreads();
        const double2 *q = sm + (tid & 15) + 272 * (tid >> 4);
#pragma unroll
        for (int i = 0; i < kRegs; ++i) v[i] = q[17 * i];
        __syncthreads();
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < kRegs; ++i) s += v[i].x + v[i].y;
    if (s == 12345.678) sink[blockIdx.x] = s;
}

// 1-bit register <-> lane swap through warp shuffles (an XY round change of one
// register bit to a lane bit): 8 of 16 registers cross to lane ^ 1
__global__ void __launch_bounds__(kThreads, 2) k_shfl_swap(int iters, double *sink) {
    const int tid = threadIdx.x;
    const bool hi = tid & 1;
    double2 v[kRegs];
#pragma unroll
    for (int i = 0; i < kRegs; ++i) v[i] = make_double2(tid + i, blockIdx.x);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < kRegs / 2; ++i) {
            const double2 send = hi ? v[i] : v[i + kRegs / 2];
            double2 r;
            r.x = __shfl_xor_sync(0xffffffffu, send.x, 1);
            r.y = __shfl_xor_sync(0xffffffffu, send.y, 1);
            if (hi) v[i] = r;
            else v[i + kRegs / 2] = r;
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < kRegs; ++i) s += v[i].x + v[i].y;
    if (s == 12345.678) sink[blockIdx.x] = s;
}

template <int C, bool WRITE>
__global__ void __launch_bounds__(kThreads, 1) k_dsmem(int iters, double *sink) {
    extern __shared__ double2 sm[];
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned rank = cluster.block_rank();
    const int tid = threadIdx.x;
    double2 *peer[C];
#pragma unroll
    for (int r = 0; r < C; ++r) peer[r] = cluster.map_shared_rank(sm, r);
    double2 v[kRegs];
#pragma unroll
    for (int i = 0; i < kRegs; ++i) v[i] = make_double2(tid + i, rank);
    cluster.sync();
    for (int it = 0; it < iters; ++it) {
        // register i belongs to cluster rank (i % C): the (C-1)/C of the registers
        // owned by other ranks cross DSMEM, the rest stays local
        if (WRITE) {
#pragma unroll
            for (int i = 0; i < kRegs; ++i) {
                const int owner = i % C;
                peer[owner][slot(tid + kThreads * (i / C) + (kTile / C) * rank)] = v[i];
            }
            cluster.sync();
#pragma unroll
            for (int i = 0; i < kRegs; ++i) v[i] = sm[slot(tid + kThreads * i)];
            cluster.sync();
        } else {
#pragma unroll
            for (int i = 0; i < kRegs; ++i) sm[slot(tid + kThreads * i)] = v[i];
            cluster.sync();
#pragma unroll
            for (int i = 0; i < kRegs; ++i) {
                const int owner = i % C;
                v[i] = peer[owner][slot(tid + kThreads * (i / C) + (kTile / C) * rank)];
            }
            cluster.sync();
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < kRegs; ++i) s += v[i].x + v[i].y;
    if (s == 12345.678) sink[blockIdx.x] = s;
}

template <typename K>
static float time_kernel(K kern, dim3 grid, size_t smem, int iters, double *sink, int cluster) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    int na = 0;
    if (cluster > 1) {
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cluster;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        na = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    CK(cudaLaunchKernelEx(&cfg, kern, 2, sink));  // warm-up
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a));
    CK(cudaLaunchKernelEx(&cfg, kern, iters, sink));
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms;
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
    double *sink;
    CK(cudaMalloc(&sink, 4096 * sizeof(double)));
    const int iters = 2000;
    const size_t smem = kPadded * sizeof(double2);
    const double tile_bytes = kTile * 16.0;
    // local transpose, 2 CTAs per SM (the pass kernel's occupancy)
    CK(cudaFuncSetAttribute(k_local, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int per_sm = 1; per_sm <= 2; ++per_sm) {
        const float ms = time_kernel(k_local, dim3(per_sm * sms), smem, iters, sink, 1);
        const double ns = ms * 1e6 / iters;  // per transpose step (the CTAs of an SM in parallel)
        const double bytes_per_sm = per_sm * 2 * tile_bytes;  // CTAs x (write + read) of 64 KiB
        printf("{\"variant\": \"local transpose\", \"ctas_per_sm\": %d, \"ns_per_step\": %.1f, "
               "\"smem_B_per_clk_per_sm\": %.1f}\n",
               per_sm, ns, bytes_per_sm / (ns * 1e-9 * clk_khz * 1e3));
    }
    for (int per_sm = 1; per_sm <= 2; ++per_sm) {
        const float ms = time_kernel(k_shfl_swap, dim3(per_sm * sms), 0, iters, sink, 1);
        const double ns = ms * 1e6 / iters;
        printf("{\"variant\": \"shuffle 1-bit swap (8 of 16 registers)\", \"ctas_per_sm\": %d, "
               "\"ns_per_step\": %.1f}\n", per_sm, ns);
    }
    auto run = [&](auto kern, int C, const char *name) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        const int grid = (sms / C) * C;
        const float ms = time_kernel(kern, dim3(grid), smem, iters, sink, C);
        const double ns = ms * 1e6 / iters;
        const double remote = tile_bytes * (C - 1) / C;  // per CTA per step over DSMEM
        printf("{\"variant\": \"%s\", \"cluster\": %d, \"ctas_per_sm\": 1, \"ns_per_step\": %.1f, "
               "\"dsmem_B_per_clk_per_sm\": %.1f, \"hbm_pass_ns_per_tile_equiv\": %.1f}\n",
               name, C, ns, remote / (ns * 1e-9 * clk_khz * 1e3),
               // an HBM pass moves 2 x 64 KiB per tile; at 6.55 TB/s over the SMs:
               2 * tile_bytes / (6.55e12 / sms) * 1e9);
    };
    run(k_dsmem<2, true>, 2, "dsmem_w");
    run(k_dsmem<4, true>, 4, "dsmem_w");
    run(k_dsmem<8, true>, 8, "dsmem_w");
    run(k_dsmem<2, false>, 2, "dsmem_r");
    run(k_dsmem<4, false>, 4, "dsmem_r");
    run(k_dsmem<8, false>, 8, "dsmem_r");
    return 0;
}
