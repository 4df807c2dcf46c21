// Feasibility microbenchmark (development only): can two consecutive passes
// over a 1 GiB state share ONE HBM round trip if the state is processed in
// L2-resident slabs by teams of CTAs (sub-pass 1 over the slab, team barrier,
// sub-pass 2 over the same slab while it is still in L2)?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_sweep l2_sweep.cu
//   ./l2_sweep            (prints ms of: 2 plain passes, sweeps at several slab / team sizes)
//
// Sub-pass k reads 16 B per amplitude and writes it back (x*1.0000001): the
// byte pattern of a tiled pass with contiguous 64 KiB tiles.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int kThreads = 256;
constexpr int kTileAmps = 4096;  // 64 KiB

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ void team_barrier(unsigned *ctr, unsigned target, int *err) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        const unsigned long long t0 = gtime();
        while (ld_acquire(ctr) < target) {
            if (gtime() - t0 > 2000000000ULL) { atomicExch(err, 1); break; }
        }
        __threadfence();
    }
    __syncthreads();
}

// mode 0: evict-normal stores; 1: intermediate stores with L2::evict_last policy
template <int MODE>
__device__ __forceinline__ void tile_rw(double2 *psi, long long base, bool from_l2, bool final_store, double f,
                                        unsigned long long pol) {
    double2 v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const double2 *p = psi + base + threadIdx.x + i * kThreads;
        v[i] = from_l2 ? __ldcg(p) : __ldcs(p);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) { v[i].x *= f; v[i].y *= f; }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        double2 *p = psi + base + threadIdx.x + i * kThreads;
        if (final_store) __stcs(p, v[i]);
        else if (MODE == 1)
            asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v[i].x), "d"(v[i].y), "l"(pol) : "memory");
        else __stcg(p, v[i]);
    }
}

// plain pass: grid-stride over tiles
__global__ void __launch_bounds__(kThreads, 2) k_plain(double2 *psi, long long n_tiles, double f) {
    for (long long t = blockIdx.x; t < n_tiles; t += gridDim.x) tile_rw<0>(psi, t * kTileAmps, false, true, f, 0);
}

// sweep: team = blockIdx.x / G; slab = tiles [s*T, (s+1)*T); sub-pass 1 then 2 per slab
template <int MODE>
__global__ void __launch_bounds__(kThreads, 2) k_sweep(double2 *psi, long long n_slabs, int tiles_per_slab, int G,
                                                       int n_teams, unsigned *ctr, int *err, double f) {
    const int team = blockIdx.x / G, tr = blockIdx.x % G;
    if (team >= n_teams) return;
    unsigned long long pol = 0;
    if (MODE == 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    unsigned nb = 0;
    for (long long s = team; s < n_slabs; s += n_teams) {
        const long long t0 = s * tiles_per_slab;
        for (int j = tr; j < tiles_per_slab; j += G) tile_rw<MODE>(psi, (t0 + j) * kTileAmps, false, false, f, pol);
        team_barrier(ctr + team * 32, (unsigned)(G * ++nb), err);
        for (int j = tr; j < tiles_per_slab; j += G) tile_rw<MODE>(psi, (t0 + j) * kTileAmps, true, true, f, pol);
    }
}

int main() {
    const long long n_amps = 1LL << 26;  // 1 GiB complex128
    double2 *psi;
    CK(cudaMalloc(&psi, n_amps * sizeof(double2)));
    CK(cudaMemset(psi, 0, n_amps * sizeof(double2)));
    unsigned *ctr;
    int *err;
    CK(cudaMalloc(&ctr, 64 * 32 * sizeof(unsigned)));
    CK(cudaMalloc(&err, sizeof(int)));
    CK(cudaMemset(err, 0, sizeof(int)));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int grid = 2 * sms;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const long long n_tiles = n_amps / kTileAmps;
    auto time_it = [&](auto fn, int reps) {
        for (int i = 0; i < 3; ++i) fn();
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        for (int i = 0; i < reps; ++i) fn();
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        return ms / reps;
    };
    const double gb = 2.0 * n_amps * 16 / 1e9;
    float plain = time_it([&] { k_plain<<<grid, kThreads>>>(psi, n_tiles, 1.0000001); }, 20);
    printf("plain pass: %.4f ms (%.0f GB/s); two passes %.4f ms\n", plain, gb / plain * 1e3, 2 * plain);
    for (int mode = 0; mode < 2; ++mode)
        for (int slab_log2_mib : {1, 2, 3, 4}) {
            const int tiles_per_slab = (1 << slab_log2_mib) * 16;  // 64 KiB tiles per slab
            for (int G : {16, 32, 37, 64, 74}) {
                const int n_teams = grid / G;
                const long long n_slabs = n_tiles / tiles_per_slab;
                float ms = time_it([&] {
                    cudaMemsetAsync(ctr, 0, 64 * 32 * sizeof(unsigned));
                    if (mode == 0)
                        k_sweep<0><<<grid, kThreads>>>(psi, n_slabs, tiles_per_slab, G, n_teams, ctr, err, 1.0000001);
                    else
                        k_sweep<1><<<grid, kThreads>>>(psi, n_slabs, tiles_per_slab, G, n_teams, ctr, err, 1.0000001);
                }, 10);
                int e = 0;
                CK(cudaMemcpy(&e, err, sizeof(int), cudaMemcpyDeviceToHost));
                printf("sweep mode=%d slab=%2d MiB G=%2d teams=%2d in-flight=%3d MiB: %.4f ms (%.2fx two passes)%s\n",
                       mode, 1 << slab_log2_mib, G, n_teams, n_teams << slab_log2_mib, ms, 2 * plain / ms,
                       e ? " TIMEOUT" : "");
                CK(cudaMemset(err, 0, sizeof(int)));
            }
        }
    return 0;
}
