// Tensor maps describing one pass tile (12 physical index bits) of a state or
// cost vector, for the one-instruction L2 tile prefetch
// (cp.async.bulk.prefetch.tensor) of the pass kernels.  Host only.
#pragma once
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "pass.cuh"

namespace fq {

// ---- tensor maps for the tile prefetch (driver entry point fetched through the runtime; no -lcuda)
static inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// Describe one tile (12 physical index bits) of a 2^n vector as a TMA box:
// runs of tile bits become box dims (full extent, <= 256 elements each), runs
// of outer bits become box-1 dims whose coordinate comes from the tile number.
// `per_amp` elements of `elem_bytes` per amplitude (state: 2 doubles).
// Returns the rank (0 if the layout cannot be expressed: rank > 5, rows or
// strides not multiples of 16 B, or no driver entry point).
static inline int build_tile_map(CUtensorMap *map, const void *gaddr, int n, const int *tile_pos, CUtensorMapDataType dt,
                          int elem_bytes, int per_amp, int *outer_shift, int *outer_bits) {
    auto fn = encode_fn();
    if (!fn || !gaddr) return 0;
    bool is_tile[64] = {};
    for (int i = 0; i < kTileBits; ++i) is_tile[tile_pos[i]] = true;
    if (!is_tile[0]) return 0;
    struct Dim { bool tile; int start, len; };
    std::vector<Dim> dims;
    const int cap0 = (per_amp == 2) ? 7 : 8;
    for (int b = 0; b < n;) {
        int e = b;
        while (e < n && is_tile[e] == is_tile[b]) ++e;
        if (is_tile[b]) {
            for (int at = b; at < e;) {
                const int len = std::min(dims.empty() ? cap0 : 8, e - at);
                dims.push_back({true, at, len});
                at += len;
            }
        } else {
            dims.push_back({false, b, e - b});
        }
        b = e;
    }
    if (dims.size() > 5) return 0;
    const int rank = (int)dims.size();
    cuuint64_t gdim[5], gstride[5];
    cuuint32_t box[5], estr[5];
    int shift = 0;
    for (int d = 0; d < rank; ++d) {
        gdim[d] = (cuuint64_t)(d == 0 ? per_amp : 1) << dims[d].len;
        box[d] = dims[d].tile ? (cuuint32_t)gdim[d] : 1u;
        estr[d] = 1;
        if (d > 0) {
            gstride[d - 1] = ((cuuint64_t)1 << dims[d].start) * per_amp * elem_bytes;
            if (gstride[d - 1] % 16) return 0;
        }
        outer_shift[d] = dims[d].tile ? 0 : shift;
        outer_bits[d] = dims[d].tile ? 0 : dims[d].len;
        if (!dims[d].tile) shift += dims[d].len;
    }
    if ((box[0] * (cuuint32_t)elem_bytes) % 16) return 0;
    for (int d = rank; d < 5; ++d) outer_shift[d] = outer_bits[d] = 0;
    CUresult r = fn(map, dt, (cuuint32_t)rank, const_cast<void *>(gaddr), gdim, gstride, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? rank : 0;
}

// Encoding a map costs a few microseconds of host time per pass; a program
// re-encodes the same (buffer, tile) pairs every call (the caching allocator
// hands back the same state buffer), so maps are memoised.
struct TileMapKey {
    const void *addr;
    int n, dt, elem_bytes, per_amp;
    long long tile_mask;
    bool operator==(const TileMapKey &o) const {
        return addr == o.addr && n == o.n && dt == o.dt && elem_bytes == o.elem_bytes && per_amp == o.per_amp &&
               tile_mask == o.tile_mask;
    }
};
struct TileMapEntry {
    TileMapKey key;
    alignas(64) CUtensorMap map;
    int rank, shift[5], bits[5];
};

static inline int cached_tile_map(CUtensorMap *map, const void *gaddr, int n, const int *tile_pos,
                                  CUtensorMapDataType dt, int elem_bytes, int per_amp, int *outer_shift,
                                  int *outer_bits) {
    static std::vector<TileMapEntry> cache;  // small: a few groups x (state, costs)
    static size_t next = 0;
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    TileMapKey key{gaddr, n, (int)dt, elem_bytes, per_amp, 0};
    for (int i = 0; i < 12; ++i) key.tile_mask |= 1LL << tile_pos[i];
    for (auto &e : cache)
        if (e.key == key) {
            *map = e.map;
            for (int d = 0; d < 5; ++d) outer_shift[d] = e.shift[d], outer_bits[d] = e.bits[d];
            return e.rank;
        }
    TileMapEntry e;
    e.key = key;
    e.rank = build_tile_map(&e.map, gaddr, n, tile_pos, dt, elem_bytes, per_amp, e.shift, e.bits);
    if (cache.size() < 64) cache.push_back(e);
    else cache[next++ % 64] = e;
    *map = e.map;
    for (int d = 0; d < 5; ++d) outer_shift[d] = e.shift[d], outer_bits[d] = e.bits[d];
    return e.rank;
}

}  // namespace fq
