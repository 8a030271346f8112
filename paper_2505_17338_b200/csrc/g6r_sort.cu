// g6r_sort.cu -- on-device stable LSD radix sort of the tile entries and
// per-tile range extraction.
//
// Replaces raster.py:376-379: np.argsort(key, kind="stable") over the 64-bit
// keys (tile << 32 | f32 depth bits) and tile_starts = cumsum(bincount(tile)).
// Stability reproduces the reference tie rule (equal keys keep splat order,
// raster.py:22-24), so the output is bit-identical to the reference.
//
// Key compression: depths are positive, so their f32 bit patterns order
// monotonically; the projection records the view's min/max depth bits and the
// sort ranks the order-preserving key' = tile << dbits | (depth_bits - dmin)
// with dbits = bits(dmax - dmin).  At 512^2 with a 1M-Gaussian orbit view that
// is ~10 + 24 bits: 4 passes of 9-bit digits instead of 6 passes of 8 bits.
// The stored keys stay the original 64-bit keys (ranges read the tile from
// them); digits are computed on the fly.  The pass count is decided on the
// device; surplus pass launches exit at once and consumers read which
// ping-pong buffer holds the result (sorted_buffer()).
//
// Each pass is reduce-then-scan over 4096-key tiles, with no inter-CTA waiting:
//   upsweep    per-tile digit counts (warp match-any aggregated smem atomics)
//              + global digit totals;
//   colscan    exclusive scan of every digit column across tiles;
//   downsweep  re-rank each tile (stable: warp-striped items, warps in order),
//              scatter to global digit offset + column prefix + local rank.
// (A decoupled look-back version was latency-bound: its inclusive-prefix
// frontier advances one probe width per L2 round trip, ~30 us per pass.)
#include <algorithm>

#include "g6r_common.cuh"
#include "g6r_internal.h"

namespace g6r {

constexpr int kWarps = kBlock / 32;
constexpr int kDigitsPerThread = kBins / kBlock;   // 2

int tile_bits(int64_t tiles) {
    int tb = 0;
    while ((1ll << tb) < tiles) ++tb;
    return tb;
}

int sort_passes(int tiles) {   // upper bound (full 32 depth bits)
    return (32 + tile_bits(tiles) + kRadixBits - 1) / kRadixBits;
}

struct SortParams {
    int64_t cap;
    int tbits;
};

__device__ __forceinline__ bool entries_valid(const int64_t *counters, int64_t cap, int64_t &e) {
    e = counters[G6R_CNT_ENTRIES];
    return !counters[G6R_CNT_OVERFLOW] && e <= cap;
}

// (dmin, dbits, passes) of this view from the projection's depth-bit extrema.
__device__ __forceinline__ void view_key_shape(const long long *internal, int tbits, unsigned &dmin,
                                               int &dbits, int &passes) {
    const unsigned lo = ~(unsigned)internal[kDepthMinInv];
    const unsigned hi = (unsigned)internal[kDepthMax];
    const unsigned span = hi >= lo ? hi - lo : 0u;
    dmin = hi >= lo ? lo : 0u;
    dbits = span ? 32 - __clz(span) : 0;
    passes = (tbits + dbits + kRadixBits - 1) / kRadixBits;
}

__device__ __forceinline__ unsigned digit_of(unsigned long long key, unsigned dmin, int dbits,
                                             int shift) {
    const unsigned long long k2 =
        ((key >> 32) << dbits) | (unsigned long long)((unsigned)key - dmin);
    return (unsigned)(k2 >> shift) & (kBins - 1);
}

__global__ void __launch_bounds__(kBlock)
k_upsweep(const unsigned long long *__restrict__ keys, const int64_t *counters, SortParams sp,
          long long *internal, int pass, unsigned *__restrict__ counts,
          unsigned *__restrict__ totals) {
    __shared__ unsigned h[kBins];
    int64_t e;
    if (!entries_valid(counters, sp.cap, e)) return;
    unsigned dmin;
    int dbits, passes;
    view_key_shape(internal, sp.tbits, dmin, dbits, passes);
    if (pass == 0 && blockIdx.x == 0 && threadIdx.x == 0) internal[kSortPasses] = passes;
    if (pass >= passes) return;
    const int64_t ntiles = ceil_div(e, kSortTile);
    const int shift = kRadixBits * pass;
    const int lane = threadIdx.x & 31;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int k = threadIdx.x; k < kBins; k += kBlock) h[k] = 0u;
        __syncthreads();
        const int64_t base = tile * kSortTile;
#pragma unroll 4
        for (int k = 0; k < kSortItems; ++k) {
            const int64_t idx = base + k * kBlock + threadIdx.x;
            const unsigned d = idx < e ? digit_of(keys[idx], dmin, dbits, shift) : (unsigned)kBins;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            if (d < (unsigned)kBins && lane == __ffs(peers) - 1) atomicAdd(&h[d], (unsigned)__popc(peers));
        }
        __syncthreads();
        for (int d = threadIdx.x; d < kBins; d += kBlock) {
            const unsigned c = h[d];
            counts[tile * kBins + d] = c;
            if (c) atomicAdd(&totals[d], c);
        }
        __syncthreads();
    }
}

// Exclusive scan of each digit column across tiles.  CTA c owns 32 digit
// columns (lane = digit); its 8 warps each sum a contiguous chunk of tiles,
// the chunk sums are scanned in smem, then each warp rewrites its chunk.
__global__ void __launch_bounds__(kBlock)
k_colscan(const int64_t *counters, SortParams sp, const long long *internal, int pass,
          unsigned *__restrict__ counts) {
    __shared__ unsigned s_sum[kWarps][32];
    int64_t e;
    if (!entries_valid(counters, sp.cap, e)) return;
    unsigned dmin;
    int dbits, passes;
    view_key_shape(internal, sp.tbits, dmin, dbits, passes);
    if (pass >= passes) return;
    const int64_t ntiles = ceil_div(e, kSortTile);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int d = blockIdx.x * 32 + lane;
    const int64_t per = ceil_div(ntiles, kWarps);
    const int64_t t0 = warp * per, t1 = std::min<int64_t>(ntiles, t0 + per);
    constexpr int U = 8;   // independent loads in flight per lane
    unsigned s = 0;
    for (int64_t t = t0; t < t1; t += U) {
        unsigned c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) c[u] = t + u < t1 ? counts[(t + u) * kBins + d] : 0u;
#pragma unroll
        for (int u = 0; u < U; ++u) s += c[u];
    }
    s_sum[warp][lane] = s;
    __syncthreads();
    unsigned run = 0;
    for (int w = 0; w < warp; ++w) run += s_sum[w][lane];
    for (int64_t t = t0; t < t1; t += U) {
        unsigned c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) c[u] = t + u < t1 ? counts[(t + u) * kBins + d] : 0u;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (t + u < t1) counts[(t + u) * kBins + d] = run;
            run += c[u];
        }
    }
}

__global__ void __launch_bounds__(kBlock)
k_downsweep(const unsigned long long *__restrict__ kin, const unsigned *__restrict__ vin,
            unsigned long long *__restrict__ kout, unsigned *__restrict__ vout,
            const int64_t *counters, SortParams sp, const long long *internal, int pass,
            const unsigned *__restrict__ counts, const unsigned *__restrict__ totals) {
    __shared__ unsigned s_goff[kBins];
    __shared__ unsigned s_wh[kWarps][kBins];
    __shared__ unsigned s_scan[kWarps];
    int64_t e;
    if (!entries_valid(counters, sp.cap, e)) return;
    unsigned dmin;
    int dbits, passes;
    view_key_shape(internal, sp.tbits, dmin, dbits, passes);
    if (pass >= passes) return;
    const int shift = kRadixBits * pass;
    const int64_t ntiles = ceil_div(e, kSortTile);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    {   // global exclusive digit offsets: thread t owns digits 2t, 2t+1
        const unsigned c0 = totals[2 * tid], c1 = totals[2 * tid + 1];
        const unsigned c = c0 + c1;
        const unsigned inc = warp_inclusive_scan(c);
        if (lane == 31) s_scan[warp] = inc;
        __syncthreads();
        unsigned pre = 0;
        for (int w = 0; w < warp; ++w) pre += s_scan[w];
        s_goff[2 * tid] = pre + inc - c;
        s_goff[2 * tid + 1] = pre + inc - c + c0;
    }
    const unsigned lanemask_lt = (1u << lane) - 1u;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int k = tid; k < kWarps * kBins; k += kBlock) (&s_wh[0][0])[k] = 0u;
        __syncthreads();
        // warp w owns the contiguous items [w*512, w*512+512) of the tile, striped
        const int64_t base = tile * kSortTile + (int64_t)warp * (32 * kSortItems);
        unsigned long long key[kSortItems];
        unsigned val[kSortItems];
        unsigned rank[kSortItems];
#pragma unroll
        for (int k = 0; k < kSortItems; ++k) {
            const int64_t idx = base + k * 32 + lane;
            const bool valid = idx < e;
            key[k] = valid ? kin[idx] : ~0ull;
            val[k] = valid ? vin[idx] : 0u;
            rank[k] = valid ? 0u : 0xffffffffu;
        }
#pragma unroll
        for (int k = 0; k < kSortItems; ++k) {
            const unsigned d =
                rank[k] == 0xffffffffu ? (unsigned)kBins : digit_of(key[k], dmin, dbits, shift);
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            const int leader = __ffs(peers) - 1;
            unsigned old = 0;
            if (d < (unsigned)kBins && lane == leader) {
                old = s_wh[warp][d];
                s_wh[warp][d] = old + (unsigned)__popc(peers);
            }
            old = __shfl_sync(0xffffffffu, old, leader);
            if (d < (unsigned)kBins) rank[k] = old + (unsigned)__popc(peers & lanemask_lt);
            __syncwarp();
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kDigitsPerThread; ++q) {   // tile base + exclusive prefix over warps
            const int d = tid + q * kBlock;
            unsigned run = s_goff[d] + counts[tile * kBins + d];
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const unsigned c = s_wh[w][d];
                s_wh[w][d] = run;
                run += c;
            }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kSortItems; ++k) {
            if (rank[k] == 0xffffffffu) continue;
            const unsigned d = digit_of(key[k], dmin, dbits, shift);
            const unsigned pos = s_wh[warp][d] + rank[k];
            kout[pos] = key[k];
            vout[pos] = val[k];
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kBlock)
k_ranges(Workspace ws, const int64_t *counters, int64_t n_tiles, int64_t *__restrict__ starts2,
         int32_t *__restrict__ entry_out) {
    int64_t e;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
    int64_t *starts = ws.tile_starts;
    if (!entries_valid(counters, ws.entry_capacity, e)) {   // overflow: empty runs everywhere
        for (int64_t t = gtid; t <= n_tiles; t += gsz) {
            starts[t] = 0;
            if (starts2) starts2[t] = 0;
        }
        return;
    }
    const int fb = sorted_buffer(ws.internal);
    const unsigned long long *keys = ws.keys[fb];
    const unsigned *vals = ws.vals[fb];
    for (int64_t i = gtid; i <= e; i += gsz) {
        const int64_t ti = i < e ? (int64_t)(keys[i] >> 32) : n_tiles;
        const int64_t tp = i > 0 ? (int64_t)(keys[i - 1] >> 32) : -1;
        for (int64_t t = tp + 1; t <= ti; ++t) {
            starts[t] = i;
            if (starts2) starts2[t] = i;
        }
        if (i < e && entry_out) entry_out[i] = (int32_t)vals[i];
    }
}

static int num_sms() {
    static int cached = 0;
    if (!cached) {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) v = 148;
        cached = v;
    }
    return cached;
}

int launch_sort(const ViewParams &vp, const Workspace &ws, const int64_t *counters, cudaStream_t st) {
    const int64_t n_tiles = (int64_t)vp.tiles_x * vp.tiles_y;
    SortParams sp{ws.entry_capacity, tile_bits(n_tiles)};
    const int max_passes = sort_passes((int)n_tiles);
    const int sms = num_sms();
    // one CTA per 4096-key tile of the capacity (idle ones exit), grid-stride beyond
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ws.sort_tiles_cap, sms * 8));
    int src = 0;
    for (int p = 0; p < max_passes; ++p) {
        unsigned *counts = ws.sort_status + (int64_t)p * ws.sort_tiles_cap * kBins;
        unsigned *totals = ws.hist + p * kBins;
        k_upsweep<<<grid, kBlock, 0, st>>>(ws.keys[src], counters, sp, ws.internal, p, counts, totals);
        k_colscan<<<kBins / 32, kBlock, 0, st>>>(counters, sp, ws.internal, p, counts);
        k_downsweep<<<grid, kBlock, 0, st>>>(ws.keys[src], ws.vals[src], ws.keys[1 - src],
                                             ws.vals[1 - src], counters, sp, ws.internal, p, counts,
                                             totals);
        src = 1 - src;
    }
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

int launch_ranges(const ViewParams &vp, const Workspace &ws, const int64_t *counters,
                  int64_t *tile_starts_out, int32_t *entry_splat_out, cudaStream_t st) {
    const int64_t n_tiles = (int64_t)vp.tiles_x * vp.tiles_y;
    const int64_t cap = ws.entry_capacity;
    const unsigned rgrid =
        (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(cap + 1, kBlock), num_sms() * 4));
    k_ranges<<<rgrid, kBlock, 0, st>>>(ws, counters, n_tiles, tile_starts_out, entry_splat_out);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

}  // namespace g6r
