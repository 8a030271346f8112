// g6r_sort.cu -- on-device stable LSD radix sort of the tile entries and
// per-tile range extraction, for a batch of views per launch.
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
// device per view; surplus work exits at once and consumers read which
// ping-pong buffer holds the result (sorted_buffer()).
//
// Each pass is reduce-then-scan over 4096-key tiles, with no inter-CTA waiting
// (grid y = view):
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

__device__ __forceinline__ bool entries_valid(const int64_t *counters, int64_t cap, int64_t &e) {
    e = counters[G6R_CNT_ENTRIES];
    return !counters[G6R_CNT_OVERFLOW] && e <= cap;
}

// (dmin, dbits, passes) of a view from the projection's depth-bit extrema.
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

// Common prologue: this view's entry count, key shape, and whether `pass` runs.
struct PassCtx {
    int64_t e, ntiles;
    unsigned dmin;
    int dbits, passes;
};

__device__ __forceinline__ bool pass_ctx(const Batch &b, int v, int tbits, int pass, PassCtx &c) {
    if (!entries_valid(b.out[v].counters, b.ws[v].entry_capacity, c.e)) return false;
    view_key_shape(b.ws[v].internal, tbits, c.dmin, c.dbits, c.passes);
    c.ntiles = ceil_div(c.e, kSortTile);
    return pass < c.passes;
}

__device__ __forceinline__ int pass_src(int pass) { return pass & 1; }

__global__ void __launch_bounds__(kBlock)
k_upsweep(const __grid_constant__ Batch b, int tbits, int pass) {
    __shared__ unsigned h[kBins];
    const int v = blockIdx.y;
    PassCtx c;
    const bool run = pass_ctx(b, v, tbits, pass, c);
    const Workspace &ws = b.ws[v];
    if (pass == 0 && blockIdx.x == 0 && threadIdx.x == 0 && c.e <= ws.entry_capacity)
        ws.internal[kSortPasses] = run ? c.passes : 0;
    if (!run) return;
    const unsigned long long *__restrict__ keys = ws.keys[pass_src(pass)];
    unsigned *counts = ws.sort_counts + (int64_t)pass * ws.sort_tiles_cap * kBins;
    unsigned *totals = ws.hist + pass * kBins;
    const int shift = kRadixBits * pass;
    const int lane = threadIdx.x & 31;
    for (int64_t tile = blockIdx.x; tile < c.ntiles; tile += gridDim.x) {
        for (int k = threadIdx.x; k < kBins; k += kBlock) h[k] = 0u;
        __syncthreads();
        const int64_t base = tile * kSortTile;
        unsigned long long key[kSortItems];
#pragma unroll
        for (int k = 0; k < kSortItems; ++k) {   // all loads in flight first
            const int64_t idx = base + k * kBlock + threadIdx.x;
            key[k] = idx < c.e ? keys[idx] : 0ull;
        }
#pragma unroll
        for (int k = 0; k < kSortItems; ++k) {
            const int64_t idx = base + k * kBlock + threadIdx.x;
            const unsigned d = idx < c.e ? digit_of(key[k], c.dmin, c.dbits, shift) : (unsigned)kBins;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            if (d < (unsigned)kBins && lane == __ffs(peers) - 1) atomicAdd(&h[d], (unsigned)__popc(peers));
        }
        __syncthreads();
        for (int d = threadIdx.x; d < kBins; d += kBlock) {
            const unsigned cnt = h[d];
            counts[tile * kBins + d] = cnt;
            if (cnt) atomicAdd(&totals[d], cnt);
        }
        __syncthreads();
    }
}

// Exclusive scan of each digit column across tiles.  CTA x owns 32 digit
// columns (lane = digit); its 8 warps each sum a contiguous chunk of tiles,
// the chunk sums are scanned in smem, then each warp rewrites its chunk.
__global__ void __launch_bounds__(kBlock)
k_colscan(const __grid_constant__ Batch b, int tbits, int pass) {
    __shared__ unsigned s_sum[kWarps][32];
    const int v = blockIdx.y;
    PassCtx c;
    if (!pass_ctx(b, v, tbits, pass, c)) return;
    const Workspace &ws = b.ws[v];
    unsigned *counts = ws.sort_counts + (int64_t)pass * ws.sort_tiles_cap * kBins;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int d = blockIdx.x * 32 + lane;
    const int64_t per = ceil_div(c.ntiles, kWarps);
    const int64_t t0 = warp * per, t1 = std::min<int64_t>(c.ntiles, t0 + per);
    constexpr int U = 8;   // independent loads in flight per lane
    unsigned s = 0;
    for (int64_t t = t0; t < t1; t += U) {
        unsigned x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = t + u < t1 ? counts[(t + u) * kBins + d] : 0u;
#pragma unroll
        for (int u = 0; u < U; ++u) s += x[u];
    }
    s_sum[warp][lane] = s;
    __syncthreads();
    unsigned run = 0;
    for (int w = 0; w < warp; ++w) run += s_sum[w][lane];
    for (int64_t t = t0; t < t1; t += U) {
        unsigned x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = t + u < t1 ? counts[(t + u) * kBins + d] : 0u;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (t + u < t1) counts[(t + u) * kBins + d] = run;
            run += x[u];
        }
    }
}

__global__ void __launch_bounds__(kBlock)
k_downsweep(const __grid_constant__ Batch b, int tbits, int pass) {
    __shared__ unsigned s_goff[kBins];
    __shared__ unsigned s_wh[kWarps][kBins];
    __shared__ unsigned s_scan[kWarps];
    const int v = blockIdx.y;
    PassCtx c;
    if (!pass_ctx(b, v, tbits, pass, c)) return;
    const Workspace &ws = b.ws[v];
    const int src = pass_src(pass);
    const unsigned long long *__restrict__ kin = ws.keys[src];
    const unsigned *__restrict__ vin = ws.vals[src];
    unsigned long long *__restrict__ kout = ws.keys[src ^ 1];
    unsigned *__restrict__ vout = ws.vals[src ^ 1];
    const unsigned *counts = ws.sort_counts + (int64_t)pass * ws.sort_tiles_cap * kBins;
    const unsigned *totals = ws.hist + pass * kBins;
    const int shift = kRadixBits * pass;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    {   // global exclusive digit offsets: thread t owns digits 2t, 2t+1
        const unsigned c0 = totals[2 * tid], c1 = totals[2 * tid + 1];
        const unsigned cc = c0 + c1;
        const unsigned inc = warp_inclusive_scan(cc);
        if (lane == 31) s_scan[warp] = inc;
        __syncthreads();
        unsigned pre = 0;
        for (int w = 0; w < warp; ++w) pre += s_scan[w];
        s_goff[2 * tid] = pre + inc - cc;
        s_goff[2 * tid + 1] = pre + inc - cc + c0;
    }
    const unsigned lanemask_lt = (1u << lane) - 1u;
    for (int64_t tile = blockIdx.x; tile < c.ntiles; tile += gridDim.x) {
        for (int k = tid; k < kWarps * kBins; k += kBlock) (&s_wh[0][0])[k] = 0u;
        __syncthreads();
        // warp w owns the contiguous items [w*512, w*512+512) of the tile, striped
        const int64_t base = tile * kSortTile + (int64_t)warp * (32 * kSortItems);
        unsigned long long key[kSortItems];
        unsigned val[kSortItems];
        unsigned dig[kSortItems];
        unsigned rank[kSortItems];
#pragma unroll
        for (int k = 0; k < kSortItems; ++k) {
            const int64_t idx = base + k * 32 + lane;
            const bool valid = idx < c.e;
            key[k] = valid ? kin[idx] : ~0ull;
            val[k] = valid ? vin[idx] : 0u;
        }
#pragma unroll
        for (int k = 0; k < kSortItems; ++k) {
            const int64_t idx = base + k * 32 + lane;
            dig[k] = idx < c.e ? digit_of(key[k], c.dmin, c.dbits, shift) : (unsigned)kBins;
        }
#pragma unroll
        for (int k = 0; k < kSortItems; ++k) {
            const unsigned d = dig[k];
            rank[k] = 0xffffffffu;
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
                const unsigned cnt = s_wh[w][d];
                s_wh[w][d] = run;
                run += cnt;
            }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kSortItems; ++k) {
            if (dig[k] >= (unsigned)kBins) continue;
            const unsigned pos = s_wh[warp][dig[k]] + rank[k];
            kout[pos] = key[k];
            vout[pos] = val[k];
        }
        __syncthreads();
    }
}

// grid y = view: tile_starts from the boundaries of the sorted keys.
__global__ void __launch_bounds__(kBlock)
k_ranges(const __grid_constant__ Batch b) {
    const int v = blockIdx.y;
    const Workspace &ws = b.ws[v];
    const ViewOut &out = b.out[v];
    const int64_t n_tiles = (int64_t)b.vp[v].tiles_x * b.vp[v].tiles_y;
    int64_t e;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
    int64_t *starts = ws.tile_starts;
    int64_t *starts2 = out.tile_starts;
    if (!entries_valid(out.counters, ws.entry_capacity, e)) {   // overflow: empty runs everywhere
        for (int64_t t = gtid; t <= n_tiles; t += gsz) {
            starts[t] = 0;
            if (starts2) starts2[t] = 0;
        }
        return;
    }
    const int fb = sorted_buffer(ws.internal);
    const unsigned long long *keys = ws.keys[fb];
    const unsigned *vals = ws.vals[fb];
    int32_t *entry_out = out.entry_splat;
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

int launch_sort(const Batch &b, cudaStream_t st) {
    if (b.nviews == 0) return G6R_OK;
    const int64_t n_tiles = (int64_t)b.vp[0].tiles_x * b.vp[0].tiles_y;
    const int tbits = tile_bits(n_tiles);
    const int max_passes = sort_passes((int)n_tiles);
    const int sms = num_sms();
    const int64_t tiles_cap = b.ws[0].sort_tiles_cap;
    // per view: one CTA per 4096-key tile of the capacity (idle ones exit), grid-stride beyond
    const unsigned gx = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>(tiles_cap, std::max<int64_t>(sms * 8 / b.nviews, 1)));
    for (int p = 0; p < max_passes; ++p) {
        k_upsweep<<<dim3(gx, b.nviews), kBlock, 0, st>>>(b, tbits, p);
        trace_mark("upsweep", st);
        k_colscan<<<dim3(kBins / 32, b.nviews), kBlock, 0, st>>>(b, tbits, p);
        trace_mark("colscan", st);
        k_downsweep<<<dim3(gx, b.nviews), kBlock, 0, st>>>(b, tbits, p);
        trace_mark("downsweep", st);
    }
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

int launch_ranges(const Batch &b, cudaStream_t st) {
    if (b.nviews == 0) return G6R_OK;
    const int64_t cap = b.ws[0].entry_capacity;
    const unsigned gx = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>(ceil_div(cap + 1, kBlock), std::max(num_sms() * 4 / b.nviews, 1)));
    k_ranges<<<dim3(gx, b.nviews), kBlock, 0, st>>>(b);
    trace_mark("ranges", st);
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

}  // namespace g6r
