// g6r_tiles.cu -- order-preserving expansion of depth-sorted splats into
// per-tile runs (the splat-level half of the hot-path sort).
//
// The reference orders every tile's run by (f32 depth bits, then entry order),
// raster.py:366-379.  Entry order follows the splat index and equal depths keep
// it, so the run of tile t is exactly "the drawn splats whose rect covers t, in
// (depth, row) order".  The hot path therefore sorts the n splat rows by depth
// once (g6r_sort.cu, splat mode: n keys instead of E entries, 8-byte items) and
// expands them here without a second sort:
//   k_chunk_count    per chunk of chunk_splats(T) sorted splats: tile histogram
//   k_chunk_colscan  per tile: exclusive prefix over chunks, tile totals
//   k_tile_scan      tile_starts = exclusive scan of the totals (+ overflow)
//   k_chunk_scatter  per chunk: each warp recounts its slice of the chunk per
//                    tile, the counts are prefixed over warps, then each warp
//                    expands its splats' entries in order and ranks them with
//                    a ballot match on the tile id against its running counters;
//                    every entry's splat row is written to tile_start + chunk
//                    prefix + warp prefix + running count + rank.
// Every step is deterministic and keeps the sorted order, so runs, tile starts
// and images are bit-identical to the entry sort's.
#include <algorithm>
#include <atomic>

#include "g6r_common.cuh"
#include "g6r_internal.h"

namespace g6r {


struct PartCtx {
    int64_t m;             // drawn splats (the first m sorted items)
    int64_t chunks;
    int chunk;             // sorted splats per chunk
    int tiles, tiles_x;
    const unsigned long long *items;   // depth-sorted (depth code << vbits | row)
    const uint2 *rect;                 // tile rects the runs are built from
};

__device__ __forceinline__ bool part_ctx(const Batch &b, int v, PartCtx &c) {
    const int64_t *cnt = b.out[v].counters;
    const Workspace &ws = b.ws[v];
    if (cnt[G6R_CNT_OVERFLOW] || cnt[G6R_CNT_ENTRIES] > ws.entry_capacity) return false;
    c.m = cnt[G6R_CNT_DRAWN];
    c.tiles_x = b.vp[v].tiles_x;
    c.tiles = b.vp[v].tiles_x * b.vp[v].tiles_y;
    c.chunk = chunk_splats(c.tiles);
    c.chunks = ceil_div(c.m, c.chunk);
    c.items = ws.keys[ws.internal[kSortPasses] & 1];
    // runs that are exported (entry_splat / tile_starts) or indexed by
    // last_contrib are the reference's; otherwise only the entries the
    // compositor can visit (same pixels, same order: bit-identical images)
    const ViewOut &o = b.out[v];
    c.rect = (o.entry_splat || o.tile_starts || o.last_contrib || !ws.crect) ? ws.rect : ws.crect;
    return true;
}

__device__ __forceinline__ void unpack_rect(uint2 r, int &x0, int &y0, int &wx, int &hy) {
    x0 = (int)(r.x & 0xffffu);
    y0 = (int)(r.x >> 16);
    wx = (int)(r.y & 0xffffu);
    hy = (int)(r.y >> 16);
}

// Load-balanced entry enumeration for a warp's group of 32 sorted splats.
// Lane i holds splat i's row, packed rect and its inclusive/exclusive entry
// prefix over the group; entry s (0 <= s < total, row-major within each rect,
// rects in lane order) is owned by the first lane whose inclusive prefix
// exceeds s, found by a 5-step shuffle search.  Every lane then decodes one
// entry, so a group costs the same whatever the spread of rect sizes.
struct EntryGroup {
    unsigned row, rx, ry;   // splat row, packed (x0 | y0 << 16), (wx | hy << 16)
    int excl, incl, total;
};

__device__ __forceinline__ EntryGroup load_group(const PartCtx &c, const Workspace &ws, int64_t sp,
                                                 int64_t end, unsigned long long vmask) {
    EntryGroup g;
    g.row = 0;
    g.rx = 0;
    g.ry = 0;
    if (sp < end) {
        g.row = (unsigned)(c.items[sp] & vmask);
        const uint2 r = c.rect[g.row];
        g.rx = r.x;
        g.ry = r.y;
    }
    const int cnt = (int)((g.ry & 0xffffu) * (g.ry >> 16));
    g.incl = warp_inclusive_scan(cnt);
    g.excl = g.incl - cnt;
    g.total = __shfl_sync(0xffffffffu, g.incl, 31);
    return g;
}

// tile of entry s of the group (any value for s >= total); row of its splat
__device__ __forceinline__ unsigned group_entry(const EntryGroup &g, int s, int tiles_x, unsigned &row) {
    int L = 0;
#pragma unroll
    for (int b = 16; b; b >>= 1) {
        const int v = __shfl_sync(0xffffffffu, g.incl, L + b - 1);
        if (v <= s) L += b;
    }
    const int k = s - __shfl_sync(0xffffffffu, g.excl, L);
    const unsigned a = __shfl_sync(0xffffffffu, g.rx, L);
    const unsigned w = __shfl_sync(0xffffffffu, g.ry, L);
    row = __shfl_sync(0xffffffffu, g.row, L);
    const int wx = (int)(w & 0xffffu);
    // k / wx: k < wx * hy <= 4096 entries, so the float quotient is never
    // within an ulp of the next integer
    const int qy = (int)__fdividef((float)k + 0.5f, (float)wx);
    const int qx = k - qy * wx;
    return (unsigned)(((int)(a >> 16) + qy) * tiles_x + (int)(a & 0xffffu) + qx);
}

// Per chunk: each warp counts the entries of its slice of the chunk (the
// slices k_chunk_scatter ranks) per tile into packed 16-bit counters; the
// counters are prefixed over the warps and written out (the scatter's starting
// offsets inside the chunk), and the chunk's tile totals go to chunk_hist.
__global__ void __launch_bounds__(kBlock)
k_chunk_count(const __grid_constant__ Batch b, unsigned long long vmask) {
    extern __shared__ unsigned s_cw[];   // [warps][tw] packed u16 counters
    const int v = blockIdx.y;
    PartCtx c;
    if (!part_ctx(b, v, c) || blockIdx.x >= c.chunks) return;
    const Workspace &ws = b.ws[v];
    const int T = c.tiles, tw = (T + 1) >> 1;
    for (int k = threadIdx.x; k < kScatterWarps * tw; k += blockDim.x) s_cw[k] = 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int per = c.chunk / kScatterWarps;
    const int64_t c0 = (int64_t)blockIdx.x * c.chunk;
    const int64_t chunk_end = c0 + c.chunk < c.m ? c0 + c.chunk : c.m;
    const int64_t w0s = c0 + (int64_t)warp * per;
    const int64_t w1s = w0s + per < chunk_end ? w0s + per : chunk_end;
    unsigned *cw = s_cw + warp * tw;
    for (int64_t sp = w0s + lane; sp < w1s; sp += 32) {
        const unsigned row = (unsigned)(c.items[sp] & vmask);
        int x0, y0, wx, hy;
        unpack_rect(c.rect[row], x0, y0, wx, hy);
        for (int yy = 0; yy < hy; ++yy)
            for (int xx = 0; xx < wx; ++xx) {
                const int t = (y0 + yy) * c.tiles_x + x0 + xx;
                atomicAdd(&cw[t >> 1], 1u << ((t & 1) * 16));
            }
    }
    __syncthreads();
    unsigned *pre = ws.warp_prefix + (int64_t)blockIdx.x * kScatterWarps * tw;
    unsigned *row_out = ws.chunk_hist + (int64_t)blockIdx.x * T;
    for (int k = threadIdx.x; k < tw; k += blockDim.x) {
        unsigned run = 0;   // packed pairs: a chunk puts < 65536 entries in a tile
#pragma unroll
        for (int w = 0; w < kScatterWarps; ++w) {
            const unsigned x = s_cw[w * tw + k];
            pre[w * tw + k] = run;
            run += x;
        }
        row_out[2 * k] = run & 0xffffu;
        if (2 * k + 1 < T) row_out[2 * k + 1] = run >> 16;
    }
}

// Exclusive prefix of every tile column over the chunks, and the tile totals.
// CTA x owns 32 tiles (lane = tile); its 8 warps each sum a contiguous range of
// chunks, the range sums are scanned in shared memory, then each warp rewrites
// its range.
__global__ void __launch_bounds__(kBlock) k_chunk_colscan(const __grid_constant__ Batch b) {
    __shared__ unsigned s_sum[kBlock / 32][32];
    const int v = blockIdx.y;
    PartCtx c;
    if (!part_ctx(b, v, c)) return;
    const Workspace &ws = b.ws[v];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kBlock / 32;
    const int t = blockIdx.x * 32 + lane;
    const bool ok = t < c.tiles;
    const int64_t per = ceil_div(c.chunks, nw);
    const int64_t a = warp * per, e = a + per < c.chunks ? a + per : c.chunks;
    constexpr int U = 8;
    unsigned sum = 0;
    for (int64_t ch = a; ch < e; ch += U) {
        unsigned x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = (ok && ch + u < e) ? ws.chunk_hist[(ch + u) * c.tiles + t] : 0u;
#pragma unroll
        for (int u = 0; u < U; ++u) sum += x[u];
    }
    s_sum[warp][lane] = sum;
    __syncthreads();
    unsigned run = 0, total = 0;
    for (int w = 0; w < nw; ++w) {
        const unsigned x = s_sum[w][lane];
        run += w < warp ? x : 0u;
        total += x;
    }
    for (int64_t ch = a; ch < e; ch += U) {
        unsigned x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = (ok && ch + u < e) ? ws.chunk_hist[(ch + u) * c.tiles + t] : 0u;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (ok && ch + u < e) ws.chunk_hist[(ch + u) * c.tiles + t] = run;
            run += x[u];
        }
    }
    if (ok && warp == 0) ws.tile_total[t] = total;
}

// one CTA per view: tile_starts (T+1) from the totals; empty runs on overflow
__global__ void __launch_bounds__(1024) k_tile_scan(const __grid_constant__ Batch b) {
    __shared__ unsigned long long s_warp[32];
    __shared__ unsigned long long s_carry;
    const int v = blockIdx.y;
    const Workspace &ws = b.ws[v];
    int64_t *starts = ws.tile_starts;
    int64_t *starts2 = b.out[v].tile_starts;
    const int tiles = b.vp[v].tiles_x * b.vp[v].tiles_y;
    PartCtx c;
    if (!part_ctx(b, v, c)) {
        for (int t = threadIdx.x; t <= tiles; t += blockDim.x) {
            starts[t] = 0;
            if (starts2) starts2[t] = 0;
        }
        return;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int t0 = 0; t0 < tiles; t0 += blockDim.x) {
        const int t = t0 + threadIdx.x;
        const unsigned long long x = t < tiles ? ws.tile_total[t] : 0ull;
        const unsigned long long inc = warp_inclusive_scan(x);
        if (lane == 31) s_warp[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            const unsigned long long w = s_warp[lane];
            s_warp[lane] = warp_inclusive_scan(w) - w;
        }
        __syncthreads();
        const unsigned long long excl = s_carry + s_warp[warp] + inc - x;
        if (t < tiles) {
            starts[t] = (int64_t)excl;
            if (starts2) starts2[t] = (int64_t)excl;
        }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_carry = excl + x;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        starts[tiles] = (int64_t)s_carry;
        if (starts2) starts2[tiles] = (int64_t)s_carry;
    }
}

// k_chunk_scatter: CTA = chunk, warp w owns the w-th eighth of the chunk's
// sorted splats (the slices k_chunk_count counted).  The warp's counters start
// at k_chunk_count's per-warp prefix (16-bit counters, two per shared word);
// tile_start + chunk prefix is kept per tile.  Each warp walks its splats in
// groups of 32, enumerates the group's entries in order 32 at a time
// (group_entry) and ranks them with a ballot match on the tile id against its own
// running counters; the leader of each tile's peers advances the counter.  No
// CTA barrier after the setup, and every position is a function of the sorted
// order alone.
__global__ void __launch_bounds__(kBlock)
k_chunk_scatter(const __grid_constant__ Batch b, unsigned long long vmask) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    const int v = blockIdx.y;
    PartCtx c;
    if (!part_ctx(b, v, c) || blockIdx.x >= c.chunks) return;
    const Workspace &ws = b.ws[v];
    const int T = c.tiles;
    const int tw = (T + 1) >> 1;   // packed counter words per warp
    unsigned *s_tb = reinterpret_cast<unsigned *>(s_raw);                  // [T] tile start + chunk prefix
    unsigned *s_cw = s_tb + ((T + 3) & ~3);                                 // [warps][tw] packed u16 counters
    const unsigned *chunk_off = ws.chunk_hist + (int64_t)blockIdx.x * T;
    for (int t = threadIdx.x; t < T; t += blockDim.x) s_tb[t] = (unsigned)ws.tile_starts[t] + chunk_off[t];
    {   // this chunk's per-warp starting counters (k_chunk_count)
        const uint4 *pre = reinterpret_cast<const uint4 *>(ws.warp_prefix + (int64_t)blockIdx.x * kScatterWarps * tw);
        uint4 *dst = reinterpret_cast<uint4 *>(s_cw);
        for (int k = threadIdx.x; k < kScatterWarps * tw / 4; k += blockDim.x) dst[k] = pre[k];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lanemask_lt = (1u << lane) - 1u;
    const int per = c.chunk / kScatterWarps;
    const int64_t c0 = (int64_t)blockIdx.x * c.chunk;
    const int64_t chunk_end = c0 + c.chunk < c.m ? c0 + c.chunk : c.m;
    const int64_t w0s = c0 + (int64_t)warp * per;
    const int64_t w1s = w0s + per < chunk_end ? w0s + per : chunk_end;
    unsigned *cw = s_cw + warp * tw;
    unsigned short *cnt16 = reinterpret_cast<unsigned short *>(cw);
    // pass 2: rank and scatter, 32 entries at a time
    unsigned *vals = ws.vals[0];
    int tbits = 0;
    while ((1 << tbits) <= T) ++tbits;   // tile ids and the invalid code T
    for (int64_t g0 = w0s; g0 < w1s; g0 += 32) {
        const EntryGroup g = load_group(c, ws, g0 + lane, w1s, vmask);
        for (int q0 = 0; q0 < g.total; q0 += 32) {
            const bool valid = q0 + lane < g.total;
            unsigned row;
            unsigned t = group_entry(g, q0 + lane, c.tiles_x, row);
            t = valid ? t : 0xffffffffu;
            // lanes with the same tile: one ballot per tile-id bit (tile ids
            // and the invalid code T; cheaper than MATCH.ANY's latency here)
            unsigned peers = 0xffffffffu;
            {
                const unsigned key = valid ? t : (unsigned)T;
                for (int bit = 0; bit < tbits; ++bit) {
                    const bool on = (key >> bit) & 1u;
                    const unsigned bl = __ballot_sync(0xffffffffu, on);
                    peers &= on ? bl : ~bl;
                }
            }

            const int leader = __ffs(peers) - 1;
            unsigned old = 0;
            if (valid && lane == leader) {
                old = cnt16[t];
                cnt16[t] = (unsigned short)(old + (unsigned)__popc(peers));
            }
            old = __shfl_sync(0xffffffffu, old, leader);
            if (valid) {
                const unsigned pos = s_tb[t] + old + (unsigned)__popc(peers & lanemask_lt);
                G6R_CHECK(t < (unsigned)T && (int64_t)pos < ws.tile_starts[t + 1] &&
                          (int64_t)pos < ws.entry_capacity);
                vals[pos] = row;
            }
        }
    }
}

// --- optional export of the sorted runs (g6r_frame.entry_splat) --------------
// The scatter stores scene rows; the reference's entry_splat holds indices
// into the compacted SplatBatch (drawn rows in ascending scene order,
// raster.py:279-288, 366-376).  cidx[row] = number of drawn rows before row:
// the projection left each 256-row block's drawn count in proj_status[block]
// (k_project, splat-keys mode); k_rank_scan turns the block counts into
// exclusive offsets, k_rank_fill ranks rows inside a block (drawn <=> the rect
// is non-empty), k_export_runs maps every entry.  cidx lives in the sort
// ping-pong buffer that does not hold the sorted items (>= 8n bytes, unused
// after the partition).  Only views whose frame asks for entry_splat run.
__device__ __forceinline__ unsigned *rank_buffer(const Workspace &ws) {
    return reinterpret_cast<unsigned *>(ws.keys[(ws.internal[kSortPasses] & 1) ^ 1]);
}

__global__ void __launch_bounds__(1024) k_rank_scan(const __grid_constant__ Batch b, int64_t nblk) {
    __shared__ unsigned long long s_warp[32];
    __shared__ unsigned long long s_carry;
    const int v = blockIdx.y;
    PartCtx c;
    if (!b.out[v].entry_splat || !part_ctx(b, v, c)) return;
    unsigned long long *cnt = b.ws[v].proj_status;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int64_t k0 = 0; k0 < nblk; k0 += blockDim.x) {
        const int64_t k = k0 + threadIdx.x;
        const unsigned long long x = k < nblk ? cnt[k] : 0ull;
        const unsigned long long inc = warp_inclusive_scan(x);
        if (lane == 31) s_warp[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            const unsigned long long w = s_warp[lane];
            s_warp[lane] = warp_inclusive_scan(w) - w;
        }
        __syncthreads();
        const unsigned long long excl = s_carry + s_warp[warp] + inc - x;
        if (k < nblk) cnt[k] = excl;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_carry = excl + x;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kBlock) k_rank_fill(const __grid_constant__ Batch b, int64_t n) {
    __shared__ unsigned s_w[kBlock / 32];
    const int v = blockIdx.y;
    PartCtx c;
    if (!b.out[v].entry_splat || !part_ctx(b, v, c)) return;
    const Workspace &ws = b.ws[v];
    const int64_t row = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    const bool drawn = row < n && ws.rect[row].y != 0u;
    const unsigned bal = __ballot_sync(0xffffffffu, drawn);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s_w[warp] = (unsigned)__popc(bal);
    __syncthreads();
    unsigned pre = 0;
    for (int w = 0; w < warp; ++w) pre += s_w[w];
    if (drawn)
        rank_buffer(ws)[row] = (unsigned)ws.proj_status[blockIdx.x] + pre +
                               (unsigned)__popc(bal & ((1u << lane) - 1u));
}

__global__ void __launch_bounds__(kBlock) k_export_runs(const __grid_constant__ Batch b) {
    const int v = blockIdx.y;
    PartCtx c;
    int32_t *out = b.out[v].entry_splat;
    if (!out || !part_ctx(b, v, c)) return;
    const Workspace &ws = b.ws[v];
    const int64_t e = b.out[v].counters[G6R_CNT_ENTRIES];
    const unsigned *cidx = rank_buffer(ws);
    const unsigned *rows = ws.vals[0];
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < e;
         k += (int64_t)gridDim.x * blockDim.x) {
        G6R_CHECK(cidx[rows[k]] < (unsigned)c.m);
        out[k] = (int32_t)cidx[rows[k]];
    }
}

static size_t scatter_smem_bytes(int tiles) {
    return (size_t)((tiles + 3) & ~3) * sizeof(unsigned) + (size_t)kScatterWarps * ((tiles + 1) / 2) * sizeof(unsigned);
}

int launch_tile_partition(const Batch &b, int64_t n, int vbits, cudaStream_t st) {
    if (b.nviews == 0) return G6R_OK;
    const int tiles = b.vp[0].tiles_x * b.vp[0].tiles_y;
    const int64_t chunks = ceil_div(n > 0 ? n : 1, chunk_splats(tiles));
    const unsigned long long vmask = (1ull << vbits) - 1ull;
    const size_t count_smem = (size_t)kScatterWarps * ((tiles + 1) / 2) * sizeof(unsigned);
    const size_t scatter_smem = scatter_smem_bytes(tiles);
    static std::atomic<unsigned long long> attrs_done{0};   // one bit per device
    if (const unsigned long long bit = device_bit(); !(attrs_done.load() & bit)) {
        cudaFuncSetAttribute(k_chunk_count, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kScatterWarps * (kMaxSplatSortTiles / 2) * sizeof(unsigned)));
        cudaFuncSetAttribute(k_chunk_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)scatter_smem_bytes(kMaxSplatSortTiles));
        attrs_done.fetch_or(bit);   // idempotent: a racing thread sets the same values
    }
    const dim3 cgrid((unsigned)chunks, (unsigned)b.nviews);
    k_chunk_count<<<cgrid, kBlock, count_smem, st>>>(b, vmask);
    trace_mark("chunk_count", st);
    k_chunk_colscan<<<dim3((unsigned)ceil_div(tiles, 32), b.nviews), kBlock, 0, st>>>(b);
    trace_mark("chunk_colscan", st);
    k_tile_scan<<<dim3(1, b.nviews), 1024, 0, st>>>(b);
    trace_mark("tile_scan", st);
    k_chunk_scatter<<<cgrid, kBlock, scatter_smem, st>>>(b, vmask);
    trace_mark("chunk_scatter", st);
    bool want_runs = false;
    for (int v = 0; v < b.nviews; ++v) want_runs = want_runs || b.out[v].entry_splat;
    if (want_runs && n > 0) {
        const int64_t nblk = ceil_div(n, kBlock);
        k_rank_scan<<<dim3(1, b.nviews), 1024, 0, st>>>(b, nblk);
        k_rank_fill<<<dim3((unsigned)nblk, b.nviews), kBlock, 0, st>>>(b, n);
        int64_t cap = b.ws[0].entry_capacity;
        const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(cap, kBlock), 1184));
        k_export_runs<<<dim3(gx, b.nviews), kBlock, 0, st>>>(b);
        trace_mark("export_runs", st);
    }
    return cudaGetLastError() == cudaSuccess ? G6R_OK : G6R_ECUDA;
}

}  // namespace g6r
