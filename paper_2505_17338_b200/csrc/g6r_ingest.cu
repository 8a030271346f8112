// g6r_ingest.cu -- scene ingest on device.
//
//   * Psi decode: the 37-channel parameter volume on the half-resolution grid
//     -> scene rows for the foreground voxels in np.nonzero (C) order
//     (priming.py:232-285 decode_param_volume);
//   * group filter: rows whose label is in a 12-bit mask, order kept
//     (priming.py:362-374 filter_scene) -- the same stream compaction.
//
// Compaction is order-preserving and deterministic: a count pass (one CTA per
// 4096-item chunk), a one-CTA exclusive scan of the chunk counts, and an emit
// pass that re-evaluates the predicate and ranks items inside the chunk with
// warp ballots.  All three kernels are HBM-bound streaming passes.
#include "g6r_common.cuh"
#include "g6r_internal.h"

namespace g6r {

constexpr int kCompactItems = 16;
constexpr int kChunk = kBlock * kCompactItems;   // 4096 items per CTA

struct VoxelPred {   // foreground voxel of the half grid
    const uint8_t *lab;
    __device__ bool operator()(int64_t i) const { return lab[i] != 0; }
};

struct LabelPred {   // row whose label bit is set in the mask
    const uint8_t *lab;
    uint32_t mask;
    __device__ bool operator()(int64_t i) const { return (mask >> (lab[i] & 31u)) & 1u; }
};

template <class Pred>
__global__ void __launch_bounds__(kBlock) k_compact_count(int64_t n, Pred pred, unsigned *counts) {
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    int c = 0;
#pragma unroll 4
    for (int k = 0; k < kCompactItems; ++k) {
        const int64_t i = base + k * kBlock + threadIdx.x;
        c += __syncthreads_count(i < n && pred(i));
    }
    if (threadIdx.x == 0) counts[blockIdx.x] = (unsigned)c;
}

// in-place exclusive scan of nb chunk counts; total -> *count
__global__ void __launch_bounds__(1024) k_compact_scan(int nb, unsigned *counts, int64_t *count) {
    __shared__ unsigned warp_tot[32];
    __shared__ unsigned long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int b0 = 0; b0 < nb; b0 += 1024) {
        const int i = b0 + threadIdx.x;
        const unsigned v = i < nb ? counts[i] : 0u;
        const unsigned inc = warp_inclusive_scan(v);
        if (lane == 31) warp_tot[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            const unsigned t = warp_tot[lane];
            warp_tot[lane] = warp_inclusive_scan(t) - t;
        }
        __syncthreads();
        const unsigned long long excl = carry + warp_tot[warp] + inc - v;
        if (i < nb) counts[i] = (unsigned)excl;
        __syncthreads();
        if (threadIdx.x == 1023) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) *count = (int64_t)carry;
}

// Rank the chunk's kept items in index order and hand (item, row) to emit.
template <class Pred, class Emit>
__global__ void __launch_bounds__(kBlock)
k_compact_emit(int64_t n, Pred pred, const unsigned *offsets, Emit emit) {
    __shared__ unsigned warp_cnt[kBlock / 32];
    const int64_t base = (int64_t)blockIdx.x * kChunk;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t row = offsets[blockIdx.x];
    for (int k = 0; k < kCompactItems; ++k) {
        const int64_t i = base + k * kBlock + threadIdx.x;
        const bool keep = i < n && pred(i);
        const unsigned ball = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) warp_cnt[warp] = __popc(ball);
        __syncthreads();
        unsigned before = 0, total = 0;
#pragma unroll
        for (int w = 0; w < kBlock / 32; ++w) {
            const unsigned c = warp_cnt[w];
            before += w < warp ? c : 0u;
            total += c;
        }
        if (keep) emit(i, row + before + __popc(ball & ((1u << lane) - 1u)));
        row += total;
        __syncthreads();
    }
}

// --- Psi decode ---------------------------------------------------------------

struct DecodeArgs {
    const void *psi;          // (37, V) f32 or f64, channel-major
    const double *base;       // (4, V) base R, G, B, A on the half grid
    const uint8_t *lab;       // (V)
    int64_t V;
    int dh, dw;               // half-grid H', W'
    double spacing[3], origin[3], dir[9];
    double *mu_p, *mu_d, *cov_raw, *sh, *opacity_raw;
    uint8_t *labels;
};

constexpr double kShC0 = 0.28209479177387814;   // core.py SH_C0

template <bool kF32>
struct DecodeEmit {
    DecodeArgs a;
    __device__ double psi(int c, int64_t v) const {
        if (kF32) return (double)static_cast<const float *>(a.psi)[c * a.V + v];
        return static_cast<const double *>(a.psi)[c * a.V + v];
    }
    __device__ void operator()(int64_t v, int64_t r) const {
        const int64_t plane = (int64_t)a.dh * a.dw;
        const int64_t z = v / plane;
        const int64_t rem = v - z * plane;
        const int64_t y = rem / a.dw;
        const int64_t x = rem - y * a.dw;
        // voxel_world_coords (priming.py:125-134): origin + (idx * spacing) @ dir^T,
        // accumulated as the reference host's OpenBLAS dgemm does (fma chain
        // from column 0; pinned by tests/golden/ingest_rotated.npz)
        const double q0 = (double)(x * 2) * a.spacing[0];
        const double q1 = (double)(y * 2) * a.spacing[1];
        const double q2 = (double)(z * 2) * a.spacing[2];
#pragma unroll
        for (int k = 0; k < 3; ++k)
            a.mu_p[r * 3 + k] = a.origin[k] + __fma_rn(q2, a.dir[k * 3 + 2],
                                                       __fma_rn(q1, a.dir[k * 3 + 1],
                                                                q0 * a.dir[k * 3 + 0]));
        a.mu_d[r * 3 + 0] = 0.0 + psi(0, v);   // DEFAULT_MU_D + pred[0:3]
        a.mu_d[r * 3 + 1] = 0.0 + psi(1, v);
        a.mu_d[r * 3 + 2] = 1.0 + psi(2, v);
#pragma unroll
        for (int k = 0; k < 3; ++k)
            a.sh[r * 12 + k] = (a.base[k * a.V + v] - 0.5) / kShC0 + psi(3 + k, v);
#pragma unroll
        for (int k = 0; k < 9; ++k) a.sh[r * 12 + 3 + k] = psi(6 + k, v);
        a.opacity_raw[r] = a.base[3 * a.V + v] + psi(15, v);
#pragma unroll
        for (int k = 0; k < 21; ++k) a.cov_raw[r * 21 + k] = psi(16 + k, v);
        a.labels[r] = a.lab[v];
    }
};

// --- group filter -------------------------------------------------------------

struct FilterArgs {
    const double *in[5];
    double *out[5];
    const uint8_t *lab;
    uint8_t *labels;
};

struct FilterEmit {
    FilterArgs a;
    __device__ void operator()(int64_t i, int64_t r) const {
        const int widths[5] = {3, 3, 21, 12, 1};
#pragma unroll
        for (int f = 0; f < 5; ++f)
            for (int k = 0; k < widths[f]; ++k) a.out[f][r * widths[f] + k] = a.in[f][i * widths[f] + k];
        a.labels[r] = a.lab[i];
    }
};

size_t compact_workspace_bytes(int64_t n) {
    const int64_t nb = ceil_div(n > 0 ? n : 1, kChunk);
    return (size_t)((nb * 4 + 255) & ~255ll);
}

template <class Pred>
static int compact_count(int64_t n, Pred p, unsigned *counts, int64_t *count, cudaStream_t st) {
    const int64_t nb = ceil_div(n > 0 ? n : 1, kChunk);
    if (nb >= (1ll << 31)) return 1;
    k_compact_count<<<(unsigned)nb, kBlock, 0, st>>>(n, p, counts);
    k_compact_scan<<<1, 1024, 0, st>>>((int)nb, counts, count);
    return cudaGetLastError() != cudaSuccess;
}

int launch_decode_count(int64_t V, const uint8_t *lab, void *ws, int64_t *count, cudaStream_t st) {
    return compact_count(V, VoxelPred{lab}, static_cast<unsigned *>(ws), count, st);
}

int launch_decode_emit(const DecodeArgsHost &h, void *ws, cudaStream_t st) {
    DecodeArgs a{};
    a.psi = h.psi;
    a.base = h.base;
    a.lab = h.lab;
    a.V = h.V;
    a.dh = h.dh;
    a.dw = h.dw;
    for (int k = 0; k < 3; ++k) {
        a.spacing[k] = h.spacing[k];
        a.origin[k] = h.origin[k];
    }
    for (int k = 0; k < 9; ++k) a.dir[k] = h.dir[k];
    a.mu_p = h.mu_p;
    a.mu_d = h.mu_d;
    a.cov_raw = h.cov_raw;
    a.sh = h.sh;
    a.opacity_raw = h.opacity_raw;
    a.labels = h.labels;
    const int64_t nb = ceil_div(h.V > 0 ? h.V : 1, kChunk);
    const unsigned *offs = static_cast<const unsigned *>(ws);
    if (h.psi_f32)
        k_compact_emit<<<(unsigned)nb, kBlock, 0, st>>>(h.V, VoxelPred{h.lab}, offs, DecodeEmit<true>{a});
    else
        k_compact_emit<<<(unsigned)nb, kBlock, 0, st>>>(h.V, VoxelPred{h.lab}, offs, DecodeEmit<false>{a});
    return cudaGetLastError() != cudaSuccess;
}

int launch_filter_rows(int64_t n, const uint8_t *lab, uint32_t mask, const double *const in[5],
                       double *const out[5], uint8_t *labels, void *ws, int64_t *count,
                       cudaStream_t st) {
    if (compact_count(n, LabelPred{lab, mask}, static_cast<unsigned *>(ws), count, st)) return 1;
    FilterArgs a{};
    for (int f = 0; f < 5; ++f) {
        a.in[f] = in[f];
        a.out[f] = out[f];
    }
    a.lab = lab;
    a.labels = labels;
    const int64_t nb = ceil_div(n > 0 ? n : 1, kChunk);
    k_compact_emit<<<(unsigned)nb, kBlock, 0, st>>>(n, LabelPred{lab, mask},
                                                    static_cast<const unsigned *>(ws), FilterEmit{a});
    return cudaGetLastError() != cudaSuccess;
}

}  // namespace g6r
