// Cell-list binning: reference bin_particles (neighbor.py:57-91).
//   1. k_cell_index : cell of every particle in fp64 (true division, clip) and an
//                     atomic per-cell count that hands back the in-cell slot;
//   2. exclusive prefix sum of the counts (warp-shuffle scan, three launches);
//   3. k_scatter    : particle index -> cell_start[cell] + slot;
//   4. k_sort_cells : ascending particle index inside every cell, which is the
//                     order the reference's stable argsort produces.
// All integer outputs are bit-exact with the reference for positions given as
// (double)hi + (double)lo.
#include <math.h>

#include "common.cuh"

namespace b2md {

constexpr int kThreads = 256;
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

struct GridD {
    int nc[3];
    double edge[3];
};

__global__ void k_cell_index(const float4 *__restrict__ pos_hi, const float4 *__restrict__ pos_lo,
                             int64_t n, GridD g, int32_t *__restrict__ cell_of,
                             int32_t *__restrict__ count, int32_t *__restrict__ slot) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    float4 h = pos_hi[i], l = pos_lo[i];
    double p[3] = {ds_to_double(h.x, l.x), ds_to_double(h.y, l.y), ds_to_double(h.z, l.z)};
    int c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        // idx = floor(pos / cell_edge), clipped to [0, nc-1]   (neighbor.py:74-75)
        double q = floor(__ddiv_rn(p[a], g.edge[a]));
        long long k = (long long)q;
        k = k < 0 ? 0 : (k > g.nc[a] - 1 ? g.nc[a] - 1 : k);
        c[a] = (int)k;
    }
    int flat = (c[0] * g.nc[1] + c[1]) * g.nc[2] + c[2];
    cell_of[i] = flat;
    slot[i] = atomicAdd(&count[flat], 1);
}

// ---- exclusive scan over int32, tiles of 4096 ------------------------------
__device__ __forceinline__ int block_exclusive_scan(int v, int *warp_sums, int &block_total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) warp_sums[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        int w = lane < (blockDim.x >> 5) ? warp_sums[lane] : 0;
        int winc = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, winc, o);
            if (lane >= o) winc += t;
        }
        warp_sums[lane] = winc - w;  // exclusive per-warp offsets
        if (lane == 31) warp_sums[32] = winc;
    }
    __syncthreads();
    block_total = warp_sums[32];
    return inc - v + warp_sums[warp];
}

// Pass 1: scan every tile locally, emit tile totals.
__global__ void __launch_bounds__(kScanThreads)
k_scan_tiles(const int32_t *__restrict__ in, int64_t n, int32_t *__restrict__ out,
             int32_t *__restrict__ tile_total) {
    __shared__ int warp_sums[33];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int v[kScanItems];
    int sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = (base + k < n) ? in[base + k] : 0;
        sum += v[k];
    }
    int total;
    int ex = block_exclusive_scan(sum, warp_sums, total);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < n) out[base + k] = ex;
        ex += v[k];
    }
    if (threadIdx.x == 0) tile_total[blockIdx.x] = total;
}

// Pass 2: one block scans the tile totals in place (<= 4096 tiles per round).
__global__ void __launch_bounds__(kScanThreads)
k_scan_totals(int32_t *tile_total, int n_tiles, int32_t *grand_total) {
    __shared__ int warp_sums[33];
    int carry = 0;
    for (int start = 0; start < n_tiles; start += kScanTile) {
        const int base = start + threadIdx.x * kScanItems;
        int v[kScanItems];
        int sum = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            v[k] = (base + k < n_tiles) ? tile_total[base + k] : 0;
            sum += v[k];
        }
        int total;
        int ex = block_exclusive_scan(sum, warp_sums, total) + carry;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            if (base + k < n_tiles) tile_total[base + k] = ex;
            ex += v[k];
        }
        carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) *grand_total = carry;
}

// Pass 3: add tile offsets; the entry one past the end gets the grand total.
__global__ void __launch_bounds__(kScanThreads)
k_scan_apply(int32_t *out, int64_t n, const int32_t *__restrict__ tile_offset,
             const int32_t *__restrict__ grand_total) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    const int off = tile_offset[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
        if (base + k < n) out[base + k] += off;
    if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = *grand_total;
}

__global__ void k_scatter(const int32_t *__restrict__ cell_of, const int32_t *__restrict__ slot,
                          const int32_t *__restrict__ cell_start, int64_t n,
                          int32_t *__restrict__ cell_particles) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    cell_particles[cell_start[cell_of[i]] + slot[i]] = (int32_t)i;
}

// One thread per cell: ascending order of its (short) occupant slice.  After a Hilbert /
// cell reorder the occupants of a cell are consecutive rows, so the slice is a permutation
// of [min, min + m): one read pass finds that out and one write pass stores min + k.
// Otherwise: insertion sort.
__global__ void k_sort_cells(const int32_t *__restrict__ cell_start, int64_t n_cells,
                             int32_t *__restrict__ cell_particles) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n_cells) return;
    const int lo = cell_start[c], hi = cell_start[c + 1];
    if (hi - lo < 2) return;
    {
        int vmin = 0x7fffffff, vmax = -1;
        bool sorted = true;
        int prev = -1;
        for (int a = lo; a < hi; ++a) {
            const int v = cell_particles[a];
            vmin = min(vmin, v);
            vmax = max(vmax, v);
            sorted = sorted && v > prev;
            prev = v;
        }
        if (sorted) return;
        if (vmax - vmin == hi - lo - 1) {           // distinct indices: a contiguous range
            for (int a = lo; a < hi; ++a) cell_particles[a] = vmin + (a - lo);
            return;
        }
    }
    for (int a = lo + 1; a < hi; ++a) {
        int v = cell_particles[a];
        int b = a - 1;
        while (b >= lo && cell_particles[b] > v) {
            cell_particles[b + 1] = cell_particles[b];
            --b;
        }
        cell_particles[b + 1] = v;
    }
}

// Single-launch scan for up to kFusedScanTiles tiles: a tile takes a ticket (so that
// every predecessor is already running), scans itself, publishes its total as one 64-bit
// word {ready, total}, then warp 0 sums the totals of all predecessors (32 per round,
// polling until each is ready) -- the tile never waits for a predecessor's PREFIX, only
// for its local total, so the wait is one block scan deep whatever the tile count.

__global__ void __launch_bounds__(kScanThreads)
k_scan_fused(const int32_t *__restrict__ in, int64_t n, int32_t *__restrict__ out,
             unsigned long long *state, int n_tiles) {
    __shared__ int warp_sums[33];
    __shared__ int s_tile, s_prefix;
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(&state[n_tiles], 1ull);
    __syncthreads();
    const int tile = s_tile;
    const int64_t base = (int64_t)tile * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int v[kScanItems];
    int sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = (base + k < n) ? in[base + k] : 0;
        sum += v[k];
    }
    int total;
    int ex = block_exclusive_scan(sum, warp_sums, total);
    if (threadIdx.x == 0) {
        *(volatile unsigned long long *)&state[tile] = (1ull << 32) | (unsigned)total;
        __threadfence();
    }
    if (threadIdx.x < 32) {
        int prefix = 0;
        for (int p0 = 0; p0 < tile; p0 += 32) {
            const int p = p0 + (int)threadIdx.x;
            int t = 0;
            if (p < tile) {
                unsigned long long w;
                do { w = *(volatile unsigned long long *)&state[p]; } while ((w >> 32) == 0ull);
                t = (int)(unsigned)w;
            }
            prefix += __reduce_add_sync(0xffffffffu, t);
        }
        if (threadIdx.x == 0) s_prefix = prefix;
    }
    __syncthreads();
    ex += s_prefix;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < n) out[base + k] = ex;
        ex += v[k];
    }
    if (tile == n_tiles - 1 && threadIdx.x == 0) out[n] = s_prefix + total;
}

// Exclusive scan of d_in[0..n) into d_out[0..n], d_out[n] = total.
// d_tiles: scan_scratch_ints(n) ints of scratch (common.cuh).
int exclusive_scan_i32(const int32_t *d_in, int32_t *d_out, int64_t n, int32_t *d_tiles,
                       cudaStream_t stream) {
    const int64_t n_tiles = (n + kScanTile - 1) / kScanTile;
    if (n_tiles > (int64_t)kScanTile * 4096) {
        set_error("exclusive_scan_i32: n=%lld too large", (long long)n);
        return -2;
    }
    if (n_tiles >= 1 && n_tiles <= kFusedScanTiles) {
        unsigned long long *state =
            (unsigned long long *)(((uintptr_t)d_tiles + 7) & ~(uintptr_t)7);
        int rc = check_cuda(cudaMemsetAsync(state, 0, sizeof(unsigned long long) * (n_tiles + 1),
                                            stream), "exclusive_scan_i32 memset");
        if (rc) return rc;
        k_scan_fused<<<(unsigned)n_tiles, kScanThreads, 0, stream>>>(d_in, n, d_out, state,
                                                                    (int)n_tiles);
        B2MD_CHECK_LAUNCH("exclusive_scan_i32");
        return 0;
    }
    k_scan_tiles<<<(unsigned)n_tiles, kScanThreads, 0, stream>>>(d_in, n, d_out, d_tiles);
    k_scan_totals<<<1, kScanThreads, 0, stream>>>(d_tiles, (int)n_tiles, d_tiles + n_tiles);
    k_scan_apply<<<(unsigned)n_tiles, kScanThreads, 0, stream>>>(d_out, n, d_tiles,
                                                                d_tiles + n_tiles);
    B2MD_CHECK_LAUNCH("exclusive_scan_i32");
    return 0;
}

}  // namespace b2md

using namespace b2md;

// neighbor.py:64-71,90 in host fp64.
B2MD_EXPORT int b2md_grid_shape(const b2md_box *box, double r_list, b2md_grid *g) {
    if (!box || !g) { set_error("b2md_grid_shape: null argument"); return -1; }
    if (!(r_list > 0.0) || !isfinite(r_list)) {
        set_error("b2md_grid_shape: r_list must be positive and finite");
        return -2;
    }
    g->n_cells = 1;
    g->fallback = 0;
    for (int a = 0; a < 3; ++a) {
        const double L = box->edge[a];
        if (L < r_list) {
            set_error("b2md_grid_shape: box edge %g < r_list %g", L, r_list);
            return -3;
        }
        long long nc = (long long)floor(L / r_list);
        if (nc < 1) nc = 1;
        if (nc > 2000000) { set_error("b2md_grid_shape: too many cells"); return -4; }
        g->ncell[a] = (int32_t)nc;
        g->cell_edge[a] = L / (double)nc;
        g->n_cells *= nc;
        if (nc < 3) g->fallback = 1;
    }
    if (g->n_cells > 2000000000LL) { set_error("b2md_grid_shape: too many cells"); return -4; }
    return 0;
}

B2MD_EXPORT int64_t b2md_bin_scratch_bytes(int64_t n, int64_t n_cells) {
    // counts (n_cells) + slot (n) + scan tiles
    return (int64_t)sizeof(int32_t) * (n_cells + n + scan_scratch_ints(n_cells)) + 256;
}

B2MD_EXPORT int b2md_bin(const void *d_pos_hi, const void *d_pos_lo, int64_t n,
                         const b2md_grid *grid, int32_t *d_cell_of, int32_t *d_cell_start,
                         int32_t *d_cell_particles, void *d_scratch, void *stream) {
    if (n <= 0 || !grid) { set_error("b2md_bin: bad arguments"); return -1; }
    if (n > 2000000000LL) { set_error("b2md_bin: n too large for int32 indices"); return -2; }
    cudaStream_t s = as_stream(stream);
    const int64_t nc = grid->n_cells;
    int32_t *count = (int32_t *)d_scratch;
    int32_t *slot = count + nc;
    int32_t *tiles = slot + n;
    int rc = check_cuda(cudaMemsetAsync(count, 0, sizeof(int32_t) * nc, s), "b2md_bin memset");
    if (rc) return rc;
    GridD g;
    for (int a = 0; a < 3; ++a) { g.nc[a] = grid->ncell[a]; g.edge[a] = grid->cell_edge[a]; }
    k_cell_index<<<blocks_for(n, kThreads), kThreads, 0, s>>>(
        (const float4 *)d_pos_hi, (const float4 *)d_pos_lo, n, g, d_cell_of, count, slot);
    B2MD_CHECK_LAUNCH("k_cell_index");
    rc = exclusive_scan_i32(count, d_cell_start, nc, tiles, s);
    if (rc) return rc;
    k_scatter<<<blocks_for(n, kThreads), kThreads, 0, s>>>(d_cell_of, slot, d_cell_start, n,
                                                           d_cell_particles);
    k_sort_cells<<<blocks_for(nc, kThreads), kThreads, 0, s>>>(d_cell_start, nc, d_cell_particles);
    B2MD_CHECK_LAUNCH("b2md_bin");
    return 0;
}
