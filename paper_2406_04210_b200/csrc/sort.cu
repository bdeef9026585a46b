// Spatial reordering: reference reorder_by_cell (neighbor.py:257-270) generalised
// to Hilbert-curve order.  Keys are 64-bit; the sort is a hand-written stable LSD
// radix sort (8-bit digits) carrying the particle index as payload; every
// per-particle array is then moved with a 16-byte (or 4-byte) row gather, so
// values are relocated bit-for-bit, never recomputed.
//
// One radix pass = three steps:
//   k_radix_hist    per-tile digit histogram (shared-memory atomics)
//                   -> hist[digit * n_tiles + tile]
//   exclusive scan  over that digit-major table (cells.cu) = global offset of
//                   every (digit, tile) bucket
//   k_radix_scatter stable rank of each key inside its tile (warp match_any +
//                   per-warp running digit counters), then the scatter.
#include "common.cuh"

namespace b2md {

int exclusive_scan_i32(const int32_t *d_in, int32_t *d_out, int64_t n, int32_t *d_tiles,
                       cudaStream_t stream);

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
#ifndef B2MD_SORT_KEYS_PER_THREAD
#define B2MD_SORT_KEYS_PER_THREAD 4
#endif
constexpr int kKeysPerThread = B2MD_SORT_KEYS_PER_THREAD;
constexpr int kSortTile = kSortThreads * kKeysPerThread;   // keys per CTA
constexpr int kRadix = 256;

// ------------------------------------------------------------------ keys
struct KeyGeom {
    double cell_edge[3];   // neighbor.py:71 cell edge, host fp64
    float inv_edge[3];     // 1 / cell_edge (sub-cell coordinate only)
    int nc[3];
    int cell_bits;         // bits per axis holding the cell coordinate
    int sub_bits;          // bits per axis refining the position inside the cell
};

// Skilling's transpose form of the Hilbert index (AIP Conf. Proc. 707, 2004),
// then bit-interleave x,y,z MSB first.
__device__ __forceinline__ uint64_t hilbert_index(uint32_t x, uint32_t y, uint32_t z, int bits) {
    uint32_t X[3] = {x, y, z};
    const uint32_t M = 1u << (bits - 1);
    for (uint32_t Q = M; Q > 1; Q >>= 1) {
        const uint32_t P = Q - 1;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            if (X[i] & Q) {
                X[0] ^= P;
            } else {
                const uint32_t t = (X[0] ^ X[i]) & P;
                X[0] ^= t;
                X[i] ^= t;
            }
        }
    }
    X[1] ^= X[0];
    X[2] ^= X[1];
    uint32_t t = 0;
    for (uint32_t Q = M; Q > 1; Q >>= 1)
        if (X[2] & Q) t ^= Q - 1;
    X[0] ^= t; X[1] ^= t; X[2] ^= t;
    uint64_t key = 0;
    for (int b = bits - 1; b >= 0; --b) {
#pragma unroll
        for (int i = 0; i < 3; ++i) key = (key << 1) | ((X[i] >> b) & 1u);
    }
    return key;
}

// Key = Hilbert index of the CELL-ALIGNED integer coordinate
//     q_a = (cell_a << sub_bits) | floor(frac_a * 2^sub_bits)
// where cell_a is exactly bin_particles' cell coordinate (fp64 division, clip;
// neighbor.py:74-75).  The Hilbert curve is hierarchical, so every cell's
// particles end up contiguous in the sorted order (cells follow the curve,
// particles inside a cell follow the refined curve).
__global__ void k_hilbert_keys(const float4 *__restrict__ pos_hi, const float4 *__restrict__ pos_lo,
                               int64_t n, KeyGeom g, uint64_t *__restrict__ keys) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 h = pos_hi[i], l = pos_lo[i];
    const double p[3] = {ds_to_double(h.x, l.x), ds_to_double(h.y, l.y), ds_to_double(h.z, l.z)};
    uint32_t q[3];
    const int sub_top = (1 << g.sub_bits) - 1;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        long long c = (long long)floor(__ddiv_rn(p[a], g.cell_edge[a]));
        c = c < 0 ? 0 : (c > g.nc[a] - 1 ? g.nc[a] - 1 : c);
        // position inside the cell, fp32 is plenty for a locality key
        const float frac =
            __double2float_rn(__dsub_rn(p[a], __dmul_rn((double)c, g.cell_edge[a]))) * g.inv_edge[a];
        int sub = (int)floorf(frac * (float)(1 << g.sub_bits));
        sub = sub < 0 ? 0 : (sub > sub_top ? sub_top : sub);
        q[a] = ((uint32_t)c << g.sub_bits) | (uint32_t)sub;
    }
    keys[i] = hilbert_index(q[0], q[1], q[2], g.cell_bits + g.sub_bits);
}

__global__ void k_cell_keys(const int32_t *__restrict__ cell_of, int64_t n,
                            uint64_t *__restrict__ keys) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) keys[i] = (uint64_t)(uint32_t)cell_of[i];
}

__global__ void k_iota(int32_t *__restrict__ v, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) v[i] = (int32_t)i;
}

// ------------------------------------------------------------- radix sort
__global__ void __launch_bounds__(kSortThreads)
k_radix_hist(const uint64_t *__restrict__ keys, int64_t n, int shift, int n_tiles,
             int32_t *__restrict__ hist) {
    __shared__ int s_hist[kRadix];
    s_hist[threadIdx.x] = 0;   // kSortThreads == kRadix
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kSortTile;
#pragma unroll
    for (int r = 0; r < kKeysPerThread; ++r) {
        const int64_t idx = base + r * kSortThreads + threadIdx.x;
        if (idx < n) atomicAdd(&s_hist[(int)((keys[idx] >> shift) & (kRadix - 1))], 1);
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * n_tiles + blockIdx.x] = s_hist[threadIdx.x];
}

__global__ void __launch_bounds__(kSortThreads)
k_radix_scatter(const uint64_t *__restrict__ keys_in, const int32_t *__restrict__ vals_in,
                int64_t n, int shift, int n_tiles, const int32_t *__restrict__ offsets,
                uint64_t *__restrict__ keys_out, int32_t *__restrict__ vals_out) {
    // per-warp running digit counts; after the prefix step: exclusive base of
    // (warp, digit) inside the tile
    __shared__ int s_count[kSortWarps][kRadix];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int d = threadIdx.x; d < kSortWarps * kRadix; d += kSortThreads)
        (&s_count[0][0])[d] = 0;
    __syncthreads();

    // warp w owns keys [w*512, (w+1)*512) of the tile, 16 rounds of 32 in order
    const int64_t wbase = (int64_t)blockIdx.x * kSortTile + (int64_t)warp * (32 * kKeysPerThread);
    uint64_t key[kKeysPerThread];
    int rank[kKeysPerThread];   // rank of the key among equal digits seen so far in this warp
    const unsigned lt_mask = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < kKeysPerThread; ++r) {
        const int64_t idx = wbase + r * 32 + lane;
        const bool ok = idx < n;
        key[r] = ok ? keys_in[idx] : ~0ull;
        const int digit = ok ? (int)((key[r] >> shift) & (kRadix - 1)) : kRadix;  // 256 = "absent"
        const unsigned peers = __match_any_sync(0xffffffffu, digit);
        const int before = ok ? s_count[warp][digit] : 0;
        rank[r] = before + __popc(peers & lt_mask);
        __syncwarp();
        if (ok && (peers & lt_mask) == 0) s_count[warp][digit] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // exclusive prefix over warps for each digit (thread d handles digit d)
    {
        const int d = threadIdx.x;
        int run = offsets[(int64_t)d * n_tiles + blockIdx.x];
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            const int c = s_count[w][d];
            s_count[w][d] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kKeysPerThread; ++r) {
        const int64_t idx = wbase + r * 32 + lane;
        if (idx < n) {
            const int digit = (int)((key[r] >> shift) & (kRadix - 1));
            const int64_t dst = (int64_t)s_count[warp][digit] + rank[r];
            keys_out[dst] = key[r];
            vals_out[dst] = vals_in[idx];
        }
    }
}

// ----------------------------------------------------------------- gathers
__global__ void k_gather16(const int4 *__restrict__ src, int4 *__restrict__ dst,
                           const int32_t *__restrict__ perm, int64_t n) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) dst[k] = __ldg(src + perm[k]);
}

__global__ void k_gather4(const int32_t *__restrict__ src, int32_t *__restrict__ dst,
                          const int32_t *__restrict__ perm, int64_t n) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) dst[k] = __ldg(src + perm[k]);
}

// Whole particle rows in one launch: five 16-byte arrays and one 4-byte array through the
// same permutation (read once), six independent loads in flight per thread.
struct GatherRows {
    const int4 *src16[5];
    int4 *dst16[5];
    const int32_t *src4;
    int32_t *dst4;
};

__global__ void __launch_bounds__(256)
k_gather_rows(const __grid_constant__ GatherRows g, const int32_t *__restrict__ perm, int64_t n) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int32_t p = perm[k];
    int4 v[5];
#pragma unroll
    for (int a = 0; a < 5; ++a) v[a] = __ldg(g.src16[a] + p);
    const int32_t w = g.src4 ? __ldg(g.src4 + p) : 0;
#pragma unroll
    for (int a = 0; a < 5; ++a) g.dst16[a][k] = v[a];
    if (g.src4) g.dst4[k] = w;
}

static inline int64_t sort_tiles(int64_t n) { return (n + kSortTile - 1) / kSortTile; }

}  // namespace b2md

using namespace b2md;

B2MD_EXPORT int b2md_hilbert_key_bits(const b2md_grid *grid, int32_t sub_bits) {
    if (!grid || sub_bits < 0) return -1;
    int mx = grid->ncell[0] > grid->ncell[1] ? grid->ncell[0] : grid->ncell[1];
    mx = mx > grid->ncell[2] ? mx : grid->ncell[2];
    int cell_bits = 1;
    while ((1 << cell_bits) < mx) ++cell_bits;
    if (cell_bits + sub_bits > 21) return -2;
    return 3 * (cell_bits + sub_bits);
}

B2MD_EXPORT int b2md_hilbert_keys(const void *d_pos_hi, const void *d_pos_lo, int64_t n,
                                  const b2md_grid *grid, int32_t sub_bits, uint64_t *d_keys,
                                  void *stream) {
    const int key_bits = b2md_hilbert_key_bits(grid, sub_bits);
    if (n <= 0 || key_bits < 0) {
        set_error("b2md_hilbert_keys: bad arguments (cell bits + sub bits must be <= 21)");
        return -1;
    }
    KeyGeom g;
    g.sub_bits = sub_bits;
    g.cell_bits = key_bits / 3 - sub_bits;
    for (int a = 0; a < 3; ++a) {
        g.nc[a] = grid->ncell[a];
        g.cell_edge[a] = grid->cell_edge[a];
        g.inv_edge[a] = (float)(1.0 / grid->cell_edge[a]);
    }
    k_hilbert_keys<<<blocks_for(n, 256), 256, 0, as_stream(stream)>>>(
        (const float4 *)d_pos_hi, (const float4 *)d_pos_lo, n, g, d_keys);
    B2MD_CHECK_LAUNCH("b2md_hilbert_keys");
    return 0;
}

B2MD_EXPORT int b2md_cell_keys(const int32_t *d_cell_of, int64_t n, uint64_t *d_keys,
                               void *stream) {
    if (n <= 0) { set_error("b2md_cell_keys: bad arguments"); return -1; }
    k_cell_keys<<<blocks_for(n, 256), 256, 0, as_stream(stream)>>>(d_cell_of, n, d_keys);
    B2MD_CHECK_LAUNCH("b2md_cell_keys");
    return 0;
}

B2MD_EXPORT int b2md_iota_i32(int32_t *d_vals, int64_t n, void *stream) {
    if (n <= 0) { set_error("b2md_iota_i32: bad arguments"); return -1; }
    k_iota<<<blocks_for(n, 256), 256, 0, as_stream(stream)>>>(d_vals, n);
    B2MD_CHECK_LAUNCH("b2md_iota_i32");
    return 0;
}

B2MD_EXPORT int64_t b2md_sort_scratch_bytes(int64_t n) {
    const int64_t tiles = sort_tiles(n < 1 ? 1 : n);
    const int64_t hist = kRadix * tiles;
    return (int64_t)sizeof(int32_t) * (2 * hist + 1 + scan_scratch_ints(hist)) + 256;
}

B2MD_EXPORT int b2md_sort_pairs_u64(uint64_t *d_keys, int32_t *d_vals, uint64_t *d_keys_tmp,
                                    int32_t *d_vals_tmp, int64_t n, int32_t key_bits,
                                    void *d_scratch, void *stream) {
    if (n <= 0 || key_bits < 1 || key_bits > 64 || !d_scratch) {
        set_error("b2md_sort_pairs_u64: bad arguments");
        return -1;
    }
    cudaStream_t s = as_stream(stream);
    const int64_t tiles = sort_tiles(n);
    if (tiles > 0x7fffffff / kRadix) { set_error("b2md_sort_pairs_u64: n too large"); return -2; }
    const int64_t hist_len = kRadix * tiles;
    int32_t *hist = (int32_t *)d_scratch;
    int32_t *offs = hist + hist_len;          // hist_len + 1 entries
    int32_t *scan_tiles = offs + hist_len + 1;
    uint64_t *kin = d_keys, *kout = d_keys_tmp;
    int32_t *vin = d_vals, *vout = d_vals_tmp;
    const int passes = (key_bits + 7) / 8;
    for (int p = 0; p < passes; ++p) {
        const int shift = 8 * p;
        k_radix_hist<<<(unsigned)tiles, kSortThreads, 0, s>>>(kin, n, shift, (int)tiles, hist);
        int rc = exclusive_scan_i32(hist, offs, hist_len, scan_tiles, s);
        if (rc) return rc;
        k_radix_scatter<<<(unsigned)tiles, kSortThreads, 0, s>>>(kin, vin, n, shift, (int)tiles,
                                                                 offs, kout, vout);
        uint64_t *tk = kin; kin = kout; kout = tk;
        int32_t *tv = vin; vin = vout; vout = tv;
    }
    B2MD_CHECK_LAUNCH("b2md_sort_pairs_u64");
    if (kin != d_keys) {
        int rc = check_cuda(cudaMemcpyAsync(d_keys, kin, sizeof(uint64_t) * n,
                                            cudaMemcpyDeviceToDevice, s), "sort copy keys");
        if (rc) return rc;
        rc = check_cuda(cudaMemcpyAsync(d_vals, vin, sizeof(int32_t) * n,
                                        cudaMemcpyDeviceToDevice, s), "sort copy vals");
        if (rc) return rc;
    }
    return 0;
}

B2MD_EXPORT int b2md_gather16(const void *d_src, void *d_dst, const int32_t *d_perm, int64_t n,
                              void *stream) {
    if (n <= 0) { set_error("b2md_gather16: bad arguments"); return -1; }
    k_gather16<<<blocks_for(n, 256), 256, 0, as_stream(stream)>>>((const int4 *)d_src,
                                                                  (int4 *)d_dst, d_perm, n);
    B2MD_CHECK_LAUNCH("b2md_gather16");
    return 0;
}

B2MD_EXPORT int b2md_gather_rows(const void *const *d_src16, void *const *d_dst16,
                                 const void *d_src4, void *d_dst4, const int32_t *d_perm,
                                 int64_t n, void *stream) {
    if (n <= 0 || !d_src16 || !d_dst16 || !d_perm || (d_src4 && !d_dst4)) {
        set_error("b2md_gather_rows: bad arguments");
        return -1;
    }
    GatherRows g;
    for (int a = 0; a < 5; ++a) {
        if (!d_src16[a] || !d_dst16[a]) { set_error("b2md_gather_rows: null array"); return -1; }
        g.src16[a] = (const int4 *)d_src16[a];
        g.dst16[a] = (int4 *)d_dst16[a];
    }
    g.src4 = (const int32_t *)d_src4;
    g.dst4 = (int32_t *)d_dst4;
    k_gather_rows<<<blocks_for(n, 256), 256, 0, as_stream(stream)>>>(g, d_perm, n);
    B2MD_CHECK_LAUNCH("b2md_gather_rows");
    return 0;
}

B2MD_EXPORT int b2md_gather4(const void *d_src, void *d_dst, const int32_t *d_perm, int64_t n,
                             void *stream) {
    if (n <= 0) { set_error("b2md_gather4: bad arguments"); return -1; }
    k_gather4<<<blocks_for(n, 256), 256, 0, as_stream(stream)>>>((const int32_t *)d_src,
                                                                 (int32_t *)d_dst, d_perm, n);
    B2MD_CHECK_LAUNCH("b2md_gather4");
    return 0;
}
