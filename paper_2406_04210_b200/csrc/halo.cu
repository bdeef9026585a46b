// Slab decomposition support (no counterpart in the reference, SPEC.md:131 lists
// spatial decomposition as a non-goal): classification of
// owned particles against the slab faces, stable stream compaction of the
// selected rows, and packing of migration / ghost records.
//
// A rank owns x in [x_lo, x_hi) of the global periodic box and keeps, behind its
// owned rows, ghost copies of neighbour-rank particles within r_ghost of its
// faces -- all in GLOBAL coordinates, so the cell, list and force kernels (which
// wrap periodically over the global box) run unchanged on owned + ghost rows.
#include "common.cuh"

namespace b2md {

int exclusive_scan_i32(const int32_t *d_in, int32_t *d_out, int64_t n, int32_t *d_tiles,
                       cudaStream_t stream);

constexpr int kThreads = 256;

// Offset of x from the slab centre, the short way round the periodic axis, in
// fp64 without contraction (a numpy restatement reproduces it bit for bit):
//     d = x - centre;  d -= L * floor(d / L + 0.5)          in [-L/2, L/2)
// A particle is inside the slab iff -half <= d < half.
//   lo_cut / hi_cut: flag_left = d < lo_cut, flag_right = d >= hi_cut
//   (migration: lo_cut = -half, hi_cut = half; ghosts: -half + r_ghost, half - r_ghost).
__global__ void k_slab_classify(const float4 *__restrict__ pos_hi, const float4 *__restrict__ pos_lo,
                                int64_t n, double centre, double Lx, double lo_cut, double hi_cut,
                                int32_t *__restrict__ left, int32_t *__restrict__ right) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x = ds_to_double(pos_hi[i].x, pos_lo[i].x);
    double d = __dsub_rn(x, centre);
    d = __dsub_rn(d, __dmul_rn(Lx, floor(__dadd_rn(__ddiv_rn(d, Lx), 0.5))));
    left[i] = d < lo_cut;
    right[i] = d >= hi_cut;
}

__global__ void k_compact_scatter(const int32_t *__restrict__ flags,
                                  const int32_t *__restrict__ offsets, int64_t n,
                                  int32_t *__restrict__ out_idx) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && flags[i]) out_idx[offsets[i]] = (int32_t)i;
}

__global__ void k_flag_not_either(const int32_t *__restrict__ a, const int32_t *__restrict__ b,
                                  int64_t n, int32_t *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = (a[i] | b[i]) ? 0 : 1;
}

// Destination slots of the fused per-step halo: dst[i] = -1 for every owned row, then
// dst[send_idx[k]] = base + k (row k of the send list lands in ghost row base + k of the
// neighbour rank).
__global__ void k_halo_slots(const int32_t *__restrict__ send_idx, int64_t n_send, int32_t base,
                             int64_t n, int32_t *__restrict__ dst, bool fill) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (fill) {
        if (i < n) dst[i] = -1;
    } else if (i < n_send) {
        dst[send_idx[i]] = base + (int32_t)i;
    }
}

}  // namespace b2md

using namespace b2md;

B2MD_EXPORT int b2md_halo_slots(const int32_t *d_send_idx, int64_t n_send, int32_t base,
                                int64_t n, int32_t *d_dst, void *stream) {
    if (n < 0 || n_send < 0 || n_send > n || base < 0 || !d_dst || (n_send && !d_send_idx)) {
        set_error("b2md_halo_slots: bad arguments");
        return -1;
    }
    if (n == 0) return 0;
    k_halo_slots<<<blocks_for(n, kThreads), kThreads, 0, as_stream(stream)>>>(
        d_send_idx, n_send, base, n, d_dst, true);
    B2MD_CHECK_LAUNCH("b2md_halo_slots");
    if (n_send) {
        k_halo_slots<<<blocks_for(n_send, kThreads), kThreads, 0, as_stream(stream)>>>(
            d_send_idx, n_send, base, n, d_dst, false);
        B2MD_CHECK_LAUNCH("b2md_halo_slots");
    }
    return 0;
}

// Kernels of the CURRENT device may load / store memory of `peer_device` afterwards
// (NVLink / NVSwitch peer access).  Same device, or already enabled: ok.
B2MD_EXPORT int b2md_enable_peer_access(int32_t peer_device) {
    int dev = -1;
    int rc = check_cuda(cudaGetDevice(&dev), "b2md_enable_peer_access");
    if (rc) return rc;
    if (dev == peer_device) return 0;
    int can = 0;
    rc = check_cuda(cudaDeviceCanAccessPeer(&can, dev, peer_device), "b2md_enable_peer_access");
    if (rc) return rc;
    if (!can) {
        set_error("b2md_enable_peer_access: device %d cannot access device %d", dev, peer_device);
        return -2;
    }
    cudaError_t err = cudaDeviceEnablePeerAccess(peer_device, 0);
    if (err == cudaErrorPeerAccessAlreadyEnabled) { cudaGetLastError(); return 0; }
    return check_cuda(err, "b2md_enable_peer_access");
}

namespace b2md {
// out[dst[i]] = rows[i] for every i with dst[i] >= 0: the halo stores of the step kernel
// on their own (start-up probe of the peer mapping, decomp.py).
__global__ void k_halo_store(const float4 *__restrict__ rows, const int32_t *__restrict__ dst,
                             int64_t n, float4 *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int slot = dst[i];
    if (slot >= 0) out[slot] = rows[i];
}
}  // namespace b2md

B2MD_EXPORT int b2md_halo_store(const void *d_rows_f4, const int32_t *d_dst, int64_t n,
                                void *d_out_f4, void *stream) {
    if (n < 0 || (n > 0 && (!d_rows_f4 || !d_dst || !d_out_f4))) {
        set_error("b2md_halo_store: bad arguments");
        return -1;
    }
    if (n == 0) return 0;
    b2md::k_halo_store<<<blocks_for(n, 256), 256, 0, as_stream(stream)>>>(
        (const float4 *)d_rows_f4, d_dst, n, (float4 *)d_out_f4);
    B2MD_CHECK_LAUNCH("b2md_halo_store");
    return 0;
}

B2MD_EXPORT int b2md_slab_classify(const void *d_pos_hi, const void *d_pos_lo, int64_t n,
                                   double centre, double box_x, double lo_cut, double hi_cut,
                                   int32_t *d_flag_left, int32_t *d_flag_right, void *stream) {
    if (n < 0 || !(box_x > 0.0)) { set_error("b2md_slab_classify: bad arguments"); return -1; }
    if (n == 0) return 0;
    k_slab_classify<<<blocks_for(n, kThreads), kThreads, 0, as_stream(stream)>>>(
        (const float4 *)d_pos_hi, (const float4 *)d_pos_lo, n, centre, box_x, lo_cut, hi_cut,
        d_flag_left, d_flag_right);
    B2MD_CHECK_LAUNCH("b2md_slab_classify");
    return 0;
}

B2MD_EXPORT int64_t b2md_compact_scratch_bytes(int64_t n) {
    return (int64_t)sizeof(int32_t) * ((n < 1 ? 1 : n) + 1 + scan_scratch_ints(n)) + 256;
}

// Stable stream compaction: d_out_idx receives, in ascending order, the indices i
// with d_flags[i] != 0 (flags must be 0/1); d_count[0] receives how many.
B2MD_EXPORT int b2md_compact_indices(const int32_t *d_flags, int64_t n, int32_t *d_out_idx,
                                     int32_t *d_count, void *d_scratch, void *stream) {
    if (n < 0 || !d_count || !d_scratch) { set_error("b2md_compact_indices: bad arguments"); return -1; }
    cudaStream_t s = as_stream(stream);
    if (n == 0) return check_cuda(cudaMemsetAsync(d_count, 0, sizeof(int32_t), s), "compact memset");
    int32_t *offsets = (int32_t *)d_scratch;        // n + 1
    int32_t *tiles = offsets + n + 1;
    int rc = exclusive_scan_i32(d_flags, offsets, n, tiles, s);
    if (rc) return rc;
    k_compact_scatter<<<blocks_for(n, kThreads), kThreads, 0, s>>>(d_flags, offsets, n, d_out_idx);
    B2MD_CHECK_LAUNCH("b2md_compact_indices");
    return check_cuda(cudaMemcpyAsync(d_count, offsets + n, sizeof(int32_t),
                                      cudaMemcpyDeviceToDevice, s), "compact count");
}

// out[i] = !(a[i] | b[i])  (the "stays" flag after a migration classification)
B2MD_EXPORT int b2md_flag_neither(const int32_t *d_a, const int32_t *d_b, int64_t n,
                                  int32_t *d_out, void *stream) {
    if (n < 0) { set_error("b2md_flag_neither: bad arguments"); return -1; }
    if (n == 0) return 0;
    k_flag_not_either<<<blocks_for(n, kThreads), kThreads, 0, as_stream(stream)>>>(d_a, d_b, n,
                                                                                   d_out);
    B2MD_CHECK_LAUNCH("b2md_flag_neither");
    return 0;
}
