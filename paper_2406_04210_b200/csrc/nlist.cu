// Verlet neighbour lists: reference build_neighbor_list (neighbor.py:185-240),
// kernels _list_cells_chunk (112-152) and _list_brute_chunk (155-182), the
// build-time snapshot (238) and needs_rebuild's reduction (243-254).
//
// The listing decision r2 < rl2 is taken in fp64 with the reference's exact
// operation sequence (no FMA) on positions (double)hi + (double)lo, so the
// neighbour SETS are bit-exact.  A cheap fp32 pre-test on the high words skips
// the fp64 arithmetic for candidates that are far outside or far inside the
// listing sphere; its guard band is wide enough that it can never change a
// decision (bound derived below).
//
// Output layout is column-major and padded: entry k of particle i lives at
// nbr[k * pitch + i], so the force kernel's per-k loads coalesce across a warp.
#include <math.h>
#include <stdlib.h>

#include "common.cuh"

namespace b2md {

constexpr int kBuildThreads = 128;

struct ListGeom {
    BoxD box;
    int nc[3];
    double rl2;
    // fp32 pre-test:  r2f < rl2_in  => certainly listed,  r2f > rl2_out => certainly not.
    float rl2_in, rl2_out;
    float rl2_in_b, rl2_out_b;   // tighter band of the ballot kernel (no fp32 min-image step)
    float Lf[3], invLf[3];
    float margin[3];   // boundary flag: within this distance of a periodic face
    float Lhi[3];
    float mid[3];      // L/2 per axis, and how far from that plane a particle must be for the
    float mid_clear[3];   // force kernel's face frame (bits 3-5 of the flag); < 0 = never
};

// One fp64 candidate test, the reference's arithmetic verbatim
// (neighbor.py:137-144): d = xi - xj; d -= L*rint(d*(1/L)); r2 = (dx*dx+dy*dy)+dz*dz.
__device__ __forceinline__ bool listed_f64(const double pi[3], const float4 hj, const float4 lj,
                                           const ListGeom &g) {
    double dx = __dsub_rn(pi[0], ds_to_double(hj.x, lj.x));
    double dy = __dsub_rn(pi[1], ds_to_double(hj.y, lj.y));
    double dz = __dsub_rn(pi[2], ds_to_double(hj.z, lj.z));
    dx = min_image_f64(dx, g.box.L[0], g.box.invL[0]);
    dy = min_image_f64(dy, g.box.L[1], g.box.invL[1]);
    dz = min_image_f64(dz, g.box.L[2], g.box.invL[2]);
    double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    return r2 < g.rl2;
}

// fp32 estimate of the same squared distance from the high words only.
// Error budget (per component, box edge L, u = 2^-24):
//   |hi - x| <= u*L for both particles, the fp32 subtraction adds <= u*L, the
//   product d*invL and the fma with L_f32 (|L - L_f32| <= u*L) add <= 3*u*L more
//   => |d_f32 - d| <= 8*u*L.  With |d| <= 1.5*r_list per component the squared
//   distance is off by at most 3 * (2*1.5*r_list*8uL + (8uL)^2) plus 3 roundings of
//   the sum (<= 4u * r2).  The host sets the band to 4x that figure.
__device__ __forceinline__ float dist2_f32(const float4 hi_i, const float4 hj, const ListGeom &g) {
    float dx = hi_i.x - hj.x, dy = hi_i.y - hj.y, dz = hi_i.z - hj.z;
    dx = fmaf(-g.Lf[0], rintf(dx * g.invLf[0]), dx);
    dy = fmaf(-g.Lf[1], rintf(dy * g.invLf[1]), dy);
    dz = fmaf(-g.Lf[2], rintf(dz * g.invLf[2]), dz);
    return fmaf(dz, dz, fmaf(dy, dy, dx * dx));
}

// Sort the kept prefix ascending (neighbor.py:152), store the count, and fold the
// row's wanted length into the status block with one atomic per warp.  Must be
// called by every thread of the warp (inactive lanes pass active = false).
__device__ __forceinline__ void finish_row(int32_t *__restrict__ nbr, int64_t pitch, int64_t i,
                                           bool active, int found, int stride, int32_t *counts,
                                           b2md_status *status) {
    if (active) {
        const int kept = found < stride ? found : stride;
        counts[i] = kept;
        for (int a = 1; a < kept; ++a) {  // rows arrive nearly sorted
            int v = nbr[(int64_t)a * pitch + i];
            int b = a - 1;
            while (b >= 0) {
                int w = nbr[(int64_t)b * pitch + i];
                if (w <= v) break;
                nbr[(int64_t)(b + 1) * pitch + i] = w;
                --b;
            }
            if (b + 1 != a) nbr[(int64_t)(b + 1) * pitch + i] = v;
        }
    }
    int mx = active ? found : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) {
        if (mx > stride) atomicExch(&status->overflow, 1);
        atomicMax(&status->max_count, mx);
    }
}

// Bit a is set when the particle is within `margin` of a periodic face on axis a:
// only then can one of its listed pairs need an image shift along that axis
// during the list's lifetime.
// Bit 3 + a is set when the particle stays clear of the mid-plane x_a = L_a / 2 for the list's
// whole lifetime by more than any listed pair can span (margin = r_list + skin, plus the
// particle's own skin / 2 of travel, rounded up to skin): every listed partner is then on
// the same side of that plane or across the periodic face, which is what the force kernel's
// face frame (force.cu, face_frame) needs.  Never set in boxes narrower than 4 x that reach.
__device__ __forceinline__ uint8_t boundary_flag(const float4 h, const ListGeom &g) {
    const float p[3] = {h.x, h.y, h.z};
    int bits = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if ((p[a] < g.margin[a]) | (p[a] > g.Lhi[a] - g.margin[a])) bits |= 1 << a;
        if (g.mid_clear[a] >= 0.0f && fabsf(p[a] - g.mid[a]) > g.mid_clear[a]) bits |= 8 << a;
    }
    return (uint8_t)bits;
}

template <bool PREFILTER>
__global__ void __launch_bounds__(kBuildThreads)
k_list_cells(const float4 *__restrict__ pos_hi, const float4 *__restrict__ pos_lo, int64_t n,
             int64_t n_rows, ListGeom g, const int32_t *__restrict__ cell_of,
             const int32_t *__restrict__ cell_start, const int32_t *__restrict__ cell_particles,
             int stride, int64_t pitch, int32_t *__restrict__ nbr, int32_t *__restrict__ counts,
             uint8_t *__restrict__ boundary, b2md_status *status) {
    const int64_t i_raw = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool active = i_raw < n_rows;
    const int64_t i = active ? i_raw : n_rows - 1;
    const float4 hi_i = pos_hi[i], lo_i = pos_lo[i];
    const double pi[3] = {ds_to_double(hi_i.x, lo_i.x), ds_to_double(hi_i.y, lo_i.y),
                          ds_to_double(hi_i.z, lo_i.z)};
    const int ci = cell_of[i];
    const int cz = ci % g.nc[2];
    const int cy = (ci / g.nc[2]) % g.nc[1];
    const int cx = ci / (g.nc[2] * g.nc[1]);
    int found = 0;
    for (int ox = -1; ox <= 1; ++ox) {
        int jx = cx + ox;
        jx = jx < 0 ? jx + g.nc[0] : (jx >= g.nc[0] ? jx - g.nc[0] : jx);
        for (int oy = -1; oy <= 1; ++oy) {
            int jy = cy + oy;
            jy = jy < 0 ? jy + g.nc[1] : (jy >= g.nc[1] ? jy - g.nc[1] : jy);
            for (int oz = -1; oz <= 1; ++oz) {
                int jz = cz + oz;
                jz = jz < 0 ? jz + g.nc[2] : (jz >= g.nc[2] ? jz - g.nc[2] : jz);
                const int cj = (jx * g.nc[1] + jy) * g.nc[2] + jz;
                const int p_end = active ? cell_start[cj + 1] : 0;
                for (int p = cell_start[cj]; p < p_end; ++p) {
                    const int j = cell_particles[p];
                    if (j == (int)i) continue;
                    const float4 hj = __ldg(&pos_hi[j]);
                    bool hit;
                    if (PREFILTER) {
                        const float r2f = dist2_f32(hi_i, hj, g);
                        if (r2f > g.rl2_out) continue;
                        hit = (r2f < g.rl2_in) || listed_f64(pi, hj, __ldg(&pos_lo[j]), g);
                    } else {
                        hit = listed_f64(pi, hj, __ldg(&pos_lo[j]), g);
                    }
                    if (hit) {
                        if (found < stride) nbr[(int64_t)found * pitch + i] = j;
                        ++found;
                    }
                }
            }
        }
    }
    if (boundary && active) boundary[i] = boundary_flag(hi_i, g);
    finish_row(nbr, pitch, i, active, found, stride, counts, status);
}

// ---------------------------------------------------------------------------
// Production build kernel: one warp per cell, lane = particle of that cell.
//
// The 27 neighbour cells are visited in the reference's order; each neighbour
// cell's occupants are staged 32 at a time in shared memory as fp32 high words
// already shifted by the periodic image of that cell (so the inner loop needs no
// minimum-image arithmetic), then every lane walks the staged candidates by
// shared-memory broadcast.  The fp32 squared distance only pre-sorts candidates
// into certainly-out / certainly-in / in-band; in-band candidates (a shell a few
// 1e-5 sigma thick) take the exact fp64 test of listed_f64, so rows are
// bit-identical to the reference.  Rows are collected in shared memory
// ([k][lane] layout, conflict-free), sorted there, and written to the
// column-major list with all lanes storing the same k together.
constexpr int kCellWarps = 4;

// Neighbour cell `slot` (0..26, reference order: x offset outermost, z innermost)
// of cell (cx,cy,cz): flat index and the periodic image shift to apply to its
// occupants so that plain differences are minimum-image differences.
__device__ __forceinline__ void neighbour_cell(const ListGeom &g, int cx, int cy, int cz, int slot,
                                               int &cj, float &sx, float &sy, float &sz) {
    int jx = cx + slot / 9 - 1, jy = cy + (slot / 3) % 3 - 1, jz = cz + slot % 3 - 1;
    sx = sy = sz = 0.f;
    if (jx < 0) { jx += g.nc[0]; sx = -g.Lf[0]; } else if (jx >= g.nc[0]) { jx -= g.nc[0]; sx = g.Lf[0]; }
    if (jy < 0) { jy += g.nc[1]; sy = -g.Lf[1]; } else if (jy >= g.nc[1]) { jy -= g.nc[1]; sy = g.Lf[1]; }
    if (jz < 0) { jz += g.nc[2]; sz = -g.Lf[2]; } else if (jz >= g.nc[2]) { jz -= g.nc[2]; sz = g.Lf[2]; }
    cj = (jx * g.nc[1] + jy) * g.nc[2] + jz;
}

// Warp-wide bitonic sort of (key, value) held one pair per lane, ascending key.
__device__ __forceinline__ void warp_sort_pairs(int &key, int &val, int lane) {
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const int okey = __shfl_xor_sync(0xffffffffu, key, stride);
            const int oval = __shfl_xor_sync(0xffffffffu, val, stride);
            const bool up = ((lane & size) == 0);
            const bool lower = ((lane & stride) == 0);
            const bool take = (lower == up) ? (okey < key || (okey == key && oval < val))
                                            : (okey > key || (okey == key && oval > val));
            if (take) { key = okey; val = oval; }
        }
    }
}

// Exact listing decision for particle pair (i, j), kept out of line so that the
// hot loops do not carry its registers.  The geometry travels BY VALUE: the callers hold it
// as a __grid_constant__ kernel parameter, and a reference would make this function read
// parameter memory through a generic pointer (legal, but compute-sanitizer cannot follow it
// into the parameter buffers of graph kernel nodes).
struct ExactGeom { BoxD box; double rl2; };

__device__ __noinline__ bool listed_exact_v(const float4 *__restrict__ pos_hi,
                                            const float4 *__restrict__ pos_lo, int i, int j,
                                            const ExactGeom e) {
    const float4 hi_i = pos_hi[i], lo_i = pos_lo[i];
    const float4 hj = pos_hi[j], lj = pos_lo[j];
    double dx = __dsub_rn(ds_to_double(hi_i.x, lo_i.x), ds_to_double(hj.x, lj.x));
    double dy = __dsub_rn(ds_to_double(hi_i.y, lo_i.y), ds_to_double(hj.y, lj.y));
    double dz = __dsub_rn(ds_to_double(hi_i.z, lo_i.z), ds_to_double(hj.z, lj.z));
    dx = min_image_f64(dx, e.box.L[0], e.box.invL[0]);
    dy = min_image_f64(dy, e.box.L[1], e.box.invL[1]);
    dz = min_image_f64(dz, e.box.L[2], e.box.invL[2]);
    const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    return r2 < e.rl2;
}

__device__ __forceinline__ bool listed_exact(const float4 *__restrict__ pos_hi,
                                             const float4 *__restrict__ pos_lo, int i, int j,
                                             const ListGeom &g) {
    ExactGeom e;
    e.box = g.box;
    e.rl2 = g.rl2;
    return listed_exact_v(pos_hi, pos_lo, i, j, e);
}

constexpr int kBandTag = (int)0x80000000;
constexpr int kCandCap = 160;      // candidates staged per batch and warp

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
k_list_cells_warp(const float4 *__restrict__ pos_hi, const float4 *__restrict__ pos_lo, int64_t n,
                  int64_t n_rows, const __grid_constant__ ListGeom g, int64_t n_cells,
                  const int32_t *__restrict__ cell_start,
                  const int32_t *__restrict__ cell_particles, int stride, int64_t pitch,
                  int32_t *__restrict__ nbr, int32_t *__restrict__ counts,
                  uint8_t *__restrict__ boundary, b2md_status *status) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float4 *s_cand = reinterpret_cast<float4 *>(smem_raw) + warp * kCandCap;
    // rows: [k][lane], k = 0 .. stride+1 (two spare slots: "one too many" + scratch)
    int32_t *s_rows = reinterpret_cast<int32_t *>(smem_raw + WARPS * kCandCap * sizeof(float4)) +
                      (size_t)warp * (stride + 2) * 32 + lane;
    const int64_t c = (int64_t)blockIdx.x * WARPS + warp;
    int wanted_max = 0;
    if (c < n_cells) {
        const int cz = (int)(c % g.nc[2]);
        const int cy = (int)((c / g.nc[2]) % g.nc[1]);
        const int cx = (int)(c / ((int64_t)g.nc[2] * g.nc[1]));
        const int i_begin = cell_start[c], i_end = cell_start[c + 1];
        const float rl2_in = g.rl2_in, rl2_out = g.rl2_out;
        if (i_begin == i_end) return;          // empty cell (whole warp leaves together)

        // Visiting order of the 27 neighbour cells.  Rows must come out ascending
        // (neighbor.py:152); cells are visited by ascending first-occupant index,
        // so for cell-contiguous particle orders the rows are born sorted and the
        // final insertion sort is a single checking pass.  Lane s holds slot s.
        int my_slot = lane, my_key = 0x7fffffff;
        if (lane < 27) {
            int cj; float sx, sy, sz;
            neighbour_cell(g, cx, cy, cz, lane, cj, sx, sy, sz);
            const int b = cell_start[cj];
            if (b < cell_start[cj + 1]) my_key = cell_particles[b];
        }
        int sorted_key = my_key, sorted_slot = my_slot;
        warp_sort_pairs(sorted_key, sorted_slot, lane);

        for (int i0 = i_begin; i0 < i_end; i0 += 32) {
            // rows exist for particles [0, n_rows) only (ghost rows are skipped)
            const int i_raw = (i0 + lane < i_end) ? cell_particles[i0 + lane] : -1;
            const bool active = i_raw >= 0 && i_raw < n_rows;
            const int i = active ? i_raw : -1;
            // inactive lanes sit at +1e30: every distance test fails
            const float4 hi_i = active ? pos_hi[i] : make_float4(1e30f, 1e30f, 1e30f, 0.f);

            // ---- pass 0 (fast): sorted visiting order, branch-free compaction.
            // Candidates are staged kCandCap at a time (several neighbour cells per
            // batch) so that the scan is one long tight loop.  Every candidate is
            // stored at the row's next free slot and the slot advances only when
            // the fp32 distance is inside the outer radius (a later candidate
            // overwrites a miss).  Entries inside the guard band carry a tag bit
            // and are settled exactly afterwards.
            int slot = 0;                               // word offset into this lane's column
            const int slot_cap = (stride + 1) * 32;
            {
                int t = 0, p = 0, p_end = 0;
                float sx = 0.f, sy = 0.f, sz = 0.f;
                bool have = false;                      // (p, p_end) describe an open cell
                for (;;) {
                    int ncand = 0;
                    __syncwarp();
                    while (ncand < kCandCap) {
                        if (!have) {
                            if (t == 27) break;
                            const int nslot = __shfl_sync(0xffffffffu, sorted_slot, t);
                            int cj;
                            neighbour_cell(g, cx, cy, cz, nslot, cj, sx, sy, sz);
                            p = cell_start[cj];
                            p_end = cell_start[cj + 1];
                            have = true;
                            ++t;
                        }
                        const int take = min(p_end - p, kCandCap - ncand);
                        for (int o = lane; o < take; o += 32) {
                            const int j = cell_particles[p + o];
                            const float4 hj = __ldg(&pos_hi[j]);
                            s_cand[ncand + o] = make_float4(hj.x + sx, hj.y + sy, hj.z + sz,
                                                            __int_as_float(j));
                        }
                        ncand += take;
                        p += take;
                        if (p == p_end) have = false;
                    }
                    if (ncand == 0) break;
                    __syncwarp();
#pragma unroll 8
                    for (int q = 0; q < ncand; ++q) {
                        const float4 cnd = s_cand[q];
                        const float dx = hi_i.x - cnd.x, dy = hi_i.y - cnd.y, dz = hi_i.z - cnd.z;
                        const float r2f = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                        const int j = __float_as_int(cnd.w);
                        const bool take = (r2f <= rl2_out) && (j != i);
                        s_rows[slot] = (r2f >= rl2_in) ? (j | kBandTag) : j;
                        slot = min(slot + (take ? 32 : 0), slot_cap);
                    }
                    if (t == 27 && !have) break;
                }
            }
            int found = slot >> 5;
            // settle guard-band entries exactly (rare), compact, and keep the row
            // ascending (neighbor.py:152; rows are born nearly sorted)
            {
                int w = 0;
                for (int k = 0; k < found; ++k) {
                    int v = s_rows[k * 32];
                    bool keep = true;
                    if (v < 0) {
                        v &= ~kBandTag;
                        keep = listed_exact(pos_hi, pos_lo, i, v, g);
                    }
                    if (keep) {
                        int b = w - 1;
                        while (b >= 0 && s_rows[b * 32] > v) {
                            s_rows[(b + 1) * 32] = s_rows[b * 32];
                            --b;
                        }
                        s_rows[(b + 1) * 32] = v;
                        ++w;
                    }
                }
                // a row that filled all stride+1 slots may have lost entries: redo exactly
                if (found <= stride) found = w;
            }
            // ---- pass 1 (only if some row may exceed the budget): reference scan
            // order with exact in-loop decisions, so that the kept prefix is the
            // reference's (first `stride` hits in its order, neighbor.py:145-149).
            const bool redo = __any_sync(0xffffffffu, found > stride);
            if (redo) {
                found = 0;
                for (int t = 0; t < 27; ++t) {
                    int cj; float sx, sy, sz;
                    neighbour_cell(g, cx, cy, cz, t, cj, sx, sy, sz);
                    const int p_begin = cell_start[cj], p_end = cell_start[cj + 1];
                    for (int p0 = p_begin; p0 < p_end; p0 += 32) {
                        const int m = min(32, p_end - p0);
                        __syncwarp();
                        if (lane < m) {
                            const int j = cell_particles[p0 + lane];
                            const float4 hj = __ldg(&pos_hi[j]);
                            s_cand[lane] = make_float4(hj.x + sx, hj.y + sy, hj.z + sz,
                                                       __int_as_float(j));
                        }
                        __syncwarp();
                        for (int q = 0; q < m; ++q) {
                            const float4 cnd = s_cand[q];
                            const float dx = hi_i.x - cnd.x, dy = hi_i.y - cnd.y,
                                        dz = hi_i.z - cnd.z;
                            const float r2f = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                            const int j = __float_as_int(cnd.w);
                            if (r2f <= rl2_out && j != i) {
                                bool hit = r2f < rl2_in;
                                if (!hit) hit = listed_exact(pos_hi, pos_lo, i, j, g);
                                if (hit) {
                                    if (found < stride) s_rows[found * 32] = j;
                                    ++found;
                                }
                            }
                        }
                    }
                }
            }
            // ---- publish (pass-1 rows still need their ascending order)
            const int kept = min(found, stride);
            if (redo) {
                for (int a = 1; a < kept; ++a) {
                    const int v = s_rows[a * 32];
                    int b = a - 1;
                    while (b >= 0 && s_rows[b * 32] > v) {
                        s_rows[(b + 1) * 32] = s_rows[b * 32];
                        --b;
                    }
                    if (b + 1 != a) s_rows[(b + 1) * 32] = v;
                }
            }
            const int kmax = __reduce_max_sync(0xffffffffu, kept);
            for (int k = 0; k < kmax; ++k)
                if (k < kept) nbr[(int64_t)k * pitch + i] = s_rows[k * 32];
            if (active) {
                counts[i] = kept;
                if (boundary) boundary[i] = boundary_flag(hi_i, g);
            }
            wanted_max = max(wanted_max, __reduce_max_sync(0xffffffffu, found));
        }
    }
    if (lane == 0 && wanted_max > 0) {
        if (wanted_max > stride) atomicExch(&status->overflow, 1);
        atomicMax(&status->max_count, wanted_max);
    }
}

// ---------------------------------------------------------------------------
// Production build kernel, second generation: one warp per cell, LANE = CANDIDATE.
//
// k_list_cells_warp keeps one particle of the cell per lane (19 of 32 lanes busy
// at rho = 0.75) and walks all 513 candidates per lane; its per-lane compaction
// and the settle / sort pass behind it made it issue-bound at ~30 instructions per
// candidate.  Here the roles are swapped: the candidates of the 27 neighbour cells
// form one stream in ascending visiting order, every lane holds one candidate of a
// 32-wide chunk (all lanes busy), and the cell's particles are walked one after the
// other by shared-memory broadcast.  The listing decision of a chunk is a ballot,
// the slot of an accepted candidate is the population count of the lower lanes, so
// rows are compacted in stream order without any per-lane state: they are born
// ascending whenever the particle order is cell-contiguous (always, after the
// Hilbert / cell reorder) -- checked while staging, else a sort pass runs.
// The fp32 distance pre-sorts as before; the rare candidate inside the guard band
// is settled on the spot with the reference's exact fp64 sequence (warp-uniform
// branch), so rows are final -- and bit-identical to the reference -- as written.
// Rows wanting more than `stride` entries send the cell through the reference-order
// rescan of k_list_cells_warp (the kept prefix must be the reference's).
constexpr int kStreamCap = 640;    // candidate indices staged per batch and warp

constexpr int kPassRows = 24;      // particles of the cell handled per pass
constexpr int kMaskPitch = kStreamCap / 32 + 1;   // ballot words per row and batch (odd)

__host__ __device__ inline size_t ballot_warp_bytes() {
    return (kPassRows / 2) * 2 * sizeof(float4) + kPassRows * kMaskPitch * sizeof(uint32_t) +
           kStreamCap * sizeof(int32_t);
}

// Ascending order of one row of the column-major list, in place (neighbor.py:152);
// insertion sort: the callers' rows are nearly sorted.
__device__ __forceinline__ void sort_row_strided(int32_t *__restrict__ row, int64_t step, int kept) {
    for (int a = 1; a < kept; ++a) {
        const int v = row[(int64_t)a * step];
        int b = a - 1;
        while (b >= 0) {
            const int w = row[(int64_t)b * step];
            if (w <= v) break;
            row[(int64_t)(b + 1) * step] = w;
            --b;
        }
        if (b + 1 != a) row[(int64_t)(b + 1) * step] = v;
    }
}
__device__ __forceinline__ void sort_row_in_list(int32_t *__restrict__ nbr, int64_t pitch, int i,
                                                 int kept) {
    sort_row_strided(nbr + i, pitch, kept);
}

// One particle's row straight into the column-major list in the reference's scan
// order (27 cells, x offset outermost; neighbor.py:126-149) with exact decisions,
// then sorted ascending in place.  Slow path of the ballot kernel for rows that
// overflow `stride` (the kept prefix must be the reference's).  Returns the unclamped
// count.
__device__ __noinline__ int scan_row_reference_order(
    const float4 *__restrict__ pos_hi, const float4 *__restrict__ pos_lo, const ListGeom &g,
    int cx, int cy, int cz, const int32_t *__restrict__ cell_start,
    const int32_t *__restrict__ cell_particles, int i, const float4 hi_i, int stride,
    int64_t pitch, int32_t *__restrict__ nbr) {
    int found = 0;
    for (int t = 0; t < 27; ++t) {
        int cj; float sx, sy, sz;
        neighbour_cell(g, cx, cy, cz, t, cj, sx, sy, sz);
        const int p_end = cell_start[cj + 1];
        for (int p = cell_start[cj]; p < p_end; ++p) {
            const int j = cell_particles[p];
            if (j == i) continue;
            const float4 hj = __ldg(&pos_hi[j]);
            const float dx = hi_i.x - (hj.x + sx), dy = hi_i.y - (hj.y + sy),
                        dz = hi_i.z - (hj.z + sz);
            const float r2f = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
            if (r2f > g.rl2_out) continue;
            if (r2f < g.rl2_in || listed_exact(pos_hi, pos_lo, i, j, g)) {
                if (found < stride) nbr[(int64_t)found * pitch + i] = j;
                ++found;
            }
        }
    }
    sort_row_in_list(nbr, pitch, i, min(found, stride));
    return found;
}

// fp32x2 helpers (FADD2 / FMUL2 / FFMA2): two particles of the cell per instruction
__device__ __forceinline__ unsigned long long nl_pk(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ unsigned long long nl_sub2(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long nl_mul2(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long nl_fma2(unsigned long long a, unsigned long long b,
                                                      unsigned long long c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
#ifndef B2MD_LIST_MIN_BLOCKS
#define B2MD_LIST_MIN_BLOCKS 4
#endif

// Position of combined rank R in the bit stream (ma[x] | mb[x]), x = 0 .. n_chunks-1: word w and
// that word with its lower-ranked bits cleared.  (R beyond the stream: word 0, harmless.)
__device__ __forceinline__ void seek_rank(const uint32_t *ma, const uint32_t *mb, int n_chunks,
                                          int R, int &w, uint32_t &um) {
    int cum = 0, w0 = 0, r0 = 0;
    for (int x = 0; x < n_chunks; ++x) {
        const int c = __popc(ma[x] | mb[x]);
        const bool here = R >= cum && R < cum + c;
        w0 = here ? x : w0;
        r0 = here ? R - cum : r0;
        cum += c;
    }
    w = w0;
    um = ma[w0] | mb[w0];
    for (int k = 0; k < r0; ++k) um &= um - 1u;
}

// PAIRS (b2md_build_pair_list): the kernel emits the force kernel's PAIR ROWS (see k_pair_rows
// below for the layout) straight from the ballot masks instead of the plain rows.  Rows 2t and
// 2t+1 that sit next to each other in a pass share one candidate stream, so their merged row is
// the set bits of (mask of 2t | mask of 2t+1) in stream order, each entry flagged with the two
// mask bits -- no merge, and the 4 c B per particle of plain rows are never written or read back.
// The pairs of a pass share the warp: each gets 32 / pairs lanes, and the lanes of a pair split
// its merged row by RANK into runs of whole int4 tiles (a lane seeks to its first entry through
// the population counts of the mask words), so they are balanced and tile-aligned by
// construction.  Rows whose partner lives in another cell or pass ("single" rows) are dealt to
// the lanes the same way and stored as plain rows -- ROW-major in this mode (row i at nbr +
// i * list_rows: 6 % of the rows, scattered over the whole list, would otherwise be one DRAM
// sector per entry for the merge that follows); k_pair_fixup merges those afterwards and pads
// every pair row to the longest row of its force-kernel warp.
struct PairOut {
    int4 *pair_nbr;
    int32_t *pair_counts;
    int64_t pair_pitch;
    int pair_tiles;
    int list_rows;      // PAIRS: single rows are stored ROW-major, row i at nbr + i * list_rows
};

template <int WARPS, bool PAIRS>
__global__ void __launch_bounds__(WARPS * 32, B2MD_LIST_MIN_BLOCKS)
k_list_cells_ballot(const float4 *__restrict__ pos_hi, const float4 *__restrict__ pos_lo,
                    int64_t n, int64_t n_rows, const __grid_constant__ ListGeom g,
                    int64_t n_cells, const int32_t *__restrict__ cell_start,
                    const int32_t *__restrict__ cell_particles, int stride, int64_t pitch,
                    int32_t *__restrict__ nbr, int32_t *__restrict__ counts,
                    uint8_t *__restrict__ boundary, b2md_status *status, int exact_prefix,
                    const __grid_constant__ PairOut po) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char *base = smem_raw + warp * ballot_warp_bytes();
    // particles of the pass, two per slot: A = (x0, x1, y0, y1), B = (z0, z1, i0, i1)
    float4 *s_pa = reinterpret_cast<float4 *>(base);
    float4 *s_pb = s_pa + kPassRows / 2;
    uint32_t *s_mask = reinterpret_cast<uint32_t *>(s_pb + kPassRows / 2);   // [row][chunk]
    int32_t *s_stream = reinterpret_cast<int32_t *>(s_mask + kPassRows * kMaskPitch);
    const int64_t c = (int64_t)blockIdx.x * WARPS + warp;
    if (c >= n_cells) return;
    const int cz = (int)(c % g.nc[2]);
    const int cy = (int)((c / g.nc[2]) % g.nc[1]);
    const int cx = (int)(c / ((int64_t)g.nc[2] * g.nc[1]));
    const int i_begin = cell_start[c], i_end = cell_start[c + 1];
    if (i_begin == i_end) return;
    const float rl2_in = g.rl2_in_b, rl2_out = g.rl2_out_b;
    // |r2 - band_mid| <= band_half is implied by rl2_in <= r2 <= rl2_out (the half width is
    // rounded up generously; a false alarm only costs the exact settle loop)
    const float band_mid = 0.5f * (rl2_in + rl2_out);
    const float band_half = 0.5f * (rl2_out - rl2_in) * 1.001f + 4.0e-7f * rl2_out;
    const unsigned long long mid2 = nl_pk(band_mid, band_mid);

    // visiting order: neighbour cells by ascending first-occupant index (lane s = slot s)
    int my_key = 0x7fffffff, my_begin = 0, my_size = 0, my_wrap = 0;
    if (lane < 27) {
        int cj; float sx, sy, sz;
        neighbour_cell(g, cx, cy, cz, lane, cj, sx, sy, sz);
        my_begin = cell_start[cj];
        my_size = cell_start[cj + 1] - my_begin;
        if (my_size > 0) my_key = cell_particles[my_begin];
        // periodic image of the whole neighbour cell: 2 bits per axis (0: -L, 1: 0, 2: +L)
        my_wrap = ((sx < 0.f) ? 0 : (sx > 0.f) ? 2 : 1) | (((sy < 0.f) ? 0 : (sy > 0.f) ? 2 : 1) << 2) |
                  (((sz < 0.f) ? 0 : (sz > 0.f) ? 2 : 1) << 4);
    }
    int sorted_key = my_key, sorted_slot = lane;
    warp_sort_pairs(sorted_key, sorted_slot, lane);
    // lane t now describes the t-th cell to visit; v_end = candidates up to and including it
    const int v_begin = __shfl_sync(0xffffffffu, my_begin, sorted_slot);
    const int v_size = __shfl_sync(0xffffffffu, my_size, sorted_slot);
    const int v_wrap = __shfl_sync(0xffffffffu, my_wrap, sorted_slot);
    int v_end = v_size;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int up = __shfl_up_sync(0xffffffffu, v_end, o);
        if (lane >= o) v_end += up;
    }
    const int n_cand = __shfl_sync(0xffffffffu, v_end, 31);
    // where the cell's own occupants sit in the stream (slot 13 = offset (0,0,0)): row
    // particle number k of the cell is stream position own_start + k -- its self test is
    // not excluded pair by pair in phase 1, its bit is cleared afterwards
    const int own_t = __ffs(__ballot_sync(0xffffffffu, sorted_slot == 13)) - 1;
    const int own_start = __shfl_sync(0xffffffffu, v_end - v_size, own_t);
    // Is the candidate stream ascending?  (Every visited cell a contiguous index range,
    // ranges in ascending order: true after every Hilbert / cell reorder.)  Rows are
    // then born sorted; otherwise they are sorted after the fact.
    bool ascending;
    {
        const int first = sorted_key;                 // first occupant of visited cell `lane`
        const int last = v_size > 0 ? cell_particles[v_begin + v_size - 1] : first;
        const int prev_last = __shfl_up_sync(0xffffffffu, last, 1);
        const bool ok = v_size == 0 ||
                        (last - first == v_size - 1 && (lane == 0 || prev_last < first));
        ascending = __all_sync(0xffffffffu, ok);
    }

    int wanted_max = 0;
    for (int i0 = i_begin; i0 < i_end; i0 += kPassRows) {
        const int ni = min(kPassRows, i_end - i0);
        const int i_raw = (lane < ni) ? cell_particles[i0 + lane] : -1;
        const bool active = i_raw >= 0 && i_raw < n_rows;    // ghost rows get no list
        const int i = active ? i_raw : -1;
        const float4 hi_i = active ? pos_hi[i] : make_float4(1e30f, 1e30f, 1e30f, 0.f);
        int found = 0;
        // PAIRS: lanes per pair / per single row of the pass (see the kernel comment)
        int a_L = 32, a_sub = 0, a_row = 0, a_i = 0, a_done = 0;
        int b_L = 32, b_sub = 0, b_row = 0, b_i = 0, b_done = 0;
        bool a_has = false, b_has = false;
        int e1 = 0, e2 = 0, e3 = 0;
        if (PAIRS) {
            const int i_next = __shfl_down_sync(0xffffffffu, i_raw, 1);
            const int i_prev = __shfl_up_sync(0xffffffffu, i_raw, 1);
            const bool lo_ok = ascending && active && !(i & 1) && lane + 1 < ni &&
                               i_next == i + 1 && i + 1 < n_rows;
            const bool hi_ok = ascending && active && (i & 1) && lane >= 1 && i_prev == i - 1;
            const unsigned lo_mask = __ballot_sync(0xffffffffu, lo_ok);
            const unsigned sg_mask = __ballot_sync(0xffffffffu, active && !lo_ok && !hi_ok);
            const int n_a = __popc(lo_mask), n_b = __popc(sg_mask);
            a_L = n_a ? 32 / n_a : 32;
            b_L = n_b ? 32 / n_b : 32;
            const int ua = lane / a_L, ub = lane / b_L;
            a_sub = lane - ua * a_L;
            b_sub = lane - ub * b_L;
            a_has = ua < n_a;
            b_has = ub < n_b;
            a_row = a_has ? (int)__fns(lo_mask, 0, ua + 1) : 0;
            b_row = b_has ? (int)__fns(sg_mask, 0, ub + 1) : 0;
            a_i = __shfl_sync(0xffffffffu, i_raw, a_row);
            b_i = __shfl_sync(0xffffffffu, i_raw, b_row);
        }
        {
            __syncwarp();
            if (lane < kPassRows) {
                float *fa = reinterpret_cast<float *>(s_pa + (lane >> 1));
                float *fb = reinterpret_cast<float *>(s_pb + (lane >> 1));
                const int h = lane & 1;
                fa[h] = hi_i.x;
                fa[2 + h] = hi_i.y;
                fb[h] = hi_i.z;
                fb[2 + h] = __int_as_float(i);
            }
            int32_t *out = nbr + (active ? i : 0);       // entry k of this row: out[k * pitch]
            for (int batch0 = 0; batch0 < n_cand; batch0 += kStreamCap) {
                const int total = min(kStreamCap, n_cand - batch0);
                const int n_chunks = (total + 31) >> 5;
                __syncwarp();
                // stage candidate indices (+ wrap code) of stream positions [batch0, +total)
                for (int m0 = 0; m0 < total; m0 += 32) {         // warp-uniform trip count
                    const int m = m0 + lane;
                    const int pos = batch0 + min(m, total - 1);
                    // visited cell holding stream position `pos`: first t with v_end[t] > pos
                    int t = 0;
#pragma unroll
                    for (int bit = 16; bit > 0; bit >>= 1) {
                        const int probe = __shfl_sync(0xffffffffu, v_end, min(t + bit - 1, 31));
                        if (probe <= pos) t += bit;
                    }
                    const int ce = __shfl_sync(0xffffffffu, v_end, t);
                    const int cs = __shfl_sync(0xffffffffu, v_size, t);
                    const int cb = __shfl_sync(0xffffffffu, v_begin, t);
                    const int cw = __shfl_sync(0xffffffffu, v_wrap, t);
                    if (m < total)
                        s_stream[m] = cell_particles[cb + (pos - (ce - cs))] | (cw << 26);
                }
                __syncwarp();
                // ---- phase 1: all particles of the pass against 32 candidates per chunk;
                // the decisions of row r on chunk w are one ballot, parked in s_mask[r][w]
                for (int w = 0; w < n_chunks; ++w) {
                    float qx = -1e30f, qy = -1e30f, qz = -1e30f;
                    int j = -2;
                    if (w * 32 + lane < total) {
                        const int code = s_stream[w * 32 + lane];
                        j = code & 0x03ffffff;
                        const float4 hj = __ldg(&pos_hi[j]);
                        qx = hj.x + (float)(((code >> 26) & 3) - 1) * g.Lf[0];
                        qy = hj.y + (float)(((code >> 28) & 3) - 1) * g.Lf[1];
                        qz = hj.z + (float)(((code >> 30) & 3) - 1) * g.Lf[2];
                    }
                    const unsigned long long qx2 = nl_pk(qx, qx), qy2 = nl_pk(qy, qy),
                                             qz2 = nl_pk(qz, qz);
                    // distance of r2 from the middle of the guard band, minimum over the
                    // rows: one packed subtract and two |.|-minimum per row pair
                    float band_min = 3.0e38f;
                    uint32_t *mask_w = s_mask + w;
#pragma unroll 2
                    for (int p = 0; p < (ni + 1) >> 1; ++p) {
                        const float4 A = s_pa[p], B = s_pb[p];               // broadcasts
                        const unsigned long long dx = nl_sub2(nl_pk(A.x, A.y), qx2);
                        const unsigned long long dy = nl_sub2(nl_pk(A.z, A.w), qy2);
                        const unsigned long long dz = nl_sub2(nl_pk(B.x, B.y), qz2);
                        const unsigned long long r2 =
                            nl_fma2(dz, dz, nl_fma2(dy, dy, nl_mul2(dx, dx)));
                        float r2a, r2b, ea, eb;
                        asm("mov.b64 {%0, %1}, %2;" : "=f"(r2a), "=f"(r2b) : "l"(r2));
                        asm("mov.b64 {%0, %1}, %2;" : "=f"(ea), "=f"(eb) : "l"(nl_sub2(r2, mid2)));
                        band_min = fminf(band_min, fminf(fabsf(ea), fabsf(eb)));
                        const unsigned ha = __ballot_sync(0xffffffffu, r2a <= rl2_out);
                        const unsigned hb = __ballot_sync(0xffffffffu, r2b <= rl2_out);
                        if (lane == 0) {
                            mask_w[(2 * p) * kMaskPitch] = ha;
                            mask_w[(2 * p + 1) * kMaskPitch] = hb;
                        }
                    }
                    const bool in_band = band_min <= band_half;
                    if (__any_sync(0xffffffffu, in_band)) {
                        // guard band (a shell ~1e-5 sigma thick): settle with the reference's
                        // exact fp64 sequence and clear the bits that fail
                        __syncwarp();
                        for (int r = 0; r < ni; ++r) {
                            const float *fa = reinterpret_cast<const float *>(s_pa + (r >> 1));
                            const float *fb = reinterpret_cast<const float *>(s_pb + (r >> 1));
                            const float dx = fa[r & 1] - qx, dy = fa[2 + (r & 1)] - qy,
                                        dz = fb[r & 1] - qz;
                            const float r2f = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
                            const int ir = __float_as_int(fb[2 + (r & 1)]);
                            if ((r2f <= rl2_out) && (j != ir) && (r2f >= rl2_in) &&
                                !listed_exact(pos_hi, pos_lo, ir, j, g))
                                atomicAnd(&mask_w[r * kMaskPitch], ~(1u << lane));
                        }
                    }
                }
                __syncwarp();
                {   // the row's own particle passed every test of phase 1 (r2 = 0): drop it
                    const int self = own_start + (i0 - i_begin) + lane - batch0;
                    if (lane < ni && self >= 0 && self < total)
                        s_mask[lane * kMaskPitch + (self >> 5)] &= ~(1u << (self & 31));
                }
                if (PAIRS) {
                    __syncwarp();      // the masks are read by other lanes than the row's own

                    // rows of this batch counted from their masks (counts[], overflow)
                    if (active) {
                        const uint32_t *mr = s_mask + lane * kMaskPitch;
                        for (int w = 0; w < n_chunks; ++w) found += __popc(mr[w]);
                    }
                    // ---- pairs: merged row = set bits of (mask A | mask B) in stream order
                    {
                        const uint32_t *ma = s_mask + a_row * kMaskPitch;
                        const uint32_t *mb = ma + kMaskPitch;
                        int T = 0;
                        if (a_has)
                            for (int w = 0; w < n_chunks; ++w) T += __popc(ma[w] | mb[w]);
                        // entries carried in sub-lane 0's registers from the previous batch
                        // (unfinished tile): that lane then takes the whole batch
                        const int carry = a_done & 3;
                        const int full = T >> 2;
                        int t0 = full * a_sub / a_L, t1 = full * (a_sub + 1) / a_L;
                        int left = 4 * (t1 - t0) + (a_sub == a_L - 1 ? (T & 3) : 0);
                        if (carry) { t0 = 0; left = a_sub == 0 ? T : 0; }
                        if (!a_has) left = 0;
                        int tile = (a_done >> 2) + t0;
                        int w = 0;
                        uint32_t um = 0u;
                        seek_rank(ma, mb, n_chunks, 4 * t0, w, um);
                        uint32_t aw = ma[w], bw = mb[w];
                        const int32_t *ps = s_stream + w * 32;
                        int4 *pt = po.pair_nbr + (a_i >> 1) + (int64_t)tile * po.pair_pitch;
                        int e0 = 0;
#define B2MD_NEXT_ENTRY()                                                                         \
    {                                                                                             \
        while (um == 0u && left > 0) {       /* (1 % of the words are empty) */                   \
            ++w;                                                                                  \
            aw = ma[w];                                                                           \
            bw = mb[w];                                                                           \
            um = aw | bw;                                                                         \
            ps += 32;                                                                             \
        }                                                                                         \
        const bool has = left > 0 && um != 0u;                                                    \
        const int bit = (__ffs(um) - 1) & 31;                                                     \
        um &= um - 1u;                                                                            \
        const int j = ps[bit] & 0x03ffffff;                                                       \
        const int e = (j << 2) | (int)((aw >> bit) & 1u) | (int)(((bw >> bit) & 1u) << 1);        \
        if (has) { e0 = e1; e1 = e2; e2 = e3; e3 = e; }                                           \
        left -= has ? 1 : 0;                                                                      \
    }
                        if (carry && a_sub == 0 && a_has) {
                            // finish the carried tile first (rare: cells with several batches)
                            int fill = carry;
                            while (fill < 4 && left > 0) {
                                const int before = left;
                                B2MD_NEXT_ENTRY();
                                fill += before - left;
                            }
                            if (fill == 4) {
                                if (tile < po.pair_tiles) *pt = make_int4(e0, e1, e2, e3);
                                pt += po.pair_pitch;
                                ++tile;
                            }
                        }
                        // Branch-free tile loop: four entries, one 16-byte store.  (The lanes of
                        // a warp are at different words and tiles; every divergent branch would
                        // be executed once per path.)
                        while (__any_sync(0xffffffffu, left > 0)) {
                            const bool whole = left >= 4;
#pragma unroll
                            for (int rep = 0; rep < 4; ++rep) B2MD_NEXT_ENTRY();
                            if (whole && tile < po.pair_tiles) *pt = make_int4(e0, e1, e2, e3);
                            pt += po.pair_pitch;
                            ++tile;
                        }
#undef B2MD_NEXT_ENTRY
                        // the unfinished tile sits in the last lane of the pair (or in sub-lane
                        // 0 when that one took the whole batch): hand it to sub-lane 0, which
                        // continues it in the next batch or flushes it
                        const int src = carry ? lane : lane - a_sub + a_L - 1;
                        const int t1e = __shfl_sync(0xffffffffu, e1, src & 31);
                        const int t2e = __shfl_sync(0xffffffffu, e2, src & 31);
                        const int t3e = __shfl_sync(0xffffffffu, e3, src & 31);
                        if (a_sub == 0) { e1 = t1e; e2 = t2e; e3 = t3e; }
                        a_done += T;
                    }
                    // ---- single rows: plain-row entries at their rank
                    if (__any_sync(0xffffffffu, b_has)) {
                        const uint32_t *mr = s_mask + b_row * kMaskPitch;
                        int T = 0;
                        if (b_has)
                            for (int w = 0; w < n_chunks; ++w) T += __popc(mr[w]);
                        const int k0 = T * b_sub / b_L, k1 = T * (b_sub + 1) / b_L;
                        int left = b_has ? k1 - k0 : 0;
                        unsigned rank = (unsigned)(b_done + k0);
                        int w = 0;
                        uint32_t um = 0u;
                        seek_rank(mr, mr, n_chunks, k0, w, um);
                        const int32_t *ps = s_stream + w * 32;
                        int32_t *pr = nbr + (int64_t)b_i * po.list_rows + rank;
                        while (__any_sync(0xffffffffu, left > 0)) {
#pragma unroll
                            for (int rep = 0; rep < 2; ++rep) {
                                if (um == 0u && left > 0) {
                                    ++w;
                                    um = mr[w];
                                    ps += 32;
                                }
                                const bool has = left > 0 && um != 0u;
                                const int bit = (__ffs(um) - 1) & 31;
                                um &= um - 1u;
                                const int j = ps[bit] & 0x03ffffff;
                                if (has && rank < (unsigned)stride) *pr = j;
                                pr += has ? 1 : 0;
                                rank += has ? 1u : 0u;
                                left -= has ? 1 : 0;
                            }
                        }
                        b_done += T;
                    }
                } else
                // ---- phase 2: lane r walks the set bits of row r in stream order
                // (= ascending j) and stores entry k of its row; all rows are at the
                // same k, so the column-major stores coalesce across the cell's particles
                {
                    const uint32_t *my_mask = s_mask + lane * kMaskPitch;
                    const int my_chunks = active ? n_chunks : 0;
                    const int32_t *my_stream = s_stream;         // advanced with the mask word
                    int left = my_chunks - 1;                    // mask words not yet fetched
                    unsigned m = active ? my_mask[0] : 0u;
                    // row index space: entry k of this row lives at nbr[k * pitch + i]
                    const unsigned row_i = (unsigned)(active ? i : 0);
                    const unsigned upitch = (unsigned)pitch;
                    const bool small = (uint64_t)pitch * (uint64_t)(stride + 1) < 0xffffffffull;
                    for (;;) {
                        if (m == 0u && left > 0) {               // next word (1 % are empty)
                            m = *++my_mask;
                            my_stream += 32;
                            --left;
                        }
                        if (!__any_sync(0xffffffffu, (m != 0u) | (left > 0))) break;
                        if (small) {
                            // branch-free body (predicated store, 32-bit element offsets):
                            // 12 instead of 21 instructions per entry
#pragma unroll
                            for (int rep = 0; rep < 4; ++rep) {  // amortise the vote
                                const bool has = m != 0u;
                                const int j = my_stream[(__ffs(m) - 1) & 31] & 0x03ffffff;
                                m &= m - 1u;
                                if (has && found < stride)
                                    nbr[(unsigned)found * upitch + row_i] = j;
                                found += has ? 1 : 0;
                            }
                        } else {
#pragma unroll
                            for (int rep = 0; rep < 3; ++rep) {
                                if (m != 0u) {
                                    const int j = my_stream[__ffs(m) - 1] & 0x03ffffff;
                                    m &= m - 1u;
                                    if (found < stride) *out = j;
                                    out += pitch;
                                    ++found;
                                }
                            }
                        }
                    }
                }
            }
        }
        if (PAIRS && a_has && a_sub == 0) {
            // flush the unfinished tile (entries first, then flag-less padding)
            int fill = a_done & 3;
            if (fill) {
                int e0 = 0;
                for (; fill < 4; ++fill) { e0 = e1; e1 = e2; e2 = e3; e3 = 0; }
                if ((a_done >> 2) < po.pair_tiles)
                    po.pair_nbr[(int64_t)(a_done >> 2) * po.pair_pitch + (a_i >> 1)] =
                        make_int4(e0, e1, e2, e3);
            }
            po.pair_counts[a_i >> 1] = a_done;
        }
        // slow path: some row wants more than `stride` entries, so the reference's scan
        // order decides which ones are kept (skipped when the caller is going to grow
        // the stride and rebuild anyway)
        if (!PAIRS && exact_prefix && __any_sync(0xffffffffu, found > stride)) {
            found = 0;
            if (active)
                found = scan_row_reference_order(pos_hi, pos_lo, g, cx, cy, cz, cell_start,
                                                 cell_particles, i, hi_i, stride, pitch, nbr);
        } else if (!ascending && active) {
            // particle order not cell-contiguous (never after a reorder; ghost rows of a
            // slab are appended unsorted): rows came out in stream order -- ascending
            // inside every cell, cells by first occupant -- so they are nearly sorted
            if (PAIRS) sort_row_strided(nbr + (int64_t)i * po.list_rows, 1, min(found, stride));
            else sort_row_in_list(nbr, pitch, i, min(found, stride));
        }
        if (active) {
            counts[i] = min(found, stride);
            if (boundary) boundary[i] = boundary_flag(hi_i, g);
        }
        wanted_max = max(wanted_max, __reduce_max_sync(0xffffffffu, found));
    }
    if (lane == 0 && wanted_max > 0) {
        if (wanted_max > stride) atomicExch(&status->overflow, 1);
        atomicMax(&status->max_count, wanted_max);
    }
}

// All-pairs scan for grids with fewer than three cells on some axis.
__global__ void __launch_bounds__(kBuildThreads)
k_list_brute(const float4 *__restrict__ pos_hi, const float4 *__restrict__ pos_lo, int64_t n,
             int64_t n_rows, ListGeom g, int stride, int64_t pitch, int32_t *__restrict__ nbr,
             int32_t *__restrict__ counts, uint8_t *__restrict__ boundary, b2md_status *status) {
    const int64_t i_raw = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool active = i_raw < n_rows;
    const int64_t i = active ? i_raw : n_rows - 1;
    const float4 hi_i = pos_hi[i], lo_i = pos_lo[i];
    const double pi[3] = {ds_to_double(hi_i.x, lo_i.x), ds_to_double(hi_i.y, lo_i.y),
                          ds_to_double(hi_i.z, lo_i.z)};
    int found = 0;
    const int64_t j_end = active ? n : 0;
    for (int64_t j = 0; j < j_end; ++j) {
        if (j == i) continue;
        if (listed_f64(pi, __ldg(&pos_hi[j]), __ldg(&pos_lo[j]), g)) {
            if (found < stride) nbr[(int64_t)found * pitch + i] = (int)j;
            ++found;
        }
    }
    if (boundary && active) boundary[i] = 7;  // tiny boxes: every pair may cross any face
    finish_row(nbr, pitch, i, active, found, stride, counts, status);
}

__global__ void k_count_boundary(const uint8_t *__restrict__ boundary, int64_t n,
                                 b2md_status *status) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int v = (i < n) ? ((boundary[i] & 7) != 0) : 0;
    v = warp_sum_i(v);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&status->n_boundary, v);
}

// Unwrapped fp64 snapshot (pos + img*L, core.py:216-219) + fp32 reference copy.
__global__ void k_snapshot(const float4 *__restrict__ pos_hi, const float4 *__restrict__ pos_lo,
                           const int4 *__restrict__ image, int64_t n, BoxD box,
                           double *__restrict__ at_build, float4 *__restrict__ ref_pos) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 h = pos_hi[i], l = pos_lo[i];
    if (at_build) {
        const int4 im = image[i];
        at_build[3 * i + 0] = __dadd_rn(ds_to_double(h.x, l.x), __dmul_rn((double)im.x, box.L[0]));
        at_build[3 * i + 1] = __dadd_rn(ds_to_double(h.y, l.y), __dmul_rn((double)im.y, box.L[1]));
        at_build[3 * i + 2] = __dadd_rn(ds_to_double(h.z, l.z), __dmul_rn((double)im.z, box.L[2]));
    }
    // w: "no displacement at the last prune" in the packing of integrate.cuh (pack_disp)
    if (ref_pos)
        ref_pos[i] = make_float4(h.x, h.y, h.z, __int_as_float(512 | (512 << 10) | (512 << 20)));
}

// Exact fp64 displacement maximum (neighbor.py:251-253).
__global__ void k_max_disp(const float4 *__restrict__ pos_hi, const float4 *__restrict__ pos_lo,
                           const int4 *__restrict__ image, int64_t n, BoxD box,
                           const double *__restrict__ at_build, b2md_status *status) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double s = 0.0;
    if (i < n) {
        const float4 h = pos_hi[i], l = pos_lo[i];
        const int4 im = image[i];
        double ux = __dadd_rn(ds_to_double(h.x, l.x), __dmul_rn((double)im.x, box.L[0]));
        double uy = __dadd_rn(ds_to_double(h.y, l.y), __dmul_rn((double)im.y, box.L[1]));
        double uz = __dadd_rn(ds_to_double(h.z, l.z), __dmul_rn((double)im.z, box.L[2]));
        double dx = __dsub_rn(ux, at_build[3 * i + 0]);
        double dy = __dsub_rn(uy, at_build[3 * i + 1]);
        double dz = __dsub_rn(uz, at_build[3 * i + 2]);
        s = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
    // non-negative doubles order like their bit patterns
    if ((threadIdx.x & 31) == 0 && s > 0.0)
        atomicMax((unsigned long long *)&status->max_disp2_f64_bits,
                  (unsigned long long)__double_as_longlong(s));
}


// ---------------------------------------------------------------------------
// Pair rows: the force kernel's own view of the list (b2md_pair_rows).
//
// Particles 2t and 2t+1 are neighbours in memory and -- after the Hilbert / cell
// reorder -- in space, so their rows overlap heavily.  Thread t merges the two
// ascending rows into one ascending "pair row": every distinct j once, with two
// flag bits saying whose row it came from,
//     entry = j << 2 | (listed for 2t) | (listed for 2t+1) << 1 .
// The pair force kernel gathers r_j once and evaluates it against both particles,
// which cuts the 16-byte position gathers per particle (the L1 data-pipe limiter
// of the one-row kernel) by about a third and the index stream with them.
//
// Layout: int4 tiles, column-major in tile units -- entries 4q .. 4q+3 of pair t
// are the int4 at d_pair_nbr[q * pair_pitch + t], so one 16-byte load per thread
// and trip fetches four entries and a warp reads 512 contiguous bytes.  Rows are
// padded with flag-less entries (j = 0) up to the longest row of the warp, so the
// force kernel needs no per-entry bound check.
__global__ void __launch_bounds__(128)
k_pair_rows(const int32_t *__restrict__ nbr, const int32_t *__restrict__ counts, int64_t pitch,
            int64_t n_rows, int4 *__restrict__ pair_nbr, int32_t *__restrict__ pair_counts,
            int64_t pair_pitch, int pair_tiles) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t n_pairs = (n_rows + 1) >> 1;
    const bool active = t < n_pairs;
    const int64_t a = 2 * t, b = 2 * t + 1;
    const int ca = active ? counts[a] : 0;
    const int cb = (active && b < n_rows) ? counts[b] : 0;
    const int32_t *ra = nbr + a, *rb = nbr + b;
    constexpr int kEnd = 0x7fffffff;
    int ia = 0, ib = 0;
    int va = ca > 0 ? ra[0] : kEnd;
    int vb = cb > 0 ? rb[0] : kEnd;
    int e0 = 0, e1 = 0, e2 = 0, e3 = 0, k = 0;
    int4 *out = pair_nbr + t;
    const int cap = pair_tiles * 4;
    while (va != kEnd || vb != kEnd) {
        const int m = min(va, vb);
        const bool from_a = va == m, from_b = vb == m;
        const int e = (m << 2) | (from_a ? 1 : 0) | (from_b ? 2 : 0);
        if (from_a) { ++ia; va = ia < ca ? ra[(int64_t)ia * pitch] : kEnd; }
        if (from_b) { ++ib; vb = ib < cb ? rb[(int64_t)ib * pitch] : kEnd; }
        e0 = e1; e1 = e2; e2 = e3; e3 = e;
        ++k;
        if ((k & 3) == 0 && k <= cap)
            out[(int64_t)((k >> 2) - 1) * pair_pitch] = make_int4(e0, e1, e2, e3);
    }
    const int total = k;                       // <= ca + cb <= capacity by construction
    // flush the partial tile, then pad to the warp's longest row (flag-less entries)
    while (k & 3) { e0 = e1; e1 = e2; e2 = e3; e3 = 0; ++k; }
    if (k > total && k <= cap)
        out[(int64_t)((k >> 2) - 1) * pair_pitch] = make_int4(e0, e1, e2, e3);
    const int tiles = k >> 2;
    const int warp_tiles = __reduce_max_sync(0xffffffffu, tiles);
    if (t < pair_pitch)
        for (int q = tiles; q < warp_tiles; ++q)
            out[(int64_t)q * pair_pitch] = make_int4(0, 0, 0, 0);
    if (t < pair_pitch) pair_counts[t] = active ? total : 0;
}

// The marked pairs after k_list_cells_ballot<.., PAIRS> (pair_counts[t] < 0: rows 2t and 2t+1
// sit in different cells or passes and went to the plain list, row-major), merged by a whole
// warp each.  (One thread per pair walking the two rows entry by entry, as k_pair_rows does, is
// a chain of ~90 dependent loads that only 6 % of the threads execute: 134 us at N = 1 M.)
// A warp takes 32 consecutive pairs and, for every marked one, stages both rows in shared
// memory (coalesced loads), finds the merged position of every element by binary search in the
// other row (an element of both rows is emitted once, by row A, with both flags), and stores
// the entries; then all 32 rows are padded to the warp's longest, exactly as k_pair_rows does.
// Same bits.
constexpr int kFixupWarps = 4;

__global__ void __launch_bounds__(kFixupWarps * 32)
k_pair_fixup(const int32_t *__restrict__ nbr, const int32_t *__restrict__ counts, int64_t pitch,
             int list_rows, int64_t n_rows, int4 *__restrict__ pair_nbr,
             int32_t *__restrict__ pair_counts, int64_t pair_pitch, int pair_tiles) {
    extern __shared__ int32_t s_fix[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t *sa = s_fix + warp * (3 * list_rows + 1);      // row A, row B, duplicate prefix of A
    int32_t *sb = sa + list_rows;
    int32_t *sp = sb + list_rows;
    const int64_t t0 = ((int64_t)blockIdx.x * kFixupWarps + warp) * 32;
    const int64_t n_pairs = (n_rows + 1) >> 1;
    if (t0 >= pair_pitch) return;
    const int64_t t = t0 + lane;
    const bool active = t < n_pairs;
    int total = active ? pair_counts[t] : 0;
    const unsigned marked = __ballot_sync(0xffffffffu, active && total < 0);
    int32_t *flat = reinterpret_cast<int32_t *>(pair_nbr);
    const int cap = pair_tiles * 4;
    for (unsigned left = marked; left; left &= left - 1u) {
        const int m_lane = __ffs(left) - 1;
        const int64_t m = t0 + m_lane;
        const int64_t a = 2 * m, b = 2 * m + 1;
        const int ca = counts[a];
        const int cb = b < n_rows ? counts[b] : 0;
        __syncwarp();
        for (int k = lane; k < ca; k += 32) sa[k] = nbr[a * list_rows + k];      // row-major
        for (int k = lane; k < cb; k += 32) sb[k] = nbr[b * list_rows + k];
        __syncwarp();
        // row A: position = k + (elements of B below x) - (common elements below x)
        int dups = 0;
        for (int k0 = 0; k0 < ca; k0 += 32) {                 // warp-uniform trip count
            const int k = k0 + lane;
            const bool in = k < ca;
            const int x = in ? sa[k] : 0x7fffffff;
            int lo = 0, hi = cb;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (sb[mid] < x) lo = mid + 1; else hi = mid;
            }
            const bool dup = in && lo < cb && sb[lo] == x;
            const unsigned dm = __ballot_sync(0xffffffffu, dup);
            const int before = dups + __popc(dm & ((1u << lane) - 1u));
            if (in) {
                sp[k] = before;
                const int pos = k + lo - before;
                if (pos < cap)
                    flat[((int64_t)(pos >> 2) * pair_pitch + m) * 4 + (pos & 3)] =
                        (x << 2) | 1 | (dup ? 2 : 0);
            }
            dups += __popc(dm);
        }
        if (lane == 0) sp[ca] = dups;
        __syncwarp();
        // row B: elements that are not in A
        for (int k0 = 0; k0 < cb; k0 += 32) {
            const int k = k0 + lane;
            const bool in = k < cb;
            const int y = in ? sb[k] : 0x7fffffff;
            int lo = 0, hi = ca;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (sa[mid] < y) lo = mid + 1; else hi = mid;
            }
            const bool dup = in && lo < ca && sa[lo] == y;
            if (in && !dup) {
                const int pos = lo + k - sp[lo];
                if (pos < cap)
                    flat[((int64_t)(pos >> 2) * pair_pitch + m) * 4 + (pos & 3)] = (y << 2) | 2;
            }
        }
        const int merged = ca + cb - dups;
        // flag-less padding of the last tile
        if (lane < ((4 - (merged & 3)) & 3)) {
            const int pos = merged + lane;
            if (pos < cap) flat[((int64_t)(pos >> 2) * pair_pitch + m) * 4 + (pos & 3)] = 0;
        }
        if (lane == m_lane) total = merged;
    }
    // pad to the warp's longest row
    const int tiles = (total + 3) >> 2;
    const int warp_tiles = min(__reduce_max_sync(0xffffffffu, tiles), pair_tiles);
    int4 *out = pair_nbr + t;
    if (t < pair_pitch) {
        for (int q = tiles; q < warp_tiles; ++q) out[(int64_t)q * pair_pitch] = make_int4(0, 0, 0, 0);
        if (!active || ((marked >> lane) & 1u)) pair_counts[t] = total;
    }
}

}  // namespace b2md

using namespace b2md;

namespace {

// pairs != nullptr: pair rows are wanted as well (b2md_build_pair_list); *pairs_done says
// whether the list kernel emitted them itself (the plain rows are then incomplete).
int build_list(const void *d_pos_hi, const void *d_pos_lo, int64_t n, const b2md_box *box,
               const b2md_grid *grid, const int32_t *d_cell_of, const int32_t *d_cell_start,
               const int32_t *d_cell_particles, double r_list, int32_t stride, int64_t pitch,
               int32_t *d_nbr, int32_t *d_counts, uint8_t *d_boundary, double boundary_margin,
               int64_t n_rows, int32_t flags, b2md_status *d_status, void *stream,
               const PairOut *pairs, bool *pairs_done) {
    if (pairs_done) *pairs_done = false;
    if (n <= 0 || !box || !grid || !d_status) { set_error("b2md_build_nlist: bad arguments"); return -1; }
    if (stride < 1) { set_error("b2md_build_nlist: stride must be >= 1"); return -2; }
    if (pitch < n) { set_error("b2md_build_nlist: pitch < n"); return -3; }
    if (n_rows < 1 || n_rows > n) { set_error("b2md_build_nlist: need 1 <= n_rows <= n"); return -4; }
    cudaStream_t s = as_stream(stream);
    ListGeom g;
    g.box = make_box_d(box);
    g.rl2 = r_list * r_list;  // neighbor.py:215
    double lmax = 0.0;
    for (int a = 0; a < 3; ++a) {
        g.nc[a] = grid->ncell[a];
        g.Lf[a] = (float)box->edge[a];
        g.Lhi[a] = (float)box->edge[a];
        g.invLf[a] = (float)(1.0 / box->edge[a]);
        g.margin[a] = (float)boundary_margin;
        g.mid[a] = (float)(0.5 * box->edge[a]);
        // reach of a listed pair (the margin) + the particle's own travel, with slack; the
        // frame needs the near-face layer (margin) and the mid-plane layer to be disjoint
        const double clear = boundary_margin + fmax(boundary_margin - r_list, 0.0) + 1e-3 * box->edge[a];
        g.mid_clear[a] = (0.5 * box->edge[a] - clear > boundary_margin) ? (float)clear : -1.0f;
        lmax = fmax(lmax, box->edge[a]);
    }
    // guard band of the fp32 pre-test (see dist2_f32)
    const double u = 5.9604644775390625e-08;  // 2^-24
    const double ed = 8.0 * u * lmax;
    const double band = 4.0 * (3.0 * (2.0 * 1.5 * r_list * ed + ed * ed) + 4.0 * u * 3.0 * g.rl2);
    g.rl2_in = (float)(g.rl2 - band) * (1.0f - 1e-6f);
    g.rl2_out = (float)(g.rl2 + band) * (1.0f + 1e-6f);
    // Ballot kernel: d = hi_i - fl(hi_j + s), s in {-L_f, 0, +L_f} from the cell image.
    // Per component, against the exact difference of the double-single positions:
    //   |lo_i|, |lo_j| <= u*L each, |L_f - L| <= u*L, rounding of hi_j + s <= u*(L + cell)
    //   <= 1.34*u*L, rounding of the subtraction <= u*|d| <= 0.34*u*L for a pair near the
    //   threshold (|d| <= r_list <= L/3)  =>  delta <= 4.7*u*L; 6*u*L is used.
    // r2: sum_k (2|d_k| delta + delta^2) <= 2*sqrt(3)*r_list*delta + 3*delta^2, plus three
    // roundings of the product / fma chain (<= 4u * r2).  The band is twice that figure
    // (the shared band above is 7x wider; every chunk with a candidate inside the band
    // pays the exact fp64 settle loop, 9 % of the kernel's instructions with the wide one).
    const double db = 6.0 * u * lmax;
    const double band_b = 2.0 * (2.0 * 1.7320508075688772 * 1.001 * r_list * db + 3.0 * db * db +
                                 4.0 * u * 3.0 * g.rl2);
    g.rl2_in_b = (float)(g.rl2 - band_b) * (1.0f - 1e-6f);
    g.rl2_out_b = (float)(g.rl2 + band_b) * (1.0f + 1e-6f);
    const bool prefilter = band < 0.05 * g.rl2;
    const unsigned blocks = blocks_for(n_rows, kBuildThreads);
    const size_t warp_smem = kCandCap * sizeof(float4) + (size_t)(stride + 2) * 32 * sizeof(int32_t);
    // 0: lane = candidate (default), 1: lane = particle; read per call, function attributes
    // set per launch (they are per device, and cheap): the library keeps no state
    const int list_kernel = env_choice("B2MD_LIST_KERNEL", 0) == 1 ? 1 : 0;
    if (grid->fallback) {
        k_list_brute<<<blocks, kBuildThreads, 0, s>>>(
            (const float4 *)d_pos_hi, (const float4 *)d_pos_lo, n, n_rows, g, stride, pitch, d_nbr,
            d_counts, d_boundary, d_status);
    } else if (prefilter && list_kernel == 0 && n < (1ll << 26)) {
        // lane = candidate; the wrap code shares the staged word with the index (26 bits)
        constexpr int kBallotWarps = 8;
        const int64_t nc = grid->n_cells;
        const size_t smem = ballot_warp_bytes() * kBallotWarps;
        if (pairs && (flags & B2MD_LIST_ANY_PREFIX) && env_choice("B2MD_LIST_PAIRS", 1) != 0 &&
            (size_t)kFixupWarps * (3 * (size_t)pairs->list_rows + 1) * sizeof(int32_t) <= 48 * 1024) {
            cudaFuncSetAttribute(k_list_cells_ballot<kBallotWarps, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            // every pair starts out marked "merge from the plain rows"
            cudaMemsetAsync(pairs->pair_counts, 0xff, sizeof(int32_t) * (size_t)pairs->pair_pitch, s);
            k_list_cells_ballot<kBallotWarps, true>
                <<<blocks_for(nc, kBallotWarps), kBallotWarps * 32, smem, s>>>(
                    (const float4 *)d_pos_hi, (const float4 *)d_pos_lo, n, n_rows, g, nc,
                    d_cell_start, d_cell_particles, stride, pitch, d_nbr, d_counts, d_boundary,
                    d_status, 0, *pairs);
            *pairs_done = true;
        } else {
            cudaFuncSetAttribute(k_list_cells_ballot<kBallotWarps, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k_list_cells_ballot<kBallotWarps, false>
                <<<blocks_for(nc, kBallotWarps), kBallotWarps * 32, smem, s>>>(
                    (const float4 *)d_pos_hi, (const float4 *)d_pos_lo, n, n_rows, g, nc,
                    d_cell_start, d_cell_particles, stride, pitch, d_nbr, d_counts, d_boundary,
                    d_status, (flags & B2MD_LIST_ANY_PREFIX) ? 0 : 1, PairOut{});
        }
    } else if (prefilter && warp_smem * 2 <= 200 * 1024) {
        // warp-per-cell kernel; fewer warps per CTA when rows are long
        const int64_t nc = grid->n_cells;
        if (warp_smem * kCellWarps <= 96 * 1024) {
            const size_t smem = warp_smem * kCellWarps;
            cudaFuncSetAttribute(k_list_cells_warp<kCellWarps>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
            k_list_cells_warp<kCellWarps><<<blocks_for(nc, kCellWarps), kCellWarps * 32, smem, s>>>(
                (const float4 *)d_pos_hi, (const float4 *)d_pos_lo, n, n_rows, g, nc, d_cell_start,
                d_cell_particles, stride, pitch, d_nbr, d_counts, d_boundary, d_status);
        } else {
            const size_t smem = warp_smem * 2;
            cudaFuncSetAttribute(k_list_cells_warp<2>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            k_list_cells_warp<2><<<blocks_for(nc, 2), 64, smem, s>>>(
                (const float4 *)d_pos_hi, (const float4 *)d_pos_lo, n, n_rows, g, nc, d_cell_start,
                d_cell_particles, stride, pitch, d_nbr, d_counts, d_boundary, d_status);
        }
    } else if (prefilter) {
        k_list_cells<true><<<blocks, kBuildThreads, 0, s>>>(
            (const float4 *)d_pos_hi, (const float4 *)d_pos_lo, n, n_rows, g, d_cell_of,
            d_cell_start, d_cell_particles, stride, pitch, d_nbr, d_counts, d_boundary, d_status);
    } else {
        k_list_cells<false><<<blocks, kBuildThreads, 0, s>>>(
            (const float4 *)d_pos_hi, (const float4 *)d_pos_lo, n, n_rows, g, d_cell_of,
            d_cell_start, d_cell_particles, stride, pitch, d_nbr, d_counts, d_boundary, d_status);
    }
    if (d_boundary)
        k_count_boundary<<<blocks_for(n_rows, 256), 256, 0, s>>>(d_boundary, n_rows, d_status);
    B2MD_CHECK_LAUNCH("b2md_build_nlist");
    return 0;
}

}  // namespace

B2MD_EXPORT int b2md_build_nlist_ex(const void *d_pos_hi, const void *d_pos_lo, int64_t n,
                                    const b2md_box *box, const b2md_grid *grid,
                                    const int32_t *d_cell_of, const int32_t *d_cell_start,
                                    const int32_t *d_cell_particles, double r_list,
                                    int32_t stride, int64_t pitch, int32_t *d_nbr,
                                    int32_t *d_counts, uint8_t *d_boundary,
                                    double boundary_margin, int64_t n_rows, int32_t flags,
                                    b2md_status *d_status, void *stream) {
    return build_list(d_pos_hi, d_pos_lo, n, box, grid, d_cell_of, d_cell_start, d_cell_particles,
                      r_list, stride, pitch, d_nbr, d_counts, d_boundary, boundary_margin, n_rows,
                      flags, d_status, stream, nullptr, nullptr);
}

B2MD_EXPORT int b2md_build_pair_list(const void *d_pos_hi, const void *d_pos_lo, int64_t n,
                                     const b2md_box *box, const b2md_grid *grid,
                                     const int32_t *d_cell_of, const int32_t *d_cell_start,
                                     const int32_t *d_cell_particles, double r_list,
                                     int32_t stride, int64_t pitch, int32_t *d_nbr,
                                     int32_t *d_counts, uint8_t *d_boundary,
                                     double boundary_margin, int64_t n_rows, int32_t flags,
                                     int32_t list_rows, int32_t *d_pair_nbr,
                                     int32_t *d_pair_counts, int64_t pair_pitch,
                                     int32_t pair_rows, b2md_status *d_status, void *stream) {
    const int64_t n_pairs = (n_rows + 1) / 2;
    if (!d_pair_nbr || !d_pair_counts || pair_pitch < n_pairs || pair_pitch % 32 != 0 ||
        pair_rows % 4 != 0 || pair_rows < 2 * list_rows || list_rows < stride) {
        set_error("b2md_build_pair_list: pair_pitch must be a multiple of 32 >= ceil(n_rows/2), "
                  "pair_rows a multiple of 4 >= 2 * list_rows, list_rows >= stride");
        return -6;
    }
    const PairOut po = {(int4 *)d_pair_nbr, d_pair_counts, pair_pitch, pair_rows / 4, list_rows};
    bool pairs_done = false;
    int rc = build_list(d_pos_hi, d_pos_lo, n, box, grid, d_cell_of, d_cell_start,
                        d_cell_particles, r_list, stride, pitch, d_nbr, d_counts, d_boundary,
                        boundary_margin, n_rows, flags, d_status, stream, &po, &pairs_done);
    if (rc) return rc;
    const unsigned blocks = blocks_for((n_pairs + 31) / 32 * 32, 128);
    const size_t fix_smem = (size_t)kFixupWarps * (3 * (size_t)list_rows + 1) * sizeof(int32_t);
    if (pairs_done)
        k_pair_fixup<<<blocks_for(pair_pitch / 32, kFixupWarps), kFixupWarps * 32, fix_smem,
                       as_stream(stream)>>>(d_nbr, d_counts, pitch, list_rows, n_rows, po.pair_nbr,
                                            d_pair_counts, pair_pitch, po.pair_tiles);
    else
        k_pair_rows<<<blocks, 128, 0, as_stream(stream)>>>(d_nbr, d_counts, pitch, n_rows,
                                                                  po.pair_nbr, d_pair_counts,
                                                                  pair_pitch, po.pair_tiles);
    B2MD_CHECK_LAUNCH("b2md_build_pair_list");
    return 0;
}

B2MD_EXPORT int b2md_build_nlist(const void *d_pos_hi, const void *d_pos_lo, int64_t n,
                                 const b2md_box *box, const b2md_grid *grid,
                                 const int32_t *d_cell_of, const int32_t *d_cell_start,
                                 const int32_t *d_cell_particles, double r_list, int32_t stride,
                                 int64_t pitch, int32_t *d_nbr, int32_t *d_counts,
                                 uint8_t *d_boundary, double boundary_margin, int64_t n_rows,
                                 b2md_status *d_status, void *stream) {
    return b2md_build_nlist_ex(d_pos_hi, d_pos_lo, n, box, grid, d_cell_of, d_cell_start,
                               d_cell_particles, r_list, stride, pitch, d_nbr, d_counts,
                               d_boundary, boundary_margin, n_rows, 0, d_status, stream);
}

B2MD_EXPORT int b2md_snapshot(const void *d_pos_hi, const void *d_pos_lo, const void *d_image,
                              int64_t n, const b2md_box *box, double *d_at_build_f64,
                              void *d_ref_pos_f4, void *stream) {
    if (n <= 0 || !box) { set_error("b2md_snapshot: bad arguments"); return -1; }
    k_snapshot<<<blocks_for(n, 256), 256, 0, as_stream(stream)>>>(
        (const float4 *)d_pos_hi, (const float4 *)d_pos_lo, (const int4 *)d_image, n,
        make_box_d(box), d_at_build_f64, (float4 *)d_ref_pos_f4);
    B2MD_CHECK_LAUNCH("b2md_snapshot");
    return 0;
}

B2MD_EXPORT int b2md_max_displacement(const void *d_pos_hi, const void *d_pos_lo,
                                      const void *d_image, int64_t n, const b2md_box *box,
                                      const double *d_at_build_f64, b2md_status *d_status,
                                      void *stream) {
    if (n <= 0 || !box || !d_status) { set_error("b2md_max_displacement: bad arguments"); return -1; }
    k_max_disp<<<blocks_for(n, 256), 256, 0, as_stream(stream)>>>(
        (const float4 *)d_pos_hi, (const float4 *)d_pos_lo, (const int4 *)d_image, n,
        make_box_d(box), d_at_build_f64, d_status);
    B2MD_CHECK_LAUNCH("b2md_max_displacement");
    return 0;
}

B2MD_EXPORT int b2md_pair_rows(const int32_t *d_nbr, const int32_t *d_counts, int64_t pitch,
                               int32_t stride, int64_t n_rows, int32_t *d_pair_nbr, int32_t *d_pair_counts,
                               int64_t pair_pitch, int32_t pair_rows, void *stream) {
    if (!d_nbr || !d_counts || !d_pair_nbr || !d_pair_counts || n_rows < 1 || pitch < n_rows) {
        set_error("b2md_pair_rows: bad arguments");
        return -1;
    }
    const int64_t n_pairs = (n_rows + 1) / 2;
    if (pair_pitch < n_pairs || pair_pitch % 32 != 0 || pair_rows % 4 != 0 ||
        pair_rows < 2 * stride) {
        set_error("b2md_pair_rows: pair_pitch must be a multiple of 32 >= ceil(n_rows/2), "
                  "pair_rows a multiple of 4 >= 2 * stride");
        return -2;
    }
    // whole warps only: the padding loop uses a warp reduction
    const unsigned blocks = blocks_for((n_pairs + 31) / 32 * 32, 128);
    k_pair_rows<<<blocks, 128, 0, as_stream(stream)>>>(d_nbr, d_counts, pitch, n_rows,
                                                              (int4 *)d_pair_nbr, d_pair_counts,
                                                              pair_pitch, pair_rows / 4);
    B2MD_CHECK_LAUNCH("b2md_pair_rows");
    return 0;
}
