/*
 * b2md.h -- C ABI of libb2md.so: the B200 (sm_100a) kernels behind the `mdbench`
 * per-step molecular-dynamics hot path (arXiv 2406.04210 artifact).
 *
 * The reference (`/root/reference/pkg/src/mdbench`, pure Python + numba) has no
 * FFI.  Its replaceable seam is the chunk-kernel contract of
 * `BackendSelector.run(kernel, n, *args)` (backend.py:63-73) underneath the
 * module-level operator functions (neighbor.py, forces.py, integrate.py,
 * observables.py).  Each entry point below replaces one such kernel / operator
 * body; the reference line it stands in for is cited on the declaration.  The
 * Python package `paper_2406_04210_b200` keeps the operator names and
 * signatures and binds these symbols with ctypes.
 *
 * Conventions
 *  - every pointer named d_* is a DEVICE pointer owned by the caller; the
 *    library keeps no state between calls except inside an explicit
 *    b2md_runner (the native step loop);
 *  - every call takes the CUDA stream (cudaStream_t as void*) it enqueues on and
 *    is asynchronous unless stated otherwise;
 *  - return value: 0 = ok, >0 = cudaError_t, <0 = argument error
 *    (b2md_last_error_string() describes the last failure of the calling thread);
 *  - data-dependent conditions (row overflow, coincident pair, displacement)
 *    are reported through a caller-owned device b2md_status, never by
 *    truncating silently (neighbor.py:145-149, forces.py:113-116).
 *
 * Packed particle layout in HBM (one row per particle, row = physical index):
 *   pos_hi float4 : x,y,z high words of the double-single position, w = species (int bits)
 *   pos_lo float4 : x,y,z low words,                                 w = particle id (int bits)
 *   vel    float4 : vx,vy,vz, w = mass
 *   force  float4 : fx,fy,fz, w = per-particle potential energy (half-shares)
 *   image  int4   : periodic image counters x,y,z, w unused
 *   virial float  : per-particle virial half-share 1/2 sum_j fr*r^2
 * A position is exactly (double)hi + (double)lo; that fp64 value is what the
 * reference's fp64 arithmetic (cells, neighbour decisions) is applied to.
 */
#ifndef B2MD_H
#define B2MD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B2MD_VERSION 108

/* Device-side status block (64 bytes).  Reset with b2md_status_reset. */
typedef struct b2md_status {
    int32_t overflow;            /* 1 if some list row wanted more than `stride` entries */
    int32_t max_count;           /* largest number of neighbours any row wanted (unclamped) */
    uint64_t singular;           /* (i << 32) | j of the lowest i with a coincident partner; ~0 if none */
    uint32_t max_disp2_bits;     /* float bits of max_i |r_i - r_i(build)|^2 (fast in-loop check) */
    int32_t rebuild_flag;        /* set by the fused integrate kernel when max_disp2 > (skin/2)^2 */
    uint64_t max_disp2_f64_bits; /* double bits of the exact fp64 displacement maximum */
    int32_t n_boundary;          /* particles flagged as able to interact across a periodic face */
    int32_t graph_steps;         /* graph mode: MD steps completed by captured step graphs */
    int32_t graph_rebuilds;      /* graph mode: list builds done inside step graphs */
    int32_t frozen;              /* graph mode: set when an in-graph build overflowed; every
                                    later kernel of the batch returns at once */
    int32_t reserved[4];
} b2md_status;

/* Orthorhombic periodic box: edge lengths in fp64 (core.py:25-57).  Inverse
 * edges are formed inside the library as 1.0/L in fp64 like the reference. */
typedef struct b2md_box {
    double edge[3];
} b2md_box;

/* Cell grid geometry (neighbor.py:67-71).  Filled on the host by b2md_grid_shape. */
typedef struct b2md_grid {
    int32_t ncell[3];
    int32_t fallback;       /* any axis with fewer than 3 cells (neighbor.py:90) */
    double cell_edge[3];
    int64_t n_cells;
} b2md_grid;

int b2md_version(void);
const char *b2md_last_error_string(void);

/* ---------------------------------------------------------------- status */
int b2md_status_reset(b2md_status *d_status, void *stream);
/* Same, but keeps the `singular` word (used when a list is rebuilt mid-run). */
int b2md_status_reset_list(b2md_status *d_status, void *stream);

/* ------------------------------------------------- HOST <-> COMPUTE formats
 * Replace TrackedBuffer's np.copyto between sides (core.py:131-137): the
 * reference-format arrays (fp64 / int64 / int32, staged in device memory)
 * are converted to / from the packed layout.  `d_ids` (pos_lo, may be NULL
 * for identity) maps physical row r to logical particle id = pos_lo[r].w. */
int b2md_pack_positions(const double *d_pos_f64, int64_t n, const void *d_ids_pos_lo,
                        void *d_pos_hi, void *d_pos_lo, void *stream);
int b2md_unpack_positions(const void *d_pos_hi, const void *d_pos_lo, int64_t n,
                          const void *d_ids_pos_lo, double *d_pos_f64, void *stream);
int b2md_pack_vec3(const double *d_src_f64, int64_t n, const void *d_ids_pos_lo,
                   void *d_dst_f4, void *stream);
int b2md_unpack_vec3(const void *d_src_f4, int64_t n, const void *d_ids_pos_lo,
                     double *d_dst_f64, void *stream);
int b2md_pack_w_f64(const double *d_src_f64, int64_t n, const void *d_ids_pos_lo,
                    void *d_dst_f4, void *stream);
int b2md_unpack_w_f64(const void *d_src_f4, int64_t n, const void *d_ids_pos_lo,
                      double *d_dst_f64, void *stream);
int b2md_pack_w_i32(const int32_t *d_src_i32, int64_t n, const void *d_ids_pos_lo,
                    void *d_dst_f4, void *stream);
int b2md_unpack_w_i32(const void *d_src_f4, int64_t n, const void *d_ids_pos_lo,
                      int32_t *d_dst_i32, void *stream);
int b2md_pack_images(const int64_t *d_src_i64, int64_t n, const void *d_ids_pos_lo,
                     void *d_image_i4, void *stream);
int b2md_unpack_images(const void *d_image_i4, int64_t n, const void *d_ids_pos_lo,
                       int64_t *d_dst_i64, void *stream);
int b2md_pack_scalar_f32(const double *d_src_f64, int64_t n, const void *d_ids_pos_lo,
                         float *d_dst_f32, void *stream);
int b2md_unpack_scalar_f32(const float *d_src_f32, int64_t n, const void *d_ids_pos_lo,
                           double *d_dst_f64, void *stream);
int b2md_set_ids(void *d_pos_lo, int64_t n, void *stream);      /* pos_lo[r].w = r */
int b2md_get_ids(const void *d_pos_lo, int64_t n, int32_t *d_ids, void *stream);

/* ------------------------------------------------------------- cell binning
 * bin_particles (neighbor.py:57-91).  b2md_grid_shape is host-only fp64.
 * b2md_bin: atomic per-cell count -> warp-shuffle prefix sum -> scatter ->
 * ascending order inside every cell (the reference's stable argsort).
 * Outputs: d_cell_of (n) int32, d_cell_start (n_cells+1) int32,
 * d_cell_particles (n) int32.  d_scratch: >= b2md_bin_scratch_bytes(). */
int b2md_grid_shape(const b2md_box *box, double r_list, b2md_grid *grid_out);
int64_t b2md_bin_scratch_bytes(int64_t n, int64_t n_cells);
int b2md_bin(const void *d_pos_hi, const void *d_pos_lo, int64_t n, const b2md_grid *grid,
             int32_t *d_cell_of, int32_t *d_cell_start, int32_t *d_cell_particles,
             void *d_scratch, void *stream);

/* ------------------------------------------------------ Verlet neighbour list
 * build_neighbor_list (neighbor.py:185-240; kernels 112-182).  Decision
 * r2 < rl2 in fp64 without FMA on (double)hi+(double)lo, 27-cell scan in the
 * reference's order (or all-pairs when grid->fallback), rows ascending.
 * Layout: column-major, entry k of particle i at d_nbr[k * pitch + i]
 * (pitch >= n, multiple of 32) so that a warp's loads coalesce.  Rows wanting
 * more than `stride` entries set status->overflow; status->max_count receives
 * the largest unclamped count.  d_boundary (n) uint8 marks particles within
 * `boundary_margin` of a periodic face (they may interact across it).  Rows are
 * built for particles [0, n_rows) only (n_rows = n, or the owned count when rows
 * [n_rows, n) are ghosts of a slab decomposition). */
int b2md_build_nlist(const void *d_pos_hi, const void *d_pos_lo, int64_t n,
                     const b2md_box *box, const b2md_grid *grid,
                     const int32_t *d_cell_of, const int32_t *d_cell_start,
                     const int32_t *d_cell_particles, double r_list,
                     int32_t stride, int64_t pitch, int32_t *d_nbr, int32_t *d_counts,
                     uint8_t *d_boundary, double boundary_margin, int64_t n_rows,
                     b2md_status *d_status, void *stream);

/* Same, with flags.  B2MD_LIST_ANY_PREFIX: when a row overflows `stride` the kept
 * entries need not be the reference's first `stride` hits in its scan order
 * (neighbor.py:145-149) -- for callers that react to status->overflow by growing the
 * stride and rebuilding (sim.py:141-149), as the native step loop does. */
#define B2MD_LIST_ANY_PREFIX 1
int b2md_build_nlist_ex(const void *d_pos_hi, const void *d_pos_lo, int64_t n,
                        const b2md_box *box, const b2md_grid *grid,
                        const int32_t *d_cell_of, const int32_t *d_cell_start,
                        const int32_t *d_cell_particles, double r_list,
                        int32_t stride, int64_t pitch, int32_t *d_nbr, int32_t *d_counts,
                        uint8_t *d_boundary, double boundary_margin, int64_t n_rows,
                        int32_t flags, b2md_status *d_status, void *stream);

/* The list build of the native step loop (sim.py:131-139 -> neighbor.py:185-240) when the
 * force kernel reads PAIR ROWS (b2md_pair_rows below): list build and pair rows in one call.
 * With B2MD_LIST_ANY_PREFIX and a cell-contiguous particle order (after b2md_gather_rows by
 * Hilbert / cell keys) the list kernel emits the merged rows of particles 2t, 2t+1 straight
 * from its per-cell decision masks, and only the pairs whose two particles sit in different
 * cells go through plain rows and a merge -- d_nbr is then SCRATCH (it holds the rows of those
 * particles only, row-major: row i at d_nbr + i * list_rows); d_counts, d_boundary and the
 * status words are complete.  Otherwise it is b2md_build_nlist_ex followed by b2md_pair_rows
 * (and d_nbr holds the full column-major list).  The pair rows are bit-identical either way.
 * list_rows: allocated rows of d_nbr (>= stride); pair_rows >= 2 * list_rows. */
int b2md_build_pair_list(const void *d_pos_hi, const void *d_pos_lo, int64_t n,
                         const b2md_box *box, const b2md_grid *grid,
                         const int32_t *d_cell_of, const int32_t *d_cell_start,
                         const int32_t *d_cell_particles, double r_list,
                         int32_t stride, int64_t pitch, int32_t *d_nbr, int32_t *d_counts,
                         uint8_t *d_boundary, double boundary_margin, int64_t n_rows,
                         int32_t flags, int32_t list_rows, int32_t *d_pair_nbr,
                         int32_t *d_pair_counts, int64_t pair_pitch, int32_t pair_rows,
                         b2md_status *d_status, void *stream);

/* Snapshot of the unwrapped positions a list was built from
 * (neighbor.py:238, core.py:216-219): exact fp64 rows (n,3) and the fp32
 * reference copy used by the in-loop displacement check. */
int b2md_snapshot(const void *d_pos_hi, const void *d_pos_lo, const void *d_image_i4,
                  int64_t n, const b2md_box *box, double *d_at_build_f64,
                  void *d_ref_pos_f4, void *stream);

/* needs_rebuild's reduction (neighbor.py:251-253), exact fp64:
 * status->max_disp2_f64_bits = max_i |(pos + img*L) - at_build|^2. */
int b2md_max_displacement(const void *d_pos_hi, const void *d_pos_lo, const void *d_image_i4,
                          int64_t n, const b2md_box *box, const double *d_at_build_f64,
                          b2md_status *d_status, void *stream);

/* ------------------------------------------------------------- LJ forces
 * compute_forces_truncated (forces.py:141-159; kernel 72-110), fp32 pair
 * arithmetic on pos_hi, per-particle energy and virial in registers.
 * table: HOST pointer to ntypes*ntypes rows {eps, sigma^2, rc^2, shift} (fp64;
 * forces.py:119-126 for one type).  `stride` = rows of d_nbr per particle (a
 * multiple of 16, zero-filled).  flags: B2MD_FORCE_SKIP_THERMO leaves e_pot / virial unwritten
 * (intermediate steps of the native loop, where nobody can observe them).
 * d_boundary (may be NULL = all) selects the exact-image-shift path per warp.
 * Writes force (xyz + e_pot in w) and virial.
 * A coincident listed pair is reported in status->singular. */
#define B2MD_FORCE_SKIP_THERMO 1
#define B2MD_FORCE_GATED 2        /* return at once when d_status->frozen is set */
#define B2MD_FORCE_SCHEDULED 4    /* pair kernels: d_pair_counts[pair_pitch ...] holds the block
                                     schedule written by b2md_pair_schedule */
#define B2MD_FORCE_ORDERED 8      /* pair kernels: follow the lane order of b2md_pair_order */
int b2md_force_lj(const void *d_pos_hi, int64_t n, const b2md_box *box,
                  const int32_t *d_nbr, const int32_t *d_counts, int64_t pitch,
                  int32_t stride, const uint8_t *d_boundary, const double *table, int32_t ntypes,
                  int32_t flags, void *d_force_f4, float *d_virial, b2md_status *d_status,
                  void *stream);

/* Pair rows -- the layout the production force kernel reads.  Thread t of
 * b2md_force_lj_pairs owns particles 2t and 2t+1 (neighbours in memory and, after
 * the Hilbert / cell reorder, in space) and walks the ascending merge of their two
 * rows of the list above: every distinct j once, entry = j << 2 | (row of 2t lists
 * j) | (row of 2t+1 lists j) << 1.  Entries 4q..4q+3 of pair t form the int4 at
 * d_pair_nbr[(q * pair_pitch + t) * 4]; rows are padded with flag-less entries to
 * the longest row of their warp.  pair_pitch: multiple of 32 >= ceil(n_rows/2);
 * pair_rows (entries per pair row): multiple of 4, >= 2 * stride, so a merge can
 * never overflow.  Derived data: the per-particle list stays the source of truth
 * (and what build_neighbor_list returns, neighbor.py:185-240). */
/* Persistent step kernel for small systems (no counterpart in the reference: it is the
 * per-step launch overhead of a device that it removes).  ONE cooperative launch runs up to
 * n_steps MD steps -- each the body of b2md_force_lj_advance (force, both half-kicks, drift,
 * wrap, displacement check), separated by grid-wide barriers -- over the per-particle list.
 * Step s reads the position high words in d_pos_a (s even) / d_pos_b (s odd) and writes the
 * other buffer; gate_a_word / gate_b_word are the status words holding the rebuild flag of
 * the positions in d_pos_a / d_pos_b.  The loop stops before a step whose input positions
 * need a new list; every completed step adds one to status word 13 (the advance counter), so
 * the caller learns how many steps ran and which buffer is live.  d_barrier:
 * B2MD_BARRIER_BYTES of device scratch, 128-byte aligned.  stride (allocated rows of the list) must be a multiple of 16 entries per
 * lane group: b2md_steps_persistent_lanes(n, stride, ntypes) returns the lanes per particle
 * the launch would use on the current device (16 or 4), 0 when the grid cannot be
 * co-resident -- b2md_steps_persistent then fails with -6 and launches nothing.
 * status->frozen != 0 afterwards: a barrier timed out (never expected; the launch is
 * cooperative) and the loop was abandoned. */
#define B2MD_BARRIER_BYTES 4096
int b2md_steps_persistent_lanes(int64_t n, int32_t stride, int32_t ntypes);
int b2md_steps_persistent(void *d_pos_a, void *d_pos_b, void *d_pos_lo, void *d_vel,
                          void *d_image_i4, int64_t n, const b2md_box *box, double dt,
                          void *d_ref_pos_f4, double half_skin2, const int32_t *d_nbr,
                          const int32_t *d_counts, int64_t pitch, int32_t stride,
                          const uint8_t *d_boundary, const double *table, int32_t ntypes,
                          int32_t gate_a_word, int32_t gate_b_word, int32_t n_steps,
                          uint32_t *d_barrier, b2md_status *d_status, void *stream);

/* Block schedule of the pair kernels (optional).  Blocks whose particles sit near a
 * periodic face (d_boundary, written by b2md_build_nlist) take the image-shift paths and run
 * up to 1.7x longer; in particle order they are dispatched last (a space-filling curve ends
 * on a face) and become the tail of every launch.  b2md_pair_schedule writes a permutation
 * of the blocks -- flagged blocks first -- behind the pair counts, at
 * d_pair_counts[pair_pitch ...] (the buffer must have pair_pitch + b2md_pair_schedule_len(n)
 * entries: the schedule and its scratch); launches that pass B2MD_FORCE_SCHEDULED follow it.
 * Results do not depend on the schedule. */
int64_t b2md_pair_schedule_len(int64_t n);
int b2md_pair_schedule(const uint8_t *d_boundary, int64_t n, int32_t *d_pair_counts,
                       int64_t pair_pitch, void *stream);

/* Lane order of the pair kernels (optional; no reference counterpart -- it changes which thread
 * evaluates the row of forces.py:72-110, not the row).  A warp of the pair kernel walks as many
 * tiles as its longest row has.  b2md_pair_order sorts the pairs of every 128-thread block by
 * row length (stable, in units of `unit` adjacent pairs: 1, 2, 4 ...; with face_key the pairs
 * that may need an image shift sort behind the others) and writes, behind the block schedule
 * (the buffer size b2md_pair_schedule_len(n) covers it), which pair of the block each thread
 * takes; rows are padded to the longest row of their new warp.  Launches that pass
 * B2MD_FORCE_ORDERED follow it; launches that do not remain legal on the same rows.  Per-particle
 * sums do not depend on the order (a thread owns its pair's row and walks it in ascending
 * order either way).  Call it after the pair rows are complete (b2md_pair_rows /
 * b2md_build_pair_list); d_boundary may be NULL when face_key is 0. */
int b2md_pair_order(const uint8_t *d_boundary, int64_t n, int32_t *d_pair_nbr,
                    int32_t *d_pair_counts, int64_t pair_pitch, int32_t pair_rows, int32_t unit,
                    int32_t face_key, void *stream);

int b2md_pair_rows(const int32_t *d_nbr, const int32_t *d_counts, int64_t pitch, int32_t stride,
                   int64_t n_rows, int32_t *d_pair_nbr, int32_t *d_pair_counts,
                   int64_t pair_pitch, int32_t pair_rows, void *stream);

/* compute_forces_truncated over pair rows (forces.py:141-159; kernel 72-110): r_j
 * is gathered once per pair-row entry and evaluated against both particles of the
 * pair; an entry only one of them lists contributes exact zeros to the other, so
 * every per-particle result is bit-identical to b2md_force_lj's.  d_nbr / d_counts
 * / pitch (the per-particle list) are only read to name a coincident pair.  Other
 * arguments as b2md_force_lj. */
int b2md_force_lj_pairs(const void *d_pos_hi, int64_t n, const b2md_box *box,
                        const int32_t *d_pair_nbr, const int32_t *d_pair_counts,
                        int64_t pair_pitch, const int32_t *d_nbr, const int32_t *d_counts,
                        int64_t pitch, const uint8_t *d_boundary, const double *table,
                        int32_t ntypes, int32_t flags, void *d_force_f4, float *d_virial,
                        b2md_status *d_status, void *stream);

/* One launch per intermediate MD step: b2md_force_lj_pairs followed, for every
 * particle and inside the same kernel, by what b2md_vv_finalize_integrate would do
 * with the forces just computed (vv_finalize of this step + vv_integrate of the next,
 * integrate.py:58-79, wrap and image counters core.py:72-93, displacement check
 * neighbor.py:243-254) -- the forces never travel through HBM and are NOT stored.
 * Position high words are read from d_pos_hi by all threads and the advanced ones
 * written to d_pos_hi_out (a different buffer, same layout; the caller swaps);
 * d_pos_lo, d_vel, d_image_i4 and d_ref_pos_f4 are updated in place.
 * Gating: the launch returns at once when int32 word `gate_in_word` of *d_status is
 * non-zero (the positions it would use already need a new list), and sets word
 * `gate_out_word` when the positions it produces do; the two must differ (5 =
 * rebuild_flag, 12 = reserved[0]).  This makes a speculative launch safe: the host
 * reads the flag while the kernel is already queued.  A launch that returns at once
 * also sets its own `gate_out_word`, so launches queued behind it return as well, and
 * every launch that does run adds 1 to word 13 (reserved[1]): the host can queue
 * several steps and learn afterwards how many were taken. */
int b2md_force_lj_pairs_advance(const void *d_pos_hi, void *d_pos_hi_out, void *d_pos_lo,
                                void *d_vel, void *d_image_i4, int64_t n, const b2md_box *box,
                                double dt, void *d_ref_pos_f4, double half_skin2,
                                const int32_t *d_pair_nbr, const int32_t *d_pair_counts,
                                int64_t pair_pitch, const int32_t *d_nbr,
                                const int32_t *d_counts, int64_t pitch,
                                const uint8_t *d_boundary, const double *table, int32_t ntypes,
                                int32_t flags, int32_t gate_in_word, int32_t gate_out_word,
                                b2md_status *d_status, void *stream);

/* b2md_force_lj_pairs_advance with the per-step halo of a slab decomposition fused into
 * it (the reference has no decomposition).  A particle i
 * with d_halo_dst_left[i] >= 0 also stores its advanced position high words (16 bytes)
 * into row d_halo_dst_left[i] of d_halo_out_left, likewise for the right side.  The
 * buffers are the ghost rows of the neighbour ranks' OUTPUT position buffers, mapped into
 * this process (CUDA IPC; peer access over NVLink when the ranks own different GPUs), so
 * the ghost layer needs no pack kernel and no send/recv: the collective that follows the
 * launch anyway (the all-reduce of the rebuild flag) orders the stores before the
 * neighbour's next launch.  A launch whose gate is closed stores nothing.  Null slot
 * arrays = no halo on that side; all four null = b2md_force_lj_pairs_advance. */
/* One-launch step over PRUNED pair rows (dynamic pruning of the Verlet list; the reference has
 * one list, neighbor.py:185-240, and evaluates every listed pair every step, forces.py:72-110).
 * The full ("outer") rows d_pair_nbr hold every pair inside r_cut + skin at the last list build;
 * only the pairs inside r_cut now contribute (forces.py:92).  A launch with prune_mode
 * B2MD_PRUNE_NOW walks the outer rows and also writes the "inner" rows: the entries either
 * particle of the pair has inside r_cut_max + delta now, same order, same layout (d_inner_nbr,
 * d_inner_counts, pair_rows entries per row), and records every particle's displacement from
 * the list snapshot in the spare word of d_ref_pos_f4.  Launches with B2MD_PRUNE_INNER walk the
 * inner rows (fewer entries; the dropped ones would have contributed exact zeros, so the forces
 * are bit-identical) and are valid while no particle has moved more than delta / 2 since the
 * prune; B2MD_PRUNE_OUTER walks the outer rows (when the inner ones are stale and a prune is
 * not legal any more).  Every launch publishes three flag bits about the positions it WRITES in
 * status word gate_out_word: 1 = they need a new list (as b2md_force_lj_pairs_advance), 2 = the
 * inner rows have expired for them, 4 = a prune is no longer legal for them (a particle is
 * further than (skin - delta) / 2 from the list snapshot, so the outer rows are not complete
 * to r_cut_max + delta).  A launch whose gate_in_word says it must not run (bit 1; bit 2 for
 * B2MD_PRUNE_INNER; bit 4 for B2MD_PRUNE_NOW) returns at once and copies the word to
 * gate_out_word.  The flag bits do not clear themselves: three status words rotate, and
 * every launch zeroes gate_clear_word (the word the next launch will write).  Status word 15
 * collects the largest squared displacement since the prune. */
#define B2MD_PRUNE_INNER 1
#define B2MD_PRUNE_NOW 2
#define B2MD_PRUNE_OUTER 3
int b2md_force_lj_pairs_advance_pruned(
    const void *d_pos_hi, void *d_pos_hi_out, void *d_pos_lo, void *d_vel, void *d_image_i4,
    int64_t n, const b2md_box *box, double dt, void *d_ref_pos_f4, double half_skin2,
    const int32_t *d_pair_nbr, const int32_t *d_pair_counts, int64_t pair_pitch,
    const int32_t *d_nbr, const int32_t *d_counts, int64_t pitch, const uint8_t *d_boundary,
    const double *table, int32_t ntypes, int32_t flags, int32_t gate_in_word,
    int32_t gate_out_word, int32_t gate_clear_word, int32_t prune_mode, int32_t *d_inner_nbr,
    int32_t *d_inner_counts, int32_t pair_rows, double r_cut_max, double skin, double delta,
    b2md_status *d_status, void *stream);

int b2md_force_lj_pairs_advance_halo(const void *d_pos_hi, void *d_pos_hi_out, void *d_pos_lo,
                                     void *d_vel, void *d_image_i4, int64_t n,
                                     const b2md_box *box, double dt, void *d_ref_pos_f4,
                                     double half_skin2, const int32_t *d_pair_nbr,
                                     const int32_t *d_pair_counts, int64_t pair_pitch,
                                     const int32_t *d_nbr, const int32_t *d_counts,
                                     int64_t pitch, const uint8_t *d_boundary,
                                     const double *table, int32_t ntypes, int32_t flags,
                                     int32_t gate_in_word, int32_t gate_out_word,
                                     const int32_t *d_halo_dst_left, void *d_halo_out_left,
                                     const int32_t *d_halo_dst_right, void *d_halo_out_right,
                                     b2md_status *d_status, void *stream);

/* The same for the thread- (or sub-warp-) per-particle kernel b2md_force_lj: small
 * systems, where a step is shorter than a host round trip, queue several of these. */
int b2md_force_lj_advance(const void *d_pos_hi, void *d_pos_hi_out, void *d_pos_lo, void *d_vel,
                          void *d_image_i4, int64_t n, const b2md_box *box, double dt,
                          void *d_ref_pos_f4, double half_skin2, const int32_t *d_nbr,
                          const int32_t *d_counts, int64_t pitch, int32_t stride,
                          const uint8_t *d_boundary, const double *table, int32_t ntypes,
                          int32_t flags, int32_t gate_in_word, int32_t gate_out_word,
                          b2md_status *d_status, void *stream);

/* compute_forces_all_to_all (forces.py:129-138; kernel 29-69): shared-memory
 * tiled all-pairs scan, same outputs. */
int b2md_force_lj_all_pairs(const void *d_pos_hi, int64_t n, const b2md_box *box,
                            const double *table, int32_t ntypes, void *d_force_f4,
                            float *d_virial, b2md_status *d_status, void *stream);

/* --------------------------------------------------------- velocity Verlet
 * vv_integrate (integrate.py:58-70 + core.py:72-93): half-kick, drift in
 * double-single, wrap, image counters.  When d_ref_pos_f4 != NULL the kernel
 * also reduces the squared displacement from the list snapshot into
 * status->max_disp2_bits and raises status->rebuild_flag when it exceeds
 * half_skin2 (neighbor.py:243-254, fp32 fast check; the exact test is
 * b2md_max_displacement). */
int b2md_vv_integrate(void *d_pos_hi, void *d_pos_lo, void *d_vel, const void *d_force_f4,
                      void *d_image_i4, int64_t n, const b2md_box *box, double dt,
                      void *d_ref_pos_f4, double half_skin2, b2md_status *d_status,
                      void *stream);
/* Same kernels, but they return immediately when d_status->frozen is set (used by
 * the captured step graph; kicks = 1 or 2 half-kicks before the drift). */
int b2md_vv_integrate_gated(void *d_pos_hi, void *d_pos_lo, void *d_vel, const void *d_force_f4,
                            void *d_image_i4, int64_t n, const b2md_box *box, double dt,
                            void *d_ref_pos_f4, double half_skin2, b2md_status *d_status,
                            int32_t kicks, void *stream);
/* vv_finalize (integrate.py:73-79). */
int b2md_vv_finalize(void *d_vel, const void *d_force_f4, int64_t n, double dt, void *stream);
/* finalize of step s fused with integrate of step s+1 (one pass over the state). */
int b2md_vv_finalize_integrate(void *d_pos_hi, void *d_pos_lo, void *d_vel,
                               const void *d_force_f4, void *d_image_i4, int64_t n,
                               const b2md_box *box, double dt, void *d_ref_pos_f4,
                               double half_skin2, b2md_status *d_status, void *stream);

/* ------------------------------------------------- Andersen thermostat + streams
 * andersen_thermostat (integrate.py:82-107) over the counter-based streams of
 * rng.py:40-66 (Philox4x64-10 keyed (seed, 0), counter (block+1, 0, stream, step),
 * u = ((raw >> 11) + 0.5) 2^-53, normals = ndtri(u)).  Particle i (LOGICAL id, taken
 * from pos_lo.w when d_ids_pos_lo != NULL) is redrawn iff uniform word i < probability;
 * its new velocity is normal words n+3i..n+3i+2 times sqrt(T / m).  d_redrawn
 * (may be NULL) receives the number of redrawn particles.
 * b2md_stream_words exposes raw words / uniforms / normals [offset, offset+count). */
int b2md_andersen(void *d_vel, const void *d_ids_pos_lo, int64_t n, uint64_t seed, uint64_t step,
                  double probability, double temperature, int32_t *d_redrawn, void *stream);
/* The finalize slots of a thermostatted step in ONE pass (sim.py:86-87): vv_finalize
 * (integrate.py:73-79), then andersen_thermostat at `step` (integrate.py:82-107; logical ids
 * from d_pos_lo.w), and with integrate_next != 0 also vv_integrate of the next step
 * (integrate.py:58-70 + core.py:72-93, displacement check as b2md_vv_integrate when
 * d_ref_pos_f4 != NULL).  Bit-identical to b2md_vv_finalize + b2md_andersen
 * [+ b2md_vv_integrate]; used by the native loops, which would otherwise spend four launches
 * on a thermostatted step. */
int b2md_vv_finalize_andersen(void *d_pos_hi, void *d_pos_lo, void *d_vel, const void *d_force_f4,
                              void *d_image_i4, int64_t n, const b2md_box *box, double dt,
                              uint64_t seed, uint64_t step, double probability,
                              double temperature, int32_t integrate_next, void *d_ref_pos_f4,
                              double half_skin2, b2md_status *d_status, void *stream);
int b2md_stream_words(uint64_t seed, uint64_t stream_id, uint64_t step, int64_t word_offset,
                      int64_t count, uint64_t *d_raw, double *d_uniform, double *d_normal,
                      void *stream);

/* ------------------------------------------------------------ observables
 * reduce_sum (observables.py:43-74): the reference's fixed pairing tree
 * (4096-value blocks, adjacent pairs, odd leftover carried), bit-exact in fp64.
 * d_scratch: ceil(n/4096) doubles (+ further levels).  Result -> d_out[0]. */
int64_t b2md_reduce_scratch_bytes(int64_t n);
int b2md_reduce_sum_f64(const double *d_values, int64_t n, double *d_scratch,
                        double *d_out, void *stream);
/* measure() (sim.py:159-174; observables.py:77-98) in one pass over vel/force/
 * virial with the same tree: d_out[0..7] = e_pot, e_kin, p_x, p_y, p_z,
 * virial, mass, n.  d_scratch: 8 * ceil(n/4096) doubles (+ further levels). */
int64_t b2md_thermo_scratch_bytes(int64_t n);
int b2md_thermo(const void *d_vel, const void *d_force_f4, const float *d_virial, int64_t n,
                double *d_scratch, double *d_out8, void *stream);

/* -------------------------------------------- reorder (Hilbert / cell order)
 * reorder_by_cell (neighbor.py:257-270) generalised: 64-bit keys, stable LSD
 * radix sort, gather of every per-particle array.
 * b2md_hilbert_keys: Hilbert index of the cell-aligned coordinate
 *   (cell << sub_bits) | floor(frac_in_cell * 2^sub_bits) per axis, cell = exactly
 *   bin_particles' cell coordinate, so each cell's particles become contiguous;
 *   b2md_hilbert_key_bits returns the number of significant key bits (<= 63).
 * b2md_cell_keys: key = flat cell index (exactly reorder_by_cell's order).
 * b2md_sort_pairs_u64: stable; on return keys/values are in d_keys/d_vals.
 * b2md_gather16 / b2md_gather4: dst[k] = src[perm[k]] for 16- / 4-byte rows. */
int b2md_hilbert_key_bits(const b2md_grid *grid, int32_t sub_bits);
int b2md_hilbert_keys(const void *d_pos_hi, const void *d_pos_lo, int64_t n,
                      const b2md_grid *grid, int32_t sub_bits, uint64_t *d_keys, void *stream);
int b2md_cell_keys(const int32_t *d_cell_of, int64_t n, uint64_t *d_keys, void *stream);
int b2md_iota_i32(int32_t *d_vals, int64_t n, void *stream);
int64_t b2md_sort_scratch_bytes(int64_t n);
int b2md_sort_pairs_u64(uint64_t *d_keys, int32_t *d_vals, uint64_t *d_keys_tmp,
                        int32_t *d_vals_tmp, int64_t n, int32_t key_bits,
                        void *d_scratch, void *stream);
int b2md_gather16(const void *d_src, void *d_dst, const int32_t *d_perm, int64_t n, void *stream);
int b2md_gather4(const void *d_src, void *d_dst, const int32_t *d_perm, int64_t n, void *stream);
/* reorder_by_cell's "every buffer through the same permutation" (neighbor.py:267-269) in one
 * launch: dst16[a][k] = src16[a][perm[k]] for five 16-byte-row arrays (host arrays of five
 * device pointers: pos_hi, pos_lo, vel, force, image), dst4[k] = src4[perm[k]] (virial;
 * may be null). */
int b2md_gather_rows(const void *const *d_src16, void *const *d_dst16, const void *d_src4,
                     void *d_dst4, const int32_t *d_perm, int64_t n, void *stream);

/* ---------------------------------------------- slab decomposition (multi-GPU)
 * No counterpart in the reference; SURVEY.md section 8e.  A rank
 * owns the x-slab of half-width `half` around `centre` of the global periodic
 * box and keeps ghost rows of neighbour ranks behind its owned rows, all in
 * global coordinates.
 * b2md_slab_classify: d = x - centre wrapped into [-L/2, L/2) (fp64, no FMA);
 *   flag_left[i] = d < lo_cut, flag_right[i] = d >= hi_cut.  Migration uses
 *   (-half, half); ghost selection (-half + r_ghost, half - r_ghost).
 * b2md_compact_indices: stable stream compaction of the indices whose flag is 1.
 * b2md_flag_neither: out = !(a | b) (rows that stay).
 * Records are then moved with b2md_gather16 and exchanged with NCCL send/recv.
 * b2md_halo_slots: destination slots of the halo fused into the step kernel
 *   (b2md_force_lj_pairs_advance_halo): d_dst[0..n) = -1, d_dst[d_send_idx[k]] = base + k.
 * b2md_enable_peer_access: kernels of the current device may access memory of
 *   peer_device afterwards (synchronous; -2 = no peer path between the two). */
int b2md_halo_slots(const int32_t *d_send_idx, int64_t n_send, int32_t base, int64_t n,
                    int32_t *d_dst, void *stream);
/* d_out[d_dst[i]] = d_rows[i] (16-byte rows) wherever d_dst[i] >= 0: the same stores the step
 * kernel issues, on their own -- the start-up probe of a peer mapping. */
int b2md_halo_store(const void *d_rows_f4, const int32_t *d_dst, int64_t n, void *d_out_f4,
                    void *stream);
int b2md_enable_peer_access(int32_t peer_device);
int b2md_slab_classify(const void *d_pos_hi, const void *d_pos_lo, int64_t n, double centre,
                       double box_x, double lo_cut, double hi_cut, int32_t *d_flag_left,
                       int32_t *d_flag_right, void *stream);
int64_t b2md_compact_scratch_bytes(int64_t n);
int b2md_compact_indices(const int32_t *d_flags, int64_t n, int32_t *d_out_idx, int32_t *d_count,
                         void *d_scratch, void *stream);
int b2md_flag_neither(const int32_t *d_a, const int32_t *d_b, int64_t n, int32_t *d_out,
                      void *stream);

/* ------------------------------------------------------------ native step loop
 * Simulation.run / SignalEngine.run_steps (core.py:262-279) with the rebuild
 * policy of Simulation._compute_forces/_rebuild (sim.py:114-149), driven from
 * C++ so that a step costs two launches and no Python:
 *
 *   (with pair rows and pos_hi_alt: one b2md_force_lj_pairs_advance launch per
 *   intermediate step, gated on the rebuild flag instead of the three launches below)
 *   [finalize(s-1) + integrate(s) fused, folds the displacement check]
 *   [async 64-byte status read-back]  [force(s), launched speculatively]
 *   host looks at the flag while the force kernel runs; only if it is set:
 *   bin -> (Hilbert/cell reorder) -> list build -> snapshot -> force again.
 * With use_graph = 1 the middle steps of a call are launches of ONE captured CUDA
 * graph per step: integrate -> gate kernel (cudaGraphSetConditional) -> IF node
 * holding the whole rebuild sequence -> force.  No host round trip per step; an
 * in-graph overflow freezes the remaining launches of the batch and is then
 * handled exactly like the ungraphed case.
 *
 * All memory is caller-owned (PyTorch tensors); per-particle arrays come in
 * pairs so a reorder can gather from one set into the other.  The runner never
 * grows a list: when a build overflows `stride_rows` it stops with
 * reason = B2MD_RUN_OVERFLOW and the caller re-creates it with bigger buffers
 * (sim.py:141-149 semantics: grow and rebuild, never truncate). */
typedef struct b2md_runner_config {
    int64_t n;
    int64_t capacity;            /* rows in every per-particle array, >= n */
    b2md_box box;
    double dt;
    double r_cut;                /* largest pair cutoff */
    double skin;
    int32_t ntypes;
    int32_t reorder_mode;        /* 0 none, 1 Hilbert, 2 cell order */
    int32_t reorder_every;       /* reorder on every k-th rebuild (>= 1) */
    int32_t hilbert_bits;        /* sub-cell bits per axis of the Hilbert key */
    const double *table;         /* HOST, ntypes*ntypes*4, copied at create */
    void *pos_hi[2], *pos_lo[2], *vel[2], *force[2], *image[2];
    float *virial[2];
    int32_t current;             /* which set of the pairs above is live */
    int32_t stride;              /* neighbour budget per particle */
    int32_t *nbr;                /* round_up(stride,16) * pitch, zero-filled */
    int64_t pitch;
    int32_t *counts;             /* pitch */
    uint8_t *boundary;           /* pitch */
    void *ref_pos;               /* float4[pitch] */
    double *at_build;            /* n*3 fp64 snapshot, may be NULL */
    int32_t *cell_of, *cell_start, *cell_particles;   /* n, n_cells+1, n */
    void *bin_scratch;           /* b2md_bin_scratch_bytes(n, n_cells) */
    uint64_t *keys, *keys_tmp;   /* n each (reorder only) */
    int32_t *perm, *perm_tmp;    /* n each (reorder only) */
    void *sort_scratch;          /* b2md_sort_scratch_bytes(n) */
    b2md_status *status;         /* device */
    void *stream;                /* the caller's stream; the runner orders its own against it */
    int32_t use_graph;           /* k >= 1: middle steps run as captured CUDA graphs of k MD
                                    steps each (conditional rebuild node per step), no
                                    per-step host round trip; 0: host-driven steps */
    int32_t pair_rows;           /* entries per pair row (multiple of 4, >= 2*round_up(stride,16));
                                    0 = one thread per particle (b2md_force_lj) */
    int32_t *pair_nbr;           /* pair_rows * pair_pitch (b2md_pair_rows layout) */
    int32_t *pair_counts;        /* pair_pitch */
    int64_t pair_pitch;          /* multiple of 32 >= ceil(n/2) */
    void *pos_hi_alt;            /* float4[capacity]: second buffer for the position high words;
                                    it lets the intermediate steps run as ONE kernel each
                                    (b2md_force_lj_pairs_advance / b2md_force_lj_advance);
                                    NULL = separate integrate and force launches */
    int32_t queue_depth;         /* one-launch steps queued per status read-back (>= 1); small
                                    systems, whose step is shorter than a host round trip,
                                    want several */
    int32_t pair_schedule;       /* != 0: pair_counts has b2md_pair_schedule_len(n) more entries.
                                    bit 0: the runner keeps a block schedule there (see above);
                                    bit 1: and a lane order (b2md_pair_order), bit 2 its face_key,
                                    bits 8-13 its unit (0 = 1) */
    int32_t persistent_steps;    /* > 0: intermediate steps of systems without pair rows run in
                                    batches of up to this many steps per launch of
                                    b2md_steps_persistent (needs pos_hi_alt, barrier and
                                    list_row_multiple = 64); 0: one launch per step */
    int32_t list_row_multiple;   /* nbr holds round_up(stride, this) rows; 0 = 16 (64 lets the
                                    persistent kernel use 16 lanes per particle) */
    uint32_t *barrier;           /* B2MD_BARRIER_BYTES of device scratch, 128-byte aligned */
    /* Optional caller-owned resources (NULL = the runner creates and destroys its own).
     * Page-locking memory and creating streams are the expensive parts of creating a
     * runner (1-7 ms measured on B200); a caller that builds many short-lived simulations
     * hands in recycled ones (the Python host passes blocks of torch's caching host
     * allocator and pooled torch streams). */
    void *h_status;              /* >= 64 bytes of page-locked host memory */
    void *run_stream;            /* cudaStream_t for the step loop (must not be `stream`) */
    void *copy_stream;           /* cudaStream_t for the status read-backs */
    /* Pruned ("inner") pair rows: with prune_delta > 0 (and pair rows, pos_hi_alt, queue_depth
     * 1) the one-launch steps walk rows pruned to r_cut + prune_delta, re-pruned from the full
     * rows whenever a particle has moved prune_delta / 2 since the last prune -- see
     * b2md_force_lj_pairs_advance_pruned.  Same shapes as pair_nbr / pair_counts. */
    int32_t *pair_nbr_inner;
    int32_t *pair_counts_inner;
    double prune_delta;
    /* Optional cudaEvent_t: the velocities (vel[current]) are still being written by work on
     * another stream (an upload from host memory) that this event follows.  The first list
     * build (b2md_runner_prepare) then touches positions and images only, and waits for the
     * event -- and brings the velocities into the new row order -- behind it, so that the
     * upload overlaps the build.  NULL: everything is ordered by `stream` as usual. */
    void *vel_ready_event;
} b2md_runner_config;

enum { B2MD_RUN_DONE = 0, B2MD_RUN_OVERFLOW = 1, B2MD_RUN_SINGULAR = 2 };

typedef struct b2md_run_report {
    int64_t steps_done;
    int32_t reason;              /* B2MD_RUN_* */
    int32_t rebuilds;            /* list builds during this call */
    int32_t reorders;
    int32_t current;             /* live buffer set after the call */
    int32_t max_count;           /* largest row length wanted by the last build */
    int32_t wasted_force_launches;
    int64_t kernel_launches;     /* kernels enqueued by this call */
    int32_t list_valid;          /* 0 if the call stopped before a usable list existed */
    int32_t n_boundary;
    double max_disp2;            /* last displacement maximum seen (fp32 check) */
    uint64_t singular;           /* status->singular when reason == B2MD_RUN_SINGULAR */
    int64_t graph_steps;         /* steps of this call that ran as captured graphs */
    /* CUDA-event phase timers (reference sim.py:114-129 force_seconds / nlist_seconds):
     * GPU time of the whole call on the runner's stream, and the part of it spent in
     * rebuild sequences (reorder + bin + list build + snapshot + pair rows).  The per-step
     * displacement test is fused into the step kernels and counts as force time. */
    double gpu_ms;
    double rebuild_gpu_ms;
} b2md_run_report;

typedef struct b2md_runner b2md_runner;

b2md_runner *b2md_runner_create(const b2md_runner_config *cfg);
void b2md_runner_destroy(b2md_runner *r);
/* Swap in bigger list buffers after B2MD_RUN_OVERFLOW (nbr: round_up(stride,16)*pitch, zero-filled). */
int b2md_runner_set_list(b2md_runner *r, int32_t *nbr, int32_t stride);
/* ... and the matching pair-row buffer (pair_rows >= 2 * round_up(stride,16)). */
int b2md_runner_set_pair_list(b2md_runner *r, int32_t *pair_nbr, int32_t pair_rows);
/* (Re)build the list for the current positions and evaluate forces
 * (Simulation.__init__'s initial _compute_forces, sim.py:90).  Synchronous. */
int b2md_runner_prepare(b2md_runner *r, b2md_run_report *report);
/* Advance n_steps.  finalize_at_end != 0 leaves velocities fully kicked
 * (state as after the reference's finalize slot); otherwise the last half-kick
 * is deferred into the next call's first fused kernel.  Synchronous on return. */
int b2md_runner_run(b2md_runner *r, int64_t n_steps, int32_t finalize_at_end,
                    b2md_run_report *report);
/* Andersen thermostat as the reference's second finalize slot (sim.py:86-87,100-102;
 * integrate.py:82-107): after the second half-kick of every step, b2md_andersen(seed,
 * step, probability, temperature) with step = first_step + steps completed so far in the
 * call.  probability = min(rate * dt, 1); 0 switches the thermostat off.  A thermostatted
 * runner launches integrate / force / finalize / thermostat separately (the thermostat
 * sits between the two half-kicks that the fused kernels merge). */
/* After a stride growth: the new inner pair rows (same shape as the new pair rows). */
int b2md_runner_set_inner_pair_list(b2md_runner *runner, int32_t *d_pair_nbr_inner);
/* Prune launches so far; *outer_steps (may be NULL) = one-launch steps that had to walk the
 * full rows because the inner ones had expired and a prune was no longer legal. */
int64_t b2md_runner_prune_count(const b2md_runner *runner, int64_t *outer_steps);
int b2md_runner_set_thermostat(b2md_runner *r, double probability, double temperature,
                               uint64_t seed);
/* Step counter (SignalEngine.step_count) of the first step of the next b2md_runner_run. */
int b2md_runner_set_step(b2md_runner *r, int64_t first_step);

/* ------------------------------------------------- native loop, all-to-all forces
 * Simulation.run with force_mode = "all_to_all", the reference's default (sim.py:62-102:
 * integrate -> compute_forces_all_to_all -> finalize [-> andersen_thermostat] per step,
 * core.py:262-279 for the loop).  n_steps MD steps are enqueued on `stream` without a host
 * round trip per step -- there is no list and no rebuild decision -- and the status block is
 * read back every 512 steps and at the end.  d_pos_hi_alt (may be NULL): a second buffer for
 * the position high words; with it an intermediate step without thermostat is ONE launch
 * (b2md_force_lj_all_pairs_advance), the final positions are copied back to d_pos_hi.  Same kernels
 * and order of operations as the operator-by-operator loop: bit-identical trajectories.
 * On return the velocities carry both half-kicks and d_force_f4 / d_virial hold the forces,
 * per-particle energies and virial of the final positions.  thermo_probability = min(rate *
 * dt, 1), 0 = no thermostat; first_step = SignalEngine.step_count before the call (index of
 * the thermostat stream).  h_status: 64 bytes of page-locked host memory.  A coincident
 * pair (forces.py:113-116) ends the call with report->reason = B2MD_RUN_SINGULAR and the
 * pair in report->singular; the state is then not meaningful.  Only steps_done, reason,
 * kernel_launches, singular and gpu_ms of the report are filled. */
int b2md_run_all_pairs(void *d_pos_hi, void *d_pos_lo, void *d_vel, void *d_force_f4,
                       void *d_image_i4, float *d_virial, int64_t n, const b2md_box *box,
                       const double *table, int32_t ntypes, double dt, int64_t n_steps,
                       double thermo_probability, double thermo_temperature,
                       uint64_t thermo_seed, int64_t first_step, void *d_pos_hi_alt,
                       b2md_status *d_status, void *h_status, void *stream,
                       b2md_run_report *report);
/* compute_forces_all_to_all + vv_finalize + vv_integrate of the next step in one launch (the
 * intermediate steps of b2md_run_all_pairs when d_pos_hi_alt != NULL; forces.py:129-138,
 * integrate.py:58-79): the thread that holds a particle's total force advances it.  Reads
 * d_pos_hi, writes the new high words to d_pos_hi_out (a different buffer); d_pos_lo, d_vel
 * and d_image_i4 are updated in place; forces are not stored.  Bit-identical to the separate
 * launches. */
int b2md_force_lj_all_pairs_advance(const void *d_pos_hi, void *d_pos_hi_out, void *d_pos_lo,
                                    void *d_vel, void *d_image_i4, int64_t n,
                                    const b2md_box *box, const double *table, int32_t ntypes,
                                    double dt, b2md_status *d_status, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* B2MD_H */
