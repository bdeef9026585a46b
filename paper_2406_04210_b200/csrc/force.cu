// Truncated / shifted Lennard-Jones forces over the Verlet list: reference
// compute_forces_truncated (forces.py:141-159), kernel _truncated_chunk (72-110);
// plus the all-pairs kernel (_all_to_all_chunk, forces.py:29-69).
//
// Three kernels over the same list:
//   k_force_lj              one thread (or sub-warp) per particle over its own row --
//                           small systems, and the reference of the bitwise tests;
//   k_force_lj_pair         one thread per particle PAIR over the pair's merged row on
//                           packed fp32x2 arithmetic -- large systems (n >= 200 000);
//   k_force_lj_pair<ADVANCE> the same, then finalize + integrate + displacement check for
//                           the particles just evaluated: one launch per MD step.
// fp32 pair arithmetic on the position high words, force / energy / virial accumulated in
// registers.  Neighbour indices stream through the column-major list (coalesced,
// evict-first); neighbour positions are 16-byte gathers served by L1/L2 because particles
// are kept in Hilbert / cell order.
//
// Minimum image.  A literal fp32 transcription of d - L*rint(d/L) loses ~ulp(L)
// on pairs that interact across a periodic face (r^-13 amplifies it past the 1e-5
// budget).  Two paths, chosen per warp:
//   * interior warps (no lane flagged `boundary` at list build): neighbours are
//     on the same side of every face for the list's whole lifetime, so
//     d = xi - xj needs no image shift at all (and is exact by Sterbenz' lemma
//     away from the origin);
//   * boundary warps: n = rint(d/L) via the 1.5*2^23 trick, then the box length
//     (as L_hi + L_lo) is subtracted from whichever coordinate is the larger one,
//     which is exact, before the difference is formed.
//
// Single-type systems defer the 24*eps, 2*eps, 12*eps prefactors to the end of the
// row; tabulated systems (Kob-Andersen) read {sigma^2, rc^2, 24 eps, 2 eps, shift/2}
// per species pair from shared memory.
//
// Coincident pairs (r2 == 0; forces.py:94-97) cost nothing in the loop: they
// turn the row's accumulators non-finite, and only then is the row rescanned to
// report (i, first j) through status->singular.
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "integrate.cuh"

namespace b2md {

constexpr int kForceThreads = 128;
#ifndef B2MD_PAIR_THREADS
#define B2MD_PAIR_THREADS 128
#endif
constexpr int kPairThreads = B2MD_PAIR_THREADS;    // CTA size of k_force_lj_pair (1024 threads per SM)
constexpr int kMaxTypes = 8;

// Lanes per particle of the row kernels (k_force_lj, its ADVANCE form and the persistent
// step kernel all take the same decision, so their per-particle sums -- partial sums of the
// lanes combined by shuffles -- are bit-identical): the widest sub-warp whose grid of n * lanes
// threads fits the device at once (148 SMs x 1024 threads; small systems are latency-bound
// serial row loops, the more lanes the shorter) and whose trips of 4 * lanes entries stay
// inside the `rows` allocated per row.  B2MD_FORCE_SUBWARP pins it (A/B runs).
inline int lanes_for(int64_t n, int rows) {
    const int pinned = env_choice("B2MD_FORCE_SUBWARP", 0);
    const int cand[4] = {16, 4, 2, 1};
    for (int k = 0; k < 4; ++k) {
        const int sub = cand[k];
        if (pinned && sub != pinned) continue;
        if (rows % (4 * sub) != 0) continue;
        if (pinned || n * sub <= (int64_t)kNumSM * 1024) return sub;
    }
    return 1;
}

struct PairParams {   // one species pair, fp32
    float sig2, rc2, c_f, c_u;   // sigma^2, rc^2, 24*eps, 2*eps
    float half_shift, c_w;       // shift/2, 12*eps
};

struct ForceArgs {
    BoxF box;
    PairParams single;
    int ntypes;
    const int32_t *schedule;    // pair kernel: block executed by blockIdx.x (null = identity)
    const uint8_t *order;       // pair kernel: pair of the block taken by threadIdx.x (null = identity)
    float4 tab_a[kMaxTypes * kMaxTypes];   // sig2, rc2, c_f, c_u
    float2 tab_b[kMaxTypes * kMaxTypes];   // half_shift, c_w
};

// 1/x to 1 ulp on the SFU (MUFU.RCP), no IEEE slow path
__device__ __forceinline__ float rcp_fast(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float rint_small(float q) {
    // round-half-even for |q| < 2^22 on the FMA pipe (no FRND / conversion pipe)
    const float magic = 12582912.0f;  // 1.5 * 2^23
    return __fsub_rn(__fadd_rn(q, magic), magic);
}

template <bool CAREFUL>
__device__ __forceinline__ float delta(float xi, float xj, float L_hi, float L_lo, float invL) {
    if (!CAREFUL) return xi - xj;
    const float d0 = xi - xj;
    const float ns = rint_small(d0 * invL);            // -1, 0 or +1 for listed pairs
    const float a = fmaf(-fmaxf(ns, 0.0f), L_hi, xi);  // shift the larger coordinate: exact
    const float b = fmaf(-fmaxf(-ns, 0.0f), L_hi, xj);
    return fmaf(-ns, L_lo, a - b);
}

struct RowAcc {
    float fx, fy, fz, u, w;
    int cnt;
};

// A load the compiler can neither hoist nor merge with an earlier load of the same address.
__device__ __forceinline__ float4 reload_f4(const float4 *p) {
    float4 v;
    asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

// Single-type pair: prefactors deferred.  `in` false => contributes exact zeros.
// THERMO = false drops the energy / virial / count accumulators (intermediate
// steps of the native loop, whose per-particle energies nobody can observe).
template <bool THERMO>
__device__ __forceinline__ void lj_pair_single(RowAcc &acc, float dx, float dy, float dz, float r2,
                                               bool valid, const PairParams &p) {
    const bool in = valid && (r2 < p.rc2);
    const float rc = rcp_fast(r2);
    const float ir2 = in ? rc : 0.0f;
    const float s2 = p.sig2 * ir2;
    const float s6 = s2 * s2 * s2;
    const float t = s6 * fmaf(2.0f, s6, -1.0f);        // s6*(2 s6 - 1) = fr*r2 / (24 eps)
    const float g = t * ir2;
    acc.fx = fmaf(g, dx, acc.fx);
    acc.fy = fmaf(g, dy, acc.fy);
    acc.fz = fmaf(g, dz, acc.fz);
    if (THERMO) {
        acc.u = fmaf(s6, s6 - 1.0f, acc.u);            // (s12 - s6)
        acc.w += t;
        acc.cnt += in ? 1 : 0;
    }
}

// Pair-row variant: `flag` is the entry's ownership bit for this particle; the
// masked reciprocal is one LOP3 (bit -> predicate), one FSETP.LT.AND and one FSEL.
__device__ __forceinline__ float masked_rcp(float r2, float rc2, int e, int bit) {
    float out;
    const float rc = rcp_fast(r2);
    asm("{\n\t.reg .pred p, q;\n\t.reg .b32 t;\n\t"
        "and.b32 t, %3, %4;\n\t"
        "setp.ne.u32 q, t, 0;\n\t"
        "setp.lt.and.f32 p, %1, %2, q;\n\t"
        "selp.f32 %0, %5, 0f00000000, p;\n\t}"
        : "=f"(out) : "f"(r2), "f"(rc2), "r"(e), "r"(bit), "f"(rc));
    return out;
}

template <bool THERMO>
__device__ __forceinline__ void lj_pair_table(RowAcc &acc, float dx, float dy, float dz, float r2,
                                              bool valid, const float4 pa, const float2 pb) {
    const bool in = valid && (r2 < pa.y);
    const float rc = rcp_fast(r2);
    const float ir2 = in ? rc : 0.0f;
    const float s2 = pa.x * ir2;
    const float s6 = s2 * s2 * s2;
    const float t = s6 * fmaf(2.0f, s6, -1.0f);
    const float g = pa.z * t * ir2;
    acc.fx = fmaf(g, dx, acc.fx);
    acc.fy = fmaf(g, dy, acc.fy);
    acc.fz = fmaf(g, dz, acc.fz);
    if (THERMO) {
        acc.u = fmaf(pa.w * s6, s6 - 1.0f, acc.u);
        acc.u += in ? pb.x : 0.0f;
        acc.w = fmaf(pb.y, t, acc.w);
    }
}

// SUB lanes cooperate on one particle ("subwarp per particle"): lane `sub` owns
// entries k = sub, sub+SUB, sub+2*SUB, ... of the row and the partial sums are
// combined with shuffles at the end.  A warp therefore covers 32/SUB consecutive
// particles and, per load instruction, SUB consecutive entries of each of them --
// a much tighter set of cache lines for the position gathers than 32 different
// particles' k-th entries (L1 wavefronts per gather were the limiter at SUB = 1).
//
// Four entries per lane per trip.  The index stream comes from HBM (it is the
// bulk of the kernel's traffic), so it is software-pipelined two trips ahead:
// while trip t does its four position gathers and the arithmetic, the indices of
// trips t+1 and t+2 are already in flight.  CHECK = false is used for the leading
// trips in which every lane still has valid entries.
// The 16-byte neighbour-position gathers go through LDG (ld.global.nc).  The LSU data pipe
// of L1 (about one 128-byte wavefront per cycle per SM) is the limiter of this kernel: a
// gather of 32 scattered float4 costs ~11 wavefronts.  (Routing half of them through the TEX
// pipe of the same cache was measured in round 1 and did not pay; the texture path and its
// process-wide object cache are gone.)
// A coherent 16-byte load (ld.global, L1-cacheable but inside the memory model): what the
// persistent step kernel gathers with -- its positions are rewritten by other blocks of the
// same launch, so the read-only path of __ldg is off limits there.
__device__ __forceinline__ float4 ld_coherent_f4(const float4 *p) {
    float4 v;
    asm volatile("ld.global.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p) : "memory");
    return v;
}

template <bool NC = true>
__device__ __forceinline__ void gather4(float4 (&pj)[4], const int (&j)[4], const float4 *pos) {
#pragma unroll
    for (int u = 0; u < 4; ++u) pj[u] = NC ? __ldg(pos + j[u]) : ld_coherent_f4(pos + j[u]);
}

// AXES: bit a set = pairs of this warp may need an image shift along axis a.
template <int SUB, int AXES, bool TABLE, bool THERMO, bool CHECK>
__device__ __forceinline__ void compute4(RowAcc &acc, const float4 pi, int cnt, int k,
                                         const float4 (&pj)[4], const ForceArgs &a,
                                         const float4 *s_tab_a, const float2 *s_tab_b,
                                         int ti_row) {
    const BoxF &b = a.box;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const float dx = delta<(AXES & 1) != 0>(pi.x, pj[u].x, b.L_hi[0], b.L_lo[0], b.invL[0]);
        const float dy = delta<(AXES & 2) != 0>(pi.y, pj[u].y, b.L_hi[1], b.L_lo[1], b.invL[1]);
        const float dz = delta<(AXES & 4) != 0>(pi.z, pj[u].z, b.L_hi[2], b.L_lo[2], b.invL[2]);
        const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
        const bool valid = CHECK ? (k + u * SUB) < cnt : true;
        if (TABLE) {
            const int t = ti_row + __float_as_int(pj[u].w);
            lj_pair_table<THERMO>(acc, dx, dy, dz, r2, valid, s_tab_a[t], s_tab_b[t]);
        } else {
            lj_pair_single<THERMO>(acc, dx, dy, dz, r2, valid, a.single);
        }
    }
}

// k0 = this lane's first entry (= sub); kmin / kmax = smallest / largest row
// length among the particles of the warp.  Rows are allocated in multiples of 16
// and zero-filled, so reads past a row's end stay inside the allocation.
// PIPE = true additionally keeps the NEXT trip's four position gathers in flight
// while the current trip is being computed (deeper memory-level parallelism at
// the price of 16 more registers).
// The index entries of the first two trips of a row (what row_loop loads before its loop):
// the persistent kernel loads them once per launch instead of once per step.
template <int SUB>
__device__ __forceinline__ void row_first_indices(int (&ja)[4], int (&jb)[4], int kmax,
                                                  const int32_t *__restrict__ col, int64_t pitch) {
    constexpr int kTrip = 4 * SUB;
    const int64_t step = (int64_t)SUB * pitch;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        ja[u] = (0 < kmax) ? __ldcs(col + u * step) : 0;
        jb[u] = (kTrip < kmax) ? __ldcs(col + (4 + u) * step) : 0;
    }
}

template <int SUB, int PIPEK, int AXES, bool TABLE, bool THERMO, bool NC = true,
          bool PRELOADED = false>
__device__ __forceinline__ void row_loop(RowAcc &acc, const float4 pi, int cnt, int k0, int kmin,
                                         int kmax, const int32_t *__restrict__ col,
                                         int64_t pitch, const float4 *pos,
                                         const ForceArgs &a,
                                         const float4 *s_tab_a, const float2 *s_tab_b,
                                         int ti_row, const int *ja0 = nullptr,
                                         const int *jb0 = nullptr) {
    constexpr bool PIPE = (PIPEK == 1);
    constexpr int kTrip = 4 * SUB;            // entries of one particle consumed per trip
    const int64_t step = (int64_t)SUB * pitch;
    int ja[4], jb[4];
    if (PRELOADED) {
#pragma unroll
        for (int u = 0; u < 4; ++u) { ja[u] = ja0[u]; jb[u] = jb0[u]; }
    } else {
        row_first_indices<SUB>(ja, jb, kmax, col, pitch);
    }
    float4 pa[4], pb[4];
    if (PIPE) gather4<NC>(pa, ja, pos);
    for (int base = 0; base < kmax; base += kTrip) {
        int jc[4];
        const bool more = base + 2 * kTrip < kmax;          // warp-uniform
#pragma unroll
        for (int u = 0; u < 4; ++u) jc[u] = more ? __ldcs(col + (8 + u) * step) : 0;
        if (PIPE) gather4<NC>(pb, jb, pos);                  // row 0 is always a valid index
        else gather4<NC>(pa, ja, pos);
        if (base + kTrip <= kmin)
            compute4<SUB, AXES, TABLE, THERMO, false>(acc, pi, cnt, base + k0, pa, a, s_tab_a,
                                                         s_tab_b, ti_row);
        else
            compute4<SUB, AXES, TABLE, THERMO, true>(acc, pi, cnt, base + k0, pa, a, s_tab_a,
                                                        s_tab_b, ti_row);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            ja[u] = jb[u];
            jb[u] = jc[u];
            if (PIPE) pa[u] = pb[u];
        }
        col += 4 * step;
    }
}

// Rare path: find the first listed j at zero separation (forces.py:94-97).
__device__ __noinline__ void report_singular(int i, const float4 pi, int cnt,
                                             const int32_t *__restrict__ col, int64_t pitch,
                                             const float4 *__restrict__ pos, const BoxF &b,
                                             b2md_status *status) {
    for (int k = 0; k < cnt; ++k) {
        const int j = col[(int64_t)k * pitch];
        const float4 pj = pos[j];
        const float dx = delta<true>(pi.x, pj.x, b.L_hi[0], b.L_lo[0], b.invL[0]);
        const float dy = delta<true>(pi.y, pj.y, b.L_hi[1], b.L_lo[1], b.invL[1]);
        const float dz = delta<true>(pi.z, pj.z, b.L_hi[2], b.L_lo[2], b.invL[2]);
        if (fmaf(dz, dz, fmaf(dy, dy, dx * dx)) == 0.0f) {
            atomicMin((unsigned long long *)&status->singular,
                      ((unsigned long long)(unsigned)i << 32) | (unsigned)j);
            return;
        }
    }
}

// The same over a pair row (entries j << 2 | flags, int4 tiles, see k_pair_rows): the pair
// kernels never look at the plain rows -- the step loop's list build writes them only for
// pairs that straddle two cells (b2md_build_pair_list).  which = 0: particle 2t, 1: 2t+1.
__device__ __noinline__ void report_singular_pair(int i, int which, const float4 pi, int cnt,
                                                  const int4 *__restrict__ col,
                                                  int64_t pair_pitch,
                                                  const float4 *__restrict__ pos, const BoxF &b,
                                                  b2md_status *status) {
    for (int k = 0; k < cnt; ++k) {
        const int e = reinterpret_cast<const int *>(col + (int64_t)(k >> 2) * pair_pitch)[k & 3];
        if (!((e >> which) & 1)) continue;
        const int j = (int)((unsigned)e >> 2);
        const float4 pj = pos[j];
        const float dx = delta<true>(pi.x, pj.x, b.L_hi[0], b.L_lo[0], b.invL[0]);
        const float dy = delta<true>(pi.y, pj.y, b.L_hi[1], b.L_lo[1], b.invL[1]);
        const float dz = delta<true>(pi.z, pj.z, b.L_hi[2], b.L_lo[2], b.invL[2]);
        if (fmaf(dz, dz, fmaf(dy, dy, dx * dx)) == 0.0f) {
            atomicMin((unsigned long long *)&status->singular,
                      ((unsigned long long)(unsigned)i << 32) | (unsigned)j);
            return;
        }
    }
}

// ADVANCE (both list kernels): the kernel also applies what the step loop does between two force
// evaluations -- both half-kicks with the forces it has just computed, the drift, the
// wrap and the displacement check (= k_integrate<2>) -- so the intermediate steps of
// the native loop are ONE launch each and the forces never travel through HBM.
// Positions are read by other threads while this one moves on, hence the new high
// words go to a second buffer (pos_out) that the next launch reads; velocities, low
// words, images and the list snapshot are private to the thread and updated in place.
// The launch is gated on status word `gate_in` ("the positions I am about to use
// already need a new list": set by the previous launch, which wrote `gate_out` of its
// own) -- a launch enqueued speculatively then returns at once and the host rebuilds.
constexpr int kWordAdvanceCount = 13;      // b2md_status::reserved[1]: advance launches that ran

struct AdvanceArgs {
    float4 *pos_out, *pos_lo, *vel, *ref_pos;
    int4 *image;
    StepConst step;
    int gate_in, gate_out;        // int32 word indices into b2md_status
    // Slab decomposition, halo fused into the step kernel: a particle whose halo_dst[s][i]
    // is >= 0 also stores its advanced high words into row halo_dst[s][i] of halo_out[s] --
    // the ghost rows of a neighbour rank's position buffer, mapped into this process
    // (peer memory over NVLink).  Null = no halo on that side.
    const int32_t *halo_dst[2];
    float4 *halo_out[2];
    // Pruned ("inner") pair rows, b2md_force_lj_pairs_advance_pruned: prune_mode 0 = none,
    // kPruneInner = walk the inner rows, kPruneNow = walk the outer rows and write the inner ones
    // (entries with r < r_cut + delta, the prune snapshot into ref_pos.w), kPruneOuter = walk the
    // outer rows but keep publishing the inner flags.  Flag bits of the gate words: 1 = the
    // positions need a new list, 2 = the inner rows have expired for them (some particle moved
    // more than delta / 2 since the prune), 4 = a prune is no longer legal for them (some
    // particle is further than (skin - delta) / 2 from the list snapshot, so the outer rows are
    // not complete to r_cut + delta any more).  gate_clear: the third word of the rotation,
    // zeroed by this launch for the next one to write.
    int prune_mode, gate_clear;
    int4 *inner_nbr;
    int32_t *inner_counts;
    float inner_rl2, inner_half2, prune_limit2;
    int inner_tiles;
};
constexpr int kPruneInner = 1, kPruneNow = 2, kPruneOuter = 3;
constexpr int kWordInnerDisp = 15;         // b2md_status::reserved[3]: max inner displacement^2

// Gate of an ADVANCE launch (see AdvanceArgs): true = this launch must not run.
__device__ __forceinline__ bool advance_gate_closed(b2md_status *status, const AdvanceArgs &adv) {
    // a launch that must not run hands the flag on, so that launches queued behind it
    // do not run either; one that runs counts itself (the host may have several queued)
    const int w = ((volatile int *)status)[adv.gate_in];
    if (adv.prune_mode) {
        // three gate words in rotation (flag bits do not clear themselves as the rebuild flag
        // does): nobody reads or writes gate_clear during this launch
        if (blockIdx.x == 0 && threadIdx.x == 0) ((int *)status)[adv.gate_clear] = 0;
        const bool closed = (w & 1) || (adv.prune_mode == kPruneInner && (w & 2)) ||
                            (adv.prune_mode == kPruneNow && (w & 4));
        if (closed) {
            if (blockIdx.x == 0 && threadIdx.x == 0) ((int *)status)[adv.gate_out] = w;
            return true;
        }
    } else if (w) {
        if (blockIdx.x == 0 && threadIdx.x == 0) ((int *)status)[adv.gate_out] = 1;
        return true;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&((int *)status)[kWordAdvanceCount], 1);
    return false;
}

// Displacement maximum of the block -> status (as k_integrate does); all threads call it.
template <int THREADS = kForceThreads>
__device__ __forceinline__ void advance_publish_disp(float d2, float *s_max, b2md_status *status,
                                                     const AdvanceArgs &adv) {
    d2 = warp_max(d2);
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = d2;
    __syncthreads();
    if (threadIdx.x < 32) {
        float m = threadIdx.x < THREADS / 32 ? s_max[threadIdx.x] : 0.0f;
        m = warp_max(m);
        if (threadIdx.x == 0 && m > 0.0f) {
            atomicMax(&status->max_disp2_bits, __float_as_uint(m));
            if (adv.prune_mode) {
                const int bits = (m > adv.step.half_skin2 ? 1 : 0) | (m > adv.prune_limit2 ? 4 : 0);
                if (bits) atomicOr(&((int *)status)[adv.gate_out], bits);
            } else if (m > adv.step.half_skin2) {
                ((int *)status)[adv.gate_out] = 1;
            }
        }
    }
}

// The same for the displacement since the last prune (flag bit 2 of the gate word).
template <int THREADS>
__device__ __forceinline__ void advance_publish_inner(float d2, float *s_max, b2md_status *status,
                                                      const AdvanceArgs &adv) {
    d2 = warp_max(d2);
    __syncthreads();                       // s_max is reused
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = d2;
    __syncthreads();
    if (threadIdx.x < 32) {
        float m = threadIdx.x < THREADS / 32 ? s_max[threadIdx.x] : 0.0f;
        m = warp_max(m);
        if (threadIdx.x == 0 && m > 0.0f) {
            atomicMax(&((unsigned *)status)[kWordInnerDisp], __float_as_uint(m));
            if (m > adv.inner_half2) atomicOr(&((int *)status)[adv.gate_out], 2);
        }
    }
}

// PIPE doubles as the occupancy knob of the experiments: 0 = 8 CTAs/SM (<= 64
// registers), 1 = gathers one trip ahead with 6 CTAs/SM, 2 = 12 CTAs/SM (<= 40).
template <int SUB, int PIPE, bool TABLE, bool THERMO, bool ADVANCE = false>
__global__ void __launch_bounds__(kForceThreads, PIPE == 1 ? 6 : (PIPE == 2 ? 12 : 8))
k_force_lj(const float4 *__restrict__ pos, int64_t n,
           const __grid_constant__ ForceArgs a,
           const int32_t *__restrict__ nbr, const int32_t *__restrict__ counts, int64_t pitch,
           const uint8_t *__restrict__ boundary, float4 *__restrict__ force,
           float *__restrict__ virial, b2md_status *status, int gated,
           const __grid_constant__ AdvanceArgs adv) {
    __shared__ float4 s_tab_a[TABLE ? kMaxTypes * kMaxTypes : 1];
    __shared__ float2 s_tab_b[TABLE ? kMaxTypes * kMaxTypes : 1];
    __shared__ float s_max[kForceThreads / 32];
    // step-graph batches: nothing to do once an in-graph list build overflowed
    if (gated && *(volatile int *)&status->frozen) return;
    if (ADVANCE && advance_gate_closed(status, adv)) return;
    if (TABLE) {
        for (int t = threadIdx.x; t < a.ntypes * a.ntypes; t += blockDim.x) {
            s_tab_a[t] = a.tab_a[t];
            s_tab_b[t] = a.tab_b[t];
        }
        __syncthreads();
    }
    constexpr int kPerBlock = kForceThreads / SUB;
    const int sub = threadIdx.x % SUB;
    const int64_t i_raw = blockIdx.x * (int64_t)kPerBlock + threadIdx.x / SUB;
    const bool active = i_raw < n;
    const int64_t i = active ? i_raw : n - 1;
    const float4 pi = pos[i];
    const int cnt = active ? counts[i] : 0;
    const int kmax = __reduce_max_sync(0xffffffffu, cnt);
    const int kmin = __reduce_min_sync(0xffffffffu, active ? cnt : 0x7fffffff);
    // which axes can need an image shift for some pair of this warp (0 = interior warp)
    const int axes = boundary ? (__reduce_or_sync(0xffffffffu, active ? (int)boundary[i] : 0) & 7) : 7;
    const int32_t *col = nbr + (int64_t)sub * pitch + i;
    const int ti_row = TABLE ? __float_as_int(pi.w) * a.ntypes : 0;

    RowAcc acc = {0.f, 0.f, 0.f, 0.f, 0.f, 0};
#define B2MD_ROW_LOOP(AXES)                                                                  \
    row_loop<SUB, PIPE, AXES, TABLE, THERMO>(acc, pi, cnt, sub, kmin, kmax, col, pitch, pos, a,  \
                                             s_tab_a, s_tab_b, ti_row)
    switch (axes) {                 // warp-uniform
        case 0: B2MD_ROW_LOOP(0); break;      // interior: plain differences
        case 1: B2MD_ROW_LOOP(1); break;      // one face family only
        case 2: B2MD_ROW_LOOP(2); break;
        case 4: B2MD_ROW_LOOP(4); break;
        default: B2MD_ROW_LOOP(7); break;     // edges / corners / tiny boxes
    }
#undef B2MD_ROW_LOOP
#pragma unroll
    for (int o = SUB >> 1; o > 0; o >>= 1) {
        acc.fx += __shfl_xor_sync(0xffffffffu, acc.fx, o);
        acc.fy += __shfl_xor_sync(0xffffffffu, acc.fy, o);
        acc.fz += __shfl_xor_sync(0xffffffffu, acc.fz, o);
        if (THERMO) {
            acc.u += __shfl_xor_sync(0xffffffffu, acc.u, o);
            acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
            acc.cnt += __shfl_xor_sync(0xffffffffu, acc.cnt, o);
        }
    }
    float d2 = 0.0f;
    if (active && sub == 0) {
        float fx, fy, fz, u, w;
        if (TABLE) {
            fx = acc.fx; fy = acc.fy; fz = acc.fz; u = acc.u; w = acc.w;
        } else {
            const PairParams &p = a.single;
            fx = p.c_f * acc.fx; fy = p.c_f * acc.fy; fz = p.c_f * acc.fz;
            u = fmaf(p.c_u, acc.u, p.half_shift * (float)acc.cnt);
            w = p.c_w * acc.w;
        }
        if (ADVANCE) {
            float4 h = pi;
            d2 = advance_particle<2>(i, h, make_float4(fx, fy, fz, u), adv.pos_lo, adv.vel,
                                     adv.image, adv.step, adv.ref_pos);
            adv.pos_out[i] = h;
        } else {
            force[i] = make_float4(fx, fy, fz, u);
            if (THERMO && virial) virial[i] = w;
        }
        if (!(isfinite(fx) && isfinite(fy) && isfinite(fz)))
            report_singular((int)i, pi, cnt, nbr + i, pitch, pos, a.box, status);
    }
    if (ADVANCE) advance_publish_disp(d2, s_max, status, adv);
}

// ---- persistent step kernel (small systems) -------------------------------------
// Below ~10^5 particles an MD step is shorter than what a launch plus a host round trip
// costs (17 us per step at N = 4096 with one gated launch per step).  Here ONE cooperative
// launch runs up to n_steps steps: every step is the body of k_force_lj<SUB, ADVANCE> --
// force, both half-kicks, drift, wrap, displacement check -- followed by a grid-wide barrier;
// the position high words ping-pong between two buffers, everything else a thread updates
// is private to its particle.  The loop ends early when the positions it is about to use
// need a new list (the flag word of those positions, exactly as the gated launches hand it
// on); the device counts the steps it took, the host reads count and flags once.
//
// Memory model: positions written by other blocks are gathered with plain ld.global (never
// the read-only path); the barrier is a release (fence + atomic add) / acquire (fence after
// the spin) pair at gpu scope, which also drops stale L1 lines of the executing SM.
// A barrier that does not complete within kBarrierTimeout clocks (it cannot, unless the grid
// is not co-resident -- the launch is cooperative -- or a block died) sets status->frozen and
// lets every block leave: a bug here must not hang the device.
struct PersistArgs {
    float4 *pos[2];           // step s reads pos[s & 1], writes pos[(s & 1) ^ 1]
    int gate[2];              // status word holding the rebuild flag of pos[0] / pos[1]
    int n_steps;
    unsigned long long *barrier;   // B2MD_BARRIER_BYTES, zeroed before the launch: per counter,
};                                 // arrivals in the low word, flagged arrivals in the high word

constexpr long long kBarrierTimeout = 4000000000ll;      // ~2 s at 1.97 GHz
#ifndef B2MD_PERSIST_THREADS
#define B2MD_PERSIST_THREADS 256
#endif
// threads per block of the persistent kernel: the grid barrier costs one atomic and one
// polling thread per BLOCK, so fewer, larger blocks make it cheaper (128 ... 512 measured
// within 10 % of each other, 1024 slower)
constexpr int kPersistThreads = B2MD_PERSIST_THREADS;

// Grid-wide barrier; thread 0 of every block arrives with `flagged` (this block saw a
// displacement beyond the threshold).  Returns -1 if the barrier timed out, else how many
// arrivals carried a flag so far -- the rebuild decision travels with the barrier, no second
// round trip.  The counter only grows: step s waits for (s + 1) x gridDim.x arrivals.  (A
// two-level version -- 16 group counters on their own cache lines, last arrival of a group
// arrives on the top counter -- was measured slower, 10.3 against 9.4 us per step at N = 4096:
// the extra dependent atomic costs more than 256 same-address atomics.)
__device__ __forceinline__ int grid_barrier(unsigned long long *counter, unsigned step,
                                            bool flagged, b2md_status *status) {
    __shared__ int s_flags;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();                                   // release: my block's stores
        atomicAdd(counter, 1ull | (flagged ? (1ull << 32) : 0ull));
        const unsigned target = gridDim.x * (step + 1u);
        const long long t0 = clock64();
        unsigned long long v;
        int out = 0;
        while ((unsigned)(v = *(volatile unsigned long long *)counter) < target) {
            if (clock64() - t0 > kBarrierTimeout || *(volatile int *)&status->frozen) {
                status->frozen = 1;
                out = -1;
                break;
            }
        }
        if (out == 0) out = (int)(v >> 32);
        __threadfence();                                   // acquire: everybody else's stores
        s_flags = out;
    }
    __syncthreads();
    return s_flags;
}

template <int SUB, bool TABLE>
__global__ void __launch_bounds__(kPersistThreads, 1024 / kPersistThreads)
k_steps_persistent(int64_t n, const __grid_constant__ ForceArgs a,
                   const int32_t *__restrict__ nbr, const int32_t *__restrict__ counts,
                   int64_t pitch, const uint8_t *__restrict__ boundary, b2md_status *status,
                   const __grid_constant__ AdvanceArgs adv, const __grid_constant__ PersistArgs ps) {
    __shared__ float4 s_tab_a[TABLE ? kMaxTypes * kMaxTypes : 1];
    __shared__ float2 s_tab_b[TABLE ? kMaxTypes * kMaxTypes : 1];
    __shared__ float s_max[kPersistThreads / 32];
    if (TABLE) {
        for (int t = threadIdx.x; t < a.ntypes * a.ntypes; t += blockDim.x) {
            s_tab_a[t] = a.tab_a[t];
            s_tab_b[t] = a.tab_b[t];
        }
        __syncthreads();
    }
    // grid-uniform: the flag of the initial positions was written by an earlier launch
    if (((volatile int *)status)[ps.gate[0]]) return;
    constexpr int kPerBlock = kPersistThreads / SUB;
    const int sub = threadIdx.x % SUB;
    const int64_t i_raw = blockIdx.x * (int64_t)kPerBlock + threadIdx.x / SUB;
    const bool active = i_raw < n;
    const int64_t i = active ? i_raw : n - 1;
    const bool owner = active && sub == 0;
    // what does not change during the launch stays in registers: the list (row length, the
    // index entries of the first two trips), and -- in the particle's owner lane -- the state
    // no other thread touches: low words, velocity, snapshot, the high words just written
    const int cnt = active ? counts[i] : 0;
    const int kmax = __reduce_max_sync(0xffffffffu, cnt);
    const int kmin = __reduce_min_sync(0xffffffffu, active ? cnt : 0x7fffffff);
    const int axes = boundary ? (__reduce_or_sync(0xffffffffu, active ? (int)boundary[i] : 0) & 7) : 7;
    const int32_t *col = nbr + (int64_t)sub * pitch + i;
    int ja0[4], jb0[4];
    row_first_indices<SUB>(ja0, jb0, kmax, col, pitch);
    float4 h = ld_coherent_f4(ps.pos[0] + i);
    float4 l = owner ? adv.pos_lo[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 v = owner ? adv.vel[i] : make_float4(0.f, 0.f, 0.f, 1.f);
    float4 r = owner ? adv.ref_pos[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    const int ti_row = TABLE ? __float_as_int(h.w) * a.ntypes : 0;

    int s = 0;
    for (; s < ps.n_steps; ++s) {
        const int w_out = ps.gate[(s & 1) ^ 1];
        const float4 *pos = ps.pos[s & 1];
        float4 *pos_out = ps.pos[(s & 1) ^ 1];
        // the particle's own position: from its owner lane
        float4 pi = h;
        if (SUB > 1) {
            const int src = (threadIdx.x & 31) & ~(SUB - 1);
            pi.x = __shfl_sync(0xffffffffu, h.x, src);
            pi.y = __shfl_sync(0xffffffffu, h.y, src);
            pi.z = __shfl_sync(0xffffffffu, h.z, src);
        }
        RowAcc acc = {0.f, 0.f, 0.f, 0.f, 0.f, 0};
#define B2MD_ROW_LOOP(AXES)                                                                     \
    row_loop<SUB, 0, AXES, TABLE, false, false, true>(acc, pi, cnt, sub, kmin, kmax, col, pitch, \
                                                      pos, a, s_tab_a, s_tab_b, ti_row, ja0, jb0)
        switch (axes) {                 // warp-uniform
            case 0: B2MD_ROW_LOOP(0); break;
            case 1: B2MD_ROW_LOOP(1); break;
            case 2: B2MD_ROW_LOOP(2); break;
            case 4: B2MD_ROW_LOOP(4); break;
            default: B2MD_ROW_LOOP(7); break;
        }
#undef B2MD_ROW_LOOP
#pragma unroll
        for (int o = SUB >> 1; o > 0; o >>= 1) {
            acc.fx += __shfl_xor_sync(0xffffffffu, acc.fx, o);
            acc.fy += __shfl_xor_sync(0xffffffffu, acc.fy, o);
            acc.fz += __shfl_xor_sync(0xffffffffu, acc.fz, o);
        }
        float d2 = 0.0f;
        if (owner) {
            float fx, fy, fz;
            if (TABLE) {
                fx = acc.fx; fy = acc.fy; fz = acc.fz;
            } else {
                const PairParams &p = a.single;
                fx = p.c_f * acc.fx; fy = p.c_f * acc.fy; fz = p.c_f * acc.fz;
            }
            const float4 before = h;
            d2 = advance_regs<2>(i, h, l, v, r, true, make_float4(fx, fy, fz, 0.0f), adv.image,
                                 adv.step);
            pos_out[i] = h;
            if (!(isfinite(fx) && isfinite(fy) && isfinite(fz)))
                report_singular((int)i, before, cnt, nbr + i, pitch, pos, a.box, status);
        }
        // displacement maximum of the block -> status; the flag of the new positions
        d2 = warp_max(d2);
        if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = d2;
        __syncthreads();
        bool flagged = false;
        if (threadIdx.x < 32) {
            float m = threadIdx.x < kPersistThreads / 32 ? s_max[threadIdx.x] : 0.0f;
            m = warp_max(m);
            if (threadIdx.x == 0 && m > 0.0f) {
                atomicMax(&status->max_disp2_bits, __float_as_uint(m));
                if (m > adv.step.half_skin2) {
                    ((int *)status)[w_out] = 1;
                    flagged = true;
                }
            }
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&((int *)status)[kWordAdvanceCount], 1);
        const int flags = grid_barrier(ps.barrier, (unsigned)s, flagged, status);
        if (flags != 0) break;           // the new positions need a list (or the barrier failed)
    }
    if (owner) {                         // the state this launch kept in registers
        adv.pos_lo[i] = l;
        adv.vel[i] = v;
        adv.ref_pos[i] = r;
    }
}

// ---- pair rows: two particles per thread -------------------------------------
// Thread t owns particles 2t and 2t+1 and walks their merged row (k_pair_rows in
// nlist.cu: ascending j, entry = j << 2 | listed-for-2t | listed-for-2t+1 << 1,
// int4 tiles).  r_j is gathered once and evaluated against both particles; an
// entry that only one of them lists contributes exact zeros to the other, so each
// particle's sums are bit-identical to the one-row kernel's (same ascending-j
// order, same fp32 sequence).  Compared with one thread per particle this needs
// about a third fewer 16-byte gathers and index bytes per particle -- the L1 data
// pipe, not HBM or issue, limits the one-row kernel -- and one 16-byte index load
// per four entries instead of four 4-byte ones.

// ---- packed fp32x2 arithmetic (FADD2 / FMUL2 / FFMA2) -------------------------
// One-species pairs: the two particles of a thread go through identical
// instruction sequences against the same r_j, so they ride in the two halves of
// sm_100's packed fp32 instructions -- half the issue slots for the same
// per-lane IEEE operations (round-to-nearest, no contraction beyond the fmas the
// scalar code has), hence the same bits as the scalar kernels.  A scalar operand
// packed with itself is encoded by ptxas as a broadcast, not a move.
typedef unsigned long long f32x2;

__device__ __forceinline__ f32x2 pk(float lo, float hi) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ f32x2 pk1(float v) { return pk(v, v); }
__device__ __forceinline__ void upk(f32x2 v, float &lo, float &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// delta<CAREFUL> for both particles of a pair against one x_j
template <bool CAREFUL>
__device__ __forceinline__ f32x2 delta2(f32x2 xi, float xj, float L_hi, float L_lo, float invL) {
    const f32x2 d0 = sub2(xi, pk1(xj));
    if (!CAREFUL) return d0;
    const float magic = 12582912.0f;  // 1.5 * 2^23 (rint_small)
    const f32x2 ns = sub2(add2(mul2(d0, pk1(invL)), pk1(magic)), pk1(magic));
    float n0, n1;
    upk(ns, n0, n1);
    // fmaf(-m, L, x) == fmaf(m, -L, x): the negation moves onto the constant
    const f32x2 sa = fma2(pk(fmaxf(n0, 0.0f), fmaxf(n1, 0.0f)), pk1(-L_hi), xi);
    const f32x2 sb = fma2(pk(fmaxf(-n0, 0.0f), fmaxf(-n1, 0.0f)), pk1(-L_hi), pk1(xj));
    return fma2(ns, pk1(-L_lo), sub2(sa, sb));
}

// ---- image shifts in the frame centred on the periodic face ---------------------
// delta2<true> derives the image number of every pair from its raw difference (rint via the
// magic constant, two max pairs, three fmas per half and axis: +22 issue slots per axis and
// entry; 14 % of the step kernel's time at N = 1 M, where 16 % of the particles sit in
// flagged warps).  When every particle of the warp lies in the outer quarters of the box
// along a flagged axis (x < L/4 or x > 3L/4; warp-uniform test, always true for a Hilbert-
// ordered fluid in a box wider than 4 (r_list + skin)), the image number of a listed pair is
// simply s_i - s_j with s = [x > L/2]: map every coordinate above L/2 down by L_hi (exact,
// Sterbenz) and correct by (s_j - s_i) L_lo.  One compare, two selects and one add on the
// scalar x_j, two packed operations more than the plain difference -- and the same bits as
// delta2<true>: same shifted operands a, b, same image number, same single rounding of
// (a - b) - n L_lo; for s_i = s_j the correction is an exact zero and the difference of the
// two exactly shifted coordinates is the difference of the unshifted ones.
__device__ __forceinline__ void face_frame(f32x2 &x2, f32x2 &corr2, float L_hi, float L_lo,
                                           float half) {
    float x0, x1;
    upk(x2, x0, x1);
    const bool s0 = x0 > half, s1 = x1 > half;
    x2 = pk(s0 ? x0 - L_hi : x0, s1 ? x1 - L_hi : x1);
    corr2 = pk(s0 ? L_lo : 0.0f, s1 ? L_lo : 0.0f);
}

// MODE 0: plain difference, 1: delta2<true>, 2: face frame (xi already mapped, corr_i = s_i L_lo)
template <int MODE>
__device__ __forceinline__ f32x2 delta2m(f32x2 xi, f32x2 corr_i, float xj, float L_hi, float L_lo,
                                         float invL, float half) {
    if (MODE == 0) return sub2(xi, pk1(xj));
    if (MODE == 1) return delta2<true>(xi, xj, L_hi, L_lo, invL);
    const bool sj = xj > half;
    const float xjm = sj ? xj - L_hi : xj;
    const float corr_j = sj ? L_lo : 0.0f;
    return add2(sub2(xi, pk1(xjm)), sub2(pk1(corr_j), corr_i));
}

// AXES: bits 0-2 = axes on delta2<true>, bits 3-5 = axes in the face frame
template <int AXES, int AXIS>
struct AxisMode { static constexpr int value = (AXES >> AXIS) & 1 ? 1 : ((AXES >> (3 + AXIS)) & 1 ? 2 : 0); };

struct PackAcc {
    f32x2 fx, fy, fz, u, w;   // halves: particle 2t, particle 2t+1
    int cnt_a, cnt_b;
};

// PRUNE launches (AdvanceArgs::prune_mode == kPruneNow) also write the "inner" pair row: the
// entries either particle of the pair still has inside r_cut + delta, ownership flags narrowed
// to the particles that do, in the same (ascending) order and the same int4 tile layout.
struct PruneOut {
    int o0, o1, o2, o3, cnt, cap;
    unsigned oq, pitch;             // element offset of the tile being filled; tiles are pitch apart
    int4 *ocol;
    float rl2;
};
// Branch-free (the lanes of a warp keep different entries; 80 % are kept): four selects shift
// the entry in, one predicated 16-byte store per fourth kept entry.
__device__ __forceinline__ void prune_keep(PruneOut &P, int e, float r2a, float r2b) {
    const bool ka = (e & 1) && r2a < P.rl2, kb = (e & 2) && r2b < P.rl2;
    const bool keep = ka || kb;
    const int ne = (e & ~3) | (ka ? 1 : 0) | (kb ? 2 : 0);
    P.o0 = keep ? P.o1 : P.o0;
    P.o1 = keep ? P.o2 : P.o1;
    P.o2 = keep ? P.o3 : P.o2;
    P.o3 = keep ? ne : P.o3;
    P.cnt += keep ? 1 : 0;
    const bool st = keep && (P.cnt & 3) == 0;
    if (st && P.cnt <= P.cap) P.ocol[P.oq] = make_int4(P.o0, P.o1, P.o2, P.o3);
    P.oq += st ? P.pitch : 0u;
}

// SIG1: sigma^2 == 1.0f, so s2 = sigma^2 * ir2 is ir2 itself (x * 1.0f is exact: same bits,
// one packed multiply less on the FMA pipe that bounds this kernel).
template <int AXES, bool THERMO, bool SIG1, bool PRUNE = false>
__device__ __forceinline__ void pair_entry_packed(PackAcc &acc, f32x2 ax, f32x2 ay, f32x2 az,
                                                  f32x2 cx, f32x2 cy, f32x2 cz,
                                                  int e, const float4 pj, const ForceArgs &a,
                                                  PruneOut *P = nullptr) {
    const BoxF &b = a.box;
    const PairParams &p = a.single;
    const f32x2 dx = delta2m<AxisMode<AXES, 0>::value>(ax, cx, pj.x, b.L_hi[0], b.L_lo[0], b.invL[0], b.half[0]);
    const f32x2 dy = delta2m<AxisMode<AXES, 1>::value>(ay, cy, pj.y, b.L_hi[1], b.L_lo[1], b.invL[1], b.half[1]);
    const f32x2 dz = delta2m<AxisMode<AXES, 2>::value>(az, cz, pj.z, b.L_hi[2], b.L_lo[2], b.invL[2], b.half[2]);
    const f32x2 r2 = fma2(dz, dz, fma2(dy, dy, mul2(dx, dx)));
    float r2a, r2b;
    upk(r2, r2a, r2b);
    if (PRUNE) prune_keep(*P, e, r2a, r2b);
    const float ia = masked_rcp(r2a, p.rc2, e, 1), ib = masked_rcp(r2b, p.rc2, e, 2);
    const f32x2 ir2 = pk(ia, ib);
    const f32x2 s2 = SIG1 ? ir2 : mul2(pk1(p.sig2), ir2);
    const f32x2 s6 = mul2(mul2(s2, s2), s2);
    const f32x2 t = mul2(s6, fma2(pk1(2.0f), s6, pk1(-1.0f)));
    const f32x2 g = mul2(t, ir2);
    acc.fx = fma2(g, dx, acc.fx);
    acc.fy = fma2(g, dy, acc.fy);
    acc.fz = fma2(g, dz, acc.fz);
    if (THERMO) {
        acc.u = fma2(s6, add2(s6, pk1(-1.0f)), acc.u);
        acc.w = add2(acc.w, t);
        acc.cnt_a += ia != 0.0f ? 1 : 0;
        acc.cnt_b += ib != 0.0f ? 1 : 0;
    }
}

// Per-pair-type tables (Kob-Andersen ...): the same packed evaluation with the
// parameters of (type of 2t, type of j) and (type of 2t+1, type of j) in the two
// halves.  Operation order per half is lj_pair_table's, so the sums stay bit-identical
// to the row kernel's.
template <int AXES, bool THERMO, bool PRUNE = false>
__device__ __forceinline__ void pair_entry_packed_table(PackAcc &acc, f32x2 ax, f32x2 ay,
                                                        f32x2 az, f32x2 cx, f32x2 cy, f32x2 cz,
                                                        int e, const float4 pj,
                                                        const ForceArgs &a,
                                                        const float4 *s_tab_a,
                                                        const float2 *s_tab_b, int ta_row,
                                                        int tb_row, PruneOut *P = nullptr) {
    const BoxF &b = a.box;
    const int tj = __float_as_int(pj.w);
    const float4 qa = s_tab_a[ta_row + tj], qb = s_tab_a[tb_row + tj];
    const f32x2 dx = delta2m<AxisMode<AXES, 0>::value>(ax, cx, pj.x, b.L_hi[0], b.L_lo[0], b.invL[0], b.half[0]);
    const f32x2 dy = delta2m<AxisMode<AXES, 1>::value>(ay, cy, pj.y, b.L_hi[1], b.L_lo[1], b.invL[1], b.half[1]);
    const f32x2 dz = delta2m<AxisMode<AXES, 2>::value>(az, cz, pj.z, b.L_hi[2], b.L_lo[2], b.invL[2], b.half[2]);
    const f32x2 r2 = fma2(dz, dz, fma2(dy, dy, mul2(dx, dx)));
    float r2a, r2b;
    upk(r2, r2a, r2b);
    if (PRUNE) prune_keep(*P, e, r2a, r2b);
    const float ia = masked_rcp(r2a, qa.y, e, 1), ib = masked_rcp(r2b, qb.y, e, 2);
    const f32x2 ir2 = pk(ia, ib);
    const f32x2 s2 = mul2(pk(qa.x, qb.x), ir2);
    const f32x2 s6 = mul2(mul2(s2, s2), s2);
    const f32x2 t = mul2(s6, fma2(pk1(2.0f), s6, pk1(-1.0f)));
    const f32x2 g = mul2(mul2(pk(qa.z, qb.z), t), ir2);
    acc.fx = fma2(g, dx, acc.fx);
    acc.fy = fma2(g, dy, acc.fy);
    acc.fz = fma2(g, dz, acc.fz);
    if (THERMO) {
        const float2 wa = s_tab_b[ta_row + tj], wb = s_tab_b[tb_row + tj];
        acc.u = fma2(mul2(pk(qa.w, qb.w), s6), add2(s6, pk1(-1.0f)), acc.u);
        acc.u = add2(acc.u, pk(ia != 0.0f ? wa.x : 0.0f, ib != 0.0f ? wb.x : 0.0f));
        acc.w = fma2(pk(wa.y, wb.y), t, acc.w);
    }
}


#ifndef B2MD_PAIR_TILE_ROTATE
#define B2MD_PAIR_TILE_ROTATE 0
#endif
#ifndef B2MD_PAIR_HALF_TILE
#define B2MD_PAIR_HALF_TILE 0
#endif

// `tiles` = longest row of the warp in int4 tiles (rows are padded that far with
// flag-less entries); the index tiles of the next two trips are kept in flight.
template <int AXES, bool TABLE, bool THERMO, bool SIG1, bool PRUNE = false>
__device__ __forceinline__ void pair_row_loop(RowAcc &A, RowAcc &B, const float4 pa,
                                              const float4 pb, int tiles,
                                              const int4 *__restrict__ col, int64_t pair_pitch,
                                              const float4 *__restrict__ pos, const ForceArgs &a,
                                              const float4 *s_tab_a, const float2 *s_tab_b,
                                              int ta_row, int tb_row, PruneOut *P = nullptr) {
    // The loop body is kept to one trip: unrolling it further (to rotate the tile
    // registers without moves) made instruction fetch the limiter -- 30 % of the
    // stall samples were "no instruction".
    int4 e0 = make_int4(0, 0, 0, 0), e1 = e0;
    if (tiles > 0) e0 = __ldcs(col);
    if (tiles > 1) e1 = __ldcs(col + pair_pitch);
    col += 2 * pair_pitch;
    PackAcc acc = {0ull, 0ull, 0ull, 0ull, 0ull, 0, 0};     // +0.0f in both halves
    f32x2 ax = pk(pa.x, pb.x), ay = pk(pa.y, pb.y), az = pk(pa.z, pb.z);
    f32x2 cx = 0ull, cy = 0ull, cz = 0ull;
    if (AXES & 8) face_frame(ax, cx, a.box.L_hi[0], a.box.L_lo[0], a.box.half[0]);
    if (AXES & 16) face_frame(ay, cy, a.box.L_hi[1], a.box.L_lo[1], a.box.half[1]);
    if (AXES & 32) face_frame(az, cz, a.box.L_hi[2], a.box.L_lo[2], a.box.half[2]);
#pragma unroll 1
    for (int q = 0; q < tiles; ++q) {
#if B2MD_PAIR_TILE_ROTATE == 0
        const int ev[4] = {e0.x, e0.y, e0.z, e0.w};
        e0 = e1;
        if (q + 2 < tiles) e1 = __ldcs(col);            // warp-uniform; a stale e1 is never used
        col += pair_pitch;
#else
        // the tile in use stays in e0 for the whole trip (no copy: four registers less in a
        // loop that runs at the register cap); the rotation happens at the bottom
        const int ev[4] = {e0.x, e0.y, e0.z, e0.w};
#endif
#if B2MD_PAIR_HALF_TILE
        // two gathers in flight at a time (eight registers less in a loop at the register cap)
#pragma unroll
        for (int h = 0; h < 4; h += 2) {
            float4 pj[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) pj[u] = __ldg(pos + ((unsigned)ev[h + u] >> 2));
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                if (TABLE)
                    pair_entry_packed_table<AXES, THERMO>(acc, ax, ay, az, cx, cy, cz, ev[h + u],
                                                          pj[u], a, s_tab_a, s_tab_b, ta_row,
                                                          tb_row);
                else
                    pair_entry_packed<AXES, THERMO, SIG1>(acc, ax, ay, az, cx, cy, cz, ev[h + u],
                                                          pj[u], a);
            }
        }
#else
        float4 pj[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) pj[u] = __ldg(pos + ((unsigned)ev[u] >> 2));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (TABLE)
                pair_entry_packed_table<AXES, THERMO, PRUNE>(acc, ax, ay, az, cx, cy, cz, ev[u],
                                                             pj[u], a, s_tab_a, s_tab_b, ta_row,
                                                             tb_row, P);
            else
                pair_entry_packed<AXES, THERMO, SIG1, PRUNE>(acc, ax, ay, az, cx, cy, cz, ev[u],
                                                             pj[u], a, P);
        }
#endif
#if B2MD_PAIR_TILE_ROTATE != 0
        e0 = e1;
        if (q + 2 < tiles) e1 = __ldcs(col);            // warp-uniform; a stale e1 is never used
        col += pair_pitch;
#endif
    }
    upk(acc.fx, A.fx, B.fx);
    upk(acc.fy, A.fy, B.fy);
    upk(acc.fz, A.fz, B.fz);
    upk(acc.u, A.u, B.u);
    upk(acc.w, A.w, B.w);
    A.cnt = acc.cnt_a;
    B.cnt = acc.cnt_b;
}

// The same loop out of line (its registers are allocated on their own): a knob of the A/B
// harness, B2MD_PAIR_OUTLINE -- see the dispatch.  ptxas' register assignment inside the
// 64-register loop decides +-10 % of this kernel (identical instruction mix, different
// operand banks), and any change elsewhere in the kernel reshuffles it.
template <int AXES, bool TABLE, bool THERMO, bool SIG1, bool PRUNE = false>
__device__ __noinline__ void pair_row_loop_outlined(RowAcc &A, RowAcc &B, const float4 pa,
                                                    const float4 pb, int tiles,
                                                    const int4 *__restrict__ col,
                                                    int64_t pair_pitch,
                                                    const float4 *__restrict__ pos,
                                                    const ForceArgs &a, const float4 *s_tab_a,
                                                    const float2 *s_tab_b, int ta_row,
                                                    int tb_row, PruneOut *P = nullptr) {
    pair_row_loop<AXES, TABLE, THERMO, SIG1, PRUNE>(A, B, pa, pb, tiles, col, pair_pitch, pos, a,
                                                    s_tab_a, s_tab_b, ta_row, tb_row, P);
}

#ifndef B2MD_PAIR_MIN_BLOCKS
#define B2MD_PAIR_MIN_BLOCKS (1024 / kPairThreads)
#endif
#ifndef B2MD_PAIR_INTERIOR_FACE
#define B2MD_PAIR_INTERIOR_FACE 0
#endif
#ifndef B2MD_PAIR_OUTLINE
#define B2MD_PAIR_OUTLINE 0      // 0: nothing, 1: fallback 7, 2: + multi-axis face variants, 3: all but 0
#endif                           // (measured, profiles/README.md: 0 is the fastest build)

// ADVANCE: 0 = forces only, 1 = one-launch step, 2 = one-launch step that also stores the
// slab halo into the neighbour ranks' ghost rows (AdvanceArgs::halo_*)
// ORDERED: the lane order (b2md_pair_order) is its own instantiation -- with the lookup in the
// common kernel, even switched off, ptxas allocated the table variant's loops differently and
// Kob-Andersen N = 262 144 went from 0.0955 to 0.111 ms per step.
template <bool TABLE, bool THERMO, bool SIG1, int ADVANCE, bool PRUNE = false, bool ORDERED = false>
__global__ void __launch_bounds__(kPairThreads, PRUNE ? 6 : B2MD_PAIR_MIN_BLOCKS)
k_force_lj_pair(const float4 *__restrict__ pos, int64_t n, const __grid_constant__ ForceArgs a,
                const int4 *__restrict__ pair_nbr, const int32_t *__restrict__ pair_counts,
                int64_t pair_pitch, const int32_t *__restrict__ nbr,
                const int32_t *__restrict__ counts, int64_t pitch,
                const uint8_t *__restrict__ boundary, float4 *__restrict__ force,
                float *__restrict__ virial, b2md_status *status, int gated,
                const __grid_constant__ AdvanceArgs adv) {
    __shared__ float4 s_tab_a[TABLE ? kMaxTypes * kMaxTypes : 1];
    __shared__ float2 s_tab_b[TABLE ? kMaxTypes * kMaxTypes : 1];
    __shared__ float s_max[kPairThreads / 32];
    // step-graph batches: nothing to do once an in-graph list build overflowed
    if ((gated & 1) && *(volatile int *)&status->frozen) return;
    if (ADVANCE && advance_gate_closed(status, adv)) return;
    if (TABLE) {
        for (int t = threadIdx.x; t < a.ntypes * a.ntypes; t += blockDim.x) {
            s_tab_a[t] = a.tab_a[t];
            s_tab_b[t] = a.tab_b[t];
        }
        __syncthreads();
    }
    const int64_t n_pairs = (n + 1) >> 1;
    // Block schedule (b2md_pair_schedule): blocks whose warps need image shifts run up to
    // 1.7x longer; dispatched last (the space-filling curve ends on a face of the box) they
    // were the tail of the launch -- 10 us of 118 at N = 1 M.  The schedule runs them first.
    const unsigned bid = a.schedule ? (unsigned)__ldg(a.schedule + blockIdx.x) : blockIdx.x;
    // Lane order (b2md_pair_order): a warp pays for its longest row, 27.7 tiles where the mean
    // row has 23.3; with the pairs of a block dealt to its warps by row length the warps walk
    // 24.6.  A thread still owns one pair and walks its row in ascending order: same sums.
    const unsigned slot = ORDERED ? (unsigned)a.order[bid * (unsigned)kPairThreads + threadIdx.x]
                                  : threadIdx.x;
    const int64_t t_raw = bid * (int64_t)blockDim.x + slot;
    const bool active = t_raw < n_pairs;
    const int64_t t = active ? t_raw : n_pairs - 1;
    const int64_t ia = 2 * t;
    const bool has_b = ia + 1 < n;
    const int64_t ib = has_b ? ia + 1 : ia;
    const float4 pa = pos[ia], pb = pos[ib];
    // pruned step loop: the rows walked are the inner ones unless this launch prunes / falls back
    const bool inner = ADVANCE == 1 && !PRUNE && adv.prune_mode == kPruneInner;
    const int cnt = active ? (inner ? adv.inner_counts : pair_counts)[t] : 0;
    int tiles = __reduce_max_sync(0xffffffffu, (cnt + 3) >> 2);
    if (gated >> 16) tiles = tiles * ((gated >> 16) - 1) / 100;   // timing experiment: shorter rows
    // boundary flags of the warp's particles (nlist.cu, boundary_flag): bits 0-2 OR-ed = axes
    // that may need an image shift, bits 3-5 AND-ed = axes on which every particle is clear
    // of the mid-plane (face frame legal)
    // (gated bit 1: timing experiment only -- every warp takes the no-image-shift path)
    int near = 7, clear = 0;                     // no flags: per-pair image numbers on all axes
    if (boundary) {
        const int fa = active ? (int)boundary[ia] : 0x38, fb = active ? (int)boundary[ib] : 0x38;
        near = (fa | fb) & 7;
        clear = (fa & fb) >> 3;
    }
    const int axes = (gated & 2) ? 0 : __reduce_or_sync(0xffffffffu, near);
    clear = __reduce_and_sync(0xffffffffu, clear);
    const int4 *col = (inner ? (const int4 *)adv.inner_nbr : pair_nbr) + t;
    PruneOut P = {0, 0, 0, 0, 0, 0, 0u, (unsigned)pair_pitch, nullptr, 0.0f};
    if (PRUNE) {
        P.cap = active ? adv.inner_tiles * 4 : 0;
        P.ocol = adv.inner_nbr + t;
        P.rl2 = adv.inner_rl2;
    }
    const int ta_row = TABLE ? __float_as_int(pa.w) * a.ntypes : 0;
    const int tb_row = TABLE ? __float_as_int(pb.w) * a.ntypes : 0;

    RowAcc A = {0.f, 0.f, 0.f, 0.f, 0.f, 0}, B = {0.f, 0.f, 0.f, 0.f, 0.f, 0};
#define B2MD_PAIR_LOOP(AXES)                                                                  \
    pair_row_loop<AXES, TABLE, THERMO, SIG1, PRUNE>(A, B, pa, pb, tiles, col, pair_pitch, pos,  \
                                                    a, s_tab_a, s_tab_b, ta_row, tb_row,      \
                                                    PRUNE ? &P : nullptr)
#define B2MD_PAIR_LOOP_OUT(AXES)                                                              \
    pair_row_loop_outlined<AXES, TABLE, THERMO, SIG1, PRUNE>(A, B, pa, pb, tiles, col,        \
                                                             pair_pitch, pos, a, s_tab_a,     \
                                                             s_tab_b, ta_row, tb_row,         \
                                                             PRUNE ? &P : nullptr)
#define B2MD_PAIR_LOOP_LVL(AXES, LVL)                                                         \
    do { if (B2MD_PAIR_OUTLINE >= LVL) B2MD_PAIR_LOOP_OUT(AXES); else B2MD_PAIR_LOOP(AXES); } while (0)
    // face frame (see face_frame): legal when every particle of the warp is clear of the
    // mid-plane on each flagged axis
    const bool face_ok = (axes & ~clear) == 0;
    int variant = face_ok ? (axes << 3) : (axes ? 7 : 0);
#if B2MD_PAIR_INTERIOR_FACE
    // Experiment knob (off): interior warps whose particles are all clear of the x mid-plane run
    // the x face-frame loop (same bits: every image number is 0 there and the correction terms
    // cancel exactly).  With the knob off, "all warps on variant 8" measured 106.9 us against
    // 113.4 us for variant 0 -- three packed operations MORE per entry, yet faster; with the knob
    // on, ptxas assigned the registers of every loop differently and both took 115 us.  The
    // +-10 % of this kernel are register-allocation luck (profiles/README.md).
    if (variant == 0 && (clear & 1)) variant = 8;
#endif
    if ((gated >> 2) & 0x3fff) {                     // timing experiments only (profiles/exp)
        const int v = ((gated >> 2) & 0x3fff) - 1;
        // 64: flagged warps run a second copy of the no-shift loop (instruction-cache probe)
        variant = v == 64 ? (axes ? 64 : 0) : v;
    }
    switch (variant) {                                     // warp-uniform
        case 0: B2MD_PAIR_LOOP(0); break;
        case 8: B2MD_PAIR_LOOP_LVL(8, 3); break;
        case 16: B2MD_PAIR_LOOP_LVL(16, 3); break;
        case 24: B2MD_PAIR_LOOP_LVL(24, 2); break;
        case 32: B2MD_PAIR_LOOP_LVL(32, 3); break;
        case 40: B2MD_PAIR_LOOP_LVL(40, 2); break;
        case 48: B2MD_PAIR_LOOP_LVL(48, 2); break;
        case 56: B2MD_PAIR_LOOP_LVL(56, 2); break;
        default: B2MD_PAIR_LOOP_LVL(7, 1); break;   // tiny boxes / unordered particles: per-pair images
    }
#undef B2MD_PAIR_LOOP
#undef B2MD_PAIR_LOOP_OUT
#undef B2MD_PAIR_LOOP_LVL
    if (PRUNE) {
        // flush the unfinished tile, pad to the warp's longest inner row (flag-less entries),
        // store the inner count -- the layout k_pair_rows produces
        const int kept = P.cnt;
        int k = kept;
        while (k & 3) { P.o0 = P.o1; P.o1 = P.o2; P.o2 = P.o3; P.o3 = 0; ++k; }
        if (k > kept && k <= P.cap) P.ocol[P.oq] = make_int4(P.o0, P.o1, P.o2, P.o3);
        const int my_tiles = active ? k >> 2 : 0;
        const int warp_tiles = min(__reduce_max_sync(0xffffffffu, my_tiles), adv.inner_tiles);
        if (t_raw < pair_pitch) {
            int4 *oc = adv.inner_nbr + t_raw;
            for (int q = my_tiles; q < warp_tiles; ++q)
                oc[(int64_t)q * pair_pitch] = make_int4(0, 0, 0, 0);
            adv.inner_counts[t_raw] = active ? kept : 0;
        }
    }
    float d2 = 0.0f, d2_inner = 0.0f;
    if (active) {
#pragma unroll
        for (int which = 0; which < 2; ++which) {
            if (which == 1 && !has_b) break;
            const RowAcc &acc = which ? B : A;
            const int64_t i = which ? ib : ia;
            float fx, fy, fz, u, w;
            if (TABLE) {
                fx = acc.fx; fy = acc.fy; fz = acc.fz; u = acc.u; w = acc.w;
            } else {
                const PairParams &p = a.single;
                fx = p.c_f * acc.fx; fy = p.c_f * acc.fy; fz = p.c_f * acc.fz;
                u = fmaf(p.c_u, acc.u, p.half_shift * (float)acc.cnt);
                w = p.c_w * acc.w;
            }
            if (ADVANCE) {
                // the particle's own position is read again (an L1 / L2 hit) instead of being
                // kept in registers across the row loop: 8 registers of slack there
                float4 h = reload_f4(pos + i);
                if (ADVANCE == 1 && adv.prune_mode) {                    // kernel-uniform
                    float di;
                    d2 = fmaxf(d2, advance_particle_pruned<2>(i, h, make_float4(fx, fy, fz, u),
                                                              adv.pos_lo, adv.vel, adv.image,
                                                              adv.step, adv.ref_pos, PRUNE, di));
                    d2_inner = fmaxf(d2_inner, di);
                } else {
                    d2 = fmaxf(d2, advance_particle<2>(i, h, make_float4(fx, fy, fz, u),
                                                       adv.pos_lo, adv.vel, adv.image, adv.step,
                                                       adv.ref_pos));
                }
                adv.pos_out[i] = h;
                if (ADVANCE == 2) {
#pragma unroll
                    for (int side = 0; side < 2; ++side)
                        if (adv.halo_dst[side]) {          // kernel-uniform
                            const int slot = __ldg(&adv.halo_dst[side][i]);
                            if (slot >= 0) adv.halo_out[side][slot] = h;
                        }
                }
            } else {
                force[i] = make_float4(fx, fy, fz, u);
                if (THERMO && virial) virial[i] = w;
            }
            if (!(isfinite(fx) && isfinite(fy) && isfinite(fz)))
                report_singular_pair((int)i, which, reload_f4(pos + i), cnt, col, pair_pitch, pos,
                                     a.box, status);
        }
    }
    if (ADVANCE) advance_publish_disp<kPairThreads>(d2, s_max, status, adv);
    if (ADVANCE == 1 && adv.prune_mode)
        advance_publish_inner<kPairThreads>(d2_inner, s_max, status, adv);
}

// ---- block schedule of the pair kernel ---------------------------------------
// k_pair_block_flags: one warp per block of the pair kernel (kPairThreads pairs = 2 kPairThreads
// particles): flag = some particle of the block near a periodic face.  k_pair_schedule: one
// block partitions the flags stably -- flagged blocks first, in their own order, the others
// behind them -- and writes schedule[position] = block.
constexpr int kScheduleThreads = 1024;

__global__ void __launch_bounds__(256)
k_pair_block_flags(const uint8_t *__restrict__ boundary, int64_t n, int n_blocks,
                   int32_t *__restrict__ flags) {
    const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (b >= n_blocks) return;
    const int lane = threadIdx.x & 31;
    const int64_t lo = (int64_t)b * 2 * kPairThreads;
    const int64_t hi = min(lo + 2 * kPairThreads, n);
    int f = 0;
    for (int64_t i = lo + lane; i < hi; i += 32) f |= boundary[i] & 7;
    f = __reduce_or_sync(0xffffffffu, f);
    if (lane == 0) flags[b] = f != 0;
}

__global__ void __launch_bounds__(kScheduleThreads)
k_pair_schedule(const int32_t *__restrict__ flags, int n_blocks, int32_t *__restrict__ schedule) {
    __shared__ int s_warp[kScheduleThreads / 32];
    __shared__ int s_base;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_base = 0;
    for (int pass = 0; pass < 2; ++pass) {          // pass 0: flagged blocks, pass 1: the rest
        for (int b0 = 0; b0 < n_blocks; b0 += kScheduleThreads) {
            __syncthreads();
            const int b = b0 + threadIdx.x;
            const int want = b < n_blocks && ((flags[b] != 0) == (pass == 0));
            const unsigned vote = __ballot_sync(0xffffffffu, want);
            if (lane == 0) s_warp[warp] = __popc(vote);
            __syncthreads();
            int before = 0, total = 0;
            for (int w = 0; w < kScheduleThreads / 32; ++w) {
                const int c = s_warp[w];
                before += w < warp ? c : 0;
                total += c;
            }
            const int base = s_base;
            if (want) schedule[base + before + __popc(vote & ((1u << lane) - 1u))] = b;
            __syncthreads();
            if (threadIdx.x == 0) s_base = base + total;
        }
    }
}


// ---- lane order of the pair kernel --------------------------------------------
// A warp of the pair kernel walks as many tiles as its longest row has.  In particle order
// that is 27.7 tiles in the molten fluid at N = 1 M against a mean row of 23.3 (row lengths
// within a block scatter by +-1.6 tiles).  k_pair_order sorts the kPairThreads pairs of every
// block by row length (stable; in units of `unit` adjacent pairs, so that a unit of 2 keeps
// 32-byte sectors of the index stream inside one warp) and stores order[block][slot] = pair of
// the block that thread `slot` takes; warps then hold rows of similar length: 24.6 tiles.
// With face_key, pairs that may need an image shift (boundary bits 0-2) sort behind all the
// others, so that the shuffle does not spread them over more warps than before.  Every row is
// padded (flag-less entries) to the longest row of its NEW warp.  The padding that
// k_pair_rows / k_pair_fixup wrote for the particle-order warps stays, so launches without
// B2MD_FORCE_ORDERED remain legal on the same rows.
__global__ void __launch_bounds__(kPairThreads)
k_pair_order(const uint8_t *__restrict__ boundary, int64_t n, int4 *__restrict__ pair_nbr,
             const int32_t *__restrict__ pair_counts, int64_t pair_pitch, int pair_tiles,
             int unit, int face_key, uint8_t *__restrict__ order) {
    __shared__ int s_key[kPairThreads];
    __shared__ int s_tiles[kPairThreads];       // by slot
    __shared__ int s_gmax[kPairThreads / 32];
    __shared__ uint8_t s_order[kPairThreads];
    const int s = threadIdx.x;
    const int64_t n_pairs = (n + 1) >> 1;
    const int64_t t = blockIdx.x * (int64_t)kPairThreads + s;
    const bool active = t < n_pairs;
    const int tiles = active ? min((pair_counts[t] + 3) >> 2, pair_tiles) : 0;
    int key = tiles;
    if (face_key && active && boundary) {
        const int64_t ia = 2 * t, ib = min(ia + 1, n - 1);
        if ((boundary[ia] | boundary[ib]) & 7) key |= 1 << 16;
    }
    s_key[s] = key;
    __syncthreads();
    const int u = s / unit, n_units = kPairThreads / unit;
    int ku = 0;
    for (int k = 0; k < unit; ++k) ku = max(ku, s_key[u * unit + k]);
    int rank = 0;
    for (int v = 0; v < n_units; ++v) {
        int kv = 0;
        for (int k = 0; k < unit; ++k) kv = max(kv, s_key[v * unit + k]);
        rank += (kv < ku) || (kv == ku && v < u);
    }
    const int slot = rank * unit + s % unit;
    s_order[slot] = (uint8_t)s;
    s_tiles[slot] = tiles;
    __syncthreads();
    const int g = __reduce_max_sync(0xffffffffu, s_tiles[s]);
    if ((s & 31) == 0) s_gmax[s >> 5] = g;
    order[blockIdx.x * (int64_t)kPairThreads + s] = s_order[s];
    __syncthreads();
    if (active) {
        int to = s_gmax[slot >> 5];
        // the idle threads behind the last pair read ITS row (k_force_lj_pair clamps t), for as
        // many tiles as their own warp walks
        if (t == n_pairs - 1)
            for (int w = 0; w < kPairThreads / 32; ++w) to = max(to, s_gmax[w]);
        int4 *out = pair_nbr + t;
        for (int q = tiles; q < to; ++q) out[(int64_t)q * pair_pitch] = make_int4(0, 0, 0, 0);
    }
}

// ---- all pairs (reference _all_to_all_chunk, forces.py:29-69) --------------------
// The paper's primary benchmark is N = 2000: one thread per particle is 16 blocks on 148 SMs.
// A thread-block CLUSTER of kAllPairsSplit blocks therefore shares one block of 128 particles
// i: block r of the cluster walks the j tiles r, r + S, r + 2S, ... (positions staged through
// shared memory, 128 at a time), and the partial sums of the S blocks are combined through
// distributed shared memory by block 0 of the cluster in the fixed order r = 0 .. S-1 -- no
// atomics, no scratch buffer, bitwise reproducible.
constexpr int kAllPairsSplit = 8;           // portable cluster size
// below these sizes: k_force_all_pairs_small with 8 / 4 warps per tile of 32 particles
constexpr int64_t kAllPairsEightWarps = 12288, kAllPairsFourWarps = 65536;

// `zeros` = partners at zero distance.  A particle meets itself exactly once (identical
// coordinates give an exact zero), so a total other than 1 means a coincident pair: the rare
// slow path (all_pairs_report_singular) then finds the partner.  Cheaper than telling "self"
// from "singular" for every pair: one predicate and one add instead of 64-bit index compares.
struct AllPairsPartial {
    float fx, fy, fz, u, w;
    int cnt;
    int zeros;
    int pad;
};

// Fixed-point coordinates of the all-pairs kernels: a coordinate x in [0, L) becomes the 32-bit
// integer round(x 2^32 / L), so that the wrapped difference of two of them IS the minimum
// image (forces.py:45-50: d - L rint(d / L)) -- one integer subtract, one conversion and one
// multiply per axis where the exact fp32 sequence (delta<true>: split box length, shifted
// operands) takes ten instructions.  Resolution L 2^-32 (3e-9 sigma at N = 2000, finer than the
// fp32 high words the kernel is given); the difference is exact, its conversion rounds to 24
// bits of the DISTANCE, so close pairs lose nothing to the size of the box.
struct FixedBox {
    double to_fixed[3];       // 2^32 / L
    float scale[3];           // L / 2^32
};

inline FixedBox make_fixed_box(const b2md_box *box) {
    FixedBox f;
    for (int c = 0; c < 3; ++c) {
        f.to_fixed[c] = 4294967296.0 / box->edge[c];
        f.scale[c] = (float)(box->edge[c] / 4294967296.0);
    }
    return f;
}

// (x, y, z, w) -> fixed-point x, y, z (mod 2^32: a coordinate equal to L is 0), w kept
__device__ __forceinline__ int4 to_fixed4(const float4 p, const FixedBox &fb) {
    int4 q;
    q.x = (int)(unsigned)__double2ll_rn((double)p.x * fb.to_fixed[0]);
    q.y = (int)(unsigned)__double2ll_rn((double)p.y * fb.to_fixed[1]);
    q.z = (int)(unsigned)__double2ll_rn((double)p.z * fb.to_fixed[2]);
    q.w = __float_as_int(p.w);
    return q;
}

__device__ __forceinline__ float fixed_delta(int a, int b, float scale) {
    return __int2float_rn((int)((unsigned)a - (unsigned)b)) * scale;
}

// forces.py:113-116 for the all-pairs kernels: lowest j != i at zero distance from particle i.
__device__ __noinline__ void all_pairs_report_singular(int i, const int4 qi,
                                                       const float4 *__restrict__ pos, int n,
                                                       const FixedBox &fb, b2md_status *status) {
    for (int j = 0; j < n; ++j) {
        if (j == i) continue;
        const int4 qj = to_fixed4(pos[j], fb);
        if (qi.x == qj.x && qi.y == qj.y && qi.z == qj.z) {
            atomicMin((unsigned long long *)&status->singular,
                      ((unsigned long long)(unsigned)i << 32) | (unsigned)j);
            return;
        }
    }
}

// One pair of the all-pairs scan (forces.py:41-66): the pair contributes iff r2 != 0.
template <bool TABLE, bool THERMO = true>
__device__ __forceinline__ void all_pairs_entry(RowAcc &acc, int &zeros, const int4 qi,
                                                const int4 qj, const FixedBox &fb,
                                                const ForceArgs &a, const float4 *s_tab_a,
                                                const float2 *s_tab_b, int ti_row) {
    const float dx = fixed_delta(qi.x, qj.x, fb.scale[0]);
    const float dy = fixed_delta(qi.y, qj.y, fb.scale[1]);
    const float dz = fixed_delta(qi.z, qj.z, fb.scale[2]);
    const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
    const bool valid = r2 != 0.0f;
    zeros += valid ? 0 : 1;
    if (TABLE) {
        const int tt = ti_row + qj.w;
        lj_pair_table<THERMO>(acc, dx, dy, dz, r2, valid, s_tab_a[tt], s_tab_b[tt]);
    } else {
        lj_pair_single<THERMO>(acc, dx, dy, dz, r2, valid, a.single);
    }
}

// ADVANCE variants of the all-pairs kernels (the intermediate steps of b2md_run_all_pairs): the
// thread that holds a particle's total force also applies vv_finalize of this step and
// vv_integrate of the next (integrate.py:58-79, the body of k_integrate<2>) -- one launch per
// MD step, forces never stored.  Every block of the launch reads the old positions, so the new
// high words go to a second buffer.
struct AllPairsAdvance {
    float4 *pos_out, *pos_lo, *vel;
    int4 *image;
    StepConst step;
};

template <bool TABLE, bool ADVANCE = false>
__global__ void __cluster_dims__(kAllPairsSplit, 1, 1) __launch_bounds__(kForceThreads)
k_force_all_pairs(const float4 *__restrict__ pos, int64_t n, const __grid_constant__ ForceArgs a,
                  const __grid_constant__ FixedBox fb, float4 *__restrict__ force,
                  float *__restrict__ virial, b2md_status *status,
                  const __grid_constant__ AllPairsAdvance adv) {
    __shared__ int4 tile[kForceThreads];
    __shared__ float4 s_tab_a[TABLE ? kMaxTypes * kMaxTypes : 1];
    __shared__ float2 s_tab_b[TABLE ? kMaxTypes * kMaxTypes : 1];
    __shared__ AllPairsPartial s_part[kForceThreads];
    if (TABLE) {
        for (int t = threadIdx.x; t < a.ntypes * a.ntypes; t += blockDim.x) {
            s_tab_a[t] = a.tab_a[t];
            s_tab_b[t] = a.tab_b[t];
        }
    }
    unsigned rank;                                   // block rank inside the cluster
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int64_t i_raw = (blockIdx.x / kAllPairsSplit) * (int64_t)blockDim.x + threadIdx.x;
    const bool active = i_raw < n;
    const int64_t i = active ? i_raw : n - 1;
    const int4 qi = to_fixed4(pos[i], fb);
    const int ti_row = TABLE ? qi.w * a.ntypes : 0;
    RowAcc acc = {0.f, 0.f, 0.f, 0.f, 0.f, 0};
    int zeros = 0;
    const int ni = (int)n;                       // (row indices are 32-bit everywhere)
    for (int base = (int)rank * kForceThreads; base < ni; base += kAllPairsSplit * kForceThreads) {
        __syncthreads();
        const int jl = base + (int)threadIdx.x;
        tile[threadIdx.x] = to_fixed4(pos[jl < ni ? jl : ni - 1], fb);
        __syncthreads();
        const int lim = min(kForceThreads, ni - base);
#pragma unroll 4
        for (int t = 0; t < lim; ++t)
            all_pairs_entry<TABLE, !ADVANCE>(acc, zeros, qi, tile[t], fb, a, s_tab_a, s_tab_b, ti_row);
    }
    AllPairsPartial mine = {acc.fx, acc.fy, acc.fz, acc.u, acc.w, acc.cnt, zeros, 0};
    s_part[threadIdx.x] = mine;
    // cluster barrier (release / acquire): every block's partial sums are in its shared memory
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (rank == 0 && active) {
        RowAcc sum = {0.f, 0.f, 0.f, 0.f, 0.f, 0};
        int zeros_all = 0;
        const unsigned local = (unsigned)__cvta_generic_to_shared(&s_part[threadIdx.x]);
#pragma unroll
        for (unsigned r = 0; r < (unsigned)kAllPairsSplit; ++r) {      // fixed order
            unsigned remote;
            asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(r));
            float fx, fy, fz, u, w;
            int cnt, zr;
            asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(fx) : "r"(remote));
            asm volatile("ld.shared::cluster.f32 %0, [%1+4];" : "=f"(fy) : "r"(remote));
            asm volatile("ld.shared::cluster.f32 %0, [%1+8];" : "=f"(fz) : "r"(remote));
            asm volatile("ld.shared::cluster.f32 %0, [%1+12];" : "=f"(u) : "r"(remote));
            asm volatile("ld.shared::cluster.f32 %0, [%1+16];" : "=f"(w) : "r"(remote));
            asm volatile("ld.shared::cluster.s32 %0, [%1+20];" : "=r"(cnt) : "r"(remote));
            asm volatile("ld.shared::cluster.s32 %0, [%1+24];" : "=r"(zr) : "r"(remote));
            sum.fx += fx; sum.fy += fy; sum.fz += fz; sum.u += u; sum.w += w; sum.cnt += cnt;
            zeros_all += zr;
        }
        float fx, fy, fz, u, w;
        if (TABLE) {
            fx = sum.fx; fy = sum.fy; fz = sum.fz; u = sum.u; w = sum.w;
        } else {
            const PairParams &p = a.single;
            fx = p.c_f * sum.fx; fy = p.c_f * sum.fy; fz = p.c_f * sum.fz;
            u = fmaf(p.c_u, sum.u, p.half_shift * (float)sum.cnt);
            w = p.c_w * sum.w;
        }
        if (ADVANCE) {
            float4 h = pos[i];
            advance_particle<2>(i, h, make_float4(fx, fy, fz, u), adv.pos_lo, adv.vel, adv.image,
                                adv.step, nullptr);
            adv.pos_out[i] = h;
        } else {
            force[i] = make_float4(fx, fy, fz, u);
            if (virial) virial[i] = w;
        }
        if (zeros_all != 1) all_pairs_report_singular((int)i, qi, pos, (int)n, fb, status);
    }
    // nobody leaves while block 0 may still read its shared memory
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Small systems (the paper's N = 2000).  With one thread per particle i a thread walks N / 8
// partners one after the other and a scheduler holds less than one warp: the launch is as long
// as that dependent chain (33 us at N = 2000 for 8 us of arithmetic).  Here the WARPS warps of
// a block share ONE tile of 32 particles i and split every staged tile of 32 WARPS partners
// between them, on top of the 8-way split over the cluster: 8 WARPS times the warps, chains
// 8 WARPS times shorter.  Partial sums are combined in fixed order -- warps 0 .. WARPS-1
// through shared memory, then blocks 0 .. 7 through distributed shared memory -- so results
// are bitwise reproducible.  The shape depends on n alone: a system always takes the same
// summation order.
template <bool TABLE, int WARPS, bool ADVANCE = false>
__global__ void __cluster_dims__(kAllPairsSplit, 1, 1) __launch_bounds__(32 * WARPS)
k_force_all_pairs_small(const float4 *__restrict__ pos, int64_t n,
                        const __grid_constant__ ForceArgs a, const __grid_constant__ FixedBox fb,
                        float4 *__restrict__ force, float *__restrict__ virial,
                        b2md_status *status, const __grid_constant__ AllPairsAdvance adv) {
    constexpr int kTile = 32 * WARPS;
    __shared__ int4 tile[kTile];
    __shared__ float4 s_tab_a[TABLE ? kMaxTypes * kMaxTypes : 1];
    __shared__ float2 s_tab_b[TABLE ? kMaxTypes * kMaxTypes : 1];
    __shared__ AllPairsPartial s_part[kTile];           // [warp][lane]
    __shared__ AllPairsPartial s_sum[32];               // the block's total per particle i
    if (TABLE) {
        for (int t = threadIdx.x; t < a.ntypes * a.ntypes; t += blockDim.x) {
            s_tab_a[t] = a.tab_a[t];
            s_tab_b[t] = a.tab_b[t];
        }
    }
    unsigned rank;                                   // block rank inside the cluster
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i_raw = (blockIdx.x / kAllPairsSplit) * 32ll + lane;
    const bool active = i_raw < n;
    const int64_t i = active ? i_raw : n - 1;
    const int4 qi = to_fixed4(pos[i], fb);
    const int ti_row = TABLE ? qi.w * a.ntypes : 0;
    RowAcc acc = {0.f, 0.f, 0.f, 0.f, 0.f, 0};
    int zeros = 0;
    const int ni = (int)n;                       // (row indices are 32-bit everywhere)
    const int my = warp * 32;                    // this warp's slice of the staged tile
    for (int base = (int)rank * kTile; base < ni; base += kAllPairsSplit * kTile) {
        __syncthreads();
        const int jl = base + (int)threadIdx.x;
        tile[threadIdx.x] = to_fixed4(pos[jl < ni ? jl : ni - 1], fb);
        __syncthreads();
        const int lim = max(0, min(32, ni - (base + warp * 32)));
#pragma unroll 4
        for (int t = 0; t < lim; ++t)
            all_pairs_entry<TABLE, !ADVANCE>(acc, zeros, qi, tile[my + t], fb, a, s_tab_a, s_tab_b, ti_row);
    }
    AllPairsPartial mine = {acc.fx, acc.fy, acc.fz, acc.u, acc.w, acc.cnt, zeros, 0};
    s_part[threadIdx.x] = mine;
    __syncthreads();
    if (warp == 0) {
        AllPairsPartial tot = s_part[lane];
#pragma unroll
        for (int w = 1; w < WARPS; ++w) {                           // fixed order
            const AllPairsPartial q = s_part[w * 32 + lane];
            tot.fx += q.fx; tot.fy += q.fy; tot.fz += q.fz; tot.u += q.u; tot.w += q.w;
            tot.cnt += q.cnt;
            tot.zeros += q.zeros;
        }
        s_sum[lane] = tot;
    }
    // cluster barrier (release / acquire): every block's sums are in its shared memory
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (rank == 0 && warp == 0 && active) {
        RowAcc sum = {0.f, 0.f, 0.f, 0.f, 0.f, 0};
        int zeros_all = 0;
        const unsigned local = (unsigned)__cvta_generic_to_shared(&s_sum[lane]);
#pragma unroll
        for (unsigned r = 0; r < (unsigned)kAllPairsSplit; ++r) {      // fixed order
            unsigned remote;
            asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(r));
            float fx, fy, fz, u, w;
            int cnt, zr;
            asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(fx) : "r"(remote));
            asm volatile("ld.shared::cluster.f32 %0, [%1+4];" : "=f"(fy) : "r"(remote));
            asm volatile("ld.shared::cluster.f32 %0, [%1+8];" : "=f"(fz) : "r"(remote));
            asm volatile("ld.shared::cluster.f32 %0, [%1+12];" : "=f"(u) : "r"(remote));
            asm volatile("ld.shared::cluster.f32 %0, [%1+16];" : "=f"(w) : "r"(remote));
            asm volatile("ld.shared::cluster.s32 %0, [%1+20];" : "=r"(cnt) : "r"(remote));
            asm volatile("ld.shared::cluster.s32 %0, [%1+24];" : "=r"(zr) : "r"(remote));
            sum.fx += fx; sum.fy += fy; sum.fz += fz; sum.u += u; sum.w += w; sum.cnt += cnt;
            zeros_all += zr;
        }
        float fx, fy, fz, u, w;
        if (TABLE) {
            fx = sum.fx; fy = sum.fy; fz = sum.fz; u = sum.u; w = sum.w;
        } else {
            const PairParams &p = a.single;
            fx = p.c_f * sum.fx; fy = p.c_f * sum.fy; fz = p.c_f * sum.fz;
            u = fmaf(p.c_u, sum.u, p.half_shift * (float)sum.cnt);
            w = p.c_w * sum.w;
        }
        if (ADVANCE) {
            float4 h = pos[i];
            advance_particle<2>(i, h, make_float4(fx, fy, fz, u), adv.pos_lo, adv.vel, adv.image,
                                adv.step, nullptr);
            adv.pos_out[i] = h;
        } else {
            force[i] = make_float4(fx, fy, fz, u);
            if (virial) virial[i] = w;
        }
        if (zeros_all != 1) all_pairs_report_singular((int)i, qi, pos, (int)n, fb, status);
    }
    // nobody leaves while block 0 may still read its shared memory
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

static int fill_args(ForceArgs &a, const b2md_box *box, const double *table, int ntypes) {
    if (!box || !table) { set_error("force: null box/table"); return -1; }
    if (ntypes < 1 || ntypes > kMaxTypes) {
        set_error("force: ntypes must be in [1, %d]", kMaxTypes);
        return -2;
    }
    a.box = make_box_f(box);
    a.ntypes = ntypes;
    a.schedule = nullptr;
    a.order = nullptr;
    for (int t = 0; t < ntypes * ntypes; ++t) {
        const double eps = table[4 * t], sig2 = table[4 * t + 1], rc2 = table[4 * t + 2],
                     shift = table[4 * t + 3];
        a.tab_a[t] = make_float4((float)sig2, (float)rc2, (float)(24.0 * eps), (float)(2.0 * eps));
        a.tab_b[t] = make_float2((float)(0.5 * shift), (float)(12.0 * eps));
    }
    a.single.sig2 = a.tab_a[0].x;
    a.single.rc2 = a.tab_a[0].y;
    a.single.c_f = a.tab_a[0].z;
    a.single.c_u = a.tab_a[0].w;
    a.single.half_shift = a.tab_b[0].x;
    a.single.c_w = a.tab_b[0].y;
    return 0;
}

}  // namespace b2md

using namespace b2md;

B2MD_EXPORT int b2md_force_lj(const void *d_pos_hi, int64_t n, const b2md_box *box,
                              const int32_t *d_nbr, const int32_t *d_counts, int64_t pitch,
                              int32_t stride, const uint8_t *d_boundary, const double *table,
                              int32_t ntypes, int32_t flags, void *d_force_f4, float *d_virial,
                              b2md_status *d_status, void *stream) {
    if (n <= 0 || !d_nbr || !d_counts || !d_status || stride < 1) {
        set_error("b2md_force_lj: bad arguments");
        return -1;
    }
    if (stride % 16 != 0) {
        set_error("b2md_force_lj: the list must be allocated with a multiple of 16 rows");
        return -3;
    }
    ForceArgs a;
    int rc = fill_args(a, box, table, ntypes);
    if (rc) return rc;
    cudaStream_t s = as_stream(stream);
    const bool thermo = (flags & B2MD_FORCE_SKIP_THERMO) == 0;
    // Defaults chosen from profiles/ (DESIGN.md section 6), measured on B200 at N = 1 M: 12 CTAs/SM
    // (<= 40 registers) beats 8 CTAs/SM by 5 %; one lane per particle beats sub-warps for
    // large systems, while small systems (few CTAs, latency-bound serial row loops) want as
    // many lanes per particle as the device holds at once (lanes_for).  The A/B knobs are
    // read per call: the library keeps no state.
    const int pipe = env_choice("B2MD_FORCE_PIPE", 2) == 0 ? 0 : 2;   // 0: 8 CTAs/SM, 2: 12
    const int sub = lanes_for(n, stride);
#define B2MD_LAUNCH_FORCE(SUB, PIPE, TABLE, THERMO)                                          \
    k_force_lj<SUB, PIPE, TABLE, THERMO>                                                     \
        <<<blocks_for(n, kForceThreads / SUB), kForceThreads, 0, s>>>(                       \
            (const float4 *)d_pos_hi, n, a, d_nbr, d_counts, pitch, d_boundary,              \
            (float4 *)d_force_f4, d_virial, d_status, (flags & B2MD_FORCE_GATED) ? 1 : 0,    \
            AdvanceArgs())
#define B2MD_DISPATCH_TT(SUB, PIPE)                                                          \
    do {                                                                                     \
        if (ntypes == 1) {                                                                   \
            if (thermo) B2MD_LAUNCH_FORCE(SUB, PIPE, false, true);                           \
            else B2MD_LAUNCH_FORCE(SUB, PIPE, false, false);                                 \
        } else {                                                                             \
            if (thermo) B2MD_LAUNCH_FORCE(SUB, PIPE, true, true);                            \
            else B2MD_LAUNCH_FORCE(SUB, PIPE, true, false);                                  \
        }                                                                                    \
    } while (0)
    if (sub == 1) {
        if (pipe == 0) B2MD_DISPATCH_TT(1, 0);
        else B2MD_DISPATCH_TT(1, 2);
    } else if (sub == 2) {
        B2MD_DISPATCH_TT(2, 0);
    } else if (sub == 4) {
        B2MD_DISPATCH_TT(4, 0);
    } else {
        B2MD_DISPATCH_TT(16, 0);
    }
#undef B2MD_DISPATCH_TT
#undef B2MD_LAUNCH_FORCE
    B2MD_CHECK_LAUNCH("b2md_force_lj");
    return 0;
}

namespace {

// adv == nullptr: forces, energies, virial stored; else the ADVANCE variant (nothing stored)
int launch_all_pairs(const void *d_pos_hi, int64_t n, const b2md_box *box, const double *table,
                     int32_t ntypes, void *d_force_f4, float *d_virial, b2md_status *d_status,
                     const AllPairsAdvance *advance, void *stream, const char *name) {
    if (n <= 0 || !d_status || !d_pos_hi) { set_error("%s: bad arguments", name); return -1; }
    ForceArgs a;
    int rc = fill_args(a, box, table, ntypes);
    if (rc) return rc;
    cudaStream_t s = as_stream(stream);
    const float4 *pos = (const float4 *)d_pos_hi;
    float4 *force = (float4 *)d_force_f4;
    const FixedBox fb = make_fixed_box(box);
    AllPairsAdvance adv = {};
    if (advance) adv = *advance;
    // Kernel shape by size (measured on B200, kernel time under ncu, profiles/README.md):
    // N = 2000: 32.8 us with one thread per particle i, 13.6 us with 8 warps per 32 particles;
    // N = 8192: 179 / 136 us; N = 32 768: 2.11 / 1.99 ms (4 warps); N = 131 072: 30.3 / 30.7 ms.
    // The choice depends on n alone, so a system always takes the same summation order.
#define B2MD_LAUNCH_SMALL(TABLE, WARPS, ADVANCE)                                               \
    k_force_all_pairs_small<TABLE, WARPS, ADVANCE>                                            \
        <<<blocks_for(n, 32) * kAllPairsSplit, 32 * WARPS, 0, s>>>(pos, n, a, fb, force,      \
                                                                   d_virial, d_status, adv)
#define B2MD_LAUNCH_BIG(TABLE, ADVANCE)                                                        \
    k_force_all_pairs<TABLE, ADVANCE>                                                         \
        <<<blocks_for(n, kForceThreads) * kAllPairsSplit, kForceThreads, 0, s>>>(             \
            pos, n, a, fb, force, d_virial, d_status, adv)
#define B2MD_LAUNCH_BY_SIZE(TABLE, ADVANCE)                                                    \
    do {                                                                                      \
        if (n < kAllPairsEightWarps) B2MD_LAUNCH_SMALL(TABLE, 8, ADVANCE);                    \
        else if (n < kAllPairsFourWarps) B2MD_LAUNCH_SMALL(TABLE, 4, ADVANCE);                \
        else B2MD_LAUNCH_BIG(TABLE, ADVANCE);                                                 \
    } while (0)
    if (advance) {
        if (ntypes == 1) B2MD_LAUNCH_BY_SIZE(false, true);
        else B2MD_LAUNCH_BY_SIZE(true, true);
    } else {
        if (ntypes == 1) B2MD_LAUNCH_BY_SIZE(false, false);
        else B2MD_LAUNCH_BY_SIZE(true, false);
    }
#undef B2MD_LAUNCH_BY_SIZE
#undef B2MD_LAUNCH_BIG
#undef B2MD_LAUNCH_SMALL
    B2MD_CHECK_LAUNCH(name);
    return 0;
}

}  // namespace

B2MD_EXPORT int b2md_force_lj_all_pairs(const void *d_pos_hi, int64_t n, const b2md_box *box,
                                        const double *table, int32_t ntypes, void *d_force_f4,
                                        float *d_virial, b2md_status *d_status, void *stream) {
    return launch_all_pairs(d_pos_hi, n, box, table, ntypes, d_force_f4, d_virial, d_status,
                            nullptr, stream, "b2md_force_lj_all_pairs");
}

B2MD_EXPORT int b2md_force_lj_all_pairs_advance(const void *d_pos_hi, void *d_pos_hi_out,
                                                void *d_pos_lo, void *d_vel, void *d_image_i4,
                                                int64_t n, const b2md_box *box,
                                                const double *table, int32_t ntypes, double dt,
                                                b2md_status *d_status, void *stream) {
    if (!d_pos_hi_out || d_pos_hi_out == d_pos_hi || !d_pos_lo || !d_vel || !d_image_i4 ||
        !box || !(dt > 0.0)) {
        set_error("b2md_force_lj_all_pairs_advance: bad arguments");
        return -1;
    }
    AllPairsAdvance adv;
    adv.pos_out = (float4 *)d_pos_hi_out;
    adv.pos_lo = (float4 *)d_pos_lo;
    adv.vel = (float4 *)d_vel;
    adv.image = (int4 *)d_image_i4;
    adv.step = make_step(box, dt, 1e30);
    return launch_all_pairs(d_pos_hi, n, box, table, ntypes, nullptr, nullptr, d_status, &adv,
                            stream, "b2md_force_lj_all_pairs_advance");
}

namespace {

int launch_pairs(const void *d_pos_hi, int64_t n, const b2md_box *box, const int32_t *d_pair_nbr,
                 const int32_t *d_pair_counts, int64_t pair_pitch, const int32_t *d_nbr,
                 const int32_t *d_counts, int64_t pitch, const uint8_t *d_boundary,
                 const double *table, int32_t ntypes, int32_t flags, void *d_force_f4,
                 float *d_virial, b2md_status *d_status, const AdvanceArgs *advance, void *stream,
                 const char *name) {
    if (n <= 0 || !d_pair_nbr || !d_pair_counts || !d_nbr || !d_counts || !d_status ||
        pair_pitch < (n + 1) / 2) {
        set_error("%s: bad arguments", name);
        return -1;
    }
    ForceArgs a;
    int rc = fill_args(a, box, table, ntypes);
    if (rc) return rc;
    cudaStream_t s = as_stream(stream);
    const bool thermo = (flags & B2MD_FORCE_SKIP_THERMO) == 0;
    AdvanceArgs adv = {};
    if (advance) adv = *advance;
#define B2MD_PAIR_ARGS                                                                        \
    (const float4 *)d_pos_hi, n, a, (const int4 *)d_pair_nbr, d_pair_counts, pair_pitch, d_nbr,   \
        d_counts, pitch, d_boundary, (float4 *)d_force_f4, d_virial, d_status,                \
        ((flags & B2MD_FORCE_GATED) ? 1 : 0) | exp_bits, adv
#define B2MD_LAUNCH_PAIR(TABLE, THERMO, SIG1, ADVANCE)                                        \
    do {                                                                                      \
        if (a.order)                                                                          \
            k_force_lj_pair<TABLE, THERMO, SIG1, ADVANCE, false, true>                        \
                <<<blocks, kPairThreads, 0, s>>>(B2MD_PAIR_ARGS);                             \
        else                                                                                  \
            k_force_lj_pair<TABLE, THERMO, SIG1, ADVANCE>                                     \
                <<<blocks, kPairThreads, 0, s>>>(B2MD_PAIR_ARGS);                             \
    } while (0)
    // Measured on B200 at N = 1 M (profiles/README.md): 8 CTAs/SM of 128 threads; 4 to 12
    // CTAs/SM, 32/64-thread CTAs, position gathers one trip ahead, L2 prefetch of the
    // index stream, L1 cache-policy hints, per-SM or per-warp work queues were all neutral
    // or slower.
    const unsigned blocks = blocks_for((n + 1) / 2, kPairThreads);
    const bool sig1 = a.single.sig2 == 1.0f;
    if (flags & B2MD_FORCE_SCHEDULED) a.schedule = d_pair_counts + pair_pitch;
    if (flags & B2MD_FORCE_ORDERED)
        a.order = reinterpret_cast<const uint8_t *>(d_pair_counts + pair_pitch + 2 * (int64_t)blocks);
    // profiles/exp only: B2MD_EXP_NO_BOUNDARY=1 -> no image shifts anywhere (wrong forces at the
    // faces), B2MD_EXP_VARIANT=v -> every warp runs image-shift variant v
    const int exp_variant = env_choice("B2MD_EXP_VARIANT", -1);
    const int exp_bits = (env_choice("B2MD_EXP_NO_BOUNDARY", 0) ? 2 : 0) |
                         (exp_variant >= 0 ? (exp_variant + 1) << 2 : 0) |
                         (env_choice("B2MD_EXP_TILES_PCT", -1) >= 0
                              ? (env_choice("B2MD_EXP_TILES_PCT", -1) + 1) << 16 : 0);
    if (advance && (adv.halo_dst[0] || adv.halo_dst[1])) {
        if (ntypes == 1) {
            if (sig1) B2MD_LAUNCH_PAIR(false, false, true, 2);
            else B2MD_LAUNCH_PAIR(false, false, false, 2);
        } else {
            B2MD_LAUNCH_PAIR(true, false, false, 2);
        }
    } else if (advance && adv.prune_mode == kPruneNow) {
#define B2MD_LAUNCH_PRUNE(TABLE, SIG1)                                                        \
    do {                                                                                      \
        if (a.order)                                                                          \
            k_force_lj_pair<TABLE, false, SIG1, 1, true, true>                                \
                <<<blocks, kPairThreads, 0, s>>>(B2MD_PAIR_ARGS);                             \
        else                                                                                  \
            k_force_lj_pair<TABLE, false, SIG1, 1, true>                                      \
                <<<blocks, kPairThreads, 0, s>>>(B2MD_PAIR_ARGS);                             \
    } while (0)
        if (ntypes == 1) {
            if (sig1) B2MD_LAUNCH_PRUNE(false, true);
            else B2MD_LAUNCH_PRUNE(false, false);
        } else {
            B2MD_LAUNCH_PRUNE(true, false);
        }
#undef B2MD_LAUNCH_PRUNE
    } else if (advance) {
        if (ntypes == 1) {
            if (sig1) B2MD_LAUNCH_PAIR(false, false, true, 1);
            else B2MD_LAUNCH_PAIR(false, false, false, 1);
        } else {
            B2MD_LAUNCH_PAIR(true, false, false, 1);
        }
    } else if (ntypes == 1) {
        if (thermo) B2MD_LAUNCH_PAIR(false, true, false, 0);
        else if (sig1) B2MD_LAUNCH_PAIR(false, false, true, 0);
        else B2MD_LAUNCH_PAIR(false, false, false, 0);
    } else {
        if (thermo) B2MD_LAUNCH_PAIR(true, true, false, 0);
        else B2MD_LAUNCH_PAIR(true, false, false, 0);
    }
#undef B2MD_LAUNCH_PAIR
#undef B2MD_PAIR_ARGS
    int rc2 = check_cuda(cudaPeekAtLastError(), name);
    return rc2;
}

}  // namespace

B2MD_EXPORT int64_t b2md_pair_schedule_len(int64_t n) {
    // the schedule + its flag scratch + the lane order (one byte per thread of the pair kernel)
    return (2 + kPairThreads / 4) * (int64_t)blocks_for((n + 1) / 2, kPairThreads);
}

B2MD_EXPORT int b2md_pair_order(const uint8_t *d_boundary, int64_t n, int32_t *d_pair_nbr,
                                int32_t *d_pair_counts, int64_t pair_pitch, int32_t pair_rows,
                                int32_t unit, int32_t face_key, void *stream) {
    if (n <= 0 || !d_pair_nbr || !d_pair_counts || pair_pitch < (n + 1) / 2 || pair_rows % 4 != 0 ||
        unit < 1 || unit > 32 || (unit & (unit - 1)) != 0) {
        set_error("b2md_pair_order: bad arguments (unit must be a power of two <= 32)");
        return -1;
    }
    const int64_t n_blocks = blocks_for((n + 1) / 2, kPairThreads);
    uint8_t *order = reinterpret_cast<uint8_t *>(d_pair_counts + pair_pitch + 2 * n_blocks);
    k_pair_order<<<(unsigned)n_blocks, kPairThreads, 0, as_stream(stream)>>>(
        d_boundary, n, (int4 *)d_pair_nbr, d_pair_counts, pair_pitch, pair_rows / 4, unit,
        face_key ? 1 : 0, order);
    B2MD_CHECK_LAUNCH("b2md_pair_order");
    return 0;
}

B2MD_EXPORT int b2md_pair_schedule(const uint8_t *d_boundary, int64_t n, int32_t *d_pair_counts,
                                   int64_t pair_pitch, void *stream) {
    if (n <= 0 || !d_pair_counts || pair_pitch < (n + 1) / 2) {
        set_error("b2md_pair_schedule: bad arguments");
        return -1;
    }
    const int n_blocks = (int)blocks_for((n + 1) / 2, kPairThreads);
    int32_t *schedule = d_pair_counts + pair_pitch, *flags = schedule + n_blocks;
    if (!d_boundary) {
        set_error("b2md_pair_schedule: no boundary flags");
        return -2;
    }
    k_pair_block_flags<<<blocks_for(n_blocks, 8), 256, 0, as_stream(stream)>>>(d_boundary, n,
                                                                                n_blocks, flags);
    k_pair_schedule<<<1, kScheduleThreads, 0, as_stream(stream)>>>(flags, n_blocks, schedule);
    B2MD_CHECK_LAUNCH("b2md_pair_schedule");
    return 0;
}

B2MD_EXPORT int b2md_force_lj_pairs(const void *d_pos_hi, int64_t n, const b2md_box *box,
                                    const int32_t *d_pair_nbr, const int32_t *d_pair_counts,
                                    int64_t pair_pitch, const int32_t *d_nbr,
                                    const int32_t *d_counts, int64_t pitch,
                                    const uint8_t *d_boundary, const double *table,
                                    int32_t ntypes, int32_t flags, void *d_force_f4,
                                    float *d_virial, b2md_status *d_status, void *stream) {
    return launch_pairs(d_pos_hi, n, box, d_pair_nbr, d_pair_counts, pair_pitch, d_nbr, d_counts,
                        pitch, d_boundary, table, ntypes, flags, d_force_f4, d_virial, d_status,
                        nullptr, stream, "b2md_force_lj_pairs");
}

namespace {

int fill_advance(AdvanceArgs &adv, const void *d_pos_hi, void *d_pos_hi_out, void *d_pos_lo,
                 void *d_vel, void *d_image_i4, const b2md_box *box, double dt,
                 void *d_ref_pos_f4, double half_skin2, int32_t gate_in_word,
                 int32_t gate_out_word, const char *name) {
    if (!d_pos_hi_out || d_pos_hi_out == d_pos_hi || !d_pos_lo || !d_vel || !d_image_i4 ||
        !d_ref_pos_f4 || !box || !(dt > 0.0) || gate_in_word == gate_out_word ||
        gate_in_word < 0 || gate_in_word >= 16 || gate_out_word < 0 || gate_out_word >= 16 ||
        gate_in_word == kWordAdvanceCount || gate_out_word == kWordAdvanceCount) {
        set_error("%s: bad arguments", name);
        return -1;
    }
    adv.pos_out = (float4 *)d_pos_hi_out;
    adv.pos_lo = (float4 *)d_pos_lo;
    adv.vel = (float4 *)d_vel;
    adv.ref_pos = (float4 *)d_ref_pos_f4;
    adv.image = (int4 *)d_image_i4;
    adv.step = make_step(box, dt, half_skin2);
    adv.gate_in = gate_in_word;
    adv.gate_out = gate_out_word;
    adv.halo_dst[0] = adv.halo_dst[1] = nullptr;
    adv.halo_out[0] = adv.halo_out[1] = nullptr;
    adv.prune_mode = 0;
    adv.gate_clear = 0;
    adv.inner_nbr = nullptr;
    adv.inner_counts = nullptr;
    adv.inner_rl2 = adv.inner_half2 = adv.prune_limit2 = 0.0f;
    adv.inner_tiles = 0;
    return 0;
}

}  // namespace

B2MD_EXPORT int b2md_force_lj_advance(
    const void *d_pos_hi, void *d_pos_hi_out, void *d_pos_lo, void *d_vel, void *d_image_i4,
    int64_t n, const b2md_box *box, double dt, void *d_ref_pos_f4, double half_skin2,
    const int32_t *d_nbr, const int32_t *d_counts, int64_t pitch, int32_t stride,
    const uint8_t *d_boundary, const double *table, int32_t ntypes, int32_t flags,
    int32_t gate_in_word, int32_t gate_out_word, b2md_status *d_status, void *stream) {
    if (n <= 0 || !d_nbr || !d_counts || !d_status || stride < 1 || stride % 16 != 0) {
        set_error("b2md_force_lj_advance: bad arguments");
        return -1;
    }
    AdvanceArgs adv;
    int rc = fill_advance(adv, d_pos_hi, d_pos_hi_out, d_pos_lo, d_vel, d_image_i4, box, dt,
                          d_ref_pos_f4, half_skin2, gate_in_word, gate_out_word,
                          "b2md_force_lj_advance");
    if (rc) return rc;
    ForceArgs a;
    if ((rc = fill_args(a, box, table, ntypes))) return rc;
    cudaStream_t s = as_stream(stream);
    const int gated = (flags & B2MD_FORCE_GATED) ? 1 : 0;
    // lanes per particle as in b2md_force_lj: small systems are latency-bound
#define B2MD_LAUNCH_ROW_ADVANCE(SUB, PIPE, TABLE)                                             \
    k_force_lj<SUB, PIPE, TABLE, false, true>                                                 \
        <<<blocks_for(n, kForceThreads / SUB), kForceThreads, 0, s>>>(                        \
            (const float4 *)d_pos_hi, n, a, d_nbr, d_counts, pitch, d_boundary, nullptr,      \
            nullptr, d_status, gated, adv)
    switch (lanes_for(n, stride)) {
        case 16:
            if (ntypes == 1) B2MD_LAUNCH_ROW_ADVANCE(16, 0, false);
            else B2MD_LAUNCH_ROW_ADVANCE(16, 0, true);
            break;
        case 4:
            if (ntypes == 1) B2MD_LAUNCH_ROW_ADVANCE(4, 0, false);
            else B2MD_LAUNCH_ROW_ADVANCE(4, 0, true);
            break;
        case 2:
            if (ntypes == 1) B2MD_LAUNCH_ROW_ADVANCE(2, 0, false);
            else B2MD_LAUNCH_ROW_ADVANCE(2, 0, true);
            break;
        default:
            if (ntypes == 1) B2MD_LAUNCH_ROW_ADVANCE(1, 2, false);
            else B2MD_LAUNCH_ROW_ADVANCE(1, 2, true);
    }
#undef B2MD_LAUNCH_ROW_ADVANCE
    B2MD_CHECK_LAUNCH("b2md_force_lj_advance");
    return 0;
}

namespace {

template <bool TABLE>
const void *persistent_kernel(int sub) {
    switch (sub) {
        case 16: return (const void *)k_steps_persistent<16, TABLE>;
        case 4: return (const void *)k_steps_persistent<4, TABLE>;
        case 2: return (const void *)k_steps_persistent<2, TABLE>;
        default: return (const void *)k_steps_persistent<1, TABLE>;
    }
}

// Lanes per particle of the persistent kernel for n particles and `rows` allocated list rows
// (lanes_for), 0 when that grid is not co-resident on the current device.
template <bool TABLE>
int persistent_lanes(int64_t n, int32_t rows, int *blocks_out) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return 0;
    // the lanes every row kernel uses for this system (bit-identical sums), provided the
    // grid really is co-resident on this device
    const int sub = lanes_for(n, rows);
    int per_sm = 0;
    const void *fn = persistent_kernel<TABLE>(sub);
    cudaError_t err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kPersistThreads, 0);
    if (err != cudaSuccess) { cudaGetLastError(); return 0; }
    const int64_t blocks = (n + kPersistThreads / sub - 1) / (kPersistThreads / sub);
    if (blocks > (int64_t)per_sm * sms) return 0;
    *blocks_out = (int)blocks;
    return sub;
}

}  // namespace

B2MD_EXPORT int b2md_steps_persistent_lanes(int64_t n, int32_t stride, int32_t ntypes) {
    int blocks = 0;
    if (n <= 0 || stride < 1) return 0;
    return ntypes == 1 ? persistent_lanes<false>(n, stride, &blocks)
                       : persistent_lanes<true>(n, stride, &blocks);
}

B2MD_EXPORT int b2md_steps_persistent(
    void *d_pos_a, void *d_pos_b, void *d_pos_lo, void *d_vel, void *d_image_i4, int64_t n,
    const b2md_box *box, double dt, void *d_ref_pos_f4, double half_skin2, const int32_t *d_nbr,
    const int32_t *d_counts, int64_t pitch, int32_t stride, const uint8_t *d_boundary,
    const double *table, int32_t ntypes, int32_t gate_a_word, int32_t gate_b_word,
    int32_t n_steps, uint32_t *d_barrier, b2md_status *d_status, void *stream) {
    if (n <= 0 || !d_nbr || !d_counts || !d_status || !d_barrier || stride < 1 || n_steps < 1 ||
        !d_pos_a || !d_pos_b || d_pos_a == d_pos_b) {
        set_error("b2md_steps_persistent: bad arguments");
        return -1;
    }
    AdvanceArgs adv;
    int rc = fill_advance(adv, d_pos_a, d_pos_b, d_pos_lo, d_vel, d_image_i4, box, dt, d_ref_pos_f4,
                          half_skin2, gate_a_word, gate_b_word, "b2md_steps_persistent");
    if (rc) return rc;
    ForceArgs a;
    if ((rc = fill_args(a, box, table, ntypes))) return rc;
    int blocks = 0;
    const int sub = ntypes == 1 ? persistent_lanes<false>(n, stride, &blocks)
                                : persistent_lanes<true>(n, stride, &blocks);
    if (sub == 0) {
        set_error("b2md_steps_persistent: the grid for %lld particles is not co-resident (or the "
                  "list rows are not a multiple of 16 entries per lane group)", (long long)n);
        return -6;
    }
    PersistArgs ps;
    ps.pos[0] = (float4 *)d_pos_a;
    ps.pos[1] = (float4 *)d_pos_b;
    ps.gate[0] = gate_a_word;
    ps.gate[1] = gate_b_word;
    ps.n_steps = n_steps;
    ps.barrier = reinterpret_cast<unsigned long long *>(d_barrier);
    cudaStream_t s = as_stream(stream);
    if ((rc = check_cuda(cudaMemsetAsync(d_barrier, 0, B2MD_BARRIER_BYTES, s), "barrier reset")))
        return rc;
    void *args[] = {(void *)&n, (void *)&a, (void *)&d_nbr, (void *)&d_counts, (void *)&pitch,
                    (void *)&d_boundary, (void *)&d_status, (void *)&adv, (void *)&ps};
    const void *fn = ntypes == 1 ? persistent_kernel<false>(sub) : persistent_kernel<true>(sub);
    return check_cuda(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(kPersistThreads), args, 0, s),
                      "b2md_steps_persistent");
}

B2MD_EXPORT int b2md_force_lj_pairs_advance(
    const void *d_pos_hi, void *d_pos_hi_out, void *d_pos_lo, void *d_vel, void *d_image_i4,
    int64_t n, const b2md_box *box, double dt, void *d_ref_pos_f4, double half_skin2,
    const int32_t *d_pair_nbr, const int32_t *d_pair_counts, int64_t pair_pitch,
    const int32_t *d_nbr, const int32_t *d_counts, int64_t pitch, const uint8_t *d_boundary,
    const double *table, int32_t ntypes, int32_t flags, int32_t gate_in_word,
    int32_t gate_out_word, b2md_status *d_status, void *stream) {
    return b2md_force_lj_pairs_advance_halo(
        d_pos_hi, d_pos_hi_out, d_pos_lo, d_vel, d_image_i4, n, box, dt, d_ref_pos_f4, half_skin2,
        d_pair_nbr, d_pair_counts, pair_pitch, d_nbr, d_counts, pitch, d_boundary, table, ntypes,
        flags, gate_in_word, gate_out_word, nullptr, nullptr, nullptr, nullptr, d_status, stream);
}

B2MD_EXPORT int b2md_force_lj_pairs_advance_pruned(
    const void *d_pos_hi, void *d_pos_hi_out, void *d_pos_lo, void *d_vel, void *d_image_i4,
    int64_t n, const b2md_box *box, double dt, void *d_ref_pos_f4, double half_skin2,
    const int32_t *d_pair_nbr, const int32_t *d_pair_counts, int64_t pair_pitch,
    const int32_t *d_nbr, const int32_t *d_counts, int64_t pitch, const uint8_t *d_boundary,
    const double *table, int32_t ntypes, int32_t flags, int32_t gate_in_word,
    int32_t gate_out_word, int32_t gate_clear_word, int32_t prune_mode, int32_t *d_inner_nbr,
    int32_t *d_inner_counts, int32_t pair_rows, double r_cut_max, double skin, double delta,
    b2md_status *d_status, void *stream) {
    AdvanceArgs adv;
    int rc = fill_advance(adv, d_pos_hi, d_pos_hi_out, d_pos_lo, d_vel, d_image_i4, box, dt,
                          d_ref_pos_f4, half_skin2, gate_in_word, gate_out_word,
                          "b2md_force_lj_pairs_advance_pruned");
    if (rc) return rc;
    if (prune_mode < kPruneInner || prune_mode > kPruneOuter || !d_inner_nbr || !d_inner_counts ||
        pair_rows < 4 || pair_rows % 4 != 0 || !(delta > 0.0) || !(delta < skin) ||
        (uint64_t)(pair_rows / 4) * (uint64_t)pair_pitch >= 0xffffffffull ||
        0.5 * (skin - delta) > 0.99 * kPruneRange || gate_clear_word == gate_in_word ||
        gate_clear_word == gate_out_word || gate_clear_word < 0 || gate_clear_word >= 16 ||
        gate_clear_word == kWordAdvanceCount || gate_clear_word == kWordInnerDisp ||
        gate_in_word == kWordInnerDisp || gate_out_word == kWordInnerDisp) {
        set_error("b2md_force_lj_pairs_advance_pruned: bad arguments (need 0 < delta < skin, "
                  "(skin - delta) / 2 <= 0.126, three distinct gate words)");
        return -1;
    }
    adv.prune_mode = prune_mode;
    adv.gate_clear = gate_clear_word;
    adv.inner_nbr = (int4 *)d_inner_nbr;
    adv.inner_counts = d_inner_counts;
    adv.inner_tiles = pair_rows / 4;
    // keep what is inside r_cut + delta now (fp32 distance of the high words: a little wider)
    adv.inner_rl2 = (float)((r_cut_max + delta) * (r_cut_max + delta) * (1.0 + 1e-5));
    // expiry: some particle moved more than delta / 2 since the prune; the packed prune
    // snapshot is off by up to kPruneStep / 2 per component
    adv.inner_half2 = shaved_bound2(box, 0.5 * delta, 0.51 * kPruneStep);
    // a prune is legal while the outer rows are complete to r_cut + delta
    adv.prune_limit2 = shaved_bound2(box, 0.5 * (skin - delta), 0.0);
    return launch_pairs(d_pos_hi, n, box, d_pair_nbr, d_pair_counts, pair_pitch, d_nbr, d_counts,
                        pitch, d_boundary, table, ntypes, flags | B2MD_FORCE_SKIP_THERMO, nullptr,
                        nullptr, d_status, &adv, stream, "b2md_force_lj_pairs_advance_pruned");
}

B2MD_EXPORT int b2md_force_lj_pairs_advance_halo(
    const void *d_pos_hi, void *d_pos_hi_out, void *d_pos_lo, void *d_vel, void *d_image_i4,
    int64_t n, const b2md_box *box, double dt, void *d_ref_pos_f4, double half_skin2,
    const int32_t *d_pair_nbr, const int32_t *d_pair_counts, int64_t pair_pitch,
    const int32_t *d_nbr, const int32_t *d_counts, int64_t pitch, const uint8_t *d_boundary,
    const double *table, int32_t ntypes, int32_t flags, int32_t gate_in_word,
    int32_t gate_out_word, const int32_t *d_halo_dst_left, void *d_halo_out_left,
    const int32_t *d_halo_dst_right, void *d_halo_out_right, b2md_status *d_status,
    void *stream) {
    AdvanceArgs adv;
    int rc = fill_advance(adv, d_pos_hi, d_pos_hi_out, d_pos_lo, d_vel, d_image_i4, box, dt,
                          d_ref_pos_f4, half_skin2, gate_in_word, gate_out_word,
                          "b2md_force_lj_pairs_advance");
    if (rc) return rc;
    if ((d_halo_dst_left && !d_halo_out_left) || (d_halo_dst_right && !d_halo_out_right)) {
        set_error("b2md_force_lj_pairs_advance_halo: destination slots without a buffer");
        return -1;
    }
    adv.halo_dst[0] = d_halo_dst_left;
    adv.halo_out[0] = (float4 *)d_halo_out_left;
    adv.halo_dst[1] = d_halo_dst_right;
    adv.halo_out[1] = (float4 *)d_halo_out_right;
    return launch_pairs(d_pos_hi, n, box, d_pair_nbr, d_pair_counts, pair_pitch, d_nbr, d_counts,
                        pitch, d_boundary, table, ntypes, flags | B2MD_FORCE_SKIP_THERMO, nullptr,
                        nullptr, d_status, &adv, stream, "b2md_force_lj_pairs_advance");
}
