// Per-particle pieces of velocity Verlet shared by the integrate kernels
// (integrate.cu) and the force kernel that advances the particles it has just
// evaluated (force.cu): reference vv_integrate (integrate.py:58-70), wrap_position
// (core.py:72-93), vv_finalize (integrate.py:73-79).
#pragma once

#include <string.h>

#include "common.cuh"

namespace b2md {

struct StepConst {
    float L_hi[3], L_lo[3], invL[3];
    float dt_hi, dt_lo, half_dt;
    float half_skin2;
};

// x (double-single) into [0, L): k = floor(x/L) with the reference's nudges
// (core.py:81-93); returns k.
__device__ __forceinline__ int wrap_ds(float &hi, float &lo, float L_hi, float L_lo, float invL) {
    if (hi >= 0.0f && hi < L_hi) return 0;          // common case (hi == L_hi handled below)
    float kf = floorf(hi * invL);
    if (kf != 0.0f) {
        // (hi, lo) -= k * (L_hi + L_lo), product formed error-free
        const float ph = kf * L_hi;
        const float pl = fmaf(kf, L_hi, -ph) + kf * L_lo;
        ds_add(hi, lo, -ph, -pl);
    }
    // value < 0 ?
    if (hi < 0.0f || (hi == 0.0f && lo < 0.0f)) {
        ds_add(hi, lo, L_hi, L_lo);
        kf -= 1.0f;
    }
    // value >= L ?
    if (hi > L_hi || (hi == L_hi && lo >= L_lo)) {
        ds_add(hi, lo, -L_hi, -L_lo);
        kf += 1.0f;
    }
    return (int)kf;
}

__device__ __forceinline__ void kick(float4 &v, const float4 f, float half_dt) {
    // v += (f / m) * (0.5*dt): divide, then multiply (integrate.py:64,79)
    const float m = v.w;
    v.x = __fadd_rn(v.x, __fmul_rn(__fdiv_rn(f.x, m), half_dt));
    v.y = __fadd_rn(v.y, __fmul_rn(__fdiv_rn(f.y, m), half_dt));
    v.z = __fadd_rn(v.z, __fmul_rn(__fdiv_rn(f.z, m), half_dt));
}

__device__ __forceinline__ void drift(float &hi, float &lo, float v, float dt_hi, float dt_lo) {
    const float ph = v * dt_hi;
    const float pl = fmaf(v, dt_lo, fmaf(v, dt_hi, -ph));   // exact product tail
    ds_add(hi, lo, ph, pl);
}

inline StepConst make_step(const b2md_box *box, double dt, double half_skin2) {
    StepConst c;
    for (int a = 0; a < 3; ++a) {
        c.L_hi[a] = (float)box->edge[a];
        c.L_lo[a] = (float)(box->edge[a] - (double)c.L_hi[a]);
        c.invL[a] = (float)(1.0 / box->edge[a]);
    }
    c.dt_hi = (float)dt;
    c.dt_lo = (float)(dt - (double)c.dt_hi);
    c.half_dt = (float)(0.5 * dt);
    // Never fire later than the exact fp64 test (neighbor.py:251-254).  The in-loop test
    // sees high words only: per component the snapshot drops its low word (<= ulp(L)/2),
    // so does the current position, and the wrap correction of the snapshot subtracts
    // k*L_hi instead of k*L (another ulp(L)/2) -- at most 2 ulp(L) on a component, 2.5 with
    // the roundings of the difference.  The squared norm of a displacement d at the
    // threshold is then off by at most 2*sqrt(3)*|d|*delta + 3*delta^2 (plus the fp32
    // roundings of the sum, 4*2^-24 relative): that much comes off the threshold.
    double lmax = 0.0;
    for (int a = 0; a < 3; ++a) lmax = box->edge[a] > lmax ? box->edge[a] : lmax;
    int e = 0;
    frexp(lmax, &e);                                   // lmax = m * 2^e, m in [0.5, 1)
    const double ulp = ldexp(1.0, e - 24);             // fp32 ulp just below lmax
    const double delta = 2.5 * ulp;
    const double half_skin = sqrt(half_skin2);
    double shaved = half_skin2 - (2.0 * 1.7320508075688772 * half_skin * delta +
                                  3.0 * delta * delta);
    shaved *= 1.0 - 1e-6;
    if (!(shaved > 0.0)) shaved = 0.0;                 // zero skin: rebuild on any motion
    c.half_skin2 = half_skin2 >= 1e29 ? (float)half_skin2 : (float)shaved;
    return c;
}

// KICKS half-kicks with force f, drift, wrap, image counters, displacement from the list
// snapshot, on a particle held in registers: h / l = position high / low words, v = velocity
// (w = mass), r = the snapshot's high words.  Image counters are touched in memory, and only on
// a face crossing.  Returns the squared displacement (0 when !have_ref).
template <int KICKS>
__device__ __forceinline__ float advance_regs(int64_t i, float4 &h, float4 &l, float4 &v, float4 &r,
                                              bool have_ref, const float4 f,
                                              int4 *__restrict__ image, const StepConst &c) {
#pragma unroll
    for (int k = 0; k < KICKS; ++k) kick(v, f, c.half_dt);
    drift(h.x, l.x, v.x, c.dt_hi, c.dt_lo);
    drift(h.y, l.y, v.y, c.dt_hi, c.dt_lo);
    drift(h.z, l.z, v.z, c.dt_hi, c.dt_lo);
    const int kx = wrap_ds(h.x, l.x, c.L_hi[0], c.L_lo[0], c.invL[0]);
    const int ky = wrap_ds(h.y, l.y, c.L_hi[1], c.L_lo[1], c.invL[1]);
    const int kz = wrap_ds(h.z, l.z, c.L_hi[2], c.L_lo[2], c.invL[2]);
    const bool wrapped = (kx | ky | kz) != 0;
    if (wrapped) {
        int4 im = image[i];
        im.x += kx; im.y += ky; im.z += kz;
        image[i] = im;
    }
    float d2 = 0.0f;
    if (have_ref) {
        if (wrapped) {
            // keep (hi - ref) equal to the unwrapped displacement
            r.x = fmaf(-(float)kx, c.L_hi[0], r.x);
            r.y = fmaf(-(float)ky, c.L_hi[1], r.y);
            r.z = fmaf(-(float)kz, c.L_hi[2], r.z);
        }
        const float dx = h.x - r.x, dy = h.y - r.y, dz = h.z - r.z;
        d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
    }
    return d2;
}

// KICKS half-kicks with force f, drift, wrap, image counters, displacement from the
// list snapshot: one particle of k_integrate.  h (position high words) comes in and
// goes out through registers; returns the squared displacement (0 without ref_pos).
template <int KICKS>
__device__ __forceinline__ float advance_particle(int64_t i, float4 &h, const float4 f,
                                                  float4 *__restrict__ pos_lo,
                                                  float4 *__restrict__ vel,
                                                  int4 *__restrict__ image, const StepConst &c,
                                                  float4 *__restrict__ ref_pos) {
    float4 v = vel[i];
#pragma unroll
    for (int k = 0; k < KICKS; ++k) kick(v, f, c.half_dt);
    vel[i] = v;
    float4 l = pos_lo[i];
    drift(h.x, l.x, v.x, c.dt_hi, c.dt_lo);
    drift(h.y, l.y, v.y, c.dt_hi, c.dt_lo);
    drift(h.z, l.z, v.z, c.dt_hi, c.dt_lo);
    const int kx = wrap_ds(h.x, l.x, c.L_hi[0], c.L_lo[0], c.invL[0]);
    const int ky = wrap_ds(h.y, l.y, c.L_hi[1], c.L_lo[1], c.invL[1]);
    const int kz = wrap_ds(h.z, l.z, c.L_hi[2], c.L_lo[2], c.invL[2]);
    pos_lo[i] = l;
    const bool wrapped = (kx | ky | kz) != 0;
    if (wrapped) {
        int4 im = image[i];
        im.x += kx; im.y += ky; im.z += kz;
        image[i] = im;
    }
    float d2 = 0.0f;
    if (ref_pos) {
        float4 r = ref_pos[i];
        if (wrapped) {
            // keep (hi - ref) equal to the unwrapped displacement
            r.x = fmaf(-(float)kx, c.L_hi[0], r.x);
            r.y = fmaf(-(float)ky, c.L_hi[1], r.y);
            r.z = fmaf(-(float)kz, c.L_hi[2], r.z);
            ref_pos[i] = r;
        }
        const float dx = h.x - r.x, dy = h.y - r.y, dz = h.z - r.z;
        d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
    }
    return d2;
}

// ---- pruned ("inner") pair rows of the step loop -------------------------------------------
// The list snapshot's spare word (ref_pos.w) holds the particle's displacement from the list
// snapshot AT THE LAST PRUNE, three 10-bit fixed-point components: the step kernel then knows
// the displacement since the prune, (h - r) - u_prune, without a second snapshot array.
// Range +-kPruneRange per component (a prune is only legal while every particle is within
// (skin - delta) / 2 <= kPruneRange of its snapshot); the rounding error, <= kPruneStep / 2 per
// component, comes off the expiry threshold (make_prune).
constexpr float kPruneRange = 0.128f;
constexpr float kPruneStep = kPruneRange / 511.0f;

__device__ __forceinline__ float pack_disp(float ux, float uy, float uz) {
    const float inv = 1.0f / kPruneStep;
    const int qx = max(-511, min(511, __float2int_rn(ux * inv))) + 512;
    const int qy = max(-511, min(511, __float2int_rn(uy * inv))) + 512;
    const int qz = max(-511, min(511, __float2int_rn(uz * inv))) + 512;
    return __int_as_float(qx | (qy << 10) | (qz << 20));
}
__device__ __forceinline__ void unpack_disp(float w, float &ux, float &uy, float &uz) {
    const int b = __float_as_int(w);
    ux = (float)((b & 1023) - 512) * kPruneStep;
    uy = (float)(((b >> 10) & 1023) - 512) * kPruneStep;
    uz = (float)(((b >> 20) & 1023) - 512) * kPruneStep;
}
inline float pack_disp_zero_host() {
    const int b = 512 | (512 << 10) | (512 << 20);
    float f;
    memcpy(&f, &b, sizeof f);
    return f;
}

// advance_particle for a step loop with pruned pair rows.  snapshot_now: this launch prunes --
// the displacement of the INPUT position (h on entry) becomes the prune snapshot.  d2_inner
// receives the squared displacement of the advanced position since the last prune.
template <int KICKS>
__device__ __forceinline__ float advance_particle_pruned(int64_t i, float4 &h, const float4 f,
                                                         float4 *__restrict__ pos_lo,
                                                         float4 *__restrict__ vel,
                                                         int4 *__restrict__ image,
                                                         const StepConst &c,
                                                         float4 *__restrict__ ref_pos,
                                                         bool snapshot_now, float &d2_inner) {
    float4 r = ref_pos[i];
    bool store_ref = false;
    if (snapshot_now) {
        r.w = pack_disp(h.x - r.x, h.y - r.y, h.z - r.z);
        store_ref = true;
    }
    float4 v = vel[i];
#pragma unroll
    for (int k = 0; k < KICKS; ++k) kick(v, f, c.half_dt);
    vel[i] = v;
    float4 l = pos_lo[i];
    drift(h.x, l.x, v.x, c.dt_hi, c.dt_lo);
    drift(h.y, l.y, v.y, c.dt_hi, c.dt_lo);
    drift(h.z, l.z, v.z, c.dt_hi, c.dt_lo);
    const int kx = wrap_ds(h.x, l.x, c.L_hi[0], c.L_lo[0], c.invL[0]);
    const int ky = wrap_ds(h.y, l.y, c.L_hi[1], c.L_lo[1], c.invL[1]);
    const int kz = wrap_ds(h.z, l.z, c.L_hi[2], c.L_lo[2], c.invL[2]);
    pos_lo[i] = l;
    if ((kx | ky | kz) != 0) {
        int4 im = image[i];
        im.x += kx; im.y += ky; im.z += kz;
        image[i] = im;
        // keep (hi - ref) equal to the unwrapped displacement
        r.x = fmaf(-(float)kx, c.L_hi[0], r.x);
        r.y = fmaf(-(float)ky, c.L_hi[1], r.y);
        r.z = fmaf(-(float)kz, c.L_hi[2], r.z);
        store_ref = true;
    }
    if (store_ref) ref_pos[i] = r;
    const float dx = h.x - r.x, dy = h.y - r.y, dz = h.z - r.z;
    float ux, uy, uz;
    unpack_disp(r.w, ux, uy, uz);
    const float ex = dx - ux, ey = dy - uy, ez = dz - uz;
    d2_inner = fmaf(ez, ez, fmaf(ey, ey, ex * ex));
    return fmaf(dz, dz, fmaf(dy, dy, dx * dx));
}

// The same never-fire-late shave as make_step's half_skin2, for an arbitrary displacement bound
// `d` (plus `extra` of known error on the displacement itself).
inline float shaved_bound2(const b2md_box *box, double d, double extra) {
    double lmax = 0.0;
    for (int a = 0; a < 3; ++a) lmax = box->edge[a] > lmax ? box->edge[a] : lmax;
    int e = 0;
    frexp(lmax, &e);
    const double delta = 2.5 * ldexp(1.0, e - 24) + extra;
    double shaved = d * d - (2.0 * 1.7320508075688772 * d * delta + 3.0 * delta * delta);
    shaved *= 1.0 - 1e-6;
    return shaved > 0.0 ? (float)shaved : 0.0f;
}

}  // namespace b2md
